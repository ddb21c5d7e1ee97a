# dbuf background reset grid size sweep (SFG_DBUF_BLOCKS) vs no dbuf
mkdir -p gpurun_out
out=gpurun_out/exp37.txt; : > $out
run() {
  envs="$1"; shift
  timeout 300 env $envs python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-extras "$@" > /tmp/o.json 2>/tmp/e.txt
  python -c "import json,sys;d=json.load(open('/tmp/o.json'));print('$envs $* ms=%.4f kernel=%.4f'%(d['ms_per_step'],d['roofline']['kernel_ms']))" >> $out 2>&1 || (echo "$envs $* FAILED" >> $out; tail -3 /tmp/e.txt >> $out)
}
for rep in 1 2; do for b in 4 16 32 148; do run "SFG_DBUF_BLOCKS=$b"; done; run "SFG_DBUF=0"; done
