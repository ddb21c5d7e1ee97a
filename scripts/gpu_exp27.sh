# C5 latency vs load: systems per GPU 1/2/4/8/16 and CTAs per SM 1/2.
mkdir -p gpurun_out
out=gpurun_out/exp27.txt; : > $out
run() {
  envs="$1"; shift
  timeout 300 env $envs python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extras "$@" > /tmp/o.json 2>/tmp/e.txt
  python -c "import json,sys;d=json.load(open('/tmp/o.json'));print('$envs $* ms=%.3f kernel=%.3f frac=%.3f'%(d['ms_per_step'],d['roofline']['kernel_ms'],d['roofline']['frac']))" >> $out 2>&1 || (echo "$envs $* FAILED" >> $out; tail -3 /tmp/e.txt >> $out)
}
for s in 2 4 8 16; do run "X=1" --systems-per-gpu $s; done
run "SFG_BLOCKS_PER_SM=1" --systems-per-gpu 8
run "SFG_BLOCKS_PER_SM=1" --systems-per-gpu 16
run "SFG_CHAIN_G=2" --systems-per-gpu 8
run "X=1" --systems-per-gpu 8 --mode fwdfwd
