# double-buffered outputs (dbuf) for the batched chain executor: full GPU tests; bench on/off (SFG_DBUF=0) both modes
mkdir -p gpurun_out
out=gpurun_out/exp36.txt; : > $out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > /tmp/t.txt 2>&1; echo "tests rc=$? $(tail -1 /tmp/t.txt)" >> $out
grep -E "FAILED|Error" /tmp/t.txt | head >> $out
run() {
  envs="$1"; shift
  timeout 300 env $envs python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-extras "$@" > /tmp/o.json 2>/tmp/e.txt
  python -c "import json,sys;d=json.load(open('/tmp/o.json'));print('$envs $* ms=%.4f kernel=%.4f e2e=%.4f value=%.1f launches=%d'%(d['ms_per_step'],d['roofline']['kernel_ms'],d['e2e']['ms_per_step'],d['value'],d['gpu_launches']))" >> $out 2>&1 || (echo "$envs $* FAILED" >> $out; tail -3 /tmp/e.txt >> $out)
}
for rep in 1 2; do run "X=1"; run "SFG_DBUF=0"; run "X=1" --mode fwdfwd; run "SFG_DBUF=0" --mode fwdfwd; done
