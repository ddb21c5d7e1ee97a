# 384-thread k_chain_sm: bwd-gate sleep sweep (env) on C5
mkdir -p gpurun_out
out=gpurun_out/exp35.txt; : > $out
run() {
  envs="$1"; shift
  timeout 300 env $envs python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extras "$@" > /tmp/o.json 2>/tmp/e.txt
  python -c "import json,sys;d=json.load(open('/tmp/o.json'));print('$envs $* ms=%.4f kernel=%.4f'%(d['ms_per_step'],d['roofline']['kernel_ms']))" >> $out 2>&1 || (echo "$envs $* FAILED" >> $out; tail -3 /tmp/e.txt >> $out)
}
for rep in 1 2; do for g in X 0 100 300 1000 3000; do if [ $g = X ]; then run "X=1"; else run "SFG_BWD_GATE=$g"; fi; done; done
