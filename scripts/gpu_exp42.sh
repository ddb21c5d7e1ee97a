# lookahead-sized warp executors: default (20 levels) vs full occupancy (SFG_FACT_LOOKAHEAD=0) and 10/30 levels; C2/C3/C4
mkdir -p gpurun_out
out=gpurun_out/exp42.txt; : > $out
run() {
  envs="$1"; shift
  timeout 300 env $envs python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras "$@" > /tmp/o.json 2>/tmp/e.txt
  python -c "import json,sys;d=json.load(open('/tmp/o.json'));print('$envs $* ms=%.4f kernel=%.4f'%(d['ms_per_step'],d['roofline']['kernel_ms']))" >> $out 2>&1 || (echo "$envs $* FAILED" >> $out; tail -3 /tmp/e.txt >> $out)
}
for c in 4 2 3; do for l in X 0 10 30; do if [ $l = X ]; then run "X=1" --config $c; else run "SFG_FACT_LOOKAHEAD=$l" --config $c; fi; done; done
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > /tmp/t.txt 2>&1; echo "tests rc=$? $(tail -1 /tmp/t.txt)" >> $out
