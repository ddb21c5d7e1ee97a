# segment-width warp executors: auto width vs SFG_TASK_WIDTH=32 (one task per warp), C2/C3/C4; full GPU tests
mkdir -p gpurun_out
out=gpurun_out/exp32.txt; : > $out
run() {
  envs="$1"; shift
  timeout 300 env $envs python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extras "$@" > /tmp/o.json 2>/tmp/e.txt
  python -c "import json,sys;d=json.load(open('/tmp/o.json'));print('$envs $* ms=%.4f kernel=%.4f unfused=%.4f'%(d['ms_per_step'],d['roofline']['kernel_ms'],d['unfused']['ms_per_step']))" >> $out 2>&1 || (echo "$envs $* FAILED" >> $out; tail -3 /tmp/e.txt >> $out)
}
for c in 2 3 4; do for rep in 1 2; do run "SFG_TASK_WIDTH=32" --config $c; run "X=1" --config $c; run "SFG_TASK_WIDTH=16" --config $c; done; done
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > /tmp/t.txt 2>&1; echo "tests rc=$? $(tail -1 /tmp/t.txt)" >> $out
grep -E "FAILED|Error" /tmp/t.txt | head >> $out
