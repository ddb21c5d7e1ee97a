mkdir -p gpurun_out
run() {
  envs="$1"; shift
  timeout 300 env $envs python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras "$@" > /tmp/o.json 2>/tmp/e.txt
  python -c "import json,sys;d=json.load(open('/tmp/o.json'));print('$envs $* ms=%.3f kernel=%.3f unfused=%.3f frac=%.3f'%(d['ms_per_step'],d['roofline']['kernel_ms'],d['unfused']['ms_per_step'],d['roofline']['frac']))" >> gpurun_out/exp19.txt 2>&1 || (echo "$envs $* FAILED" >> gpurun_out/exp19.txt; tail -3 /tmp/e.txt >> gpurun_out/exp19.txt)
}
for q in 2 3; do for pr in 1 2 4; do run "SFG_EXECUTOR=ws SFG_WS_SLOTS=$q SFG_WS_PAIRS=$pr" --config 5; done; done
