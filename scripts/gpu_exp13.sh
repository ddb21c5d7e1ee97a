mkdir -p gpurun_out
run() {
  envs="$1"; shift
  timeout 300 env $envs python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras "$@" > /tmp/o.json 2>/tmp/e.txt
  python -c "import json,sys;d=json.load(open('/tmp/o.json'));print('$envs $* ms=%.3f kernel=%.3f unfused=%.3f frac=%.3f'%(d['ms_per_step'],d['roofline']['kernel_ms'],d['unfused']['ms_per_step'],d['roofline']['frac']))" >> gpurun_out/exp13.txt 2>&1 || (echo "$envs $* FAILED" >> gpurun_out/exp13.txt; tail -3 /tmp/e.txt >> gpurun_out/exp13.txt)
}
for sl in 0 20 50 100 200 400; do run "SFG_SLEEP_CAP=$sl" --config 5; done
run "SFG_SLEEP_CAP=100 SFG_BLOCKS_PER_SM=1" --config 5
