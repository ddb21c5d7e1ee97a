mkdir -p gpurun_out
run() {
  envs="$1"; shift
  timeout 300 env $envs python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras "$@" > /tmp/o.json 2>/tmp/e.txt
  python -c "import json,sys;d=json.load(open('/tmp/o.json'));print('$envs $* ms=%.3f kernel=%.3f unfused=%.3f'%(d['ms_per_step'],d['roofline']['kernel_ms'],d['unfused']['ms_per_step']))" >> gpurun_out/exp23.txt 2>&1 || (echo "$envs $* FAILED" >> gpurun_out/exp23.txt; tail -3 /tmp/e.txt >> gpurun_out/exp23.txt)
}
for cap in 0; do run "SFG_SLEEP_CAP=$cap" --config 4; run "SFG_SLEEP_CAP=$cap" --config 2; run "SFG_SLEEP_CAP=$cap" --config 3; done
