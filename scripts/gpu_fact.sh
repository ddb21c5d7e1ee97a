mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_fact.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_fact.log
run() {
  envs="$1"; shift
  timeout 300 env $envs python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras "$@" > /tmp/o.json 2>/tmp/e.txt
  python -c "import json,sys;d=json.load(open('/tmp/o.json'));print('$envs $* ms=%.3f kernel=%.3f unfused=%.3f e2e=%.3f'%(d['ms_per_step'],d['roofline']['kernel_ms'],d['unfused']['ms_per_step'],d['e2e']['ms_per_step']))" >> gpurun_out/fact.txt 2>&1 || (echo "$envs $* FAILED" >> gpurun_out/fact.txt; tail -3 /tmp/e.txt >> gpurun_out/fact.txt)
}
for cfg in 4 2 3; do
  run "SFG_X=0" --config $cfg
  run "SFG_SLEEP_CAP=0" --config $cfg
done
run "SFG_EXECUTOR=levels" --config 4
