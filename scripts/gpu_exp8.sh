mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
run() {
  envs="$1"; shift
  timeout 300 env $envs python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras "$@" > /tmp/o.json 2>/tmp/e.txt
  python -c "import json,sys;d=json.load(open('/tmp/o.json'));print('$envs $* ms=%.3f kernel=%.3f unfused=%.3f frac=%.3f e2e=%.2f clk=%s'%(d['ms_per_step'],d['roofline']['kernel_ms'],d['unfused']['ms_per_step'],d['roofline']['frac'],d['e2e']['ms_per_step'],d['clocks']['sm_mhz']))" >> gpurun_out/exp8.txt 2>&1 || (echo "$envs $* FAILED" >> gpurun_out/exp8.txt; tail -3 /tmp/e.txt >> gpurun_out/exp8.txt)
}
run "SFG_X=0" --config 5
run "SFG_ELL=0" --config 5
run "SFG_X=0" --config 5 --systems-per-gpu 16
run "SFG_X=0" --config 5 --systems-per-gpu 4
