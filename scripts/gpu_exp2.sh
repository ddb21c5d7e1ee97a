mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
run() {
  envs="$1"; shift
  timeout 300 env $envs python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras "$@" > /tmp/o.json 2>/tmp/e.txt
  python -c "import json,sys;d=json.load(open('/tmp/o.json'));print('$envs $* ms=%.3f kernel=%.3f unfused=%.3f frac=%.3f'%(d['ms_per_step'],d['roofline']['kernel_ms'],d['unfused']['ms_per_step'],d['roofline']['frac']))" >> gpurun_out/exp2.txt 2>&1 || (echo "$envs $* FAILED" >> gpurun_out/exp2.txt; tail -3 /tmp/e.txt >> gpurun_out/exp2.txt)
}
for B in 512 1024 2048; do run "SFG_BSF_B=$B" --config 5; done
run "SFG_EXECUTOR=levels SFG_SLEEP_CAP=0" --config 5
for B in 1024 4096 8192 16384; do run "SFG_BSF_B=$B" --config 1; done
run "SFG_EXECUTOR=levels SFG_SLEEP_CAP=0" --config 1
