mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_schedules.py tests/test_dropin.py tests/test_cpp_api.py -m gpu -q -p no:cacheprovider -x > gpurun_out/t_sched.txt 2>&1; echo sched_rc=$?; tail -15 gpurun_out/t_sched.txt
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "structures or config5_batch" --durations=10 > gpurun_out/t_struct.txt 2>&1; echo struct_rc=$?; tail -15 gpurun_out/t_struct.txt
