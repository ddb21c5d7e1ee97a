# Round-start check on a B200: GPU parity suite, default bench line.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputests.txt 2>&1; echo tests_rc=$?; tail -3 gpurun_out/gputests.txt
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_base.json 2> gpurun_out/bench_base.err; echo bench_rc=$?
tail -c 1500 gpurun_out/bench_base.json
