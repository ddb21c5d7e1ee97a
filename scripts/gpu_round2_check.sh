# full GPU suite, default bench line, reference arm
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/gputests_r2.txt 2>&1; echo tests_rc=$?; tail -3 gpurun_out/gputests_r2.txt
t0=$(date +%s); timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_r2.json 2> gpurun_out/bench_r2.err; echo bench_rc=$? secs=$(( $(date +%s) - t0 )); tail -3 gpurun_out/bench_r2.err
t0=$(date +%s); timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref_r2.json 2> gpurun_out/ref_r2.err; echo ref_rc=$? secs=$(( $(date +%s) - t0 )); tail -3 gpurun_out/ref_r2.err; tail -c 700 gpurun_out/ref_r2.json
