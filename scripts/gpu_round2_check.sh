# full GPU suite, default bench line, reference arm, per-GPU batch sizes of the sharded config 5
mkdir -p gpurun_out
nproc; free -g | head -2
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/gputests_r2.txt 2>&1; echo tests_rc=$?; tail -3 gpurun_out/gputests_r2.txt
/usr/bin/time -v timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_r2.json 2> gpurun_out/bench_r2.err; echo bench_rc=$?; grep -E "Elapsed|Maximum resident" gpurun_out/bench_r2.err
/usr/bin/time -v timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref_r2.json 2> gpurun_out/ref_r2.err; echo ref_rc=$?; grep -E "Elapsed|Maximum resident" gpurun_out/ref_r2.err; tail -c 600 gpurun_out/ref_r2.json
for S in 1 2 4; do timeout 600 python bench.py --steps 20 --warmup 3 --systems-per-gpu $S --no-cpu-baseline --no-extras > gpurun_out/bench_S$S.json 2>gpurun_out/bench_S$S.err; python -c "import json;d=json.load(open('gpurun_out/bench_S$S.json'));print('S=$S', d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['kernel'], d['parity'])"; done
