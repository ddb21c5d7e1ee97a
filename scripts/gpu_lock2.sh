mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "config5 or multisystem or batch or edge or irregular or combo8 or fwd_bwd" > gpurun_out/lock_tests.txt 2>&1; echo tests_rc=$?; tail -3 gpurun_out/lock_tests.txt
timeout 300 python scripts/trace_lock.py > gpurun_out/trace_lock.txt 2>&1; grep -v "  L=" gpurun_out/trace_lock.txt
SFG_EXECUTOR=lock timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/lock_bench_lock.json 2> gpurun_out/lock_bench_lock.err
python - <<P
import json
d=json.load(open('gpurun_out/lock_bench_lock.json'))
print('lock', d['ms_per_step'], d['roofline']['kernel_ms'], d['parity'], d.get('unfused'))
P
