# lockstep executor (lock.cu) vs k_chain_sm on C5: parity subset, then A/B timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "config5 or multisystem or batch or edge or irregular or combo8 or fwd_bwd" > gpurun_out/lock_tests.txt 2>&1; echo tests_rc=$?; tail -5 gpurun_out/lock_tests.txt
for ex in lock chain; do
  SFG_EXECUTOR=$ex timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/lock_bench_$ex.json 2> gpurun_out/lock_bench_$ex.err; echo "$ex rc=$?"
  python - <<P
import json
d=json.load(open('gpurun_out/lock_bench_$ex.json'))
print('$ex', d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['kernel'], d['parity'], d.get('unfused'))
P
done
