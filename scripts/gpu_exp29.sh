# paired waits in the factorization executors: new build vs old_lib/prev on C2/C3/C4 + parity of the new build
mkdir -p gpurun_out
for c in 2 3 4; do AB_TESTS="nothing_matches_xyz" bash scripts/gpu_ab.sh ab29_c$c.txt prev --config $c; done
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/exp29_tests.txt 2>&1; echo rc=$? >> gpurun_out/exp29_tests.txt
cat gpurun_out/ab29_c*.txt | grep -v parity; tail -2 gpurun_out/exp29_tests.txt
