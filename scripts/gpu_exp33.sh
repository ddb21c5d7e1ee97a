# next-task header prefetched across the phases of the current task: new build vs old_lib/prev, C2/C3/C4; full GPU tests
mkdir -p gpurun_out
for c in 2 3 4; do AB_TESTS="nothing_matches_xyz" bash scripts/gpu_ab.sh ab33_c$c.txt prev --config $c; done
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/exp33_tests.txt 2>&1; echo rc=$? >> gpurun_out/exp33_tests.txt
cat gpurun_out/ab33_c*.txt | grep -v parity; tail -2 gpurun_out/exp33_tests.txt
