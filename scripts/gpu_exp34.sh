# ILU0 factorization software-pipelined across tasks vs old_lib/hp (header prefetch only): C3; full GPU tests
mkdir -p gpurun_out
AB_TESTS="nothing_matches_xyz" bash scripts/gpu_ab.sh ab34_c3.txt hp --config 3
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/exp34_tests.txt 2>&1; echo rc=$? >> gpurun_out/exp34_tests.txt
cat gpurun_out/ab34_c3.txt | grep -v parity; tail -2 gpurun_out/exp34_tests.txt; grep -E "FAILED|Error" gpurun_out/exp34_tests.txt | head
