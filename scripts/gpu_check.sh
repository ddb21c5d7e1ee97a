# Round re-entry check: full GPU test suite, smoke, short default bench.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/check_tests.txt 2>&1; echo rc=$? >> gpurun_out/check_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/check_smoke.txt 2>&1; echo rc=$? >> gpurun_out/check_smoke.txt
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/check_bench.json 2> gpurun_out/check_bench.err; echo rc=$? >> gpurun_out/check_bench.err
