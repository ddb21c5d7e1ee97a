mkdir -p gpurun_out
set -x
nproc; lscpu | grep -E "Model name|Socket|Thread|Core" ; free -g | head -2
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo bench_rc=$?
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo launches_rc=$?
timeout 300 $CMD > gpurun_out/plain2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_trsv_pair -s 2 -c 1 -o gpurun_out/prof_c5 $CMD > gpurun_out/ncu_full.log 2>&1; echo full_rc=$?
ls -la gpurun_out
