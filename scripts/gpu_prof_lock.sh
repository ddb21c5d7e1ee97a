# ncu --set full with source counters of the lockstep kernel (one launch).
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras"
timeout 300 $CMD > gpurun_out/plain_lock.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_lock -s 3 -c 1 -f -o gpurun_out/prof_lock $CMD > gpurun_out/ncu_lock.log 2>&1; echo rc=$?
