# ncu --set full with source counters of the C5 chain kernel (one launch).
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras"
timeout 300 $CMD > gpurun_out/plain_c5.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_chain_sm -s 3 -c 1 -o gpurun_out/prof_c5src $CMD > gpurun_out/ncu_c5src.log 2>&1; echo rc=$? >> gpurun_out/ncu_c5src.log
