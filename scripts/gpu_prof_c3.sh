# ncu --set full of the C3 (ILU0 -> unit solve) warp executor, one launch
mkdir -p gpurun_out
CMD="python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-extras"
timeout 300 $CMD > gpurun_out/plain_c3.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_ilu0_warp -s 3 -c 1 -o gpurun_out/prof_c3 $CMD > gpurun_out/ncu_c3.log 2>&1; echo rc=$? >> gpurun_out/ncu_c3.log
CMD2="python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --no-extras"
timeout 300 $CMD2 > gpurun_out/plain_c2.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_ic0_warp -s 3 -c 1 -o gpurun_out/prof_c2 $CMD2 > gpurun_out/ncu_c2.log 2>&1; echo rc=$? >> gpurun_out/ncu_c2.log
