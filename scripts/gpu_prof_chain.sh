mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras"
timeout 300 $CMD > gpurun_out/plain_chain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain_ell -s 2 -c 1 -o gpurun_out/prof_chain $CMD > gpurun_out/ncu_chain.log 2>&1; echo rc=$?
