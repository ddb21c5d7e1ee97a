mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras --size 64"
for B in 2048; do
  SFG_BSF_B=$B timeout 300 $CMD > gpurun_out/bsf64_plain.json 2>&1
  SFG_BSF_B=$B SFG_EXECUTOR=levels SFG_SLEEP_CAP=0 timeout 300 $CMD > gpurun_out/lev64_plain.json 2>&1
done
SFG_BSF_B=2048 timeout 300 $CMD > gpurun_out/plain3.log 2>&1 && SFG_BSF_B=2048 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bsf -s 2 -c 1 -o gpurun_out/prof_bsf64 $CMD > gpurun_out/ncu_bsf.log 2>&1; echo rc=$?
