# Round evidence (final refresh): default bench line, reference arm, C5 launch list, ncu full of C5/C4/C3/C2 hot kernels.
mkdir -p gpurun_out
nproc > gpurun_out/host.txt
timeout 1200 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench_rc=$? >> gpurun_out/host.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$? >> gpurun_out/host.txt
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo launches_rc=$? >> gpurun_out/host.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain_sm -s 3 -c 1 -o gpurun_out/prof_c5 $CMD > gpurun_out/ncu_c5.log 2>&1; echo c5_rc=$? >> gpurun_out/host.txt
for c in 4 3 2; do
  K=k_ic0_warp; [ $c = 3 ] && K=k_ilu0_warp
  CMDc="python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-extras"
  timeout 300 $CMDc > gpurun_out/plain_c$c.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/prof_c$c $CMDc > gpurun_out/ncu_c$c.log 2>&1; echo c${c}_rc=$? >> gpurun_out/host.txt
done
