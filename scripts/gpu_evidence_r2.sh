# Round-2 evidence: default bench line, reference arm, C5 launch list, ncu --set full of each config's hot kernel.
mkdir -p gpurun_out/ev
E=gpurun_out/ev
nproc > $E/host.txt; nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv >> $E/host.txt
timeout 1200 python bench.py > $E/bench_default.json 2> $E/bench_default.err; echo bench_rc=$? >> $E/host.txt
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $E/bench_ref.json 2> $E/bench_ref.err; echo ref_rc=$? >> $E/host.txt
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras"
timeout 300 $CMD > $E/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $E/launches_c5.csv $CMD > $E/ncu_launch.log 2>&1; echo launches_rc=$? >> $E/host.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain_sm -s 3 -c 1 -o $E/prof_c5 -f $CMD > $E/ncu_c5.log 2>&1; echo c5_rc=$? >> $E/host.txt
for c in 1 2 3 4; do
  case $c in 1) K=k_mline1;; 2) K=k_ic0_pipe;; 3) K=k_ilu0_pack;; 4) K=k_ic0_warp;; esac
  CMDc="python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-extras"
  timeout 300 $CMDc > $E/plain_c$c.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o $E/prof_c$c -f $CMDc > $E/ncu_c$c.log 2>&1; echo c${c}_rc=$? >> $E/host.txt
done
cat $E/host.txt
