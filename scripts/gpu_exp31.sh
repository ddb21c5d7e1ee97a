# ticket claims in chunks of 2 / 4 (one atomic per chunk) vs 1, C2/C3/C4
mkdir -p gpurun_out
for c in 2 3 4; do AB_TESTS="golden or config_full_size or set_values or breakdown or batch" bash scripts/gpu_ab.sh ab31_c$c.txt "claim2 claim4" --config $c; done
cat gpurun_out/ab31_c*.txt
