# fact executors compiled for 3 / 4 resident blocks per SM vs default, C2/C3/C4
mkdir -p gpurun_out
for c in 2 3 4; do AB_TESTS="golden or config_full_size or set_values or breakdown" bash scripts/gpu_ab.sh ab30_c$c.txt "minb3 minb4" --config $c; done
cat gpurun_out/ab30_c*.txt
