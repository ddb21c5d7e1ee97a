# occupancy variants: ILU0 4-slot at 4 blocks/SM (C3); IC0 combo 5 with 4-slot batches at 3 blocks/SM or unbounded (C2); parity of each
mkdir -p gpurun_out
AB_TESTS="golden or config_full_size or combos_2_3 or ilu0 or set_values or batch or breakdown or pcg" bash scripts/gpu_ab.sh ab40_c3.txt ilu4 --config 3
AB_TESTS="golden or config_full_size or set_values or batch or breakdown or pcg" bash scripts/gpu_ab.sh ab40_c2.txt "ic5a ic5b" --config 2
cat gpurun_out/ab40_c3.txt gpurun_out/ab40_c2.txt
