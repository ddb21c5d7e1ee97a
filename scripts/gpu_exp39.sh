# ILU0 warp kernel with 4 update slots (88 regs, 2 blocks/SM) vs 8 slots (SFG_ILU_MAXU8) vs 4 slots at 3 blocks/SM (old_lib/ilu3); C3
mkdir -p gpurun_out
out=gpurun_out/exp39.txt; : > $out
run() {
  envs="$1"; shift
  timeout 300 env $envs python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extras "$@" > /tmp/o.json 2>/tmp/e.txt
  python -c "import json,sys;d=json.load(open('/tmp/o.json'));print('$envs $* ms=%.4f kernel=%.4f'%(d['ms_per_step'],d['roofline']['kernel_ms']))" >> $out 2>&1 || (echo "$envs $* FAILED" >> $out; tail -3 /tmp/e.txt >> $out)
}
for rep in 1 2; do run "X=1" --config 3; run "SFG_ILU_MAXU8=1" --config 3; run "SFG_LIB=old_lib/ilu3/libsfgpu.so" --config 3; done
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "golden or config_full_size or combos_2_3 or ilu0 or set_values or batch" > /tmp/t.txt 2>&1; echo "tests rc=$? $(tail -1 /tmp/t.txt)" >> $out
SFG_LIB=old_lib/ilu3/libsfgpu.so timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "golden or config_full_size or combos_2_3 or ilu0 or set_values or batch" > /tmp/t.txt 2>&1; echo "ilu3 tests rc=$? $(tail -1 /tmp/t.txt)" >> $out
