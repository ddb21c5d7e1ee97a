# C4 (k_ic0_warp<7>, 64 regs, 4 blocks/SM by default): resident blocks sweep
mkdir -p gpurun_out
out=gpurun_out/exp41.txt; : > $out
run() {
  envs="$1"; shift
  timeout 300 env $envs python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras "$@" > /tmp/o.json 2>/tmp/e.txt
  python -c "import json,sys;d=json.load(open('/tmp/o.json'));print('$envs $* ms=%.4f kernel=%.4f'%(d['ms_per_step'],d['roofline']['kernel_ms']))" >> $out 2>&1 || (echo "$envs $* FAILED" >> $out; tail -3 /tmp/e.txt >> $out)
}
for rep in 1 2; do for b in 0 1 2 3; do if [ $b = 0 ]; then run "X=1" --config 4; else run "SFG_BLOCKS_PER_SM=$b" --config 4; fi; done; done
for b in 0 2; do if [ $b = 0 ]; then run "X=1" --config 2; run "X=1" --config 3; else run "SFG_BLOCKS_PER_SM=$b" --config 2; run "SFG_BLOCKS_PER_SM=$b" --config 3; fi; done
