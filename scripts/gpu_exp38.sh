# C1 (k_mline1): CTAs (2 warps each) per SM sweep
mkdir -p gpurun_out
out=gpurun_out/exp38.txt; : > $out
run() {
  envs="$1"; shift
  timeout 300 env $envs python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-extras "$@" > /tmp/o.json 2>/tmp/e.txt
  python -c "import json,sys;d=json.load(open('/tmp/o.json'));print('$envs $* ms=%.4f kernel=%.4f'%(d['ms_per_step'],d['roofline']['kernel_ms']))" >> $out 2>&1 || (echo "$envs $* FAILED" >> $out; tail -3 /tmp/e.txt >> $out)
}
for rep in 1 2; do for b in 0 2 4 6 8 12 16; do if [ $b = 0 ]; then run "X=1" --config 1; else run "SFG_BLOCKS_PER_SM=$b" --config 1; fi; done; done
