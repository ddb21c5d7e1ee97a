# Factorization executors: resident warps per SM (contention) sweep on C2/C3/C4.
mkdir -p gpurun_out
out=gpurun_out/exp28.txt; : > $out
run() {
  envs="$1"; shift
  timeout 300 env $envs python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras "$@" > /tmp/o.json 2>/tmp/e.txt
  python -c "import json,sys;d=json.load(open('/tmp/o.json'));print('$envs $* ms=%.4f kernel=%.4f'%(d['ms_per_step'],d['roofline']['kernel_ms']))" >> $out 2>&1 || (echo "$envs $* FAILED" >> $out; tail -3 /tmp/e.txt >> $out)
}
for cfg in 4 2 3; do
  for b in 0 1 2 3 4 6; do
    if [ $b = 0 ]; then run "X=1" --config $cfg; else run "SFG_BLOCKS_PER_SM=$b" --config $cfg; fi
  done
done
