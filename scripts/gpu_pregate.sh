mkdir -p gpurun_out
out=gpurun_out/pregate.txt; : > $out
for rep in 1 2; do for g in 0 100 300 1000; do for mode in fwdbwd fwdfwd; do
  timeout 300 env SFG_PRE_GATE=$g python bench.py --steps 30 --warmup 3 --mode $mode --no-cpu-baseline --no-extras > /tmp/o.json 2>/tmp/e.txt
  python -c "import json;d=json.load(open('/tmp/o.json'));print('pre_gate=$g $mode ms=%.4f kernel=%.4f parity=%s'%(d['ms_per_step'],d['roofline']['kernel_ms'],d['parity']['bit_exact']))" >> $out 2>&1 || (echo FAILED >> $out; tail -3 /tmp/e.txt >> $out)
done; done; done
cat $out
