mkdir -p gpurun_out
out=gpurun_out/ab_ff.txt; : > $out
for rep in 1 2; do for lib in base prev; do for mode in fwdfwd fwdbwd; do
  if [ $lib = base ]; then E="X=1"; else E="SFG_LIB=old_lib/$lib/libsfgpu.so"; fi
  timeout 300 env $E python bench.py --steps 30 --warmup 3 --mode $mode --no-cpu-baseline --no-extras > /tmp/o.json 2>/tmp/e.txt
  python -c "import json;d=json.load(open('/tmp/o.json'));print('$lib $mode ms=%.4f kernel=%.4f'%(d['ms_per_step'],d['roofline']['kernel_ms']))" >> $out 2>&1 || (echo FAILED >> $out; tail -3 /tmp/e.txt >> $out)
done; done; done
cat $out
