# fused fwd->bwd with the in-kernel vout reset vs the prep reset (SFG_PREP_VOUT=1)
mkdir -p gpurun_out
out=gpurun_out/reset.txt; : > $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_schedules.py -m gpu -q -x -p no:cacheprovider -k "config5 or multisystem or batch or batched or edge or mline_executor or irregular or canonical" > /tmp/t.txt 2>&1; echo "tests rc=$? $(tail -1 /tmp/t.txt)" >> $out
for rep in 1 2; do for v in 0 1; do
  if [ $v = 1 ]; then E="SFG_PREP_VOUT=1"; else E="X=1"; fi
  timeout 300 env $E python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-extras > /tmp/o.json 2>/tmp/e.txt
  python -c "import json;d=json.load(open('/tmp/o.json'));print('prep_vout=$v ms=%.4f kernel=%.4f unfused=%.4f speedup=%.4f parity=%s'%(d['ms_per_step'],d['roofline']['kernel_ms'],d['unfused']['ms_per_step'],d['unfused']['fused_speedup'],d['parity']['bit_exact']))" >> $out 2>&1 || (echo FAILED >> $out; tail -3 /tmp/e.txt >> $out)
done; done
cat $out
