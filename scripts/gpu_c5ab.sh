mkdir -p gpurun_out; out=gpurun_out/c5_ab.txt; : > $out
run() { name=$1; lib=$2; shift 2
  if [ "$lib" = base ]; then L="X=1"; else L="SFG_LIB=old_lib/$lib/libsfgpu.so"; fi
  timeout 300 env $L "$@" python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extras > /tmp/o.json 2>/tmp/e.txt
  python -c "import json;d=json.load(open('/tmp/o.json'));print('$name ms=%.4f kernel=%.4f exact=%s unfused=%.4f'%(d['ms_per_step'],d['roofline']['kernel_ms'],d['parity']['bit_exact'],d['unfused']['ms_per_step']))" >> $out 2>&1 || (echo "$name FAILED" >> $out; tail -3 /tmp/e.txt >> $out)
}
for rep in 1 2; do run base base X=1; for l in $ALTS; do run $l $l X=1; done; done
cat $out
