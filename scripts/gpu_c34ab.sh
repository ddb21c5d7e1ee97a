mkdir -p gpurun_out; out=gpurun_out/c34_ab.txt; : > $out
run() { name=$1; lib=$2; cfg=$3; shift 3
  if [ "$lib" = base ]; then L="X=1"; else L="SFG_LIB=old_lib/$lib/libsfgpu.so"; fi
  timeout 300 env $L "$@" python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-extras > /tmp/o.json 2>/tmp/e.txt
  python -c "import json;d=json.load(open('/tmp/o.json'));print('$name c$cfg ms=%.4f kernel=%.4f exact=%s'%(d['ms_per_step'],d['roofline']['kernel_ms'],d['parity']['bit_exact']))" >> $out 2>&1 || (echo "$name FAILED" >> $out; tail -3 /tmp/e.txt >> $out)
}
for rep in 1 2; do for c in 2 3 4; do run base base $c X=1; for l in $ALTS; do run $l $l $c X=1; done; done; done
cat $out
