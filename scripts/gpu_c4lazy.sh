mkdir -p gpurun_out; out=gpurun_out/c4_lazy.txt; : > $out
run() { name=$1; shift
  timeout 300 env "$@" python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline --no-extras > /tmp/o.json 2>/tmp/e.txt
  python -c "import json;d=json.load(open('/tmp/o.json'));print('$name ms=%.4f kernel=%.4f exact=%s'%(d['ms_per_step'],d['roofline']['kernel_ms'],d['parity']['bit_exact']))" >> $out 2>&1 || (echo "$name FAILED" >> $out; tail -3 /tmp/e.txt >> $out)
}
run base X=1
for ns in 50 100 200 400 800; do run lazy$ns SFG_IC_LAZY=$ns; done
for b in 1 3; do run bps$b SFG_BLOCKS_PER_SM=$b; run bps${b}_lazy200 SFG_BLOCKS_PER_SM=$b SFG_IC_LAZY=200; done
run base2 X=1
cat $out
