# lockstep knobs: sleep on miss, DX, warps
mkdir -p gpurun_out; out=gpurun_out/lock_knobs.txt; : > $out
run() { # name lib envs...
  name=$1; lib=$2; shift 2
  if [ "$lib" = base ]; then L="X=1"; else L="SFG_LIB=old_lib/$lib/libsfgpu.so"; fi
  timeout 300 env $L "$@" python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras > /tmp/o.json 2>/tmp/e.txt
  python -c "import json;d=json.load(open('/tmp/o.json'));print('$name ms=%.4f kernel=%.4f exact=%s'%(d['ms_per_step'],d['roofline']['kernel_ms'],d['parity']['bit_exact']))" >> $out 2>&1 || (echo "$name FAILED" >> $out; tail -3 /tmp/e.txt >> $out)
}
run notrace notrace X=1
for ns in 100 200 400 800 1600; do run notrace_sleep$ns notrace SFG_LOCK_SLEEP=$ns; done
run dx1 dx1 X=1
for ns in 100 200 400 800; do run dx1_sleep$ns dx1 SFG_LOCK_SLEEP=$ns; done
run w4 w4 X=1
run w4_sleep400 w4 SFG_LOCK_SLEEP=400
cat $out
