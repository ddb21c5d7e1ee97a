# A/B: default build vs alternative builds under old_lib/<name> on C5 (and an
# optional config), each alternated twice; parity of each alt on config-5 tests.
# usage: bash scripts/gpu_ab.sh OUT "alt1 alt2 ..." [bench args]
mkdir -p gpurun_out
out=gpurun_out/$1; shift
alts=$1; shift
: > $out
run() {
  lib="$1"; shift
  if [ "$lib" = base ]; then envs="X=1"; else envs="SFG_LIB=old_lib/$lib/libsfgpu.so"; fi
  timeout 300 env $envs python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extras "$@" > /tmp/o.json 2>/tmp/e.txt
  python -c "import json,sys;d=json.load(open('/tmp/o.json'));print('$lib $* ms=%.4f kernel=%.4f frac=%.3f'%(d['ms_per_step'],d['roofline']['kernel_ms'],d['roofline']['frac']))" >> $out 2>&1 || (echo "$lib $* FAILED" >> $out; tail -3 /tmp/e.txt >> $out)
}
for rep in 1 2; do
  run base "$@"
  for a in $alts; do run $a "$@"; done
done
kexpr=${AB_TESTS:-"config5 or multisystem or golden_outputs"}
for a in $alts; do
  SFG_LIB=old_lib/$a/libsfgpu.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -m gpu -x -q -p no:cacheprovider -k "$kexpr" > /tmp/t.txt 2>&1; echo "$a parity rc=$? $(tail -1 /tmp/t.txt)" >> $out
done
