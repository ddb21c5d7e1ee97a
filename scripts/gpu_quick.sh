# quick GPU round: selected GPU tests + a list of bench runs.
# usage: bash scripts/gpu_quick.sh OUT "pytest -k expr" "bench args 1" "bench args 2" ...
mkdir -p gpurun_out
out=gpurun_out/$1; shift
kexpr=$1; shift
: > $out
if [ -n "$kexpr" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "$kexpr" > /tmp/t.txt 2>&1; echo "tests rc=$? $(tail -1 /tmp/t.txt)" >> $out
  grep -E "FAILED|Error|assert" /tmp/t.txt | head -20 >> $out
fi
for args in "$@"; do
  timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extras $args > /tmp/o.json 2>/tmp/e.txt
  python -c "import json,sys;d=json.load(open('/tmp/o.json'));u=d.get('unfused',{});print('$args ms=%.4f kernel=%.4f frac=%.3f unfused=%s'%(d['ms_per_step'],d['roofline']['kernel_ms'],d['roofline']['frac'],u.get('ms_per_step')))" >> $out 2>&1 || (echo "$args FAILED" >> $out; tail -3 /tmp/e.txt >> $out)
done
