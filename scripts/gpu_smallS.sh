# config 5 per-GPU batch sizes: executor / tile height per S
mkdir -p gpurun_out
out=gpurun_out/smallS.txt; : > $out
run() { tag=$1; S=$2; shift 2
  timeout 300 env "$@" python bench.py --steps 20 --warmup 3 --systems-per-gpu $S --no-cpu-baseline --no-extras > /tmp/o.json 2>/tmp/e.txt
  python -c "import json;d=json.load(open('/tmp/o.json'));print('$tag S=$S ms=%.3f kernel=%.3f %s parity=%s'%(d['ms_per_step'],d['roofline']['kernel_ms'],d['roofline']['kernel'],d['parity']['bit_exact']))" >> $out 2>&1 || (echo "$tag S=$S FAILED" >> $out; tail -3 /tmp/e.txt >> $out); }
run mline 1 X=1
for G in 1 2 4 8; do run chainG$G 1 SFG_EXECUTOR=chain SFG_CHAIN_G=$G; done
for G in 2 4 8 16; do run G$G 2 SFG_CHAIN_G=$G; done
for G in 2 4 8; do run G$G 4 SFG_CHAIN_G=$G; done
for G in 2 4; do run G$G 8 SFG_CHAIN_G=$G; done
cat $out
