# chain tile skew per level (SFG_CHAIN_SKEW) on C5, fwd->bwd and fwd->fwd; parity of each
mkdir -p gpurun_out
out=gpurun_out/skew.txt; : > $out
for rep in 1 2; do for K in 1 2 3; do for mode in fwdbwd fwdfwd; do
  timeout 300 env SFG_CHAIN_SKEW=$K python bench.py --steps 20 --warmup 3 --mode $mode --no-cpu-baseline --no-extras > /tmp/o.json 2>/tmp/e.txt
  python -c "import json;d=json.load(open('/tmp/o.json'));print('skew=$K $mode ms=%.4f kernel=%.4f unfused=%.4f parity=%s'%(d['ms_per_step'],d['roofline']['kernel_ms'],d['unfused']['ms_per_step'],d['parity']['bit_exact']))" >> $out 2>&1 || (echo "skew=$K FAILED" >> $out; tail -3 /tmp/e.txt >> $out)
done; done; done
for K in 2 3; do SFG_CHAIN_SKEW=$K timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "config5 or multisystem or mline_executor" > /tmp/t.txt 2>&1; echo "skew=$K tests rc=$? $(tail -1 /tmp/t.txt)" >> $out; done
cat $out
