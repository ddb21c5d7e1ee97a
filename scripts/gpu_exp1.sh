mkdir -p gpurun_out
timeout 120 ./scripts/micro_hop > gpurun_out/micro_hop.txt 2>&1
for cfg in 5 1 2; do
for cap in 160 0 40; do
for bps in 0 1; do
  SFG_SLEEP_CAP=$cap SFG_BLOCKS_PER_SM=$bps timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-extras > /tmp/o.json 2>&1
  python -c "import json;d=json.load(open('/tmp/o.json'));print('cfg=$cfg cap=$cap bps=$bps ms=%.3f kernel=%.3f unfused=%.3f frac=%.3f'%(d['ms_per_step'],d['roofline']['kernel_ms'],d['unfused']['ms_per_step'],d['roofline']['frac']))" >> gpurun_out/exp1.txt 2>&1 || tail -3 /tmp/o.json >> gpurun_out/exp1.txt
done; done; done
