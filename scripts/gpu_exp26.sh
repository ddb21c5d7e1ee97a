mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "config5 or multisystem or golden_outputs" > gpurun_out/exp26.txt 2>&1; echo rc=$? >> gpurun_out/exp26.txt
run() {
  envs="$1"; shift
  timeout 300 env $envs python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extras "$@" > /tmp/o.json 2>/tmp/e.txt
  python -c "import json,sys;d=json.load(open('/tmp/o.json'));print('$envs $* ms=%.3f kernel=%.3f unfused=%.3f frac=%.3f'%(d['ms_per_step'],d['roofline']['kernel_ms'],d['unfused']['ms_per_step'],d['roofline']['frac']))" >> gpurun_out/exp26.txt 2>&1 || (echo "$envs $* FAILED" >> gpurun_out/exp26.txt; tail -3 /tmp/e.txt >> gpurun_out/exp26.txt)
}
for g in 0 500 0 500; do run "SFG_BWD_GATE=$g" --config 5; done
