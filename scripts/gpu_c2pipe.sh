mkdir -p gpurun_out; out=gpurun_out/c2_pipe.txt; : > $out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x --timeout 120 > gpurun_out/c2pipe_tests.txt 2>&1; echo tests_rc=$? >> $out; tail -3 gpurun_out/c2pipe_tests.txt >> $out
run() { name=$1; shift
  timeout 300 env "$@" python bench.py --config 2 --steps 20 --warmup 3 --no-cpu-baseline --no-extras > /tmp/o.json 2>/tmp/e.txt
  python -c "import json;d=json.load(open('/tmp/o.json'));print('$name ms=%.4f kernel=%.4f exact=%s unfused=%.4f'%(d['ms_per_step'],d['roofline']['kernel_ms'],d['parity']['bit_exact'],d['unfused']['ms_per_step']))" >> $out 2>&1 || (echo "$name FAILED" >> $out; tail -3 /tmp/e.txt >> $out)
}
for rep in 1 2; do run pipe X=1; run old SFG_IC5_PIPE=0; done
for b in 2 4; do run pipe_bps$b SFG_BLOCKS_PER_SM=$b; done
cat $out
