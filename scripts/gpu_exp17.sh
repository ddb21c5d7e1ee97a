mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "batch" > gpurun_out/exp17.txt 2>&1; echo rc=$? >> gpurun_out/exp17.txt
timeout 600 python bench.py --no-cpu-baseline --no-extras > /tmp/o.json 2>> gpurun_out/exp17.txt
python -c "import json;d=json.load(open('/tmp/o.json'));print('C5 value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e'])" >> gpurun_out/exp17.txt 2>&1
timeout 600 python bench.py --config 1 --no-cpu-baseline --no-extras > /tmp/o1.json 2>> gpurun_out/exp17.txt
python -c "import json;d=json.load(open('/tmp/o1.json'));print('C1 value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e'])" >> gpurun_out/exp17.txt 2>&1
