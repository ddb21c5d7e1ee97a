mkdir -p gpurun_out
SFG_EXECUTOR=ws timeout 120 python -c "
import numpy as np, sys
sys.path.insert(0, '.')
import paper_2111_12238_b200 as sf
from oracle.oracle import Oracle, Csc
orc = Oracle()
M, vals = sf.config5_systems(size=16, nsys=8)
n, nnz = M.n, M.nnz
st = sf.make_state(8, M, nsys=8, values=vals)
st.execute_fused()
got = st.collect_outputs().reshape(8, 2 * n)
for s in range(8):
    Ms = Csc(n, M.colptr, M.rowidx, vals[s * nnz:(s + 1) * nnz])
    want = orc.run_sequential(8, Ms, 7 + s)
    print(s, np.array_equal(got[s], want), float(np.max(np.abs(got[s] - want))))
" > gpurun_out/exp18.txt 2>&1; echo smoke_rc=$? >> gpurun_out/exp18.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "mline_executor" >> gpurun_out/exp18.txt 2>&1; echo rc=$? >> gpurun_out/exp18.txt
run() {
  envs="$1"; shift
  timeout 300 env $envs python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras "$@" > /tmp/o.json 2>/tmp/e.txt
  python -c "import json,sys;d=json.load(open('/tmp/o.json'));print('$envs $* ms=%.3f kernel=%.3f unfused=%.3f frac=%.3f'%(d['ms_per_step'],d['roofline']['kernel_ms'],d['unfused']['ms_per_step'],d['roofline']['frac']))" >> gpurun_out/exp18.txt 2>&1 || (echo "$envs $* FAILED" >> gpurun_out/exp18.txt; tail -3 /tmp/e.txt >> gpurun_out/exp18.txt)
}
run "SFG_EXECUTOR=ws SFG_WS_SLOTS=3" --config 5
run "SFG_EXECUTOR=ws SFG_WS_SLOTS=2" --config 5
run "SFG_X=0" --config 5
