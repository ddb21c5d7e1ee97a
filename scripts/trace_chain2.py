"""(The chain kernels record their timeline only in a build with -DSFG_CHAIN_TRACE=1:
bash scripts/build_alt.sh trace "-DSFG_CHAIN_TRACE=1", then SFG_LIB=old_lib/trace/libsfgpu.so.)
Cycle-level split of the chain executor's tiles (S >= 2 kernel):
wait phase (cp.async wait + polls + sums) and carry phase, per tile."""
import os, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_12238_b200 as sf
out = "/tmp/trace.bin"
os.environ["SFG_TRACE"] = out
M, vals = sf.config5_systems(size=int(sys.argv[1]) if len(sys.argv) > 1 else None, nsys=8)
st = sf.make_state(8, M, nsys=8, values=vals)
st.inspect()
for _ in range(3):
    st.execute_fused()
print("kernel ms", st.bench(1)[1])
st.close()
raw = np.fromfile(out, dtype=np.int64)
items, tiles, nf = raw[:3]
d = raw[3:3 + items * tiles * 3].view(np.uint64).reshape(items, tiles, 3)
valid = d[:, :, 2] > 0
wait = (d[:, :, 1] >> 32).astype(np.float64)[valid]
carry = (d[:, :, 1] & 0xffffffff).astype(np.float64)[valid]
print("wait cycles p10/50/90", np.percentile(wait, [10, 50, 90]).round())
print("carry cycles p10/50/90", np.percentile(carry, [10, 50, 90]).round())
ends = d[:, :, 2].astype(np.float64)
t0 = ends[valid].min()
for i in [0, 1, 2, 100, int(nf)//2]:
    nt = int(valid[i].sum())
    e = (ends[i, :nt] - t0) / 1e3
    print(f"item {i}: tile period us", np.round(np.diff(e)[:8], 2).tolist(),
          "wait", (d[i, :8, 1] >> 32).tolist(), "carry", (d[i, :8, 1] & 0xffffffff).tolist())
