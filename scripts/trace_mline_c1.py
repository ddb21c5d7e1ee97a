"""(k_mline1 records its timeline only in a build with -DSFG_ML1_TRACE=1:
bash scripts/build_alt.sh ml1trace "-DSFG_ML1_TRACE=1", then SFG_LIB=old_lib/ml1trace/libsfgpu.so.)
Multi-line executor timeline on the C1 matrix (one forward solve pair)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_12238_b200 as sf
out = "/tmp/mtrace1.bin"
os.environ["SFG_TRACE"] = out
os.environ["SFG_EXECUTOR"] = "mline"
os.environ["SFG_MLINE_STATS"] = "1"
M = sf.config_matrix(1)
st = sf.make_state(1, M, seed=7)
st.inspect()
for _ in range(3):
    st.execute_fused()
print("kernel ms", st.bench(1)[1])
st.close()
raw = np.fromfile(out, dtype=np.int64)
items, w, nf = raw[:3]
d = raw[3:3 + items * 4].view(np.uint64).reshape(items, 4)
t0 = d[:, 0].min()
for i in range(items):
    c, f, e = (d[i, :3] - t0) / 1e3
    print(f"item {i:3d}: claim {c:8.1f} first {f:8.1f} end {e:8.1f} dur {e - f:8.1f} hi_cyc {int(d[i,3] >> 32):9d} poll_cyc {int(d[i,3] & 0xffffffff):9d}")
