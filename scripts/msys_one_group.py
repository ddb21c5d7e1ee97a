"""k_msys on a 2-D 9-point grid of 128 x 32 lines: one 32-chain group whose
only dependencies are in-group (ring) -- the free-running step cost."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_12238_b200 as sf

nx, ny, S = 128, int(sys.argv[1]) if len(sys.argv) > 1 else 32, 8
n = nx * ny
cols = []
for j in range(n):
    x, y = j % nx, j // nx
    ent = []
    for dy in (-1, 0, 1):
        for dx in (-1, 0, 1):
            xx, yy = x + dx, y + dy
            if 0 <= xx < nx and 0 <= yy < ny:
                k = yy * nx + xx
                ent.append((k, 9.0 if k == j else -1.0))
    ent.sort()
    cols.append(ent)
colptr = np.zeros(n + 1, dtype=np.int64)
colptr[1:] = np.cumsum([len(e) for e in cols])
rowidx = np.array([k for e in cols for k, _ in e], dtype=np.int64)
vals1 = np.array([v for e in cols for _, v in e])
M = sf.CscMatrix(n, colptr, rowidx, vals1)
vals = np.concatenate([vals1 * (1 + 0.01 * s) for s in range(S)])
vin = np.concatenate([sf.gen_vector(n, 7 + s) for s in range(S)])
out = "/tmp/m1trace.bin"
mode = sys.argv[2] if len(sys.argv) > 2 else "trace"
if mode == "trace":
    os.environ["SFG_TRACE"] = out
os.environ["SFG_EXECUTOR"] = "msys"
os.environ["SFG_MLINE_STATS"] = "1"
st = sf.make_state(1, M, seed=7, nsys=S, values=vals, vin=vin).inspect()
for _ in range(3):
    st.execute_fused()
got = st.collect_outputs()
print("kernel ms", st.bench(3)[1] / 3)
st.close()
os.environ.pop("SFG_EXECUTOR")
os.environ.pop("SFG_TRACE", None)
ref = sf.make_state(1, M, seed=7, nsys=S, values=vals, vin=vin)
ref.execute_fused()
print("equal", np.array_equal(got, ref.collect_outputs()))
if mode == "trace":
    raw = np.fromfile(out, dtype=np.int64)
    items = raw[0]
    d = raw[3:3 + items * 4].view(np.uint64).reshape(items, 4)
    t0 = d[:, 0].min()
    for i in range(min(items, 8)):
        c, f, e = (d[i, :3].astype(np.int64) - int(t0)) / 1e3
        print(f"item {i}: first {f:8.1f} end {e:8.1f} dur {e - f:8.1f} late_cyc {int(d[i,3] >> 32)} poll {int(d[i,3] & 0xffffffff)}")
