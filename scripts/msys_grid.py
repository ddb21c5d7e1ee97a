"""k_msys vs the chain executor on 27-point grids nx x ny x nz (lines along
x): isolates the cost of group-to-group hops in y (ny > 32) and z (nz > 1)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_12238_b200 as sf


def grid(nx, ny, nz):
    n = nx * ny * nz
    idx = np.arange(n).reshape(nz, ny, nx)
    rows, cols = [], []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                src = idx[max(0, -dz):nz - max(0, dz), max(0, -dy):ny - max(0, dy), max(0, -dx):nx - max(0, dx)]
                dst = idx[max(0, dz):nz - max(0, -dz), max(0, dy):ny - max(0, -dy), max(0, dx):nx - max(0, -dx)]
                rows.append(dst.ravel())
                cols.append(src.ravel())
    r = np.concatenate(rows)
    c = np.concatenate(cols)
    order = np.lexsort((r, c))
    r, c = r[order], c[order]
    v = np.where(r == c, 27.0, -1.0)
    colptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(c, minlength=n), out=colptr[1:])
    return sf.CscMatrix(n, colptr, r.astype(np.int64), v)


S = 8
for spec in sys.argv[1:]:
    nx, ny, nz = (int(t) for t in spec.split("x"))
    M = grid(nx, ny, nz)
    vals = np.concatenate([M.values * (1 + 0.01 * s) for s in range(S)])
    vin = np.concatenate([sf.gen_vector(M.n, 7 + s) for s in range(S)])
    res = {}
    for ex in ("msys", None):
        if ex:
            os.environ["SFG_EXECUTOR"] = ex
        else:
            os.environ.pop("SFG_EXECUTOR", None)
        st = sf.make_state(1, M, seed=7, nsys=S, values=vals, vin=vin).inspect()
        st.execute_fused()
        out = st.collect_outputs()
        st.bench(2)
        res[ex] = (out, st.bench(5)[1] / 5)
        st.close()
    print(f"{spec}: msys {res['msys'][1]:.3f} ms chain {res[None][1]:.3f} ms "
          f"equal={np.array_equal(res['msys'][0], res[None][0])}", flush=True)
