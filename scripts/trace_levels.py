"""(The chain kernels record their timeline only in a build with -DSFG_CHAIN_TRACE=1:
bash scripts/build_alt.sh trace "-DSFG_CHAIN_TRACE=1", then SFG_LIB=old_lib/trace/libsfgpu.so.)
Per-level timing of the C5 chain executor from SFG_TRACE: tile-end times
(globaltimer) per chain level, the per-level lag and the in-chain tile period."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
out = "/tmp/trace.bin"
os.environ["SFG_TRACE"] = out
os.environ.setdefault("SFG_TRACE_TILES", "40")
import paper_2111_12238_b200 as sf
M, vals = sf.config5_systems(size=int(os.environ.get("C5_SIZE", "0")) or None, nsys=8)
st = sf.make_state(8, M, nsys=8, values=vals)
st.inspect()
for _ in range(3):
    st.execute_fused()
print("kernel ms", st.bench(1)[1])
st.close()
raw = np.fromfile(out, dtype=np.int64)
items, tiles, nf = (int(v) for v in raw[:3])
d = raw[3:3 + items * tiles * 3].view(np.uint64).reshape(items, tiles, 3)
lev = np.frombuffer(raw[3 + items * tiles * 3:].tobytes(), dtype=np.int32)[:items]
ends = d[:, :, 2].astype(np.int64)
valid = ends > 0
t0 = ends[valid].min()
e = np.where(valid, ends - t0, -1).astype(np.float64) / 1e3  # us
claim = (d[:, 0, 0].astype(np.int64) - t0) / 1e3  # stage-D entry of tile 0
entry = np.where(valid, d[:, :, 0].astype(np.int64) - t0, -1).astype(np.float64) / 1e3
wait = ((d[:, :, 1] >> 22) & ((1 << 22) - 1)).astype(np.float64) * 1.965  # ns -> cycles
carry = (d[:, :, 1] & ((1 << 22) - 1)).astype(np.float64)
dd = np.diff(np.unique(ends[valid][:200000]))
print("globaltimer min step ns", dd[dd > 0].min() if dd.size else None)
ntile = valid.sum(1)
for part, sl in (("fwd", slice(0, nf)), ("bwd", slice(nf, items))):
    L = lev[sl]
    E = e[sl]
    nt = ntile[sl]
    first = E[:, 0]
    last = np.array([E[i, nt[i] - 1] for i in range(E.shape[0])])
    mid = np.array([E[i, min(16, nt[i] - 1)] for i in range(E.shape[0])])
    print(f"{part}: items {E.shape[0]} levels {L.min()}..{L.max()} tiles/chain median {np.median(nt)}")
    rows = []
    for l in range(L.min(), L.max() + 1):
        m = L == l
        if not m.any():
            continue
        rows.append((l, m.sum(), np.median(first[m]), np.max(first[m]), np.median(mid[m]), np.median(last[m]), np.max(last[m]),
                     np.median(claim[sl][m])))
    rows = np.array(rows)
    for r in rows[::max(1, len(rows) // 25)]:
        print("  L=%4d n=%3d first med %8.1f max %8.1f  mid %8.1f  last med %8.1f max %8.1f  claim %8.1f" % tuple(r))
    lag = np.diff(rows[:, 2])
    print("  per-level lag of first-tile end: median %.2f us, mean %.2f" % (np.median(lag), lag.mean()))
    lag = np.diff(rows[:, 4])
    print("  per-level lag of tile-16 end: median %.2f us, mean %.2f" % (np.median(lag), lag.mean()))
    # by tile skew class (level mod 4): a level whose skew wraps to 0 needs its producers' NEXT tile
    lv = rows[1:, 0].astype(int)
    for col, nm in ((2, "first-tile"), (4, "tile-16"), (5, "last-tile")):
        d = np.diff(rows[:, col])
        print("  lag of %s end by level mod 4:" % nm, [round(float(np.median(d[lv % 4 == m])), 2) for m in range(4)])
    per = np.concatenate([np.diff(E[i, :nt[i]]) for i in range(0, E.shape[0], 7)])
    print("  in-chain tile period us p10/50/90", np.percentile(per, [10, 50, 90]).round(2))
    # split of one tile: gap (previous tile end -> stage-D entry: stages A-C and the copy wait),
    # wait phase (polls + sum), carry
    gaps = np.concatenate([entry[sl][i, 1:nt[i]] - E[i, :nt[i] - 1] for i in range(0, E.shape[0], 7)])
    print("  gap prev-end -> stage-D entry us p10/50/90", np.percentile(gaps, [10, 50, 90]).round(2))
    ready = E - carry[sl] / 1965.0 / 1e3 * 1e3 / 1e3
    rl = []
    for l in range(L.min(), L.max() + 1):
        m = L == l
        if m.any():
            rl.append(np.median(ready[m, 8]))
    print("  per-level lag of tile-8 ready (summed) time: median %.2f" % np.median(np.diff(rl)))
    # level-1 chain alone (nothing to wait for)
    i1 = np.where(L == L.min())[0][0]
    print("  source chain: entry-gap", np.round(entry[sl][i1, 1:8] - E[i1, :7], 2).tolist(),
          "wait us", np.round(wait[sl][i1, :8] / 1965.0, 2).tolist(), "carry us", np.round(carry[sl][i1, :8] / 1965.0, 2).tolist())
    W = wait[sl][valid[sl]] / 1965.0
    C = carry[sl][valid[sl]] / 1965.0
    print("  wait-phase us p10/50/90", np.percentile(W, [10, 50, 90]).round(2), " carry us", np.percentile(C, [10, 50, 90]).round(2))
