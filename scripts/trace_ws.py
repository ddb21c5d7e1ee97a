"""Timeline of the warp-specialised chain executor (SFG_TRACE diagnostics):
per tile {slot ready, dependencies ready, published}; lag between chain
levels and where each tile's time goes."""
import os, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_12238_b200 as sf
out = "/tmp/wstrace.bin"
os.environ["SFG_TRACE"] = out
os.environ["SFG_TRACE_TILES"] = "33"
os.environ.setdefault("SFG_EXECUTOR", "ws")
M, vals = sf.config5_systems(nsys=8)
st = sf.make_state(8, M, nsys=8, values=vals)
st.inspect()
for _ in range(3):
    st.execute_fused()
print("kernel ms", st.bench(1)[1])
st.close()
raw = np.fromfile(out, dtype=np.int64)
items, tiles, nf = raw[:3]
d = raw[3:3 + items * tiles * 3].view(np.uint64).reshape(items, tiles, 3).astype(np.float64)
lev = raw[3 + items * tiles * 3:].view(np.int32)[:items]
valid = d[:, :, 2] > 0
t0 = d[valid][:, 0].min()
d = (d - t0) / 1e3
wait = (d[:, :, 1] - d[:, :, 0])[valid]
comp = (d[:, :, 2] - d[:, :, 1])[valid]
per = np.diff(d[:, :, 2], axis=1)[valid[:, 1:] & valid[:, :-1]]
print(json.dumps({"span_us": float(d[valid][:, 2].max()),
                  "dep_wait_us_p10_50_90": np.percentile(wait, [10, 50, 90]).round(3).tolist(),
                  "compute_us_p10_50_90": np.percentile(comp, [10, 50, 90]).round(3).tolist(),
                  "tile_period_us_p10_50_90": np.percentile(per, [10, 50, 90]).round(3).tolist()}))
# lag between levels, fwd solve: median publish time of tile 16 per level
for seg, sl in (("fwd", slice(0, nf)), ("bwd", slice(nf, items))):
    L = lev[sl]; D = d[sl]; V = valid[sl]
    levels = np.unique(L)
    med = []
    for l in levels:
        m = (L == l) & V[:, 16]
        if m.any():
            med.append((l, float(np.median(D[m, 16, 2]))))
    med = np.array(med)
    lag = np.diff(med[:, 1])
    print(seg, "levels", len(levels), "lag per level us p10/50/90",
          np.percentile(lag, [10, 50, 90]).round(3).tolist(), "first/last", med[0], med[-1])
# one chain's tiles in detail
for i in (0, 1, 100, int(nf) // 2):
    nt = int(valid[i].sum())
    print(f"item {i} level {lev[i]}: wait", np.round((d[i, :8, 1] - d[i, :8, 0]), 2).tolist(),
          "compute", np.round((d[i, :8, 2] - d[i, :8, 1]), 2).tolist(),
          "period", np.round(np.diff(d[i, :9, 2]), 2).tolist())
# split the lag: producer publish (level l-1) -> consumer deps ready (level l) -> consumer publish
for seg, sl in (("fwd", slice(0, nf)),):
    L = lev[sl]; D = d[sl]; V = valid[sl]
    rows = []
    for l in np.unique(L):
        m = (L == l) & V[:, 16]
        if m.any():
            rows.append((l, np.median(D[m, 16, 0]), np.median(D[m, 16, 1]), np.median(D[m, 16, 2])))
    rows = np.array(rows)
    hop = rows[1:, 2] - rows[:-1, 3]   # deps ready(l) - published(l-1)
    car = rows[1:, 3] - rows[1:, 2]    # published(l) - deps ready(l)
    slot = rows[1:, 2] - rows[1:, 1]   # deps ready - slot ready
    print(seg, "detect-after-producer us p10/50/90", np.percentile(hop, [10, 50, 90]).round(3).tolist(),
          "carry us p50", float(np.median(car)), "deps wait after slot ready p50", float(np.median(slot)))
    early = rows[1:, 1] <= rows[:-1, 3]
    print("slot ready before producer published (fraction of levels)", float(early.mean()))
