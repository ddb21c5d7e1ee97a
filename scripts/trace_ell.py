"""Timeline of the chain-ELL executor (SFG_TRACE): per-level lag and tile
period, to locate the critical path (diagnostics only)."""
import os, sys, json
import numpy as np
import warnings
warnings.filterwarnings('ignore')
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_12238_b200 as sf
out = "/tmp/trace_ell.bin"
os.environ["SFG_TRACE"] = out
os.environ.setdefault("SFG_TRACE_TILES", "40")
size = int(sys.argv[1]) if len(sys.argv) > 1 else None
M, vals = sf.config5_systems(size=size, nsys=8)
st = sf.make_state(8, M, nsys=8, values=vals)
st.inspect()
for _ in range(3):
    st.execute_fused()
print("kernel ms", st.bench(1)[1])
st.close()
raw = np.fromfile(out, dtype=np.uint8)
hdr = raw[:24].view(np.int64)
items, tiles, nf = (int(x) for x in hdr)
data = raw[24:24 + items * tiles * 8].view(np.uint64).reshape(items, tiles).astype(np.float64)
lev = raw[24 + items * tiles * 3 * 8:].view(np.int32)[:items]
G = 4
valid = data > 0
t0 = data[valid].min()
T = np.where(valid, (data - t0) / 1e3, np.nan)
for seg, lo, hi in (("fwd", 0, nf), ("bwd", nf, items)):
    L = lev[lo:hi]
    TT = T[lo:hi]
    nL = L.max()
    # absolute tile index A = u + L // G
    maxA = tiles + nL // G + 1
    acc = np.full((nL + 1, maxA), np.nan)
    for l in range(1, nL + 1):
        rows = TT[L == l]
        if rows.size == 0:
            continue
        sh = l // G
        m = np.nanmean(rows, axis=0)
        acc[l, sh:sh + tiles] = m[:maxA - sh]
    lag = np.nanmean(np.diff(acc, axis=0), axis=1)
    period = np.nanmedian(np.diff(TT, axis=1))
    end = np.nanmax(TT, axis=1)
    start = TT[:, 0]
    print(seg, json.dumps({"levels": int(nL), "span_us": float(np.nanmax(TT) - np.nanmin(TT)),
                           "lag_us_p50": float(np.nanmedian(lag)), "lag_us_mean": float(np.nanmean(lag)),
                           "tile_period_us_p50": float(period),
                           "chain_us_p50": float(np.nanmedian(end - start)),
                           "first_tile_vs_level_us": [round(float(np.nanmean(start[L == l])), 1) for l in (1, 2, 10, 50, 100, 200, 300, nL)]}))
