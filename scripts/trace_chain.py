"""(The chain kernels record their timeline only in a build with -DSFG_CHAIN_TRACE=1:
bash scripts/build_alt.sh trace "-DSFG_CHAIN_TRACE=1", then SFG_LIB=old_lib/trace/libsfgpu.so.)
Runs one traced execution of a config on the GPU and summarises the
chain executor's timeline (diagnostics; SFG_TRACE)."""
import os, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_12238_b200 as sf

cfg = int(sys.argv[1]); size = int(sys.argv[2]) if len(sys.argv) > 2 else None
out = sys.argv[3] if len(sys.argv) > 3 else "gpurun_out/trace.bin"
os.environ["SFG_TRACE"] = out
if cfg == 5:
    M, vals = sf.config5_systems(size=size, nsys=8)
    st = sf.make_state(8, M, nsys=8, values=vals)
else:
    M = sf.config_matrix(cfg, size=size)
    st = sf.make_state({1: 4}[cfg], M)
st.inspect()
for _ in range(3):
    st.execute_fused()
tot, ker = st.bench(1)
print("kernel ms", ker)
st.close()
raw = np.fromfile(out, dtype=np.int64)
items, tiles, nf = raw[:3]
d = raw[3:3 + items * tiles * 3].view(np.uint64).reshape(items, tiles, 3).astype(np.float64)
valid = d[:, :, 2] > 0
t0 = d[valid][:, 0].min()
d = (d - t0) / 1e3  # us
claim = np.where(valid.any(1), d[:, 0, 0], np.nan)
first_part = d[:, 0, 1]
ntiles = valid.sum(1)
end = np.array([d[i, ntiles[i] - 1, 2] if ntiles[i] else np.nan for i in range(items)])
tile_wait = (d[:, 1:, 1] - d[:, :-1, 2])[valid[:, 1:]]
carry = (d[:, :, 2] - d[:, :, 1])[valid]
print(json.dumps({
    "items": int(items), "fwd_items": int(nf), "span_us": float(np.nanmax(end)),
    "claim_us_p50": float(np.nanmedian(np.diff(np.sort(claim)))),
    "chain_duration_us_p50": float(np.nanmedian(end - claim)),
    "first_partial_wait_us_p50": float(np.nanmedian(first_part - claim)),
    "tile_partial_us_p50": float(np.median(tile_wait)), "tile_partial_us_p90": float(np.percentile(tile_wait, 90)),
    "carry_us_p50": float(np.median(carry)), "carry_us_p90": float(np.percentile(carry, 90)),
    "concurrent_chains_p50": float(np.median([((claim <= t) & (end >= t)).sum() for t in np.linspace(0, np.nanmax(end), 200)])),
}, indent=1))
# progress of fwd items in claim order: end time vs item index
for q in (0.1, 0.25, 0.5, 0.75, 0.9, 1.0):
    i = min(items - 1, int(q * nf))
    print("fwd item", i, "claim", round(claim[i], 1), "end", round(end[i], 1))
# per-tile completion times of a few chains (in claim order)
for i in [0, 1, 2, 3, 10, 100, int(nf) // 2]:
    if i >= items:
        continue
    nt = int(ntiles[i])
    ends = d[i, :nt, 2]
    parts = d[i, :nt, 1]
    print(f"item {i}: claim {claim[i]:.1f} tiles {nt} first ends", np.round(ends[:6], 2).tolist(),
          "partial->end", np.round((ends - parts)[:6], 2).tolist(), "last end", round(float(ends[-1]), 1) if nt else None)
