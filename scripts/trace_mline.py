"""(k_mline1 records its timeline only in a build with -DSFG_ML1_TRACE=1:
bash scripts/build_alt.sh ml1trace "-DSFG_ML1_TRACE=1", then SFG_LIB=old_lib/ml1trace/libsfgpu.so.)
Timeline of the multi-chain executor (SFG_TRACE diagnostics): group
durations, step times and where the steps stall."""
import os, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_12238_b200 as sf
out = "/tmp/mtrace.bin"
os.environ["SFG_TRACE"] = out
os.environ["SFG_MLINE_STATS"] = "1"
nsys = int(sys.argv[1]) if len(sys.argv) > 1 else 8
M, vals = sf.config5_systems(nsys=nsys)
st = sf.make_state(8, M, nsys=nsys, values=vals)
st.inspect()
for _ in range(3):
    st.execute_fused()
print("kernel ms", st.bench(1)[1])
st.close()
raw = np.fromfile(out, dtype=np.int64)
items, w, nf = raw[:3]
d = raw[3:3 + items * 4].view(np.uint64).reshape(items, 4)
t0 = d[:, 0].min()
claim = (d[:, 0] - t0) / 1e3
first = (d[:, 1] - t0) / 1e3
end = (d[:, 2] - t0) / 1e3
waitc = (d[:, 3] >> 32).astype(np.float64)
pollc = (d[:, 3] & 0xffffffff).astype(np.float64)
dur = end - first
print(json.dumps({
  "items": int(items), "fwd": int(nf), "span_us": float(end.max()),
  "fwd_end_us": float(end[:nf].max()), "bwd_first_claim_us": float(claim[nf:].min()),
  "group_dur_us_p10_50_90": np.percentile(dur, [10, 50, 90]).round(1).tolist(),
  "prologue_us_p50": float(np.median(first - claim)),
  "wait_cycles_per_group_p50": float(np.median(waitc)), "poll_cycles_per_group_p50": float(np.median(pollc)),
}, indent=1))
order = np.argsort(claim[:nf])
for q in (0, 0.1, 0.25, 0.5, 0.75, 0.9, 0.99):
    i = order[min(int(q * nf), nf - 1)]
    print(f"fwd q{q}: claim {claim[i]:.1f} first {first[i]:.1f} end {end[i]:.1f} dur {dur[i]:.1f} wait {waitc[i]:.0f} poll {pollc[i]:.0f}")
for i in [0, 1, 2, 3, 4, 8, 16, 32, 64, 128, 1000, 2000, 4000]:
    if i < items:
        print(f"item {i}: claim {claim[i]:.1f} first {first[i]:.1f} end {end[i]:.1f} dur {dur[i]:.1f} wait {waitc[i]:.0f} poll {pollc[i]:.0f}")
