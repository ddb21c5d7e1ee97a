"""Timeline of the lockstep executor (lock.cu) on C5 from SFG_TRACE: per
chain level the end of step 0, the per-level lag, the in-chain step period,
the re-poll rounds per step and the wait-entry -> step-end time."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
out = "/tmp/trace_lock.bin"
os.environ["SFG_TRACE"] = out
os.environ.setdefault("SFG_TRACE_TILES", "33")
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
d = raw[3:3 + items * tiles * 3].reshape(items, tiles, 3)
lev = np.frombuffer(raw[3 + items * tiles * 3:].tobytes(), dtype=np.int32)[:items]
ent, rnd, end = d[:, :, 0], d[:, :, 1] & 0xFFFF, d[:, :, 2]
ck = [(d[:, :, 1] >> sh) & 0xFFFF for sh in (16, 32, 48)]
valid = end > 0
t0 = end[valid].min()
print("launch span us", (end[valid].max() - t0) / 1e3)
for part, sl in (("fwd", slice(0, nf)), ("bwd", slice(nf, items))):
    L, E, EN, R, V = lev[sl], (end[sl] - t0) / 1e3, (ent[sl] - t0) / 1e3, rnd[sl], valid[sl]
    nt = V.sum(1)
    print(f"{part}: items {E.shape[0]} levels {L.min()}..{L.max()} span {E[V].min():.1f}..{E[V].max():.1f} us")
    rows = []
    for l in range(L.min(), L.max() + 1):
        m = (L == l) & (nt > 0)
        if m.any():
            last = np.array([E[i, nt[i] - 1] for i in np.nonzero(m)[0]])
            rows.append((l, m.sum(), np.median(E[m, 0]), np.median(last)))
    rows = np.array(rows)
    for r in rows[::max(1, len(rows) // 20)]:
        print("  L=%4d items=%3d step0 end %8.1f  last sampled end %8.1f" % tuple(r))
    lag = np.diff(rows[:, 2]) / np.diff(rows[:, 0])
    print("  per-level lag (step-0 end): median %.2f mean %.2f us" % (np.median(lag), lag.mean()))
    per = np.concatenate([np.diff(E[i, :nt[i]]) for i in range(E.shape[0]) if nt[i] > 1]) / 4
    print("  step period us p10/50/90/mean", np.percentile(per, [10, 50, 90]).round(3), per.mean().round(3))
    print("  re-poll rounds per sampled step: mean %.2f, zero %.0f%%, p90 %d" %
          (R[V].mean(), 100 * (R[V] == 0).mean(), np.percentile(R[V], 90)))
    w = (E - EN)[V]
    print("  wait entry -> step end us p10/50/90", np.percentile(w, [10, 50, 90]).round(3))
    w0 = (E - EN)[V & (R == 0)]
    if w0.size:
        print("  same, steps without re-poll p10/50/90", np.percentile(w0, [10, 50, 90]).round(3))
    for name, k in (("copy wait", 0), ("wait end -> published", 1), ("published -> body end", 2)):
        print("  cycles", name, "p10/50/90", np.percentile(ck[k][sl][V], [10, 50, 90]))
    l1 = np.nonzero((L == L.min()) & (nt > 1))[0]
    if l1.size:
        i = l1[0]
        print("  first-level item cycles (wait, compute, rest):", [ck[k][sl][i, 1:6].tolist() for k in range(3)])
    if l1.size:
        i = l1[0]
        print("  first-level item: step period", (np.diff(E[i, :nt[i]]) / 4).round(3)[:12])
