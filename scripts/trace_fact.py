"""(The warp executors record their timeline only in a build with -DSFG_FACT_TRACE=1:
bash scripts/build_alt.sh trace "-DSFG_FACT_TRACE=1", then SFG_LIB=old_lib/trace/libsfgpu.so.)
Per-level timing of the factorization warp executors (configs 2, 3, 4)
from SFG_TRACE: per task {start, summed, factor published, solve published}."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
out = "/tmp/ftrace.bin"
os.environ["SFG_TRACE"] = out
import paper_2111_12238_b200 as sf
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
combo = {2: 5, 3: 6, 4: 7}[cfg]
M = sf.config_matrix(cfg)
st = sf.make_state(combo, M, seed=7).inspect()
for _ in range(3):
    st.execute_fused()
print("config", cfg, "kernel ms", st.bench(1)[1])
lev1 = st.level_info(1).level.astype(np.int64)  # kernel-1 DAG levels (1-based)
st.close()
raw = np.fromfile(out, dtype=np.int64)
items = int(raw[0])
d = raw[3:3 + items * 5].view(np.uint64).reshape(items, 5).astype(np.int64)
task, start, summed, facp, solp = d.T
ok = start > 0
t0 = start[ok].min()
start, summed, facp = (start - t0) / 1e3, (summed - t0) / 1e3, (facp - t0) / 1e3
solp = np.where(solp > 0, (solp - t0) / 1e3, np.nan)
L = lev1[task]
print("tasks", items, "levels", L.min(), L.max())
print("task phases (us) p10/50/90: start->summed", np.percentile(summed - start, [10, 50, 90]).round(2),
      " summed->fac published", np.percentile(facp - summed, [10, 50, 90]).round(2))
if np.isfinite(solp).any():
    print("  fac published -> solve published", np.nanpercentile(solp - facp, [10, 50, 90]).round(2))
rows = []
for l in range(L.min(), L.max() + 1):
    m = L == l
    if m.any():
        rows.append((l, m.sum(), np.median(start[m]), np.median(summed[m]), np.max(facp[m]),
                     np.nanmax(solp[m]) if np.isfinite(solp[m]).any() else np.nan))
rows = np.array(rows)
for r in rows[::max(1, len(rows) // 12)]:
    print("  L=%5d n=%5d start med %8.1f summed med %8.1f fac max %8.1f solve max %8.1f" % tuple(r))
print("per-level lag: fac-published max %.2f us, solve max %.2f us" % (
    np.median(np.diff(rows[:, 4])), np.nanmedian(np.diff(rows[:, 5]))))
# how early were tasks claimed relative to when their inputs were ready
print("start -> summed (waiting) by level band:", [round(float(np.median((summed - start)[(L >= a) & (L < a + 20)])), 2)
                                                     for a in range(int(L.min()), int(L.max()), max(1, int(L.max()) // 8))])
