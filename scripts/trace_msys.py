"""k_msys timeline: per work item (group, system pair) claim / first step /
end (us) and cycles in cp.async waits and re-polls."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_12238_b200 as sf
size = int(sys.argv[1]) if len(sys.argv) > 1 else 24
S = int(sys.argv[2]) if len(sys.argv) > 2 else 2
combo = int(sys.argv[3]) if len(sys.argv) > 3 else 1
out = "/tmp/mstrace.bin"
os.environ["SFG_TRACE"] = out
os.environ["SFG_EXECUTOR"] = "msys"
os.environ["SFG_MLINE_STATS"] = "1"
M5, vals = sf.config5_systems(size=size, nsys=S)
st = sf.make_state(combo, M5, seed=7, nsys=S, values=vals).inspect()
for _ in range(3):
    st.execute_fused()
print("kernel ms", st.bench(1)[1])
st.close()
raw = np.fromfile(out, dtype=np.int64)
items, w, nf = raw[:3]
d = raw[3:3 + items * 4].view(np.uint64).reshape(items, 4)
t0 = d[:, 0].min()
tt = (d[:, :3].astype(np.int64) - int(t0)) / 1e3
polls = (d[:, 3] & 0xffffffff).astype(np.int64)
dur = tt[:, 2] - tt[:, 1]
print(f"items {items}: mean dur {dur.mean():.1f} us  min {dur.min():.1f} max {dur.max():.1f}  "
      f"mean polled steps {polls.mean():.1f}")
for i in list(range(0, items, max(1, items // 40))) + [items - 1]:
    c, f, e = tt[i]
    print(f"item {i:5d}: claim {c:8.1f} first {f:8.1f} end {e:8.1f} dur {e - f:7.1f} polled_steps {polls[i]}")
# concurrency profile
ts = np.linspace(0, tt[:, 2].max(), 20)
act = [int(((tt[:, 1] <= x) & (tt[:, 2] > x)).sum()) for x in ts]
print("active items over time:", act)
