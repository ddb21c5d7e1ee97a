"""Isolated step time of the lockstep kernel: C5 pattern at a small size run by
ONE warp (SFG_LOCK_GRID=1 with a 1-warp build), so no item ever waits."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SFG_LOCK_GRID"] = "1"
import paper_2111_12238_b200 as sf
size = int(os.environ.get("C5_SIZE", "32"))
M, vals = sf.config5_systems(size=size, nsys=8)
st = sf.make_state(8, M, nsys=8, values=vals)
st.inspect()
for _ in range(2):
    st.execute_fused()
ms = st.bench(3)[1]
rows = 2 * M.n
print("size %d kernel ms %.3f  rows/4 per warp-step -> us per step %.3f" % (size, ms, ms * 1e3 / (rows / 4)))
