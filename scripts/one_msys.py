"""One k_msys execution (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_12238_b200 as sf
size = int(sys.argv[1]) if len(sys.argv) > 1 else 24
S = int(sys.argv[2]) if len(sys.argv) > 2 else 2
combo = int(sys.argv[3]) if len(sys.argv) > 3 else 1
os.environ["SFG_EXECUTOR"] = os.environ.get("SFG_EXECUTOR", "msys")
M5, vals = sf.config5_systems(size=size, nsys=S)
st = sf.make_state(combo, M5, seed=7, nsys=S, values=vals).inspect()
for _ in range(2):
    st.execute_fused()
st.synchronize()
print("ok", st.bench(3))
