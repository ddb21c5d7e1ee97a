import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_12238_b200 as sf
os.environ["SFG_EXECUTOR"] = "mline"
M = sf.config_matrix(1)
st = sf.make_state(1, M, seed=7).inspect()
for _ in range(4):
    st.execute_fused()
print(st.bench(3))
