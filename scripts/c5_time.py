"""Config 5 fused time (ms per execution), the bench's inputs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_12238_b200 as sf
M, v = sf.config5_systems(nsys=8)
vin = __import__("numpy").concatenate([sf.gen_vector(M.n, 7 + s) for s in range(8)])
st = sf.make_state(8, M, seed=7, nsys=8, values=v, vin=vin).inspect()
st.bench(3)
t, k = st.bench(20)
print(os.environ.get("SFG_LIB", "in-tree"), round(t / 20, 3), "ms", flush=True)
