"""C1 and C5 matrices under the chain and multi-line executors (diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2111_12238_b200 as sf
M = sf.config_matrix(1)
def run(label, combo, M, **kw):
    st = sf.make_state(combo, M, seed=7, **kw).inspect()
    st.bench(3)
    tot, ker = st.bench(10)
    print(f"{label:28s} combo {combo}: {tot / 10:.3f} ms/exec (kernel {ker:.3f})", flush=True)
    st.close()
os.environ["SFG_EXECUTOR"] = "mline"
for dx in ("2", "4"):
    os.environ["SFG_MLINE_DX"] = dx
    run(f"C1 mline dx={dx}", 1, M)
M5, vals = sf.config5_systems(nsys=8)
for dx in ("2", "4"):
    os.environ["SFG_MLINE_DX"] = dx
    run(f"C5 mline dx={dx}", 8, M5, nsys=8, values=vals)
os.environ["SFG_EXECUTOR"] = "chain"
run("C5 chain", 8, M5, nsys=8, values=vals)
