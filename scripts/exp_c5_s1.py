"""C5 (27-pt 128^3, combo 8) at one system: multi-line vs chain executors --
the critical path of the lane-per-chain scheme without the batch."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_12238_b200 as sf


def run(label, combo, M, **kw):
    st = sf.make_state(combo, M, seed=7, **kw).inspect()
    st.bench(3)
    tot, ker = st.bench(10)
    print(f"{label:34s} combo {combo}: {tot / 10:.3f} ms/exec (kernel {ker:.3f})", flush=True)
    st.close()


M5, vals = sf.config5_systems(nsys=8)
v1 = vals[:M5.nnz]
for ex in ("mline", "chain"):
    os.environ["SFG_EXECUTOR"] = ex
    run(f"C5 S=1 {ex}", 8, M5, nsys=1, values=v1)
    run(f"C5 S=1 {ex} fwd only(combo1)", 1, M5, nsys=1, values=v1)
for S in (2, 4):
    os.environ["SFG_EXECUTOR"] = "chain"
    run(f"C5 S={S} chain", 8, M5, nsys=S, values=vals[:S * M5.nnz])
