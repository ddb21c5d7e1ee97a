"""k_msys (lane-per-chain, system pairs) vs the chain executor on C5: parity
of the outputs and time per execution."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2111_12238_b200 as sf

size = int(sys.argv[1]) if len(sys.argv) > 1 else 128
sizes = [int(a) for a in sys.argv[2].split(",")] if len(sys.argv) > 2 else [8, 2, 4]


def run(ex, combo, M, **kw):
    if ex:
        os.environ["SFG_EXECUTOR"] = ex
    else:
        os.environ.pop("SFG_EXECUTOR", None)
    st = sf.make_state(combo, M, seed=7, **kw).inspect()
    st.execute_fused()
    out = st.collect_outputs()
    st.bench(3)
    tot, ker = st.bench(10)
    st.close()
    return out, tot / 10


for S in sizes:
    M5, vals = sf.config5_systems(size=size, nsys=S)
    for combo in (8, 1):
        ref, t_ref = run(None, combo, M5, nsys=S, values=vals)
        got, t = run("msys", combo, M5, nsys=S, values=vals)
        print(f"S={S} combo {combo}: chain {t_ref:.3f} ms  msys {t:.3f} ms  "
              f"equal={np.array_equal(ref, got)}", flush=True)
