"""Configs 2-4 (factorization pairs) and config 1: ms per fused execution."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_12238_b200 as sf
COMBO = {1: 4, 2: 5, 3: 6, 4: 7}
for cfg in [int(a) for a in (sys.argv[1:] or ["2", "3", "4", "1"])]:
    M = sf.config_matrix(cfg)
    st = sf.make_state(COMBO[cfg], M, seed=7).inspect()
    st.bench(3)
    tot, ker = st.bench(20)
    ut, uk = st.bench(10, unfused=True)
    print(f"config {cfg} (combo {COMBO[cfg]}): fused {tot / 20:.3f} ms  unfused {ut / 10:.3f} ms", flush=True)
    st.close()
