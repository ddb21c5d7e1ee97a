"""PCG timing probe on the config-2 matrix: per-iteration time at check
intervals 1 and 10, and the fused preconditioner solve (combo 8, 1 system) alone."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_12238_b200 as sf
M = sf.config_matrix(2)
b = sf.gen_vector(M.n, 7)
pcg = sf.PCG(M)
for check in (1, 10, 25):
    pcg.solve(b, rtol=1e-10, maxit=1000, check=check)
    x, it, rr, ms = pcg.solve(b, rtol=1e-10, maxit=1000, check=check)
    print(f"check={check}: {it} iterations, relres {rr:.2e}, {ms:.3f} ms, {ms / it:.4f} ms/iteration")
pcg.close()
# the preconditioner's fused pair alone: combo 8 on the IC0 factor of the same matrix
st5 = sf.make_state(5, M, seed=7).inspect()
st5.execute_fused()
fac = st5.collect_outputs()[:st5.output_len - M.n] if hasattr(st5, "output_len") else None
st5.close()
st8 = sf.make_state(8, M, seed=7).inspect()
st8.bench(3)
tot, ker = st8.bench(50)
print(f"combo 8 (1 system, config-2 pattern) fused: {tot / 50:.4f} ms per execution, kernel {ker:.4f} ms")
st8.close()
