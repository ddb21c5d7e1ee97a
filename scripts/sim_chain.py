"""Discrete-event model of the C5 chain executor (forward solve, 27-point 128^3,
chains = grid lines of 4-row tiles): tile end = max(previous tile end + gap +
wait, latest producer tile end + hop) + carry, each phase log-normal with the
given coefficient of variation.  usage: sim_chain.py gap wait carry hop cv (us)"""
import numpy as np, sys
N=128; G=4
gap, w0, carry, hop, cv = [float(v) for v in sys.argv[1:6]]
rng=np.random.default_rng(1)
def smp(m): return m*np.exp(rng.normal(0, cv)) / np.exp(cv*cv/2)
end = {}
order = sorted([(y+2*z, y, z) for y in range(N) for z in range(N)])
tot=0
def tile_of(L, o): return (o + L % G) // G
for _, y, z in order:
    L = y + 2*z + 1; sk = L % G; nt = (N + sk + G - 1) // G
    deps = [(a,b) for a,b in [(y-1,z),(y-1,z-1),(y,z-1),(y+1,z-1)] if 0 <= a < N and 0 <= b < N]
    E = np.zeros(nt); prev = 0.0
    for t in range(nt):
        o_hi = min(N-1, G*t - sk + G - 1); hi = min(N-1, o_hi + 1)
        ready = max([end[(a,b)][tile_of(a+2*b+1, hi)] for a,b in deps], default=-1e9)
        ok = max(prev + smp(gap) + smp(w0), ready + smp(hop))
        E[t] = ok + smp(carry); prev = E[t]
    end[(y,z)] = E; tot = max(tot, E[-1])
print("cv",cv,"sim per solve us", round(tot,1), " per level", round(tot/382,2))
