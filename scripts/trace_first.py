"""(The chain kernels record their timeline only in a build with -DSFG_CHAIN_TRACE=1:
bash scripts/build_alt.sh trace "-DSFG_CHAIN_TRACE=1", then SFG_LIB=old_lib/trace/libsfgpu.so.)
C5 chain executor: where a level's lag goes, first tile vs a middle tile.
For every forward chain (27-point grid line (y, z)) and tile t in {0, 16}:
  hop   = consumer 'all words summed' - latest producer tile end it needs
  after = consumer tile end - consumer 'all words summed' (the carry)
  lag   = consumer tile end - latest producer tile end
  entry = consumer stage-D entry - latest producer tile end (< 0: it waited)
(SFG_TRACE timelines of k_chain_sm; globaltimer ns.)"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
out = "/tmp/trace.bin"
os.environ["SFG_TRACE"] = out
os.environ.setdefault("SFG_TRACE_TILES", "40")
import paper_2111_12238_b200 as sf
N = int(os.environ.get("C5_SIZE", "128"))
M, vals = sf.config5_systems(size=N, nsys=8)
st = sf.make_state(8, M, nsys=8, values=vals)
st.inspect()
for _ in range(3):
    st.execute_fused()
print("kernel ms", st.bench(1)[1])
st.close()
raw = np.fromfile(out, dtype=np.int64)
items, tiles, nf = (int(v) for v in raw[:3])
d = raw[3:3 + items * tiles * 3].view(np.uint64).reshape(items, tiles, 3)
lev = np.frombuffer(raw[3 + items * tiles * 3:].tobytes(), dtype=np.int32)[:items]
G = 4
entry = d[:, :, 0].astype(np.int64)
w1 = d[:, :, 1]
ready = entry + ((w1 >> 22) & ((1 << 22) - 1)).astype(np.int64)
chain = (w1 >> 44).astype(np.int64)[:, 0]
end = d[:, :, 2].astype(np.int64)
valid = end > 0
item_of = {int(chain[i]): i for i in range(nf)}
res = {0: [], 1: [], 16: []}
for i in range(nf):
    c = int(chain[i]); y, z = c % N, c // N
    L = int(lev[i]); sk = L % G
    deps = [(y - 1, z), (y - 1, z - 1), (y, z - 1), (y + 1, z - 1)]
    deps = [item_of[a + N * b] for a, b in deps if 0 <= a < N and 0 <= b < N]
    if not deps:
        continue
    for t in res:
        if not valid[i, t]:
            continue
        o_hi = min(N - 1, G * t - sk + G - 1)
        if o_hi < 0:
            continue
        need = min(N - 1, o_hi + 1)
        de, crit = 0, -1
        for j in deps:
            La = int(lev[j]); ta = (need + La % G) // G
            if end[j, ta] > de:
                de, crit = int(end[j, ta]), j
        res[t].append((ready[i, t] - de, end[i, t] - ready[i, t], end[i, t] - de, entry[i, t] - de,
                       int(lev[i]) - int(lev[crit])))
for t, r in res.items():
    a = np.array(r, dtype=np.float64)
    if not len(a):
        continue
    print(f"tile {t}: n={len(a)}")
    for k, name in enumerate(("hop (summed - producer end)", "after (end - summed)", "lag (end - producer end)",
                              "entry - producer end")):
        print(f"   {name:30s} ns p10/50/90 {np.percentile(a[:, k], [10, 50, 90]).round()}")
    print("   critical producer level diff: ", {int(v): int((a[:, 4] == v).sum()) for v in np.unique(a[:, 4])})
