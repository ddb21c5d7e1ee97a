"""(The chain kernels record their timeline only in a build with -DSFG_CHAIN_TRACE=1:
bash scripts/build_alt.sh trace "-DSFG_CHAIN_TRACE=1", then SFG_LIB=old_lib/trace/libsfgpu.so.)
Effective hop inside the C5 chain executor (forward solve, natural-order
27-point grid): for every tile, the time from the last producer tile it
depends on ending to the consumer having summed all its terms.
Chain c is grid line (y, z) = (c % N, c // N)."""
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
carry = (w1 & ((1 << 22) - 1)).astype(np.float64) / 1965.0 * 1e3  # ns
end = d[:, :, 2].astype(np.int64)
valid = end > 0
item_of = {}
for i in range(nf):
    item_of[int(chain[i])] = i
hops, waits, carries, late = [], [], [], []
for i in range(nf):
    c = int(chain[i]); y, z = c % N, c // N
    L = int(lev[i]); sk = L % G
    deps = [(y - 1, z), (y - 1, z - 1), (y, z - 1), (y + 1, z - 1)]
    deps = [item_of[a + N * b] for a, b in deps if 0 <= a < N and 0 <= b < N]
    if not deps:
        continue
    nt = int(valid[i].sum())
    for t in range(nt):
        o_hi = min(N - 1, G * t - sk + G - 1)
        if o_hi < 0:
            continue
        need = min(N - 1, o_hi + 1)
        de = 0
        for j in deps:
            La = int(lev[j]); ta = (need + La % G) // G
            de = max(de, int(end[j, ta]))
        if entry[i, t] < de:  # consumer was waiting when the producer finished
            hops.append(ready[i, t] - de)
            carries.append(carry[i, t])
        else:
            late.append(entry[i, t] - de)
hops = np.array(hops); late = np.array(late)
print("tiles: consumer waiting %d, consumer late %d" % (hops.size, late.size))
print("producer end -> consumer summed (ns) p10/50/90:", np.percentile(hops, [10, 50, 90]).round())
print("consumer carry (ns) p10/50/90:", np.percentile(carries, [10, 50, 90]).round())
print("late consumers: entry after producer end by (ns) p10/50/90:", np.percentile(late, [10, 50, 90]).round() if late.size else None)
