"""Per-source-line instruction counts and stall samples of one kernel from
an ncu report: joins `ncu --page source --print-source sass --csv` (per SASS
address) with `nvdisasm -g` line info of the cubin.
usage: sass_lines.py SASS_CSV NVDISASM_G_OUTPUT KERNEL_SUBSTR SOURCE_FILE [N]"""
import collections
import csv
import re
import sys

sass_csv, disasm, kname, srcfile = sys.argv[1:5]
N = int(sys.argv[5]) if len(sys.argv) > 5 else 40
txt = open(disasm).read().split('\n')
start = next(i for i, l in enumerate(txt) if l.strip().startswith('.section') and '.text.' in l and kname in l)
line, addr2line = None, {}
base = srcfile.split('/')[-1]
for l in txt[start + 1:]:
    if l.strip().startswith('.section') and '.text.' in l:
        break
    m = re.search(r'//## File "(.*)", line (\d+)', l)
    if m:
        line = int(m.group(2)) if m.group(1).endswith(base) else -int(m.group(2))
        continue
    m = re.search(r'/\*([0-9a-f]{4,})\*/', l)
    if m and line is not None:
        addr2line[int(m.group(1), 16)] = line
rows = list(csv.reader(open(sass_csv)))
h = rows[1]
ia, ie = h.index('Address'), h.index('Instructions Executed')
iss = h.index('Warp Stall Sampling (All Samples)')
addrs = []
for r in rows[2:]:
    try:
        addrs.append((int(r[ia], 16), float(r[ie] or 0), float(r[iss] or 0)))
    except (ValueError, IndexError):
        pass
a0 = min(a for a, _, _ in addrs)
cnt, smp = collections.Counter(), collections.Counter()
for a, e, s in addrs:
    ln = addr2line.get(a - a0, 0)
    cnt[ln] += e
    smp[ln] += s
src = open(srcfile).read().split('\n')
tot, tsm = sum(cnt.values()), sum(smp.values())
print(f"total instructions {tot/1e6:.1f}M, stall samples {tsm:.0f}")
for ln, e in sorted(cnt.items(), key=lambda x: -x[1])[:N]:
    text = src[ln - 1].strip()[:80] if ln > 0 else ('(other file line %d)' % -ln if ln < 0 else '?')
    print(f"{ln:5d} {e/1e6:8.1f}M {100*e/tot:5.1f}% smp {100*smp[ln]/tsm:5.1f}%  {text}")
