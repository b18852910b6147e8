"""Summarise an `ncu -i X --page source --csv --print-source sass` dump: stall reasons, and
instruction / stall-sample shares grouped by execution count (loop bodies)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
ia, isrc = hdr.index("Address"), hdr.index("Source")
iall, iex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = collections.Counter()
for d in data:
    for r in reasons:
        tot[r] += float(d[hdr.index(r)] or 0)
S = sum(tot.values())
print("stall reasons (share of warp samples):")
for r, v in tot.most_common():
    if v > 0.002 * S:
        print(f"  {r:26s} {100 * v / S:5.1f}%")
g = collections.defaultdict(lambda: [0, 0, 0.0, None])
for d in data:
    e = int(d[iex] or 0)
    if e == 0:
        continue
    g[e][0] += 1
    g[e][1] += e
    g[e][2] += float(d[iall] or 0)
    g[e][3] = g[e][3] or d[isrc][:40]
ti = sum(v[1] for v in g.values())
ts = sum(v[2] for v in g.values())
print(f"instructions executed: {ti}; groups by execution count:")
for e, v in sorted(g.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    print(f"  exec {e:10d} x {v[0]:4d} instr  {100 * v[1] / ti:5.1f}% of instr  {100 * v[2] / ts:5.1f}% of samples  ({v[3]})")
