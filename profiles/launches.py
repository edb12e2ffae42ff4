"""Summarise an ncu --metrics gpu__time_duration.sum CSV: the last lockstep's kernels."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
gi = hdr.index("Grid Size")
seq = [(int(r[ii]), r[ki].split("(")[0][:48], float(r[vi].replace(",", "")) / 1e3, r[gi])
       for r in rows[h + 1:] if r[mi] == "gpu__time_duration.sum"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 16
tot = sum(s[2] for s in seq[-n:])
for s in seq[-n:]:
    print(f"{s[0]:5d} {s[1]:48s} {s[2]:8.1f} us {100 * s[2] / tot:5.1f}%  grid {s[3]}")
print(f"total {tot:.1f} us over the last {n} launches")

if "--by-name" in sys.argv:
    # share of every kernel name over the whole capture (the bench's launch list)
    agg = {}
    for s in seq:
        a = agg.setdefault(s[1], [0, 0.0])
        a[0] += 1
        a[1] += s[2]
    allt = sum(a[1] for a in agg.values())
    print(f"\nby kernel over all {len(seq)} launches ({allt / 1e3:.2f} ms):")
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"  {k:48s} {c:6d} launches {t / 1e3:9.3f} ms {100 * t / allt:5.1f}%")
