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
