"""Print the last `k` launches of an ncu launch-list CSV (one solver iteration) with
durations (dev tool). Usage: python tools/iter_kernels.py launches.csv [k]"""
import csv
import sys

path = sys.argv[1]
k = int(sys.argv[2]) if len(sys.argv) > 2 else 30
rows = [r for r in csv.reader(open(path)) if r]
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
ks = [(r[ki].split("(")[0][:70], float(r[vi].replace(",", "")) * (1e-3 if r[ui].startswith("n") else 1.0))
      for r in rows[hi + 1:]]
tot = 0.0
for name, us in ks[-k:]:
    print(f"{us:9.2f} us  {name}")
    tot += us
print(f"sum {tot:.1f} us over {min(k, len(ks))} launches")
