"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) into a per-kernel table.
Usage: python tools/launch_summary.py launches.csv "command" > summary.md"""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
cmd = sys.argv[2] if len(sys.argv) > 2 else ""
rows = [r for r in csv.reader(open(path)) if r]
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
unit_i = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
agg = defaultdict(lambda: [0, 0.0])
for r in rows[hdr_i + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    unit = r[unit_i] if unit_i is not None else "nsecond"
    ms = v / 1e6 if unit.startswith("n") else (v / 1e3 if unit.startswith("u") else v)
    name = r[ki].split("(")[0] if r[ki].startswith("sknr::k_") else r[ki]
    agg[name][0] += 1
    agg[name][1] += ms
total = sum(v[1] for v in agg.values())
print("# Launch list (ncu --metrics gpu__time_duration.sum --clock-control none)\n")
print(f"Command: `{cmd}`. Times are ncu's serialised per-launch durations (cold-cache); compare shares, "
      "not absolutes.\n")
print("| kernel | launches | total ms | share | avg us |\n|---|---|---|---|---|")
for name, (cnt, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"| `{name}` | {cnt} | {ms:.3f} | {100 * ms / total:.1f}% | {1000 * ms / cnt:.1f} |")
