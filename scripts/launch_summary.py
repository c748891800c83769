"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list (shares per kernel).

    python scripts/launch_summary.py gpurun_out/launches.csv > profiles/r01_launches_summary.txt
"""
import collections
import csv
import sys

path = sys.argv[1]
lines = [l for l in open(path) if l.startswith('"')]
rows = list(csv.reader(lines))
hdr = rows[0]
ki, mi, ui, vi = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    us = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    tot[r[ki]] += us
    cnt[r[ki]] += 1
all_us = sum(tot.values())
fill = sum(v for k, v in tot.items() if "fill_kernel" in k)
print("# launch list: ncu --metrics gpu__time_duration.sum --clock-control none -c 400")
print("# command: " + (sys.argv[2] if len(sys.argv) > 2 else "python bench.py --steps 2 --warmup 1 (scripts/profile_round.sh)")
      + "   (prod, V=152064, 1,008,179 rows/step, chunk 131072)")
print("# per-launch times are cold-cache and serialised: compare SHARES, not absolutes")
print("# share_of_all  share_excl_input_fill  launches  total_us  kernel")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    ex = "" if "fill_kernel" in k else f"{100 * v / (all_us - fill):7.2f}%"
    print(f"{100 * v / all_us:6.2f}%  {ex:>8s}  {cnt[k]:6d}  {v:12.1f}  {k[:90]}")
