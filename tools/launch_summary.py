"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python tools/launch_summary.py gpurun_out/launches_bench.csv
"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
head = next(r for r in rows if "Kernel Name" in r)
body = rows[rows.index(head) + 1:]
ik, im, iv = head.index("Kernel Name"), head.index("Metric Name"), head.index("Metric Value")
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in body:
    if len(r) > iv and r[im] == "gpu__time_duration.sum":
        v = float(r[iv].replace(",", ""))
        unit = r[head.index("Metric Unit")] if "Metric Unit" in head else "ns"
        us = v / 1000 if unit in ("nsecond", "ns") else v if unit in ("usecond", "us") else v * 1000
        tot[r[ik]] += us
        cnt[r[ik]] += 1
all_us = sum(tot.values())
print(f"{'launches':>8} {'total_us':>9} {'share':>6} {'avg_us':>7}  kernel")
for k, us in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{cnt[k]:8d} {us:9.1f} {us / all_us:6.1%} {us / cnt[k]:7.1f}  {k[:100]}")
