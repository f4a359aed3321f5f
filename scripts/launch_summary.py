"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel (dev tool):
python scripts/launch_summary.py gpurun_out/launches.csv [frames]"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
frames = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
tot, cnt = collections.Counter(), collections.Counter()
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0].replace("void ", "")
    tot[name] += float(r[vi]) / 1e3
    cnt[name] += 1
T = sum(tot.values())
print(f"total {T / frames:.1f} us per frame, {sum(cnt.values()) / frames:.0f} launches")
for k, v in tot.most_common(25):
    print(f"{v / frames:9.1f} us  {v / T:6.3f}  {cnt[k] / frames:5.1f}x  {k}")
