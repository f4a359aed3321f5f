"""Summarise an ncu --metrics gpu__time_duration.sum launch-list CSV for the last frame (dev tool)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[hi]
data = [dict(zip(hdr, r)) for r in rows[hi + 1:] if len(r) == len(hdr)]
idx = max(i for i, d in enumerate(data) if "chw_to_hwc" in d["Kernel Name"])
tot, agg, cnt = 0.0, {}, {}
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 1e9
for d in data[idx:]:
    us = float(d["Metric Value"]) / 1e3
    tot += us
    nm = d["Kernel Name"].split("(")[0].replace("void ", "")[:44]
    agg[nm] = agg.get(nm, 0) + us
    cnt[nm] = cnt.get(nm, 0) + 1
    if us > thr:
        print(f"  {nm:46s} {d['Grid Size']:>16s} {us:9.1f}")
print(f"total {tot:.1f} us over {sum(cnt.values())} launches")
for k, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"  {k:46s} {v:9.1f} us  x{cnt[k]}")
