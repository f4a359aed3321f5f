"""Summaries of ncu outputs for profiles/ (dev tool)."""
import csv, collections, json, subprocess, sys

def launch_summary(path, frame_marker="chw_to_hwc"):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    data = [dict(zip(hdr, r)) for r in rows[hi + 1:] if len(r) == len(hdr)]
    idx = max(i for i, d in enumerate(data) if frame_marker in d["Kernel Name"])
    last = data[idx:]
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for d in last:
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        tot[name] += float(d["Metric Value"]) / 1e3
        cnt[name] += 1
    total = sum(tot.values())
    return {"frame_total_us": total, "launches": len(last),
            "kernels": [{"kernel": k, "us": round(v, 1), "share": round(v / total, 4), "launches": cnt[k]}
                        for k, v in sorted(tot.items(), key=lambda x: -x[1])]}

def full_summary(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    keys = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
            "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
            "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"]
    res = []
    for d in data:
        res.append({k: (d[hdr.index(k)] + (" " + units[hdr.index(k)] if units[hdr.index(k)] else "")) for k in keys if k in hdr})
    return res

if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    print(json.dumps(launch_summary(path) if kind == "launches" else full_summary(path), indent=1))
