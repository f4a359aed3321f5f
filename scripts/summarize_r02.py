"""Summaries of the round-2 ncu outputs for profiles/ (dev tool):
python scripts/summarize_r02.py gpurun_out profiles [tag]"""
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from summarize_ncu import launch_summary  # noqa: E402

KEYS = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic"]


def full(path, top=3):
    rows = list(csv.reader(open(path)))
    if len(rows) < 3:
        return []
    hdr, units, data = rows[0], rows[1], rows[2:]
    t = hdr.index("gpu__time_duration.sum")
    data.sort(key=lambda d: -float(d[t].replace(",", "")))
    out = []
    for d in data[:top]:
        rec = {k: d[hdr.index(k)] + (" " + units[hdr.index(k)] if units[hdr.index(k)] else "") for k in KEYS if k in hdr}
        stalls = sorted(((k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
                          float(d[hdr.index(k)].replace(",", "")))
                         for k in hdr if k.startswith("smsp__average_warps_issue_stalled_")
                         and k.endswith("_per_issue_active.ratio")), key=lambda x: -x[1])[:6]
        rec["top_stalls_per_issue"] = {k: round(v, 3) for k, v in stalls}
        rec["launches_captured"] = len(data)
        out.append(rec)
    return out


def main(src, dst, tag="r02"):
    for c in ("config2", "config3"):
        p = os.path.join(src, f"{tag}_launches_{c}.csv")
        if os.path.exists(p):
            json.dump(launch_summary(p), open(os.path.join(dst, f"{tag}_launch_summary_{c}.json"), "w"), indent=1)
        for k in ("k_fact2", "k_mlp_pair", "k_tail", "k_fine_rows", "k_render", "k_conflict_expand", "k_layer",
                  "k_cols", "k_gather", "k_mixed_words", "k_coarse_bits4", "k_xline_extents", "k_chw_to_hwc64"):
            p = os.path.join(src, f"{tag}_raw_{k}_{c}.csv")
            if os.path.exists(p):
                json.dump(full(p), open(os.path.join(dst, f"{tag}_ncu_full_{k}_{c}.json"), "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], *(sys.argv[3:4]))
