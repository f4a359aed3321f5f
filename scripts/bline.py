"""Summarise bench.py JSON lines (dev aid): python scripts/bline.py gpurun_out/b.log ..."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads([l for l in open(f).read().splitlines() if l.startswith("{")][-1])
    except Exception as e:
        print(f, "no line", e)
        continue
    s = d.get("secondary", {})
    nf = max(1, s.get("profiled_frames", 1))
    out = {"value": round(d["value"], 1), "single_p50": round(d["single_frame_latency_ms"]["p50"], 3),
           "frac": round(d.get("roofline", {}).get("frac", 0), 3),
           "fact_ms/f": round(d.get("roofline", {}).get("avg_launch_ms", 0) * d.get("roofline", {}).get("launches", 0) / nf, 3),
           "chain_ms/f": round(s.get("conflict_chain", {}).get("ms_per_frame", 0), 3),
           "tex_ms/f": round(s.get("texture_mlp", {}).get("ms", 0) / nf, 3),
           "tex_frac": round(s.get("texture_mlp", {}).get("frac_of_burst", 0), 3),
           "dense_ms/f": round(s.get("dense_passes", {}).get("ms", 0) / nf, 3),
           "render_ms/f": round(s.get("render", {}).get("ms", 0) / nf, 3),
           "evals": s.get("evals_per_frame"), "clk": (d.get("clocks") or {}).get("sm_mhz")}
    if d.get("e2e"):
        out["e2e"] = round(d["e2e"]["value"], 1)
    print(f, out)
