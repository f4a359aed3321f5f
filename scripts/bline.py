"""Print the headline numbers of a bench log (dev tool): python scripts/bline.py gpurun_out/b3.log"""
import json, sys
for f in sys.argv[1:]:
    d = json.loads([x for x in open(f) if x.startswith("{")][-1])
    c = d["config"]
    print(f, "value %.1f" % d["value"], "ms/step %.3f" % d["ms_per_step"], "single p50 %.3f" % c["single_frame_latency_ms"]["p50"],
          "e2e %.1f" % d["e2e"]["value"], "fact_frac %.3f" % d["roofline"].get("executed_frac", 0),
          "clk", d["clocks"]["sm_mhz"])
