"""One-line summary of a bench.py JSON line read from stdin (dev tool): tag value latency."""
import json, sys
line = [l for l in sys.stdin.read().splitlines() if l.startswith("{")][-1]
d = json.loads(line)
c = d["config"]
print(sys.argv[1] if len(sys.argv) > 1 else "", "value %.1f" % d["value"], "single-frame p50 %.3f ms" % c["single_frame_latency_ms"]["p50"],
      "in-flight p50 %.2f ms" % c["frame_latency_ms"]["p50"], "e2e", (d.get("e2e") or {}).get("value"))
