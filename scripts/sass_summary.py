"""Per-kernel SASS instruction summary of the built library (dev tool; the tcgen05 / TMA
mnemonics prove the tensor-core path):  python scripts/sass_summary.py > profiles/r02_sass_summary.json"""
import collections
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["UTCHMMA", "UTCBAR", "UTMALDG", "UTMASTG", "UTMAPF", "UBLKCP", "UBLKPF", "LDTM", "STTM", "UTCATOMSWS", "SYNCS", "MEMBAR", "HMMA", "DFMA",
        "FFMA", "LDG", "STG", "LDS", "STS", "ATOMG", "RED", "SHFL"]

txt = subprocess.run(["cuobjdump", "-sass", os.path.join(ROOT, "paper_2007_13988_b200", "libisocull_b200.so")],
                     capture_output=True, text=True).stdout
out = {}
for f in re.split(r"\n\s*Function : ", txt)[1:]:
    name = f.split("\n", 1)[0].strip()
    m = re.search(r"(k_[a-z0-9_]+)", name)
    short = m.group(1) if m else name
    tmpl = re.findall(r"ILi(\d+)E", name)
    if tmpl:
        short += "<" + ",".join(tmpl) + ">"
    if "ILb1E" in name:
        short += "<x3>"
    elif "ILb0E" in name:
        short += "<bf16>"
    cnt = {k: len(re.findall(r"\b" + re.escape(k) + r"[.\s]", f)) for k in KEYS}
    out[short] = {"instructions": len(re.findall(r"/\*[0-9a-f]{4,}\*/\s+[A-Z@]", f)), **{k: v for k, v in cnt.items() if v}}
print(json.dumps(out, indent=1, sort_keys=True))
