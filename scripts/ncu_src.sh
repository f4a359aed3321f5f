#!/bin/bash
# Source-level ncu capture of the longest launch of one kernel in one eager frame (dev tool; run
# on the GPU box, writes gpurun_out/):   scripts/ncu_src.sh <kernel-regex> <config> <tag>
# exports the per-SASS source page (stall samples per instruction) and the raw metrics.
set -u
k=$1; c=$2; tag=${3:-src}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:$k --csv \
    python scripts/one_frame.py $c 0 > /tmp/${tag}_list.csv 2>/dev/null
skip=$(python - "$tag" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(f"/tmp/{sys.argv[1]}_list.csv")) if len(r) > 10 and r[-1].replace('.', '').isdigit()]
d = [float(r[-1]) for r in rows]
print(max(range(len(d)), key=lambda i: d[i]) if d else 0)
PY
)
echo "longest launch index $skip" > gpurun_out/${tag}.log
ncu -f --set full --clock-control none --import-source on -k regex:$k --launch-skip $skip --launch-count 1 \
    -o /tmp/${tag} python scripts/one_frame.py $c 0 >> gpurun_out/${tag}.log 2>&1
ncu -i /tmp/${tag}.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_sass.csv 2>/dev/null
ncu -i /tmp/${tag}.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>/dev/null
