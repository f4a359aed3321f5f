#!/bin/bash
# ncu captures of one frame per bench config (dev tool; run on the GPU box, writes gpurun_out/):
#   launch list (gpu__time_duration, cold caches, serialised) of a warm frame, and a --set full
#   capture of every k_fact2 launch of one eager frame, exported as raw CSV (the .ncu-rep of the
#   longest launch is kept only when small).
set -u
mkdir -p gpurun_out
for c in ${@:-config2 config3}; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_r02_$c.csv \
      python scripts/one_frame.py $c 2 > gpurun_out/ncu_l_$c.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:k_fact2 --launch-count 12 \
      -o /tmp/r02_fact2_$c python scripts/one_frame.py $c 0 > gpurun_out/ncu_f_$c.log 2>&1
  ncu -i /tmp/r02_fact2_$c.ncu-rep --page raw --csv > gpurun_out/r02_fact2_${c}_raw.csv 2>/dev/null
  ncu -i /tmp/r02_fact2_$c.ncu-rep --page details --csv > gpurun_out/r02_fact2_${c}_details.csv 2>/dev/null
  ls -la /tmp/r02_fact2_$c.ncu-rep >> gpurun_out/ncu_f_$c.log
done
