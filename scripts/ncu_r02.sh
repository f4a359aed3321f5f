#!/bin/bash
# Round-2 ncu evidence (dev tool; run on the GPU box, writes gpurun_out/): per bench config a
# launch list of one warm frame (gpu__time_duration, cold caches, serialised) and --set full
# captures of the frame's main kernels in one eager frame, exported as raw CSV (reps stay in /tmp).
set -u
T=${TAG:-r02}
mkdir -p gpurun_out
for c in ${@:-config2 config3}; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_$c.csv \
      python scripts/one_frame.py $c 2 > gpurun_out/${T}_ncu_l_$c.log 2>&1
  for k in ${KERNELS:-k_fact2 k_mlp_pair k_tail k_fine_rows k_render k_conflict_expand k_layer k_cols k_gather}; do
    ncu --set full --clock-control none --import-source on -k regex:$k --launch-count 40 \
        -f -o /tmp/${T}_${k}_$c python scripts/one_frame.py $c 0 > gpurun_out/${T}_ncu_${k}_$c.log 2>&1
    ncu -i /tmp/${T}_${k}_$c.ncu-rep --page raw --csv > gpurun_out/${T}_raw_${k}_$c.csv 2>/dev/null
  done
done
ls -la gpurun_out
