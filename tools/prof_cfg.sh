#!/bin/bash
# Launch lists (ncu gpu__time_duration) of the timed operation of the given configs.
for c in "$@"; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg${c}.csv python tools/run_cfg.py $c 1 > gpurun_out/ncu_l$c.log 2>&1
done
