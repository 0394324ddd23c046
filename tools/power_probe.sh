#!/bin/bash
# Sample SM clock / power / throttle reasons while one config runs in a loop.
O=gpurun_out
for c in "$@"; do
  nvidia-smi --query-gpu=timestamp,clocks.sm,clocks.mem,power.draw,power.limit,temperature.gpu,clocks_throttle_reasons.active --format=csv -lms 100 > $O/power_cfg$c.csv &
  P=$!
  timeout 300 python tools/run_cfg.py $c 60 > $O/power_run$c.log 2>&1
  kill $P
done
