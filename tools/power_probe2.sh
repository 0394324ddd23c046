#!/bin/bash
# nvidia-smi samples (clock, power, throttle reasons) while one config loops.
O=gpurun_out
for c in "$@"; do
  nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv -lms 50 > $O/power2_cfg$c.csv &
  P=$!
  timeout 300 python tools/run_cfg.py $c 40 > /dev/null 2>&1
  kill $P
done
