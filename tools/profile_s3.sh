#!/bin/bash
# Profiling pass: launch lists of cfg0/3/4 + one ncu --set full of the cfg3 tcgen05 passes.
O=gpurun_out
for c in 0 3 4 2; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg${c}.csv python tools/run_cfg.py $c 1 > $O/ncu_l$c.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16x3 -c 3 -o $O/ncu_tc_cfg3 python tools/run_cfg.py 3 1 > $O/ncu_tc.log 2>&1
ls -la $O
