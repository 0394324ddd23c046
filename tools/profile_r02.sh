#!/bin/bash
# Round-2 profiling pass (run on the GPU box from the repo root; outputs in gpurun_out/).
# Every command ran clean without ncu first; numbers printed under ncu are not bench values.
set -x
O=gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-configs --no-e2e --no-cpu --no-nccl-check"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_r02.csv $B > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cs_gather_kernel -s 4 -c 1 -o $O/ncu_cs_gather_r02 $B > $O/ncu_gather.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rbf_tc_digits|gram_i8_kernel" -s 2 -c 2 -o $O/ncu_cfg4_r02 python tools/run_cfg.py 4 2 > $O/ncu_cfg4.log 2>&1
for c in 0 3 4; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg${c}_r02.csv python tools/run_cfg.py $c 1 > /dev/null 2>&1
done
ls -la $O
