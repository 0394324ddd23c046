#!/bin/bash
# Round-2 profiling pass (second half). Every command ran clean without ncu first;
# numbers printed under ncu are not bench values.
O=gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-configs --no-e2e --no-cpu --no-nccl-check"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_r02.csv $B > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"oz_gemm|cs_gather" -s 2 -c 2 -o $O/ncu_cfg1_r02 $B > $O/ncu_cfg1.log 2>&1
for c in 0 2 3 4; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg${c}_r02.csv python tools/run_cfg.py $c 1 > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"jacobi|gemm_skinny" -c 3 -o $O/ncu_cfg0_r02 python tools/run_cfg.py 0 1 > /dev/null 2>&1
ls -la $O
