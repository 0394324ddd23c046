"""Print the key counters and warp stall breakdown of an ncu --set full report: python tools/ncu_stalls.py REP"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
for v in rows[2:]:
    d = dict(zip(h, v))
    print(d.get("Kernel Name", "")[:90], d.get("gpu__time_duration.sum"))
    stall = {k: v for k, v in d.items() if k.startswith("smsp__average_warps_issue_stalled_")
             and k.endswith("_per_issue_active.ratio")}
    for k, vv in sorted(stall.items(), key=lambda x: -float(x[1] or 0))[:10]:
        print(f"  stall {k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]:30s} {vv}")
    for k in ["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
              "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
              "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
              "launch__grid_size", "launch__registers_per_thread", "smsp__inst_executed.sum",
              "l1tex__t_bytes_pipe_lsu_mem_global_op_ld.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]:
        if k in d:
            print(f"  {k:70s} {d[k]}")
