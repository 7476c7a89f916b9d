"""Summarise an ncu report: SOL, occupancy, DRAM bytes, bank conflicts, stall reasons, with the
units ncu reports (one block per captured kernel launch) (dev aid).

python scripts/ncu_summary.py report.ncu-rep
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, units = rows[0], rows[1]
keys = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_cluster_pct", "launch__cluster_max_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
        "sm__cycles_active.avg", "gpc__cycles_elapsed.max"]
for v in rows[2:]:
    d = dict(zip(h, v))
    u = dict(zip(h, units))
    name = d.get("Kernel Name", "?")
    print(f"== {name[:110]}")
    for k in keys:
        if k in d:
            print(f"{k:70s} {d[k]:>22s} {u.get(k, '')}")
    st = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(d[k].replace(",", "") or 0)) for k in h
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
    tot = sum(x for _, x in st) or 1
    print("stalls:", ", ".join(f"{k} {100*x/tot:.1f}%" for k, x in sorted(st, key=lambda kv: -kv[1])[:10]))
