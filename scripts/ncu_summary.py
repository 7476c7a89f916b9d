"""Summarise an ncu report: SOL, occupancy, stall reasons, instruction mix (dev aid)."""
import csv, collections, subprocess, sys
rep = sys.argv[1]
def page(args):
    out = subprocess.run(["ncu", "-i", rep] + args, capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))
r = page(["--page", "raw", "--csv"])
h, v = r[0], r[2]
d = dict(zip(h, v))
keys = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_cluster_pct", "launch__cluster_max_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
        "sm__cycles_active.avg", "gpc__cycles_elapsed.max"]
for k in keys:
    if k in d: print(f"{k:70s} {d[k]}")
st = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(d[k].replace(",", "") or 0)) for k in h
      if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
tot = sum(x for _, x in st)
print("stalls:", ", ".join(f"{k} {100*x/tot:.1f}%" for k, x in sorted(st, key=lambda kv: -kv[1])[:10]))
