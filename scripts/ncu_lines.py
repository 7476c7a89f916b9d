"""Top CUDA source lines by warp-stall samples for one kernel of an ncu report (dev aid).

python scripts/ncu_lines.py report.ncu-rep kernel_regex [n]
"""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
S, I = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
data = []
for r in rows[hi + 1:]:
    if len(r) < len(h) or not r[0]:
        continue
    try:
        data.append((float(r[S] or 0), float(r[I] or 0), r[0], r[1].strip()[:95]))
    except ValueError:
        pass
tot = sum(d[0] for d in data) or 1
itot = sum(d[1] for d in data) or 1
for samp, inst, line, src in sorted(data, reverse=True)[:n]:
    print(f"{100 * samp / tot:5.1f}% stall  {100 * inst / itot:5.1f}% inst  L{line:5s} {src}")
