"""Top CUDA source lines by excessive shared-memory wavefronts (bank conflicts) for one kernel of
an ncu report (dev aid).  python scripts/ncu_smem_lines.py report.ncu-rep kernel_regex [n]"""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
E, W, I = h.index("L1 Wavefronts Shared Excessive"), h.index("L1 Wavefronts Shared"), h.index("L1 Wavefronts Shared Ideal")
data = []
for r in rows[hi + 1:]:
    if len(r) < len(h) or not r[0]:
        continue
    try:
        data.append((float(r[E] or 0), float(r[W] or 0), float(r[I] or 0), r[0], r[1].strip()[:90]))
    except ValueError:
        pass
tot = sum(d[0] for d in data) or 1
print(f"excessive shared wavefronts: {tot:.3g} of {sum(d[1] for d in data):.3g}")
for ex, wf, ideal, line, src in sorted(data, reverse=True)[:n]:
    print(f"{100 * ex / tot:5.1f}%  wf {wf:10.3g} ideal {ideal:10.3g}  L{line:5s} {src}")
