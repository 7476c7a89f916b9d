"""Per-step kernel table from an ncu launch list of bench.py (dev aid; feeds profiles/traffic.json).

python scripts/traffic_from_launches.py LAUNCHES.csv [--update profiles/traffic.json]

The launch list is `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--clock-control none --csv` of `bench.py --steps 2 --warmup 3 --no-cpu-baseline`.  A step starts at
the first k_code_fused launch that follows a non-fused launch; the last complete step before the
e2e phase is taken (the 4th step of the device-timed loop).  Prints the per-kernel table and, with
--update, rewrites the step fields of the traffic file (other keys kept).
"""
import csv
import json
import sys
from collections import OrderedDict


def load(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    head, data = rows[0], rows[1:]
    k = OrderedDict()
    for r in data:
        d = dict(zip(head, r))
        key = int(d["ID"])
        e = k.setdefault(key, {"id": key, "kernel": d["Kernel Name"].split("(")[0]})
        try:
            e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
        except ValueError:
            pass
    return list(k.values())


def steps(launches):
    """Split into steps: a step begins at a k_code_fused launch preceded by a non-fused one."""
    out, cur, prev_fused = [], [], False
    for l in launches:
        fused = "k_code_fused" in l["kernel"]
        if fused and not prev_fused and cur:
            out.append(cur)
            cur = []
        cur.append(l)
        prev_fused = fused
    if cur:
        out.append(cur)
    return out


def main():
    path = sys.argv[1]
    st = [s for s in steps(load(path)) if any("k_code_fused" in l["kernel"] for l in s)]
    step = st[3] if len(st) > 4 else st[-2]
    # the 256 MiB L2 flush between steps runs outside the timed events
    step = [l for l in step if not ("FillFunctor" in l["kernel"] and l.get("dram__bytes_write.sum", 0) > 2e8)]
    tot = sum(l.get("gpu__time_duration.sum", 0) for l in step)  # ns
    ks = []
    for l in step:
        us = l.get("gpu__time_duration.sum", 0) / 1e3
        mb = (l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0)) / 1e6
        ks.append({"id": l["id"], "kernel": l["kernel"], "us": us, "dram_MB": mb, "share": us * 1e3 / tot})
    fused = [k for k in ks if "k_code_fused" in k["kernel"]]
    fb = sum(k["dram_MB"] for k in fused) * 1e6
    for k in ks:
        print(f"{k['id']:5d} {k['kernel'][:60]:60s} {k['us']:10.1f} us {k['dram_MB']:9.2f} MB {100 * k['share']:5.1f} %")
    print(f"step {tot / 1e3:.1f} us serialised; fused {sum(k['us'] for k in fused):.1f} us, {fb / 1e6:.2f} MB")
    if "--update" in sys.argv:
        out = sys.argv[sys.argv.index("--update") + 1]
        d = json.load(open(out))
        d["kernels"] = ks
        d["step_us_serialised"] = tot / 1e3
        d["fused_dram_bytes_per_step"] = fb
        d["fused_bytes_per_batch_iter"] = fb / 300.0
        d["fused_note"] = (f"all {len(fused)} k_code_fused launches of the step (main + tail cluster shapes), "
                           f"300 ADMM iterations each")
        json.dump(d, open(out, "w"), indent=1)
        print("updated", out)


if __name__ == "__main__":
    main()
