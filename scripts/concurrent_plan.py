"""Dev aid: makespan of two fused launches running concurrently on two streams (config 1).

python scripts/concurrent_plan.py A_N A_CS A_DREG B_N B_CS B_DREG
Launch A codes samples [0, A_N) with cluster size A_CS (register-resident D if A_DREG), launch B
codes [A_N, A_N + B_N) with B_CS / B_DREG on a second stream at the same time.  Prints the time of
A alone, B alone and both together (each shape's plan is pinned through OCSC_FUSED_CS /
OCSC_FUSED_DREG before its first use in this process)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1706_06972_b200 as ob  # noqa: E402
from paper_1706_06972_b200 import _lib  # noqa: E402
from paper_1706_06972_b200.transforms import rfft2_dev  # noqa: E402
from paper_1706_06972_b200.workloads import synth_images  # noqa: E402

an, acs, adr, bn, bcs, bdr = (int(v) for v in sys.argv[1:7])
B = an + bn
X = synth_images(B, (32, 32), (42, 42), 20, seed=1).reshape(B, -1)
tr = ob.OnlineTrainer(ob.SignalShape((42, 42), (11, 11)), ob.TrainConfig(n_filters=100, dtype="float32",
                      batch_size=B, stop_tol=0.0))
tr._buffers(B, False)  # (no partial_fit: every launch plan below is pinned fresh)
xs = torch.as_tensor(X.reshape(B, 42, 42), dtype=torch.float32).cuda()
xh = rfft2_dev(xs, tr.shape)
buf = tr._buf
uh = tr._uh
obj = torch.empty(B, dtype=torch.float64, device="cuda")
lib = _lib.load()
info = (__import__("ctypes").c_int32 * 8)()


def pin(n, cs, dreg):
    os.environ["OCSC_FUSED_CS"], os.environ["OCSC_FUSED_DREG"] = str(cs), str(dreg)
    lib.ocsc_code_fused_info(4, 42, 42, 100, n, info)
    print(f"  plan n={n}: cs={info[0]} threads={info[1]} smem={info[2]} regs={info[3]} active={info[4]} "
          f"b_main={info[5]} tail={info[6]}", flush=True)


pin(an, acs, adr)
pin(bn, bcs, bdr)
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()


def go(which):
    """which: "A", "B", "AB" (A enqueued first) or "BA" (B enqueued first)."""
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    done = []
    jobs = {"A": (0, an, sa), "B": (an, bn, sb)}
    for name in which:
        b0, n, st = jobs[name]
        st.wait_event(e0)
        with torch.cuda.stream(st):
            tr._code_fused(xh, buf, uh, obj, b0, b0 + n)
            ev = torch.cuda.Event()
            ev.record()
            done.append(ev)
    for ev in done:
        torch.cuda.current_stream().wait_event(ev)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


for which in ("A", "B", "AB", "BA", "BA"):
    print(f"{which}: {go(which):.2f} ms", flush=True)
