"""Event timeline of one config-1 mini-batch with the overlapped history inverse (dev aid):
trainer marks (CUDA events) and per-sample start/end of the fused kernel (globaltimer)."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_06972_b200 as ob  # noqa: E402
from paper_1706_06972_b200 import _lib  # noqa: E402
from paper_1706_06972_b200.workloads import CONFIGS, synth_images  # noqa: E402

c = CONFIGS[1]
B = 50
X = synth_images(4 * B, c["dims0"], c["grid"], c["K0"], seed=1).reshape(4 * B, -1)
lib = _lib.load()
for overlap in (True, False):
    tr = ob.OnlineTrainer(ob.SignalShape(c["grid"], (11, 11)),
                          ob.TrainConfig(n_filters=100, dtype="float32", batch_size=B, stop_tol=0.0, rho_dict=1.0,
                                         overlap=overlap))
    for m in range(3):
        tr.partial_fit(X[m * B:(m + 1) * B])
    torch.cuda.synchronize()
    tl = torch.zeros(2 * B, dtype=torch.int64, device="cuda")
    lib.ocsc_debug_fused_timeline(ctypes.c_void_p(tl.data_ptr()))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tr._tl = []
    e0.record()
    tr.partial_fit(X[3 * B:4 * B])
    e1.record()
    torch.cuda.synchronize()
    lib.ocsc_debug_fused_timeline(ctypes.c_void_p(0))
    print(f"overlap={overlap}: path={tr.last_path} split={tr._split_plan(B)} step {e0.elapsed_time(e1):.2f} ms")
    for label, ev in tr._tl:
        print(f"   {label:18s} {e0.elapsed_time(ev):8.3f} ms")
    t = tl.view(B, 2).cpu()
    t0 = int(t[:, 0].min())
    for b in range(B):
        print(f"   sample {b:2d}: {(int(t[b, 0]) - t0) / 1e6:7.3f} -> {(int(t[b, 1]) - t0) / 1e6:7.3f} ms")
for b in (9, 41, 50):
    info = (ctypes.c_int32 * 8)()
    side = (ctypes.c_int32 * 8)()
    lib.ocsc_code_fused_info(4, 42, 42, 100, b, info)
    lib.ocsc_code_fused_side_info(4, 42, 42, 100, b, side)
    print(f"B={b}: plan", list(info), "side", list(side))
