"""Anatomy of one training step of a BASELINE config (dev aid): trainer marks (CUDA events)
relative to the step start, with the divergence check on (the API default) and off.

python scripts/step_anatomy.py [config]   (1: 42x42 K=100 B=50; 2: 100x100 K=100 B=10)
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1706_06972_b200 as ob
from paper_1706_06972_b200.workloads import CONFIGS, synth_images

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 1
c = CONFIGS[cid]
B = c["B"]
X = torch.as_tensor(synth_images(8 * B, c["dims0"], c["grid"], c["K0"], seed=1).reshape(8, B, -1).astype(np.float32)).cuda()
for check in (True, False):
    tr = ob.OnlineTrainer(ob.SignalShape(c["grid"], (11, 11)),
                          ob.TrainConfig(n_filters=c["K"], beta=c["beta"], dtype="float32", batch_size=B, stop_tol=0.0,
                                         rho_dict=1.0))
    for m in range(3):
        tr.partial_fit(X[m], check=check)
    torch.cuda.synchronize()
    for m in range(3, 6):
        e0 = torch.cuda.Event(enable_timing=True)
        tr._tl = []
        t0 = time.perf_counter()
        e0.record()
        tr.partial_fit(X[m], check=check)
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record()
        torch.cuda.synchronize()
        cpu = (time.perf_counter() - t0) * 1e3
        marks = " ".join(f"{lab}={e0.elapsed_time(ev):.2f}" for lab, ev in tr._tl)
        print(f"check={check} step {e0.elapsed_time(e1):.2f} ms (host {cpu:.2f}): {marks}")
    tr._tl = None
