"""Objective trace of an online run at BASELINE config 1 (dev aid): N images in mini-batches of 50."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_06972_b200 as ob  # noqa: E402
from oracle import ocsc_oracle as O  # noqa: E402
from paper_1706_06972_b200.workloads import CONFIGS, synth_images  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
B = 50
c = CONFIGS[1]
X = synth_images(N, c["dims0"], c["grid"], c["K0"], seed=11).reshape(N, -1).astype(np.float32)
tr = ob.OnlineTrainer(ob.SignalShape(c["grid"], (11, 11)),
                      ob.TrainConfig(n_filters=100, dtype="float32", batch_size=B, stop_tol=0.0, rho_dict=1.0))
Xd = torch.as_tensor(X).cuda()
t0 = time.perf_counter()
means = []
for m in range(N // B):
    res = tr.partial_fit(Xd[m * B:(m + 1) * B])
    means.append(float(np.mean(res.objectives)))
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"{N} images in {dt:.2f} s ({N / dt:.0f} img/s wall, first-call setup included)")
for m in list(range(0, 5)) + list(range(5, N // B, max(1, (N // B) // 8))) + [N // B - 1]:
    print(f"  mini-batch {m:3d}: mean objective {means[m]:.4f}")
