"""Run the cfg1 mini-batch step a few times (profiling target for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1706_06972_b200 as ob
from oracle import ocsc_oracle as O
from paper_1706_06972_b200.workloads import CONFIGS, synth_images  # noqa: E402
c = CONFIGS[1]
B = int(os.environ.get("B", 50))
X = synth_images(B * 2, c["dims0"], c["grid"], c["K0"], seed=1).reshape(B * 2, -1)
cfg = ob.TrainConfig(n_filters=100, beta=1.0, rho_code=1.0, rho_dict=1.0, inner_iters=10, seed=0,
                     dtype="float32", history_dtype="float64", batch_size=B, stop_tol=0.0)
tr = ob.OnlineTrainer(ob.SignalShape(c["grid"], (11, 11)), cfg)
for m in range(2):
    r = tr.partial_fit(X[m * B:(m + 1) * B])
torch.cuda.synchronize()
print("ok", r.objectives[:2], r.iterations[:2])
