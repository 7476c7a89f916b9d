"""Two cfg3-shaped mini-batches with 2 code iterations (profiling target for the history /
dictionary kernels at K=256, 266x266; dev aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1706_06972_b200 as ob  # noqa: E402

H, K, B = 266, 256, 32
shape = ob.SignalShape((H, H), (11, 11))
cfg = ob.TrainConfig(n_filters=K, beta=0.5, rho_code=1.0, rho_dict=1.0, inner_iters=10, dtype="float32",
                     history_dtype="float64", batch_size=B, stop_tol=0.0, code_max_iters=2)
tr = ob.OnlineTrainer(shape, cfg)
x = torch.randn(B, H * H, dtype=torch.float32, device="cuda")
for _ in range(2):
    tr.partial_fit(x)
torch.cuda.synchronize()
print("ok")
