"""Launch list of a few generic (cuFFT) code-ADMM iterations at a given grid (dev aid).

python scripts/prof_generic.py H W K B iters
"""
import sys

import numpy as np
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_1706_06972_b200 as ob  # noqa: E402
from paper_1706_06972_b200.coding import CodeBuffers, infer_codes  # noqa: E402
from paper_1706_06972_b200.transforms import rfft2_dev  # noqa: E402

H, W, K, B, iters = (int(a) for a in sys.argv[1:6])
shape = ob.SignalShape((H, W), (11, 11))
tr = ob.OnlineTrainer(shape, ob.TrainConfig(n_filters=K, dtype="float32", history_dtype="float64", batch_size=B,
                                            fused=False))
x = torch.randn(B, H, W, dtype=torch.float32, device="cuda")
xh = rfft2_dev(x, shape)
buf = tr._buffers(B, False)
cc = ob.CodingConfig(max_iters=iters, rel_tol=0.0)
for _ in range(2):
    infer_codes(xh, tr.Wh, tr.den, shape, cc, buf, B, poll=0)
torch.cuda.synchronize()
print("done")
