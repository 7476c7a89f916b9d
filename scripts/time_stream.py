"""Event-timed streaming code-ADMM iterations (dev aid): python scripts/time_stream.py H K B iters"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_06972_b200 as ob  # noqa: E402
from paper_1706_06972_b200.coding import CodeBuffers, infer_codes_stream  # noqa: E402
from paper_1706_06972_b200.transforms import rfft2_dev  # noqa: E402

H, K, B, iters = (int(a) for a in sys.argv[1:5])
shape = ob.SignalShape((H, H), (11, 11))
tr = ob.OnlineTrainer(shape, ob.TrainConfig(n_filters=K, dtype="float32", batch_size=B))
x = torch.randn(B, H, H, dtype=torch.float32, device="cuda")
xh = rfft2_dev(x, shape)
buf = CodeBuffers(shape, K, B, torch.float32)
cc = ob.CodingConfig(max_iters=iters, rel_tol=0.0)
infer_codes_stream(xh, tr.Wh, tr.den, shape, cc, buf, B, poll=0)
ts = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    infer_codes_stream(xh, tr.Wh, tr.den, shape, cc, buf, B, poll=0)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"{H}x{H} K={K} B={B}: {iters} iterations {min(ts):.2f} ms = {min(ts) / iters * 1e3:.1f} us/iter")
