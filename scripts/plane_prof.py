"""Per-phase clock64 stamps of the plane-resident streaming kernel (dev aid).

python scripts/plane_prof.py [H K B]   (default 100 100 10: BASELINE config 2)
Prints the median cycles of each phase of CTA (0, 0) over its first planes, and the event
time of one code-ADMM iteration.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_06972_b200 as ob  # noqa: E402
from paper_1706_06972_b200 import _lib  # noqa: E402
from paper_1706_06972_b200.coding import CodeBuffers, infer_codes_stream  # noqa: E402
from paper_1706_06972_b200.transforms import rfft2_dev  # noqa: E402

H, K, B = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (100, 100, 10)
shape = ob.SignalShape((H, H), (11, 11))
tr = ob.OnlineTrainer(shape, ob.TrainConfig(n_filters=K, dtype="float32", batch_size=B))
x = torch.randn(B, H, H, dtype=torch.float32, device="cuda")
xh = rfft2_dev(x, shape)
buf = CodeBuffers(shape, K, B, torch.float32)
iters = 50
cc = ob.CodingConfig(max_iters=iters, rel_tol=0.0)
infer_codes_stream(xh, tr.Wh, tr.den, shape, cc, buf, B, poll=0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
infer_codes_stream(xh, tr.Wh, tr.den, shape, cc, buf, B, poll=0)
e1.record()
torch.cuda.synchronize()
print(f"{iters} iterations: {e0.elapsed_time(e1):.3f} ms ({e0.elapsed_time(e1) / iters * 1e3:.1f} us/iter)")
pb = torch.zeros(64, dtype=torch.int64, device="cuda")
_lib.call("ocsc_debug_plane_profile", pb.data_ptr())
infer_codes_stream(xh, tr.Wh, tr.den, shape, cc, buf, B, poll=0)
torch.cuda.synchronize()
_lib.call("ocsc_debug_plane_profile", None)
t = pb.cpu().numpy().reshape(4, 16).astype(np.int64)
names = ["w prefetch issue", "col inv s1(cdg)+a", "col inv b", "herm pre+row s1", "row inv a", "row inv b",
         "w wait", "update", "row fwd s1", "row fwd a", "row fwd b+post", "col fwd s1", "col fwd a",
         "col fwd b+partial"]
d = np.diff(t[:, :15], axis=1)
print("cycles per phase (median over the CTA's first 4 planes):")
for i, n in enumerate(names):
    print(f"  {n:16s} {int(np.median(d[:, i])):7d}")
print(f"  plane            {int(np.median(t[:, 14] - t[:, 0])):7d}")
