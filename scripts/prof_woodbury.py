"""Time ocsc_history_woodbury at config-1 sizes (K=100, 924 frequencies, nb=5) (dev aid)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1706_06972_b200 import _lib  # noqa: E402

K, nb = 100, int(sys.argv[1]) if len(sys.argv) > 1 else 5
nf = int(os.environ.get("WB_NF", "924"))
npk = K * (K + 1) // 2
inv = torch.randn(nf, npk, dtype=torch.complex128, device="cuda")
z = torch.randn(nb, K, nf, dtype=torch.complex64, device="cuda")
out = torch.empty(nf, npk, dtype=torch.complex64, device="cuda")
info = torch.zeros(1, dtype=torch.int32, device="cuda")
S = torch.zeros(nf, npk, dtype=torch.complex128, device="cuda")
c = torch.zeros(nf, K, dtype=torch.complex128, device="cuda")
x = torch.randn(nb, nf, dtype=torch.complex64, device="cuda")
fold = len(sys.argv) > 2
args = (_lib.F32, _lib.F32, K, nf, nb, _lib.ptr(inv), _lib.ptr(z), K * nf, nf, 1, _lib.ptr(out), _lib.ptr(info),
        _lib.ptr(x) if fold else None, nf, 1, _lib.ptr(S) if fold else None, _lib.ptr(c) if fold else None,
        _lib.stream())
for _ in range(3):
    _lib.call("ocsc_history_woodbury", *args)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    _lib.call("ocsc_history_woodbury", *args)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"woodbury K={K} nf={nf} nb={nb}: {ms * 1e3:.1f} us, {(nf * npk * 24) / ms / 1e6:.0f} GB/s (f64 in + f32 out)")
