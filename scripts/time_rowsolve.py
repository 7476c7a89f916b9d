"""Event-timed dictionary row solve (packed Hermitian inverse GEMV per frequency; dev aid).

python scripts/time_rowsolve.py [K nfreq]   (default 100 5100: BASELINE config 2; 924: config 1)
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1706_06972_b200 import _lib  # noqa: E402

K, nf = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (100, 5100)
npk = K * (K + 1) // 2
g = torch.Generator(device="cuda").manual_seed(0)
inv = torch.randn(nf, npk, dtype=torch.complex64, device="cuda", generator=g)
c = torch.randn(nf, K, dtype=torch.complex128, device="cuda", generator=g)
V = torch.randn(K, nf, dtype=torch.complex64, device="cuda", generator=g)
T = torch.randn(K, nf, dtype=torch.complex64, device="cuda", generator=g)
D = torch.empty_like(V)
args = lambda: (_lib.F32, _lib.F64, _lib.F32, K, nf, _lib.ptr(inv), _lib.ptr(c), 2.0, _lib.ptr(V), _lib.ptr(T), nf, 1,
                _lib.ptr(D), _lib.stream())
for _ in range(3):
    _lib.call("ocsc_dict_rowsolve", *args())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    _lib.call("ocsc_dict_rowsolve", *args())
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"K={K} nfreq={nf}: {ms * 1e3:.1f} us per row solve, {inv.numel() * 8 / ms / 1e6:.0f} GB/s on the inverse")
