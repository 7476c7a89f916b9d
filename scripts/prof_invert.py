"""Time the history inverse (K x K Hermitian per frequency) in isolation (dev aid).

python scripts/prof_invert.py [K nfreq dtype]   (default 100 924 f64: BASELINE config 1)
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1706_06972_b200 import _lib  # noqa: E402

K, nf = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (100, 924)
dt = sys.argv[3] if len(sys.argv) > 3 else "f64"
cd = torch.complex128 if dt == "f64" else torch.complex64
npk = K * (K + 1) // 2
g = torch.Generator(device="cuda").manual_seed(0)
Z = torch.randn(nf, K, 2 * K, dtype=cd, device="cuda", generator=g)
A = Z @ Z.conj().transpose(1, 2)
ii, jj = torch.tril_indices(K, K)
S = A[:, ii, jj].contiguous()  # packed lower triangle, row-major (i >= j)
inv = torch.empty_like(S)
info = torch.zeros(1, dtype=torch.int32, device="cuda")
code = _lib.code(S.dtype)
for _ in range(2):
    _lib.call("ocsc_history_invert", code, code, K, nf, _lib.ptr(S), 1.0, 1.0, _lib.ptr(inv), _lib.ptr(info),
              _lib.stream())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    _lib.call("ocsc_history_invert", code, code, K, nf, _lib.ptr(S), 1.0, 1.0, _lib.ptr(inv), _lib.ptr(info),
              _lib.stream())
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
flops = 8.0 * K ** 3 * nf
print(f"K={K} nfreq={nf} {dt}: {ms:.3f} ms, {flops / ms / 1e9:.2f} TFLOP/s (8 K^3 per matrix), info={int(info.item())}")
full = torch.zeros(nf, K, K, dtype=cd, device="cuda")
full[:, ii, jj] = inv
full = full + full.conj().transpose(1, 2) - torch.diag_embed(torch.diagonal(full, dim1=1, dim2=2))
Ar = A + torch.eye(K, dtype=cd, device="cuda")
err = (Ar @ full - torch.eye(K, dtype=cd, device="cuda")).abs().max().item()
print(f"max |A A^-1 - I| = {err:.2e}")
