"""Phase stamps of the blocked Cholesky (CTA 0) at config-4 shapes (development aid).

python scripts/chol_prof.py [K ...]
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1706_06972_b200 as ob
from paper_1706_06972_b200 import _lib

_lib.load()
dev = torch.device("cuda", 0)
P, B = 128 * 128, 64
for K in [int(a) for a in sys.argv[1:]] or [256, 512]:
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    z = torch.complex(torch.randn(B, P, K, device=dev, generator=g), torch.randn(B, P, K, device=dev, generator=g)) / np.sqrt(2)
    x = torch.complex(torch.randn(B, P, device=dev, generator=g), torch.randn(B, P, device=dev, generator=g)) / np.sqrt(2)
    h = ob.HistoryState(ob.SignalShape((P,), (1,)), K, 1.0 / P, dtype=torch.complex64, solver="chol")
    h.accumulate(z, (P * K, 1, K), x, (P, 1), B)
    h.count = 1
    h.factor(check=False)  # warm-up
    buf = torch.zeros(80, dtype=torch.int64, device=dev)
    _lib.call("ocsc_debug_chol_profile", buf.data_ptr())
    h._inv_count = -1  # force a second factorisation
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(); h.factor(check=False); e1.record(); torch.cuda.synchronize()
    _lib.call("ocsc_debug_chol_profile", None)
    t = buf.cpu().numpy()
    nb = (K + 31) // 32
    print(f"K={K}: factor {e0.elapsed_time(e1):.2f} ms; CTA 0 lifetime {t[2 + 4 * (nb - 2) + 4] - t[0]} cycles "
          f"(expand {t[1] - t[0]}, diag0 {t[2] - t[1]})")
    prev = t[2]
    for kb in range(nb - 1):
        a, b_, c, d = t[3 + 4 * kb: 7 + 4 * kb]
        print(f"  kb={kb:2d} R={K - 32 * (kb + 1):3d}: panel {a - prev:7d}  next diagonal done {c - b_:7d}  "
              f"trailing {d - b_:7d}  step {d - prev:7d}")
        prev = d
    del z, x, h
    torch.cuda.empty_cache()
