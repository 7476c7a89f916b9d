"""Dev aid: print the fused code-ADMM launch plans (ocsc_code_fused_info / _side_info)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1706_06972_b200 import _lib  # noqa: E402

lib = _lib.load()
torch.cuda.init()
cases = [(4, 42, 100, 50), (4, 42, 100, 41), (4, 42, 100, 9), (4, 42, 100, 1), (8, 42, 100, 50),
         (8, 10, 5, 3), (4, 30, 33, 2), (4, 42, 100, 200)]
for (dt, N, K, B) in cases:
    info = (ctypes.c_int32 * 8)()
    side = (ctypes.c_int32 * 8)()
    lib.ocsc_code_fused_info(dt, N, N, K, B, info)
    lib.ocsc_code_fused_side_info(dt, N, N, K, B, side)
    print(dict(dtype=dt, N=N, K=K, B=B, cs=info[0], threads=info[1], smem=info[2], regs=info[3], active=info[4],
               b_split=info[5], rest_cs=info[6], rest_active=info[7], side_cs=side[0], n_side=side[1],
               side_dreg=side[2], n_main=side[3], rows=side[4], main_dreg=side[5], model=side[6] / 1000,
               concurrent=side[7]), flush=True)
