import ctypes, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1706_06972_b200 import _lib
lib = _lib.load(); torch.cuda.init()
for (dt, N, K, B) in [(4, 42, 100, 50), (8, 10, 5, 3), (4, 30, 33, 2)]:
    info = (ctypes.c_int32 * 8)()
    lib.ocsc_code_fused_info(dt, N, N, K, B, info)
    print(dict(dtype=dt, N=N, K=K, B=B, cs=info[0], threads=info[1], smem=info[2], regs=info[3], active=info[4], b_main=info[5], tail_cs=info[6], tail_active=info[7]))
