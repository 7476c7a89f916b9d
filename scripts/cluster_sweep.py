"""Time the fused code ADMM (BASELINE config 1 batch) for each cluster size (dev aid).

python scripts/cluster_sweep.py [cs ...]   -- every size runs in its own process with
OCSC_FUSED_CS=cs (the plan is cached per process); prints active clusters and launch time.
"""
import ctypes
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import ctypes, os, sys
sys.path.insert(0, %r)
import torch
import paper_1706_06972_b200 as ob
from paper_1706_06972_b200 import _lib
from oracle import ocsc_oracle as O
from paper_1706_06972_b200.workloads import synth_images  # noqa: E402
from paper_1706_06972_b200.transforms import rfft2_dev
B = 50
X = synth_images(B, (32, 32), (42, 42), 20, seed=1).reshape(B, -1)
tr = ob.OnlineTrainer(ob.SignalShape((42, 42), (11, 11)), ob.TrainConfig(n_filters=100, dtype="float32", batch_size=B,
                      stop_tol=0.0))
tr.partial_fit(X)
info = (ctypes.c_int32 * 8)()
_lib.load().ocsc_code_fused_info(4, 42, 42, 100, B, info)
xs = torch.as_tensor(X.reshape(B, 42, 42), dtype=torch.float32).cuda()
xh = rfft2_dev(xs, tr.shape)
buf = tr._buf
obj = torch.empty(B, dtype=torch.float64, device="cuda")
cc = tr.coding_config
ts = []
for rep in range(4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _lib.call("ocsc_code_fused", 4, 42, 42, 100, B, xh.data_ptr(), tr.Wh.data_ptr(), tr.den.data_ptr(), cc.beta,
              cc.rho, cc.max_iters, cc.rel_tol, buf.u.data_ptr(), None, tr._uh.data_ptr(), obj.data_ptr(), None,
              buf.iters.data_ptr(), buf.status.data_ptr(), _lib.stream())
    e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"cs={info[0]:2d} threads={info[1]} smem={info[2]} regs={info[3]} active={info[4]} b_main={info[5]} "
      f"tail_cs={info[6]} tail_active={info[7]}  launch {min(ts[1:]):.2f} ms")
''' % HERE

sizes = [int(a) for a in sys.argv[1:]] or [0] + list(range(2, 17))
for cs in sizes:
    env = dict(os.environ)
    if cs:
        env["OCSC_FUSED_CS"] = str(cs)
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    out = (r.stdout.strip().splitlines() or [""])[-1]
    print(f"[{'auto' if not cs else cs}] {out}" if r.returncode == 0 else f"[{cs}] failed: {r.stderr.strip()[-300:]}",
          flush=True)
