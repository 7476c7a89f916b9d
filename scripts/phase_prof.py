import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1706_06972_b200 as ob
from paper_1706_06972_b200 import _lib
from oracle import ocsc_oracle as O
c = O.CONFIGS[1]; B = 50
X = O.synth_images(B, c["dims0"], c["grid"], c["K0"], seed=1).reshape(B, -1)
tr = ob.OnlineTrainer(ob.SignalShape(c["grid"], (11, 11)), ob.TrainConfig(n_filters=100, rho_dict=1.0, dtype="float32", batch_size=B, stop_tol=0.0))
tr.partial_fit(X)
buf = torch.zeros(64, dtype=torch.int64, device="cuda")
_lib.call("ocsc_debug_fused_profile", buf.data_ptr())
tr.partial_fit(X); torch.cuda.synchronize()
_lib.call("ocsc_debug_fused_profile", None)
t = buf.cpu().numpy().reshape(8, 8)
names = ["colF", "reduce+cs1", "exchange+decide", "(it++)", "cs2", "colI+row", "norm-push+sync"]
d = np.diff(t, axis=1)
print("cycles per phase (median over iters 8..14):")
for i, n in enumerate(names): print(f"  {n:12s} {int(np.median(d[:7, i]))}")
print("  iteration  ", int(np.median(np.diff(t[:, 0]))))
# wall-clock of the fused launch alone (events) to convert cycles -> time
from paper_1706_06972_b200.transforms import rfft2_dev
xs = torch.as_tensor(X.reshape(B, 42, 42), dtype=torch.float32).cuda()
xh = rfft2_dev(xs, tr.shape)
buf = tr._buf
obj = torch.empty(B, dtype=torch.float64, device="cuda")
cc = tr.coding_config
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rep in range(3):
    e0.record()
    _lib.call("ocsc_code_fused", 4, 42, 42, 100, B, xh.data_ptr(), tr.Wh.data_ptr(), tr.den.data_ptr(), cc.beta, cc.rho,
              cc.max_iters, cc.rel_tol, buf.u.data_ptr(), None, tr._uh.data_ptr(), obj.data_ptr(), None,
              buf.iters.data_ptr(), buf.status.data_ptr(), _lib.stream())
    e1.record(); torch.cuda.synchronize()
    print(f"fused launch {e0.elapsed_time(e1):.2f} ms")
import subprocess
print(subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active", "--format=csv"], capture_output=True, text=True).stdout)
tlb = torch.zeros(2 * B, dtype=torch.int64, device="cuda")
_lib.call("ocsc_debug_fused_timeline", tlb.data_ptr())
_lib.call("ocsc_code_fused", 4, 42, 42, 100, B, xh.data_ptr(), tr.Wh.data_ptr(), tr.den.data_ptr(), cc.beta, cc.rho,
          cc.max_iters, cc.rel_tol, buf.u.data_ptr(), None, tr._uh.data_ptr(), obj.data_ptr(), None,
          buf.iters.data_ptr(), buf.status.data_ptr(), _lib.stream())
torch.cuda.synchronize()
_lib.call("ocsc_debug_fused_timeline", None)
t = tlb.cpu().numpy().reshape(B, 2).astype(np.float64)
t -= t[:, 0].min()
for b in range(B):
    print(f"sample {b:2d}: start {t[b,0]/1e6:7.3f} ms  dur {(t[b,1]-t[b,0])/1e6:6.3f} ms")
