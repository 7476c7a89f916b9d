import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1706_06972_b200 as ob
from paper_1706_06972_b200 import _lib
from oracle import ocsc_oracle as O
from paper_1706_06972_b200.workloads import CONFIGS, synth_images  # noqa: E402
c = CONFIGS[1]; B = 50
X = synth_images(B, c["dims0"], c["grid"], c["K0"], seed=1).reshape(B, -1)
tr = ob.OnlineTrainer(ob.SignalShape(c["grid"], (11, 11)), ob.TrainConfig(n_filters=100, rho_dict=1.0, dtype="float32", batch_size=B, stop_tol=0.0))
tr.partial_fit(X)
from paper_1706_06972_b200.transforms import rfft2_dev
xs = torch.as_tensor(X.reshape(B, 42, 42), dtype=torch.float32).cuda()
xh = rfft2_dev(xs, tr.shape)
buf = tr._buf
obj = torch.empty(B, dtype=torch.float64, device="cuda")
cc = tr.coding_config
pbuf = torch.zeros(64, dtype=torch.int64, device="cuda")
_lib.call("ocsc_debug_fused_profile", pbuf.data_ptr())
# one direct launch of the whole batch (its own plan: main waves + tail, b0 = 0 for the main)
_lib.call("ocsc_code_fused", 4, 42, 42, 100, B, xh.data_ptr(), tr.Wh.data_ptr(), tr.den.data_ptr(), cc.beta, cc.rho,
          cc.max_iters, cc.rel_tol, buf.u.data_ptr(), None, tr._uh.data_ptr(), obj.data_ptr(), None,
          buf.iters.data_ptr(), buf.status.data_ptr(), _lib.stream())
torch.cuda.synchronize()
_lib.call("ocsc_debug_fused_profile", None)
t = pbuf.cpu().numpy().reshape(8, 8)
# stamp slots in time order (code_fused.cu OCSC_STAMP): 0 colF start, 1 after colF barrier,
# 3 after reduce_push, 2 after the partials wait, 4 after g push, 5 after the g wait,
# 7 after COL_I + its barrier, 6 after rows + norm push (then the end-of-iteration barrier)
order = [0, 1, 3, 2, 4, 5, 7, 6]
names = ["colF+bar", "reduce_push", "wait partials", "decide+g push", "Dprefetch+wait g", "colI+bar", "rows+norms"]
tt = t[:, order]
d = np.diff(tt, axis=1)
print("cycles per phase, CTA 0 thread 0 (median over iters 8..14):")
for i, n in enumerate(names): print(f"  {n:18s} {int(np.median(d[:7, i]))}")
print("  iteration  ", int(np.median(np.diff(t[:, 0]))))
# wall-clock of the fused launch alone (events) to convert cycles -> time
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
# per-iteration wall time and SM clock rate of CTA 0 (globaltimer vs clock64)
itb = torch.zeros(1024, dtype=torch.int64, device="cuda")
_lib.call("ocsc_debug_fused_iterations", itb.data_ptr())
_lib.call("ocsc_code_fused", 4, 42, 42, 100, B, xh.data_ptr(), tr.Wh.data_ptr(), tr.den.data_ptr(), cc.beta, cc.rho,
          cc.max_iters, cc.rel_tol, buf.u.data_ptr(), None, tr._uh.data_ptr(), obj.data_ptr(), None,
          buf.iters.data_ptr(), buf.status.data_ptr(), _lib.stream())
torch.cuda.synchronize()
_lib.call("ocsc_debug_fused_iterations", None)
a = itb.cpu().numpy().astype(np.float64)
ns, ck = a[:300], a[512:812]
dns, dck = np.diff(ns), np.diff(ck)
print(f"iteration ns: median {np.median(dns):.0f} p10 {np.percentile(dns, 10):.0f} p90 {np.percentile(dns, 90):.0f} "
      f"max {dns.max():.0f}; clock64/ns = {np.sum(dck) / np.sum(dns):.3f} GHz; iters 0-299 span {(ns[-1] - ns[0]) / 1e6:.3f} ms")
for lo in range(0, 300, 50):
    print(f"  iters {lo:3d}-{lo + 49:3d}: median {np.median(dns[lo:lo + 49]):.0f} ns, {np.median(dck[lo:lo + 49]):.0f} clk")
allns = a[:512]
last = int(np.nonzero(allns)[0].max())
print(f"iterations recorded: {last + 1}; span all {(allns[last] - allns[0]) / 1e6:.3f} ms; "
      f"timeline sample 0 dur {(t[0, 1] - t[0, 0]) / 1e6:.3f} ms")
fin = a[505:510]
print("final stage (ns after the last iteration start):", [int(x - allns[last]) for x in fin])
