"""Quick timing of the cfg1 mini-batch step (development aid, not the bench)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1706_06972_b200 as ob
from oracle import ocsc_oracle as O
from paper_1706_06972_b200.workloads import CONFIGS, synth_images  # noqa: E402

c = CONFIGS[1]
B = 50
X = synth_images(B * 4, c["dims0"], c["grid"], c["K0"], seed=1).reshape(B * 4, -1)
shape = ob.SignalShape(c["grid"], (11, 11))
cfg = ob.TrainConfig(n_filters=100, beta=1.0, rho_code=1.0, rho_dict=1.0, inner_iters=10, seed=0,
                     dtype="float32", history_dtype=os.environ.get("HD", "float64"), batch_size=B, stop_tol=0.0)
tr = ob.OnlineTrainer(shape, cfg)
for m in range(2):
    r = tr.partial_fit(X[m * B:(m + 1) * B])
torch.cuda.synchronize()
print("iters", r.iterations[:5], "obj", r.objectives[:3])
t0 = time.perf_counter()
for m in range(2, 4):
    r = tr.partial_fit(X[m * B:(m + 1) * B])
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 2
print(f"cfg1 step {dt*1e3:.2f} ms -> {B/dt:.1f} img/s")
# phase split
from paper_1706_06972_b200.coding import infer_codes
xs = torch.as_tensor(X[:B].reshape(B, 42, 42), dtype=torch.float32).cuda()
from paper_1706_06972_b200.transforms import rfft2_dev
xh = rfft2_dev(xs, shape)
buf = tr._buf
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); infer_codes(xh, tr.Wh, tr.den, shape, tr.coding_config, buf, B, poll=0); e1.record(); torch.cuda.synchronize()
print(f"code admm {e0.elapsed_time(e1):.2f} ms ({e0.elapsed_time(e1)/300*1e3:.1f} us/iter)")
e0.record(); tr._dictionary_update(); e1.record(); torch.cuda.synchronize()
print(f"dict update {e0.elapsed_time(e1):.2f} ms")
e0.record(); tr.history._inv_count = -1; tr.history.inverse(check=False); e1.record(); torch.cuda.synchronize()
print(f"hist invert {e0.elapsed_time(e1):.2f} ms")
