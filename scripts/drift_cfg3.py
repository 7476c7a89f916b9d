"""Long-horizon float32 drift at BASELINE config 3 (266x266, K = 256, beta = 0.5, B = 32): the
product path in float32 with the complex64 history (the BASELINE sizes: 9.4 GB packed) and the
blocked Cholesky, beside the same build in float64 with the complex128 history (pinned to the
reference at 1e-9 on the config-3 grid by tests/test_config_parity_gpu.py).  Prints, per
checkpoint, the max relative objective error over the mini-batches so far and the relative
Frobenius error of the final filters (north_star bars: 1e-4 and 1e-3).

python scripts/drift_cfg3.py [n_samples [config]]   (default 2,000 = the whole config-3 stream;
config 2: 100x100, K = 100, B = 10, the float64 history and Gauss-Jordan inverse in both builds)
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_06972_b200 as ob  # noqa: E402
from paper_1706_06972_b200.workloads import CONFIGS, synth_images  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000
cid = int(sys.argv[2]) if len(sys.argv) > 2 else 3
c = CONFIGS[cid]
B = c["B"]
kw = dict(n_filters=c["K"], beta=c["beta"], rho_code=1.0, rho_dict=1.0, inner_iters=10, seed=0,
          code_max_iters=300, code_rel_tol=1e-3, batch_size=B, stop_tol=0.0)
if cid == 3:
    kw["history_solver"] = "chol"
shape = ob.SignalShape(c["grid"], (11, 11))
t32 = ob.OnlineTrainer(shape, ob.TrainConfig(dtype="float32", history_dtype="float32" if cid == 3 else "float64", **kw))
t64 = ob.OnlineTrainer(shape, ob.TrainConfig(dtype="float64", history_dtype="float64", **kw))


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


worst, t0, done = 0.0, time.perf_counter(), 0
for start in range(0, n, 256):
    X = synth_images(min(256, n - start), c["dims0"], c["grid"], c["K0"], seed=2024, start=start)
    X = X.reshape(X.shape[0], -1)
    for m in range(0, X.shape[0], B):
        a = t32.partial_fit(X[m:m + B]).objectives
        b = t64.partial_fit(X[m:m + B]).objectives
        worst = max(worst, float(np.max(np.abs(a - b) / np.abs(b))))
    done = start + X.shape[0]
    if done % 512 == 0 or done == n:
        print(f"{done:5d} samples: max rel objective err so far {worst:.2e}; final filters "
              f"{rel(t32.final_filters(), t64.final_filters()):.2e}; {time.perf_counter() - t0:.0f} s", flush=True)
