"""Long-horizon float32 drift at BASELINE config 1 ("drift over 50,000 float32
samples is unmeasured").

python scripts/drift_long.py [n_samples]   (default 50,000 = the whole config-1 pass)

Two trainers learn from the same seeded 32x32 -> 42x42 stream, B = 50: the product path in
float32 (fused cluster kernel, tail split, overlapped float64 history inverse) and the same
build in float64 (pinned to the reference at 1e-9 by tests/test_config_parity_gpu.py, so it is
the reference's trajectory to ~1e-9 and the only reference trajectory that can be run to 50,000
samples: the numpy reference needs ~7 s per sample).  Prints, at checkpoints, the max relative
objective error over the mini-batches so far and the relative Frobenius error of the final and
coding filters (north_star bars: 1e-4 and 1e-3).
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_06972_b200 as ob  # noqa: E402
from paper_1706_06972_b200.workloads import CONFIGS, synth_images  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 50_000
c = CONFIGS[1]
B = 50
kw = dict(n_filters=100, beta=1.0, rho_code=1.0, rho_dict=1.0, inner_iters=10, seed=0, code_max_iters=300,
          batch_size=B, stop_tol=0.0)
shape = ob.SignalShape(c["grid"], (11, 11))
t32 = ob.OnlineTrainer(shape, ob.TrainConfig(dtype="float32", **kw))
t64 = ob.OnlineTrainer(shape, ob.TrainConfig(dtype="float64", **kw))


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


checkpoints = {1_000, 5_000, 10_000, 25_000, 50_000, n}
worst, t0 = 0.0, time.perf_counter()
print(f"float32 path: {t32._split_plan(B) and 'fused+split'}; float64 path: fused={t64.use_fused(B)}", flush=True)
for start in range(0, n, 1000):  # generate in chunks of 1000 images (20 mini-batches)
    X = synth_images(min(1000, n - start), c["dims0"], c["grid"], c["K0"], seed=2024, start=start)
    X = X.reshape(X.shape[0], -1)
    for m in range(0, X.shape[0], B):
        a = t32.partial_fit(X[m:m + B]).objectives
        b = t64.partial_fit(X[m:m + B]).objectives
        worst = max(worst, float(np.max(np.abs(a - b) / np.abs(b))))
    done = start + X.shape[0]
    if done in checkpoints:
        print(f"{done:6d} samples: max rel objective err so far {worst:.2e}; final filters "
              f"{rel(t32.final_filters(), t64.final_filters()):.2e}; coding filters "
              f"{rel(t32.coding_filters(), t64.coding_filters()):.2e}; {time.perf_counter() - t0:.0f} s",
              flush=True)
