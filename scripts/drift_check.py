"""Float32 prefix-drift check against the CPU oracle at BASELINE config 1 (dev aid).

python scripts/drift_check.py [n_batches B]  (default 2 x 50): the B200 trainer (fused code
ADMM, overlapped history inverse) and the oracle's composed mini-batch (float64 reference
algorithm) learn from the same seeded images; prints the max relative objective error per
mini-batch and the final filter error (float32 drift over long prefixes).
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_06972_b200 as ob  # noqa: E402
from oracle import ocsc_oracle as O  # noqa: E402
from paper_1706_06972_b200.workloads import CONFIGS, synth_images  # noqa: E402

nb, B = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (2, 50)
c = CONFIGS[1]
X = synth_images(nb * B, c["dims0"], c["grid"], c["K0"], seed=7).reshape(nb * B, -1)
kw = dict(beta=1.0, rho_code=1.0, rho_dict=1.0, inner_iters=10, seed=0, code_max_iters=300)
ora = O.Trainer(c["grid"], (11, 11), K=100, **kw)
tr = ob.OnlineTrainer(ob.SignalShape(c["grid"], (11, 11)),
                      ob.TrainConfig(n_filters=100, dtype="float32", batch_size=B, stop_tol=0.0, **kw))
print(f"split plan: main {tr._split_plan(B)} of {B}")
for m in range(nb):
    t0 = time.perf_counter()
    want = np.array([o for _, o in ora.step_batch(X[m * B:(m + 1) * B])])
    t1 = time.perf_counter()
    got = tr.partial_fit(X[m * B:(m + 1) * B]).objectives
    err = float(np.max(np.abs(got - want) / np.abs(want)))
    print(f"mini-batch {m}: max rel objective err {err:.2e} (oracle {t1 - t0:.0f} s)", flush=True)
ff = float(np.linalg.norm(tr.final_filters() - ora.final_filters()) / np.linalg.norm(ora.final_filters()))
print(f"final filters rel Frobenius err {ff:.2e} after {nb * B} samples (tolerances: 1e-4 objective, 1e-3 filters)")
