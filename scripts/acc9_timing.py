"""Dev aid: timing anatomy of reference acceptance criterion 9 (online vs batch wall time) on
this build -- batch outer-iteration time, per-step online latency, crossing index."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [os.path.join(ROOT, "tests", "ref_suite", "shim"), ROOT]
import torch  # noqa: E402

from ocsc import SignalShape, TrainConfig  # noqa: E402
from ocsc.evaluate import evaluate_dictionary  # noqa: E402
from ocsc.synthetic import synth_generate  # noqa: E402
from ocsc.training import OnlineTrainer, train  # noqa: E402

shape = SignalShape((64, 64), (8, 8))
k = 8
for seed in (0, 1, 2):
    data = synth_generate(shape, k, 54, seed=100 + seed, noise=0.01)
    train_x, test_x = data.consistent[:50], data.consistent[50:]
    cfg = TrainConfig(n_filters=k, beta=1.0, max_passes=1, stop_tol=0.0, code_max_iters=100, code_rel_tol=1e-3,
                      seed=seed)
    batch = train("batch", train_x, shape, cfg, test_samples=test_x)
    target = batch.records[0].test_obj
    tr = OnlineTrainer(shape, cfg)
    order = tr.rng.permutation(50)
    snaps, times, el = [], [], 0.0
    for j in range(12):
        t0 = time.perf_counter()
        st = tr.step(train_x[order[j % 50]])
        el += time.perf_counter() - t0
        times.append(el)
        snaps.append(tr.coding_filters().copy())
    cross = next((j for j in range(12) if evaluate_dictionary(snaps[j], test_x, shape, cfg.coding()).test_objective
                  <= target), None)
    steps = [times[0]] + [b - a for a, b in zip(times, times[1:])]
    print(f"seed {seed}: batch {batch.records[0].time_s * 1e3:.1f} ms, steps ms {[round(s * 1e3, 2) for s in steps]}, "
          f"crossing {cross}, last iterations {st.iterations}", flush=True)
