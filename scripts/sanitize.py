"""Small invocations of the risky kernels for compute-sanitizer (racecheck / synccheck / memcheck).

    compute-sanitizer --tool racecheck python scripts/sanitize.py fused|claim|tc|stream|chol

fused  : k_code_fused on a 14x14 grid, 3-CTA clusters (DSMEM push model, cluster barriers)
claim  : ocsc_history_invert_claim, two launches sharing the claim counter (persistent GJ)
tc     : k_hist_accum_tc (tcgen05 3xTF32: TMEM, mbarriers, async MMA)
stream : the streaming row/column kernels + k_plane (100x100, float32)
chol   : blocked Cholesky + row solve with a padded K (K = 40)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1706_06972_b200 as ob  # noqa: E402
from paper_1706_06972_b200 import _lib  # noqa: E402
from paper_1706_06972_b200.workloads import synth_images  # noqa: E402

what = sys.argv[1]
if what == "fused":
    os.environ["OCSC_FUSED_CS"] = "3"
    shape = ob.SignalShape((14, 14), (3, 3))
    X = synth_images(2, (14, 14), (14, 14), 3, filter_dims=(3, 3), seed=1, density=0.05).reshape(2, -1)
    tr = ob.OnlineTrainer(shape, ob.TrainConfig(n_filters=7, batch_size=2, dtype="float32", code_max_iters=8,
                                                inner_iters=1, stop_tol=0.0))
    assert tr.use_fused(2)
    print(tr.partial_fit(X).objectives)
elif what == "claim":
    K, nf = 40, 7
    g = torch.Generator(device="cuda").manual_seed(3)
    Z = torch.randn(nf, K, 2 * K, dtype=torch.complex128, device="cuda", generator=g)
    A = Z @ Z.conj().transpose(1, 2)
    ii, jj = torch.tril_indices(K, K)
    S = A[:, ii, jj].contiguous()
    inv = torch.empty_like(S)
    info = torch.zeros(2, dtype=torch.int32, device="cuda")
    ctr = torch.zeros(1, dtype=torch.int32, device="cuda")
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        _lib.call("ocsc_history_invert_claim", _lib.F64, _lib.F64, K, nf, _lib.ptr(S), 3.0, 1.0, _lib.ptr(inv),
                  _lib.ptr(info), _lib.ptr(ctr), 2, _lib.stream())
    _lib.call("ocsc_history_invert_claim", _lib.F64, _lib.F64, K, nf, _lib.ptr(S), 3.0, 1.0, _lib.ptr(inv),
              _lib.ptr(info), _lib.ptr(ctr), 8, _lib.stream())
    torch.cuda.synchronize()
    print(int(info[0]), float(inv.abs().max()))
elif what == "tc":
    K, B, nf = 128, 16, 3
    g = torch.Generator(device="cuda").manual_seed(1)
    z = torch.complex(torch.randn(B, nf, K, device="cuda", generator=g), torch.randn(B, nf, K, device="cuda", generator=g))
    x = torch.complex(torch.randn(B, nf, device="cuda", generator=g), torch.randn(B, nf, device="cuda", generator=g))
    h = ob.HistoryState(ob.SignalShape((nf,), (1,)), K, 1.0, nfreq=nf, dtype=torch.complex128)
    h.accumulate(z, (nf * K, 1, K), x, (nf, 1), B)
    torch.cuda.synchronize()
    print(float(h.S.abs().max()))
elif what == "stream":
    shape = ob.SignalShape((100, 100), (11, 11))
    X = synth_images(2, (90, 90), (100, 100), 3, seed=5).reshape(2, -1)
    tr = ob.OnlineTrainer(shape, ob.TrainConfig(n_filters=8, batch_size=2, dtype="float32", code_max_iters=4,
                                                inner_iters=1, stop_tol=0.0))
    print(tr.partial_fit(X).objectives, tr.last_path)
elif what == "chol":
    K, nf, B = 40, 3, 5
    h = ob.HistoryState(ob.SignalShape((nf,), (1,)), K, 1.0, solver="chol")
    rng = np.random.default_rng(0)
    z = torch.as_tensor(rng.normal(size=(B, nf, K)) + 1j * rng.normal(size=(B, nf, K)), device="cuda")
    x = torch.as_tensor(rng.normal(size=(B, nf)) + 1j * rng.normal(size=(B, nf)), device="cuda")
    h.accumulate(z, (nf * K, 1, K), x, (nf, 1), B)
    v = torch.zeros(nf, K, dtype=torch.complex128, device="cuda")
    print(float(h.rowsolve(v, v, 1, K, torch.empty_like(v)).abs().max()))
else:
    raise SystemExit(f"unknown case {what}")
