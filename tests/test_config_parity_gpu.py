"""BASELINE configurations' own device paths against the reference (golden vectors).

Golden files `cfg1_mb`, `cfg2_mb`, `cfg3_mb` (tests/golden/make_golden.py) hold the composed
mini-batch semantics computed by the REFERENCE package in float64 on each
config's shapes; `cfg0` is the reference's `OnlineTrainer.step` at config 0's full size.  Every
test asserts which device path ran (`OnlineTrainer.last_path`) so the parity claim is about
the product kernels of that configuration:

  cfg0  100x100, K=100, f64, B=1   streaming FFT kernels (k_rows / k_cols_f / k_cols_i)
  cfg1  42x42,  K=100, B=50        fused cluster kernel + tail split + overlapped inverse (f32)
  cfg2  100x100, K=100, B=10       f32: plane-resident k_plane + inverse beside coding; f64: stream
  cfg3  266x266, K=32 (chol), B=4  streaming 266-point kernels + blocked Cholesky (c64 / c128)
  cfg3  266x266, K=256, B=32       full size, float32 + complex64 history vs the float64 build

Bars (north_star): float64 1e-9 relative; float32 objective trace 1e-4, filters 1e-3 relative
Frobenius.  Reference semantics: coding.py:67-119, dictionary.py:73-114, 176-215,
training.py:128-155.
"""

import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - collected on CPU boxes
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1706_06972_b200 as ob  # noqa: E402
from paper_1706_06972_b200.workloads import synth_images  # noqa: E402
from tests._layout import rel  # noqa: E402

TOL64 = 1e-9
TOL32_OBJ, TOL32_FILT = 1e-4, 1e-3


def _inputs(g):
    B, nb = int(g["B"]), len(g["objectives"]) // int(g["B"])
    X = synth_images(B * nb, tuple(g["dims0"]), tuple(g["grid"]), int(g["K0"]), seed=int(g["seed"]))
    assert hashlib.sha256(X.tobytes()).hexdigest() == str(g["x_sha256"]), "workload generator drifted"
    return X.reshape(B * nb, -1), B, nb


def _trainer(g, dtype, **kw):
    shape = ob.SignalShape(tuple(int(d) for d in g["grid"]), (11, 11))
    hist = kw.pop("history_dtype", "float64")
    cfg = ob.TrainConfig(n_filters=int(g["K"]), beta=float(g["beta"]), rho_code=1.0, rho_dict=1.0, inner_iters=10,
                         seed=0, code_max_iters=300, code_rel_tol=1e-3, batch_size=int(g["B"]), stop_tol=0.0,
                         dtype=dtype, history_dtype=hist, **kw)
    return ob.OnlineTrainer(shape, cfg)


def _run(g, tr, path, tol_obj, tol_filt, exact_iters):
    X, B, nb = _inputs(g)
    objs, iters = [], []
    for m in range(nb):
        res = tr.partial_fit(X[m * B:(m + 1) * B])
        if path is not None:
            assert tr.last_path == path, f"expected the {path} path, ran {tr.last_path}"
        objs.extend(res.objectives)
        iters.extend(res.iterations)
        assert rel(tr.final_filters(), g["batch_filters"][m]) < tol_filt, f"filters after mini-batch {m}"
    want = g["objectives"]
    err = np.max(np.abs(np.asarray(objs) - want) / np.abs(want))
    assert err < tol_obj, f"objective trace rel err {err:.3e}"
    if exact_iters:
        assert np.array_equal(np.asarray(iters), g["iterations"])
    assert rel(tr.final_filters(), g["final_filters"]) < tol_filt
    assert rel(tr.coding_filters(), g["coding_filters"]) < tol_filt
    return err


# ----------------------------------------------------------------- config 0 --

def test_config0_stream_path_matches_reference(golden):
    """Config 0 (100x100, K=100, f64, B=1) through partial_fit -- the float64 streaming kernels,
    not the want_z cuFFT path `step` uses -- against the reference's OnlineTrainer.step."""
    g = golden("cfg0")
    shape = ob.SignalShape((100, 100), (11, 11))
    cfg = ob.TrainConfig(n_filters=100, beta=1.0, rho_code=1.0, rho_dict=1.0, inner_iters=10, seed=0)
    tr = ob.OnlineTrainer(shape, cfg)
    res = tr.partial_fit(g["X"][0])
    assert tr.last_path == "stream"
    assert int(res.iterations[0]) == int(g["iterations"][0])
    assert abs(res.objectives[0] - g["objectives"][0]) <= TOL64 * abs(g["objectives"][0])
    code = np.zeros(shape.size * 100)
    code[g["code_idx"]] = g["code_val"]
    got = res.codes[0].reshape(100, -1).cpu().numpy().T.ravel()
    assert rel(got, code) < TOL64
    assert rel(tr.final_filters(), g["final_filters"]) < TOL64
    assert rel(tr.coding_filters(), g["coding_filters"]) < TOL64


# ----------------------------------------------------------------- config 1 --

def test_config1_headline_plan_matches_reference(golden):
    """The headline plan (float32 fused cluster kernel, 45 + 5 split, side-stream inverse of the
    main part, Woodbury refresh with the tail; float64 history) on two full B=50 mini-batches."""
    g = golden("cfg1_mb")
    tr = _trainer(g, "float32")
    assert tr._split_plan(50) > 0
    _run(g, tr, "fused+split", TOL32_OBJ, TOL32_FILT, exact_iters=False)


def test_config1_float64_matches_reference(golden):
    g = golden("cfg1_mb")
    tr = _trainer(g, "float64")
    _run(g, tr, None, TOL64, TOL64, exact_iters=True)   # fused f64 cluster kernel or cuFFT, whichever fits


# ----------------------------------------------------------------- config 2 --

def test_config2_plane_kernel_with_inverse_beside_matches_reference(golden):
    """Config 2 float32: k_plane (a (sample, filter) plane per CTA on chip) with the persistent
    Gauss-Jordan inverse on the idle SMs and the Woodbury fold."""
    g = golden("cfg2_mb")
    tr = _trainer(g, "float32")
    assert tr._invert_beside_plan(10) > 0
    _run(g, tr, "stream+beside", TOL32_OBJ, TOL32_FILT, exact_iters=False)


def test_config2_float64_stream_matches_reference(golden):
    g = golden("cfg2_mb")
    tr = _trainer(g, "float64")
    _run(g, tr, "stream", TOL64, TOL64, exact_iters=True)


# ----------------------------------------------------------------- config 3 --

def test_config3_grid_cholesky_complex64_matches_reference(golden):
    """Config 3's 266x266 grid, float32 codes, complex64 history (BASELINE's history precision),
    blocked Cholesky solver (the K=256 path), on a K the reference can hold in memory."""
    g = golden("cfg3_mb")
    tr = _trainer(g, "float32", history_dtype="float32", history_solver="chol")
    assert tr.history.solver == "chol" and tr.history.S.dtype == torch.complex64
    _run(g, tr, "stream", TOL32_OBJ, TOL32_FILT, exact_iters=False)


def test_config3_grid_float64_cholesky_matches_reference(golden):
    g = golden("cfg3_mb")
    tr = _trainer(g, "float64", history_solver="chol")
    _run(g, tr, "stream", TOL64, TOL64, exact_iters=True)


def test_config3_full_size_float32_against_float64():
    """BASELINE config 3 at its full size (266x266, K = 256, B = 32: the 9.4 GB complex64 history and
    the 128-wide blocked Cholesky of the product path) for two mini-batches against the float64 /
    complex128 build of the same path, whose 266x266 kernels and Cholesky are pinned to the
    reference above (test_config3_grid_float64_cholesky_matches_reference).  north_star float32 bars;
    scripts/drift_cfg3.py runs the whole 2,000-sample stream (profiles/r2_drift_cfg3.txt)."""
    from paper_1706_06972_b200.workloads import CONFIGS

    c = CONFIGS[3]
    shape = ob.SignalShape(c["grid"], (11, 11))
    kw = dict(n_filters=c["K"], beta=c["beta"], rho_code=1.0, rho_dict=1.0, inner_iters=10, seed=0,
              code_max_iters=300, code_rel_tol=1e-3, batch_size=c["B"], stop_tol=0.0, history_solver="chol")
    t32 = ob.OnlineTrainer(shape, ob.TrainConfig(dtype="float32", history_dtype="float32", **kw))
    t64 = ob.OnlineTrainer(shape, ob.TrainConfig(dtype="float64", history_dtype="float64", **kw))
    X = synth_images(2 * c["B"], c["dims0"], c["grid"], c["K0"], seed=2024).reshape(2 * c["B"], -1)
    for m in range(2):
        xb = X[m * c["B"]:(m + 1) * c["B"]]
        a = t32.partial_fit(xb)
        b = t64.partial_fit(xb)
        assert t32.last_path == "stream" and t64.last_path == "stream"
        assert np.max(np.abs(a.objectives - b.objectives) / np.abs(b.objectives)) < TOL32_OBJ
    assert rel(t32.final_filters(), t64.final_filters()) < TOL32_FILT
    del t32, t64
    torch.cuda.empty_cache()
