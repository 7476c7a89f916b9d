"""Pin the CPU oracle (oracle/ocsc_oracle.py) to golden vectors the reference produced.

CPU-only: these run in `pytest -m "not gpu"`.  The golden files were written
by tests/golden/make_golden.py with the reference `ocsc` package imported.
"""

import numpy as np
import pytest

from oracle import ocsc_oracle as O
from paper_1706_06972_b200.workloads import synth_images
from tests._layout import cols_to_planes, hw, planes_to_cols, rel


def test_primitives(golden):
    g = golden("primitives")
    # solve_code_rows works per row; the oracle takes planes -> use a (K, 1, P) view
    d, x, t = g["d"], g["x"], g["t"]
    got = O.code_solve(d.T[:, None, :], x[None, :], t.T[:, None, :], float(g["rho"]))
    assert np.abs(got[:, 0, :].T - g["rows"]).max() < 1e-12
    assert np.array_equal(O.shrink(g["v"], float(g["kappa"])), g["st"])
    H, W = hw(g["dims"])
    planes = cols_to_planes(g["cols"], g["dims"])
    assert np.abs(planes_to_cols(O.fwd(planes)) - g["fcols"]).max() < 1e-12
    M0, M1 = hw(g["fdims"])
    padded = O.pad(g["filt"], H, W, M0, M1)
    assert np.array_equal(planes_to_cols(padded), g["padded"])
    proj = O.project(O.fwd(padded * 3.0), M0, M1)
    assert np.abs(planes_to_cols(proj) - g["proj"]).max() < 1e-12


@pytest.mark.parametrize("name", ["code_2d", "code_1d", "code_odd"])
def test_code_admm(golden, name):
    g = golden(name)
    H, W = hw(g["dims"])
    dh = cols_to_planes(g["dict_freq"], g["dims"])
    trace = []
    st = O.code_admm(g["x"], dh, float(g["beta"]), float(g["rho"]), int(g["max_iters"]),
                     float(g["rel_tol"]),
                     monitor=lambda it, c: trace.append(O.objective(g["x"], dh, c, float(g["beta"]))))
    assert st["iterations"] == int(g["iterations"])
    assert rel(planes_to_cols(st["code"]), g["code"]) < 1e-11
    assert rel(planes_to_cols(st["dual"]), g["dual"]) < 1e-11
    assert rel(planes_to_cols(st["zh"]), g["z_freq"]) < 1e-11
    assert np.allclose(trace, g["trace"], rtol=1e-12, atol=1e-14)


def test_history_sequence(golden):
    g = golden("history")
    H, W = hw(g["dims"])
    K = int(g["K"])
    h = O.History(K, H, W, float(g["rho"]))
    for i in range(len(g["z"])):
        h.fold(cols_to_planes(g["z"][i], g["dims"]), g["x"][i].reshape(H, W))
        assert np.abs(planes_to_cols(h.cross) - g["cross"][i]).max() < 1e-13
        assert np.abs(h.inv.reshape(H * W, K, K) - g["inv"][i]).max() < 1e-13
    hc = O.History(2, 1, 5, 0.8)
    for zc, xc in zip(g["zc"], g["xc"]):
        hc.fold(zc.T.reshape(2, 1, 5), xc.reshape(1, 5))
    assert np.abs(hc.inv.reshape(5, 2, 2) - g["inv_c"]).max() < 1e-13


def test_history_rejects_nonfinite():
    h = O.History(2, 1, 4, 1.0)
    bad = np.ones((2, 1, 4), complex)
    bad[0, 0, 0] = np.nan
    with pytest.raises(O.OracleDivergence):
        h.fold(bad, np.ones((1, 4), complex))
    assert h.count == 0


def test_dictionary_admm(golden):
    g = golden("dictionary")
    H, W = hw(g["dims"])
    M0, M1 = hw(g["fdims"])
    K = int(g["K"])
    h = O.History(K, H, W, float(g["rho"]))
    for z, x in zip(g["z"], g["x"]):
        h.fold(cols_to_planes(z, g["dims"]), x.reshape(H, W))
    v0 = O.pad(g["filters"], H, W, M0, M1)
    rounds = []
    dh, v, th = O.dict_admm(O.fwd(v0), v0, h, 5, M0, M1, monitor=lambda t, f, vv: rounds.append(f))
    assert rel(planes_to_cols(dh), g["freq"]) < 1e-12
    assert rel(planes_to_cols(v), g["v"]) < 1e-12
    assert rel(planes_to_cols(th), g["dual"]) < 1e-11
    for a, b in zip(rounds, g["rounds"]):
        assert rel(planes_to_cols(a), b) < 1e-12
    rows = O.dict_rows(h, cols_to_planes(g["rows_v"], g["dims"]), cols_to_planes(g["rows_dual"], g["dims"]))
    assert rel(planes_to_cols(rows), g["rows"]) < 1e-12


def test_dictionary_requires_history():
    h = O.History(2, 1, 4, 1.0)
    with pytest.raises(O.OracleUninitialized):
        O.dict_admm(np.zeros((2, 1, 4), complex), np.zeros((2, 1, 4)), h, 3, 1, 2)


def _trainer_from(g):
    return O.Trainer(tuple(g["dims"]), tuple(g["fdims"]), K=int(g["K"]), beta=float(g["beta"]),
                     rho_code=float(g["rho_code"]), rho_dict=float(g["rho_dict"]),
                     inner_iters=int(g["inner_iters"]), seed=int(g["seed"]),
                     code_max_iters=int(g["code_max_iters"]), code_rel_tol=float(g["code_rel_tol"]))


@pytest.mark.parametrize("name", ["train_2d", "train_odd", "train_14"])
def test_trainer_steps(golden, name):
    g = golden(name)
    tr = _trainer_from(g)
    for i, x in enumerate(g["X"]):
        (st, obj), = tr.step_batch(x[None])
        assert st["iterations"] == int(g["iterations"][i])
        assert abs(obj - g["objectives"][i]) <= 1e-11 * abs(g["objectives"][i])
        assert rel(planes_to_cols(st["code"]), g["codes"][i]) < 1e-10
    assert rel(tr.final_filters(), g["final_filters"]) < 1e-11
    assert rel(tr.coding_filters(), g["coding_filters"]) < 1e-11
    assert rel(planes_to_cols(tr.working), g["working_freq"]) < 1e-11
    K = int(g["K"])
    assert rel(tr.hist.inv.reshape(-1, K, K), g["inv_gram"]) < 1e-11
    assert abs(tr.dict_change - float(g["dict_change"])) < 1e-9


def test_minibatch_composition(golden):
    g = golden("minibatch")
    tr = _trainer_from(g)
    B = int(g["B"])
    objs = []
    for m in range(len(g["X"]) // B):
        objs.extend(o for _, o in tr.step_batch(g["X"][m * B:(m + 1) * B]))
    assert np.allclose(objs, g["objectives"], rtol=1e-11)
    assert rel(tr.final_filters(), g["final_filters"]) < 1e-11


def test_train_online_passes(golden):
    g = golden("train_online")
    kw = dict(K=2, beta=0.5, seed=3, inner_iters=5, code_max_iters=100, rho_dict=10.0)
    rep = O.train_online(g["X"], tuple(g["dims"]), tuple(g["fdims"]), max_passes=3, stop_tol=1e-12, **kw)
    assert np.allclose([r[1] for r in rep["records"]], g["train_obj"], rtol=1e-11)
    assert rel(rep["filters"], g["filters"]) < 1e-10
    rep2 = O.train_online(g["X"], tuple(g["dims"]), tuple(g["fdims"]), max_passes=5, stop_tol=0.5, **kw)
    assert rep2["stopped_early"] == bool(g["stopped2"])
    assert np.allclose([r[1] for r in rep2["records"]], g["train_obj2"], rtol=1e-11)


def test_synth_images_standardised():
    X = synth_images(3, (32, 32), (42, 42), 20, seed=0)
    assert X.shape == (3, 42, 42)
    core = X[:, :32, :32].reshape(3, -1)
    assert np.allclose(core.mean(axis=1), 0, atol=1e-12)
    assert np.allclose(core.std(axis=1), 1, atol=1e-12)
    assert not X[:, 32:, :].any() and not X[:, :, 32:].any()
    assert np.array_equal(X, synth_images(3, (32, 32), (42, 42), 20, seed=0))


def test_oracle_config0_full_size(golden):
    """BASELINE config 0 (100x100, K=100, f64, rho=1) step 1: the oracle vs the reference run (~50 s)."""
    g = golden("cfg0")
    tr = O.Trainer((100, 100), (11, 11), K=100, beta=1.0, rho_code=1.0, rho_dict=1.0, inner_iters=10, seed=0)
    (st, obj), = tr.step_batch(g["X"][:1])
    assert st["iterations"] == int(g["iterations"][0])
    assert abs(obj - g["objectives"][0]) <= 1e-12 * abs(g["objectives"][0])
    code = np.zeros(100 * 100 * 100)
    code[g["code_idx"]] = g["code_val"]
    assert rel(planes_to_cols(st["code"]).ravel(), code) < 1e-11
    assert rel(tr.final_filters(), g["final_filters"]) < 1e-11


def test_oracle_preprocessing_matches_reference(golden):
    g = golden("preprocess")

    def close(a, b):
        return np.abs(a - b).max() <= 1e-12 * max(np.abs(b).max(), 1.0)

    assert close(O.gray(g["rgb"]), g["gray_rgb"])
    assert close(O.preprocess(g["rgb"], seed=3), g["pre_rgb"])
    assert close(O.preprocess(g["gray"]), g["pre_gray"])
    assert close(O.preprocess(g["tiny"], seed=1), g["pre_tiny"])  # window > image: repeated reflection
    assert close(O.lcn(g["gray"], 8, 2.0), g["lcn_even"])  # even window, off-centre kernel
    assert close(O.lcn(g["tiny"], 9, 3.0, 1e-2), g["lcn_tiny"])
    assert close(O.taper(g["small"], 7, 1.5), g["taper_small"])
    assert close(O.taper(g["gray"], 6, 1.0), g["taper_even"])
    for i, im in enumerate(g["stack"]):
        assert close(O.preprocess(im, seed=5 + i), g["pre_stack"][i])


@pytest.mark.parametrize("name", ["cfg1_mb", "cfg2_mb", "cfg3_mb"])
def test_config_golden_inputs_regenerate(golden, name):
    """The BASELINE-config golden files store no images: the seeded workload generator must
    reproduce the exact inputs the reference was run on (sha256 pinned at generation)."""
    import hashlib
    import os

    from tests.conftest import GOLDEN

    if not os.path.exists(os.path.join(GOLDEN, f"{name}.npz")):
        pytest.skip(f"{name} not generated")
    g = golden(name)
    B, n = int(g["B"]), len(g["objectives"])
    X = synth_images(n, tuple(g["dims0"]), tuple(g["grid"]), int(g["K0"]), seed=int(g["seed"]))
    assert hashlib.sha256(X.tobytes()).hexdigest() == str(g["x_sha256"])
    assert n % B == 0 and g["batch_filters"].shape[0] == n // B
