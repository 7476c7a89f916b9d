"""Generate golden vectors by running the REFERENCE package `ocsc` itself.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

Every input and output lands in tests/golden/*.npz, so the checks that read
them (tests/test_oracle_golden.py on CPU, tests/test_parity_gpu.py on the
B200) never need /root/reference at run time.  Reference layouts are kept:
columns are (P, K) with K fastest, spectra are full complex, inv_gram is
(P, K, K).
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import ocsc  # noqa: E402  (the reference, via PYTHONPATH)
from ocsc.training import OnlineTrainer  # noqa: E402

from paper_1706_06972_b200.workloads import synth_images  # noqa: E402  (inputs only)

assert "reference" in ocsc.__file__, f"expected the reference ocsc, got {ocsc.__file__}"


def save(name, **arrays):
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} B)")


def case_primitives():
    rng = np.random.default_rng(1001)
    P, K = 7, 4
    d = rng.normal(size=(P, K)) + 1j * rng.normal(size=(P, K))
    x = rng.normal(size=P) + 1j * rng.normal(size=P)
    t = rng.normal(size=(P, K)) + 1j * rng.normal(size=(P, K))
    rows = ocsc.solve_code_rows(d, x, t, 1.7)
    v = rng.normal(size=50) * 2
    st = ocsc.soft_threshold(v, 0.6)
    shape = ocsc.SignalShape((6, 5), (2, 3))
    cols = rng.normal(size=(30, 3))
    fcols = ocsc.forward_dft_cols(cols, shape)
    filt = rng.normal(size=(6, 3))
    padded = ocsc.pad_filter_cols(filt, shape)
    proj = ocsc.project_filter_cols(ocsc.forward_dft_cols(padded * 3.0, shape), shape)
    save("primitives", d=d, x=x, t=t, rho=1.7, rows=rows, v=v, kappa=0.6, st=st,
         dims=shape.dims, fdims=shape.filter_dims, cols=cols, fcols=fcols,
         filt=filt, padded=padded, proj=proj)


def case_code(name, dims, fdims, K, seed, cfg, x_scale=1.0):
    rng = np.random.default_rng(seed)
    shape = ocsc.SignalShape(dims, fdims)
    filters = rng.normal(size=(shape.filter_size, K))
    filters /= np.linalg.norm(filters, axis=0)
    x = rng.normal(size=shape.size) * x_scale
    dict_freq = ocsc.forward_dft_cols(ocsc.pad_filter_cols(filters, shape), shape)
    trace = []
    st = ocsc.infer_code(x, dict_freq, shape, cfg,
                         monitor=lambda it, code: trace.append(
                             ocsc.coding_objective(x, dict_freq, code, shape, cfg.beta)))
    obj = ocsc.coding_objective(x, dict_freq, st.code, shape, cfg.beta)
    save(name, dims=shape.dims, fdims=shape.filter_dims, filters=filters, x=x,
         dict_freq=dict_freq, beta=cfg.beta, rho=cfg.rho, max_iters=cfg.max_iters,
         rel_tol=cfg.rel_tol, z_freq=st.z_freq, code=st.code, dual=st.dual,
         iterations=st.iterations, trace=np.array(trace), objective=obj)


def case_history():
    rng = np.random.default_rng(1003)
    shape = ocsc.SignalShape((6,), (2,))
    K, T, rho = 3, 4, 1.5
    h = ocsc.empty_history(shape, K, rho=rho)
    zs, xs, crosses, invs = [], [], [], []
    for _ in range(T):
        zf = ocsc.forward_dft_cols(rng.normal(size=(shape.size, K)), shape)
        xf = ocsc.forward_dft(rng.normal(size=shape.size), shape)
        ocsc.update_history(h, zf, xf)
        zs.append(zf), xs.append(xf), crosses.append(h.cross.copy()), invs.append(h.inv_gram.copy())
    # arbitrary (non-Hermitian) complex spectra exercise the full-spectrum API path
    h2 = ocsc.empty_history(ocsc.SignalShape((5,), (2,)), 2, rho=0.8)
    zc, xc = [], []
    for _ in range(3):
        zf = rng.normal(size=(5, 2)) + 1j * rng.normal(size=(5, 2))
        xf = rng.normal(size=5) + 1j * rng.normal(size=5)
        ocsc.update_history(h2, zf, xf)
        zc.append(zf), xc.append(xf)
    save("history", dims=shape.dims, fdims=shape.filter_dims, K=K, rho=rho,
         z=np.array(zs), x=np.array(xs), cross=np.array(crosses), inv=np.array(invs),
         zc=np.array(zc), xc=np.array(xc), cross_c=h2.cross, inv_c=h2.inv_gram)


def case_dictionary():
    rng = np.random.default_rng(1004)
    shape = ocsc.SignalShape((8, 6), (3, 2))
    K, rho = 3, 2.0
    h = ocsc.empty_history(shape, K, rho=rho)
    zs, xs = [], []
    for _ in range(4):
        zf = ocsc.forward_dft_cols(rng.normal(size=(shape.size, K)), shape)
        xf = ocsc.forward_dft(rng.normal(size=shape.size), shape)
        ocsc.update_history(h, zf, xf)
        zs.append(zf), xs.append(xf)
    filters = ocsc.init_dictionary(shape, K, 7)
    d0 = ocsc.dict_state_from_filters(filters, shape)
    rounds = []
    d1 = ocsc.update_dictionary(d0, h, 5, monitor=lambda tau, f, v: rounds.append(f.copy()))
    rows = ocsc.solve_dict_rows(h, d0.freq * 0.5, d0.freq * 0.1)
    save("dictionary", dims=shape.dims, fdims=shape.filter_dims, K=K, rho=rho,
         z=np.array(zs), x=np.array(xs), filters=filters, freq=d1.freq, v=d1.v,
         dual=d1.dual, rounds=np.array(rounds), rows=rows,
         rows_v=d0.freq * 0.5, rows_dual=d0.freq * 0.1)


def case_trainer(name, dims, fdims, K, n, steps, seed=0, **cfgkw):
    shape = ocsc.SignalShape(dims, fdims)
    grid = dims if len(dims) == 2 else (1, dims[0])
    X = synth_images(n, grid, grid, 3, filter_dims=fdims if len(fdims) == 2 else (1, fdims[0]),
                     seed=seed + 11, density=0.05).reshape(n, -1)
    cfg = ocsc.TrainConfig(n_filters=K, seed=seed, **cfgkw)
    tr = OnlineTrainer(shape, cfg)
    objs, codes, iters = [], [], []
    for i in range(steps):
        st = tr.step(X[i])
        objs.append(tr.last_objective), codes.append(st.code), iters.append(st.iterations)
    save(name, dims=shape.dims, fdims=shape.filter_dims, K=K, X=X[:steps],
         beta=cfg.beta, rho_code=cfg.rho_code, rho_dict=cfg.rho_dict,
         inner_iters=cfg.inner_iters, code_max_iters=cfg.code_max_iters,
         code_rel_tol=cfg.code_rel_tol, seed=seed,
         objectives=np.array(objs), codes=np.array(codes), iterations=np.array(iters),
         final_filters=tr.final_filters(), coding_filters=tr.coding_filters(),
         working_freq=tr.working_freq, cross=tr.history.cross, inv_gram=tr.history.inv_gram,
         code_change=tr.code_change, dict_change=tr.dict_change)


def case_minibatch(name, dims, fdims, K, B, nbatches, seed=0, **cfgkw):
    """Composed mini-batch semantics built from reference calls only."""
    shape = ocsc.SignalShape(dims, fdims)
    X = synth_images(B * nbatches, dims, dims, 3, filter_dims=fdims, seed=seed + 5,
                     density=0.05).reshape(B * nbatches, -1)
    cfg = ocsc.TrainConfig(n_filters=K, seed=seed, **cfgkw)
    tr = OnlineTrainer(shape, cfg)
    coding = cfg.coding()
    objs, codes = [], []
    for m in range(nbatches):
        batch = X[m * B:(m + 1) * B]
        states = [ocsc.infer_code(x, tr.working_freq, shape, coding) for x in batch]
        for x, st in zip(batch, states):
            objs.append(ocsc.coding_objective(x, tr.working_freq, st.code, shape, cfg.beta))
            codes.append(st.code)
        for x, st in zip(batch, states):
            ocsc.update_history(tr.history, ocsc.forward_dft_cols(st.code, shape),
                                ocsc.forward_dft(x, shape))
        tr.dict_state = ocsc.update_dictionary(tr.dict_state, tr.history, cfg.inner_iters)
        tr.working_freq = ocsc.forward_dft_cols(tr.dict_state.v, shape)
    save(name, dims=shape.dims, fdims=shape.filter_dims, K=K, B=B, X=X,
         beta=cfg.beta, rho_code=cfg.rho_code, rho_dict=cfg.rho_dict,
         inner_iters=cfg.inner_iters, code_max_iters=cfg.code_max_iters,
         code_rel_tol=cfg.code_rel_tol, seed=seed, objectives=np.array(objs),
         codes=np.array(codes), final_filters=tr.final_filters(),
         coding_filters=tr.coding_filters())


def case_train_online():
    shape = ocsc.SignalShape((32,), (4,))
    X = synth_images(8, (1, 32), (1, 32), 2, filter_dims=(1, 4), seed=19, density=0.1).reshape(8, 32)
    cfg = ocsc.TrainConfig(n_filters=2, beta=0.5, seed=3, max_passes=3, stop_tol=1e-12,
                           inner_iters=5, code_max_iters=100)
    rep = ocsc.train_online(X, shape, cfg)
    cfg2 = ocsc.TrainConfig(n_filters=2, beta=0.5, seed=3, max_passes=5, stop_tol=0.5,
                            inner_iters=5, code_max_iters=100)
    rep2 = ocsc.train_online(X, shape, cfg2)
    save("train_online", dims=shape.dims, fdims=shape.filter_dims, X=X,
         train_obj=np.array([r.train_obj for r in rep.records]), filters=rep.filters,
         snapshot=np.array([r.snapshot_id for r in rep.records]),
         train_obj2=np.array([r.train_obj for r in rep2.records]), filters2=rep2.filters,
         stopped2=rep2.stopped_early)


def case_cfg0(steps=1):
    """Config 0 at full size (100x100, K=100, f64, B=1, rho=1): the 1e-9 parity target."""
    from paper_1706_06972_b200.workloads import CONFIGS
    c = CONFIGS[0]
    X = synth_images(steps, c["dims0"], c["grid"], c["K0"], seed=0).reshape(steps, -1)
    shape = ocsc.SignalShape(c["grid"], (11, 11))
    cfg = ocsc.TrainConfig(n_filters=c["K"], beta=c["beta"], rho_code=1.0, rho_dict=1.0,
                           inner_iters=10, seed=0)
    tr = OnlineTrainer(shape, cfg)
    objs, iters, nz_idx, nz_val = [], [], [], []
    for i in range(steps):
        t0 = time.time()
        st = tr.step(X[i])
        print(f"cfg0 step {i}: {time.time() - t0:.1f}s, iters {st.iterations}")
        objs.append(tr.last_objective), iters.append(st.iterations)
        idx = np.flatnonzero(st.code)
        nz_idx.append(idx), nz_val.append(st.code.ravel()[idx])
    save("cfg0", X=X, objectives=np.array(objs), iterations=np.array(iters),
         code_idx=np.concatenate(nz_idx), code_val=np.concatenate(nz_val),
         code_counts=np.array([len(i) for i in nz_idx]),
         final_filters=tr.final_filters(), coding_filters=tr.coding_filters())


def case_config_minibatch(name, cfg_id, K, B, nbatches, seed, beta=None, dims0=None, grid=None, K0=None):
    """A BASELINE config's own shapes, composed mini-batch semantics built from
    reference calls only, in the reference's float64.  X is regenerated from the seed by
    paper_1706_06972_b200.workloads.synth_images (its sha256 is stored to pin the generator)."""
    import hashlib

    from paper_1706_06972_b200.workloads import CONFIGS
    c = CONFIGS[cfg_id]
    dims0, grid, K0 = dims0 or c["dims0"], grid or c["grid"], K0 or c["K0"]
    beta = c["beta"] if beta is None else beta
    X = synth_images(B * nbatches, dims0, grid, K0, seed=seed).reshape(B * nbatches, -1)
    shape = ocsc.SignalShape(grid, (11, 11))
    cfg = ocsc.TrainConfig(n_filters=K, beta=beta, rho_code=1.0, rho_dict=1.0, inner_iters=10, seed=0,
                           code_max_iters=300, code_rel_tol=1e-3)
    tr = OnlineTrainer(shape, cfg)
    coding = cfg.coding()
    objs, iters, filt = [], [], []
    for m in range(nbatches):
        t0 = time.time()
        batch = X[m * B:(m + 1) * B]
        states = [ocsc.infer_code(x, tr.working_freq, shape, coding) for x in batch]
        for x, st in zip(batch, states):
            objs.append(ocsc.coding_objective(x, tr.working_freq, st.code, shape, cfg.beta))
            iters.append(st.iterations)
        for x, st in zip(batch, states):
            ocsc.update_history(tr.history, ocsc.forward_dft_cols(st.code, shape), ocsc.forward_dft(x, shape))
        tr.dict_state = ocsc.update_dictionary(tr.dict_state, tr.history, cfg.inner_iters)
        tr.working_freq = ocsc.forward_dft_cols(tr.dict_state.v, shape)
        filt.append(tr.final_filters())
        print(f"{name} mini-batch {m}: {time.time() - t0:.1f}s", flush=True)
    save(name, cfg_id=cfg_id, dims0=dims0, grid=grid, K0=K0, K=K, B=B, seed=seed, beta=beta,
         x_sha256=hashlib.sha256(X.tobytes()).hexdigest(), objectives=np.array(objs), iterations=np.array(iters),
         batch_filters=np.array(filt), final_filters=tr.final_filters(), coding_filters=tr.coding_filters())


if __name__ == "__main__":
    which = sys.argv[1:] or ["all"]
    run_all = "all" in which
    if run_all or "primitives" in which:
        case_primitives()
    if run_all or "code" in which:
        case_code("code_2d", (12, 10), (3, 3), 4, 1002, ocsc.CodingConfig(beta=0.3))
        case_code("code_1d", (16,), (3,), 3, 1005, ocsc.CodingConfig(beta=0.2, max_iters=500, rel_tol=1e-5))
        case_code("code_odd", (9, 7), (3, 2), 3, 1006, ocsc.CodingConfig(beta=0.5, max_iters=40, rel_tol=0.0))
    if run_all or "history" in which:
        case_history()
    if run_all or "dictionary" in which:
        case_dictionary()
    if run_all or "trainer" in which:
        case_trainer("train_2d", (12, 12), (5, 5), 6, 4, 4, rho_dict=1.0, inner_iters=4,
                     code_max_iters=60, beta=0.3)
        case_trainer("train_odd", (9, 7), (3, 3), 3, 3, 3, rho_dict=10.0, inner_iters=3,
                     code_max_iters=80, beta=0.4)
    if run_all or "trainer" in which or "train_14" in which:
        case_trainer("train_14", (14, 14), (3, 3), 5, 3, 3, rho_dict=1.0, inner_iters=4,
                     code_max_iters=120, beta=0.3)
    if run_all or "minibatch" in which:
        case_minibatch("minibatch", (10, 10), (3, 3), 5, 3, 2, rho_dict=1.0, inner_iters=4,
                       code_max_iters=50, beta=0.3)
    if run_all or "train_online" in which:
        case_train_online()
    if run_all or "train_batch" in which:
        X = synth_images(5, (1, 24), (1, 24), 2, filter_dims=(1, 4), seed=21, density=0.1).reshape(5, 24)
        shape = ocsc.SignalShape((24,), (4,))
        cfg = ocsc.TrainConfig(n_filters=3, beta=0.4, seed=2, max_passes=3, stop_tol=1e-12,
                               code_max_iters=150, batch_dict_iters=60, batch_dict_tol=1e-6)
        rep = ocsc.train_batch(X, shape, cfg)
        X2 = synth_images(4, (8, 10), (8, 10), 2, filter_dims=(3, 3), seed=22, density=0.1).reshape(4, 80)
        shape2 = ocsc.SignalShape((8, 10), (3, 3))
        rep2 = ocsc.train_batch(X2, shape2, ocsc.TrainConfig(n_filters=4, beta=0.3, seed=1, max_passes=2,
                                                             code_max_iters=120, batch_dict_iters=40))
        save("train_batch", X=X, train_obj=np.array([r.train_obj for r in rep.records]), filters=rep.filters,
             X2=X2, train_obj2=np.array([r.train_obj for r in rep2.records]), filters2=rep2.filters)
    if run_all or "preprocess" in which:
        from ocsc import preprocessing as P

        rng = np.random.default_rng(31)
        rgb = rng.integers(0, 256, size=(37, 53, 3)).astype(np.float64)
        gray = 128.0 + 40.0 * rng.normal(size=(20, 16))
        tiny = rng.uniform(0, 255, size=(3, 4))
        small = rng.normal(size=(5, 6))
        stack = rng.integers(0, 256, size=(4, 32, 32, 3)).astype(np.float64)
        save("preprocess", rgb=rgb, gray=gray, tiny=tiny, small=small, stack=stack,
             gray_rgb=P.grayscale(rgb),
             pre_rgb=P.preprocess(rgb, P.PreprocessSpec(seed=3)),
             pre_gray=P.preprocess(gray),
             pre_tiny=P.preprocess(tiny, P.PreprocessSpec(seed=1)),
             lcn_even=P.local_contrast_normalize(gray, window=8, sigma=2.0),
             lcn_tiny=P.local_contrast_normalize(tiny, window=9, sigma=3.0, epsilon=1e-2),
             taper_small=P.edge_taper(small, size=7, sigma=1.5),
             taper_even=P.edge_taper(gray, size=6, sigma=1.0),
             pre_stack=np.stack([P.preprocess(im, P.PreprocessSpec(seed=5 + i)) for i, im in enumerate(stack)]))
    if run_all or "files" in which:
        rng = np.random.default_rng(1007)
        ocsc.save_dictionary(rng.normal(size=(6, 3)), (2, 3), os.path.join(HERE, "dict_2x3_k3.dic"))
        ocsc.save_sample(rng.normal(size=20), (4, 5), os.path.join(HERE, "sample_4x5.smp"))
        print("wrote dict_2x3_k3.dic, sample_4x5.smp")
    if "cfg0" in which:
        case_cfg0()
    # BASELINE configs' own shapes through the composed mini-batch oracle (reference float64)
    if "cfg1_mb" in which:   # headline: 42x42, K=100, B=50, two mini-batches
        case_config_minibatch("cfg1_mb", 1, K=100, B=50, nbatches=2, seed=101)
    if "cfg2_mb" in which:   # 100x100, K=100, B=10, two mini-batches
        case_config_minibatch("cfg2_mb", 2, K=100, B=10, nbatches=2, seed=102)
    if "cfg3_mb" in which:   # 266x266 grid, K=32 (the reference's (P, K, K) inverse of K=256 is 74 GB), B=4
        case_config_minibatch("cfg3_mb", 3, K=32, B=4, nbatches=2, seed=103)
