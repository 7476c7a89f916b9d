"""CPU oracle for the OCSC hot path -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

This module restates, in plain numpy/float64, the algorithm of the reference
package `ocsc` (arXiv 1706.06972, /root/reference/pkg/src/ocsc) for the path
the B200 build accelerates: code ADMM -> history fold -> dictionary ADMM,
driven by the online trainer, extended to mini-batches with the composed
semantics of SURVEY.md section 8(c).

Only `tests/`, `__graft_entry__.smoke()` and `bench.py` (its `cpu_baseline`
leg and `--impl reference`) may import this module, and only as the checker /
the reported CPU baseline.  The product package `paper_1706_06972_b200`
never imports it.

Layout differs from the reference on purpose: planes are (K, H, W) with the
full complex spectrum per plane (the reference uses (P, K) columns, K
fastest).  A 1-D signal of length W is the H = 1 grid.  The arithmetic is the
reference's: full complex FFTs (numpy pocketfft), the rank-one code solve,
the exact O(K^3) incremental inverse, and J rounds of dictionary ADMM.

Pinning: tests/test_oracle_golden.py checks this module against golden
vectors produced by the reference itself (tests/golden/make_golden.py,
run in the build container where /root/reference is importable).
"""

from __future__ import annotations

import numpy as np

# transforms.py:21 -- scaled bound on the imaginary residue of an inverse DFT
RESIDUE_TOL = 1e-8


class OracleDivergence(ArithmeticError):
    """Non-finite iterate (coding.py:105-106, dictionary.py:89-90)."""


class OracleUninitialized(RuntimeError):
    """Dictionary update at t = 0 (dictionary.py:194-195)."""


class OracleResidue(ArithmeticError):
    """Inverse DFT with a non-negligible imaginary part (transforms.py:102-109)."""


# ---------------------------------------------------------------- geometry --

def grid_of(dims) -> tuple[int, int]:
    """(H, W) of a 1-D or 2-D signal; 1-D maps to H = 1 (SignalShape, transforms.py:24-61)."""
    dims = tuple(int(d) for d in dims)
    return (1, dims[0]) if len(dims) == 1 else dims


def fdims_of(filter_dims) -> tuple[int, int]:
    f = tuple(int(d) for d in filter_dims)
    return (1, f[0]) if len(f) == 1 else f


# -------------------------------------------------------------- transforms --

def fwd(planes: np.ndarray) -> np.ndarray:
    """Unnormalised 2-D DFT over the last two axes (transforms.py:82-87, 148-158)."""
    return np.fft.fft2(np.asarray(planes, dtype=np.float64), axes=(-2, -1))


def inv(spec: np.ndarray) -> np.ndarray:
    """Inverse DFT with 1/P, real part after the residue guard (transforms.py:90-109, 161-176)."""
    spec = np.asarray(spec, dtype=np.complex128)
    out = np.fft.ifft2(spec, axes=(-2, -1))
    if out.size:
        residue = np.abs(out.imag).max()
        bound = RESIDUE_TOL * (1.0 + np.abs(spec).max())
        if residue > bound:
            raise OracleResidue(f"imaginary residue {residue:.3e} exceeds {bound:.3e}")
    return out.real


def pad(filters_mk: np.ndarray, H: int, W: int, M0: int, M1: int) -> np.ndarray:
    """(M, K) filters -> (K, H, W) zero-padded planes, support top-left (transforms.py:179-196)."""
    K = filters_mk.shape[1]
    out = np.zeros((K, H, W))
    out[:, :M0, :M1] = filters_mk.T.reshape(K, M0, M1)
    return out


def crop(planes: np.ndarray, M0: int, M1: int) -> np.ndarray:
    """(K, H, W) -> (M, K) leading support (transforms.py:199-211)."""
    K = planes.shape[0]
    return planes[:, :M0, :M1].reshape(K, M0 * M1).T.copy()


# ------------------------------------------------------------------ coding --

def shrink(v, kappa):
    """sign(v) * max(|v| - kappa, 0) (coding.py:45-48)."""
    v = np.asarray(v)
    return np.sign(v) * np.maximum(np.abs(v) - kappa, 0.0)


def code_solve(dh: np.ndarray, xh: np.ndarray, th: np.ndarray, rho: float) -> np.ndarray:
    """Per-frequency rank-one + ridge solve, all frequencies (coding.py:51-64).

    dh, th: (K, H, W) complex; xh: (H, W) complex.
    """
    rhs = np.conj(dh) * xh[None] + rho * th
    s = (dh * rhs).sum(axis=0)
    den = rho + (dh * np.conj(dh)).real.sum(axis=0)
    return (rhs - np.conj(dh) * (s / den)[None]) / rho


def code_admm(x, dh, beta, rho, max_iters, rel_tol, warm=None, monitor=None):
    """ADMM sparse coding of one (H, W) sample (coding.py:67-119).

    Returns dict(zh, code, dual, iterations); raises OracleDivergence with the
    iteration number on a non-finite code.
    """
    K, H, W = dh.shape
    x = np.asarray(x, dtype=np.float64).reshape(H, W)
    xh = fwd(x)
    if warm is not None:
        code, dual = warm["code"].copy(), warm["dual"].copy()
    else:
        code, dual = np.zeros((K, H, W)), np.zeros((K, H, W))
    zh = np.zeros((K, H, W), dtype=np.complex128)
    kappa = beta / rho
    iterations = 0
    for it in range(1, max_iters + 1):
        iterations = it
        zh = code_solve(dh, xh, fwd(code - dual), rho)
        z = inv(zh)
        fresh = shrink(z + dual, kappa)
        if not np.isfinite(fresh).all():
            raise OracleDivergence(f"code solver diverged at iteration {it}")
        dual = dual + z - fresh
        moved = np.linalg.norm(fresh - code)
        size = np.linalg.norm(fresh)
        code = fresh
        if monitor is not None:
            monitor(it, code)
        gap = np.linalg.norm(z - code)
        gap_scale = max(size, np.linalg.norm(dual), 1e-12)
        if moved <= rel_tol * max(size, 1e-12) and gap <= rel_tol * gap_scale:
            break
    return {"zh": zh, "code": code, "dual": dual, "iterations": iterations}


def reconstruction(dh, code):
    """Sum over k of d_k (*) code_k (coding.py:122-126)."""
    return inv((dh * fwd(code)).sum(axis=0))


def objective(x, dh, code, beta) -> float:
    """0.5 ||x - recon||^2 + beta ||code||_1 (coding.py:129-134)."""
    r = np.asarray(x, dtype=np.float64).reshape(dh.shape[1:]) - reconstruction(dh, code)
    return 0.5 * float((r * r).sum()) + beta * float(np.abs(code).sum())


# ----------------------------------------------------------------- history --

class History:
    """Averaged cross term and exact regularised inverse Gram per frequency.

    Restates HistoryState / update_history (dictionary.py:30-114): cross is
    (K, H, W) = (1/t) sum conj(xh) zh; inv is (H, W, K, K) =
    ((1/t) sum zh zh^H + rho P I)^-1 with the reference's orientation
    (G[j, k] = z_j conj(z_k)).
    """

    def __init__(self, K: int, H: int, W: int, rho: float):
        self.K, self.H, self.W = K, H, W
        self.P = H * W
        self.rho = float(rho)
        self.count = 0
        self.cross = np.zeros((K, H, W), dtype=np.complex128)
        self.inv = np.zeros((H, W, K, K), dtype=np.complex128)

    @staticmethod
    def _herm(m):
        return 0.5 * (m + np.conj(np.swapaxes(m, -1, -2)))

    def fold(self, zh: np.ndarray, xh: np.ndarray) -> None:
        zh = np.asarray(zh, dtype=np.complex128)
        xh = np.asarray(xh, dtype=np.complex128)
        if not (np.isfinite(zh).all() and np.isfinite(xh).all()):
            raise OracleDivergence("non-finite spectrum rejected before history update")
        t = self.count + 1
        ridge = self.rho * self.P
        self.cross = (1.0 - 1.0 / t) * self.cross + (1.0 / t) * np.conj(xh)[None] * zh
        z = np.moveaxis(zh, 0, -1)                      # (H, W, K)
        outer = z[..., :, None] * np.conj(z)[..., None, :]
        eye = np.eye(self.K)
        if t == 1:
            scale = ridge + (z * np.conj(z)).real.sum(axis=-1)
            new = (eye - outer / scale[..., None, None]) / ridge
        else:
            g = (1.0 - 1.0 / t) * eye + (ridge / t) * self.inv
            base = self._herm(np.linalg.solve(g, self.inv))
            w = np.einsum("hwjk,hwk->hwj", base, z)
            s = np.einsum("hwk,hwk->hw", np.conj(z), w).real
            new = base - w[..., :, None] * np.conj(w)[..., None, :] / (t + s)[..., None, None]
        self.inv = self._herm(new)
        self.count = t


def dict_rows(hist: History, vh, th):
    """Row solve (conj(cross) + rho P (v - theta)) . inv (dictionary.py:134-142)."""
    ridge = hist.rho * hist.P
    q = np.moveaxis(np.conj(hist.cross) + ridge * (vh - th), 0, -1)   # (H, W, K)
    d = np.einsum("hwk,hwkj->hwj", q, hist.inv)
    return np.moveaxis(d, -1, 0)


def project(xh, M0: int, M1: int):
    """Crop to support, scale into the unit ball, re-pad (dictionary.py:145-154)."""
    K, H, W = xh.shape
    alpha = crop(inv(xh), M0, M1)
    alpha = alpha / np.maximum(np.linalg.norm(alpha, axis=0), 1.0)
    return pad(alpha, H, W, M0, M1)


def dict_admm(dh_prev, v_prev, hist: History, J: int, M0: int, M1: int, tol=None, monitor=None):
    """DictOCSC inner ADMM (dictionary.py:176-215); returns (dh, v, theta)."""
    if hist.count == 0:
        raise OracleUninitialized("dictionary update requested at t=0")
    if J == 0:
        return dh_prev, v_prev, None
    v = np.array(v_prev, dtype=np.float64)
    vh = fwd(v)
    th = np.zeros_like(vh)
    dh = np.array(dh_prev, dtype=np.complex128)
    for tau in range(1, J + 1):
        dh = dict_rows(hist, vh, th)
        v = project(dh + th, M0, M1)
        vh = fwd(v)
        th = th + dh - vh
        if monitor is not None:
            monitor(tau, dh, v)
        if tol is not None:
            gaps = np.linalg.norm((dh - vh).reshape(dh.shape[0], -1), axis=1)
            scales = np.maximum(np.linalg.norm(dh.reshape(dh.shape[0], -1), axis=1), 1e-12)
            if (gaps / scales).max() < tol:
                break
    return dh, v, th


# ----------------------------------------------------------------- trainer --

def init_filters(M: int, K: int, seed: int) -> np.ndarray:
    """Seeded Gaussian (M, K) filters with unit columns (training.py:91-95)."""
    f = np.random.default_rng(seed).normal(size=(M, K))
    return f / np.linalg.norm(f, axis=0)


class Trainer:
    """Online trainer (training.py:102-169) generalised to mini-batches.

    A mini-batch step is the composed reference semantics of SURVEY.md 8(c):
    all B samples are coded (cold start) against the same working spectrum,
    folded into the history one by one in order, then one dictionary ADMM
    call of J rounds runs and the working spectrum becomes F(V).  For B = 1
    this is exactly OnlineTrainer.step.
    """

    def __init__(self, dims, filter_dims, K=100, beta=1.0, rho_code=1.0, rho_dict=10.0,
                 inner_iters=10, seed=0, code_max_iters=300, code_rel_tol=1e-3, stop_tol=1e-3):
        self.H, self.W = grid_of(dims)
        self.M0, self.M1 = fdims_of(filter_dims)
        self.K = K
        self.beta, self.rho_code, self.rho_dict = beta, rho_code, rho_dict
        self.J, self.max_iters, self.rel_tol = inner_iters, code_max_iters, code_rel_tol
        self.stop_tol = stop_tol
        f = init_filters(self.M0 * self.M1, K, seed)
        self.initial_filters = f
        self.v = pad(f, self.H, self.W, self.M0, self.M1)
        self.dh = fwd(self.v)
        self.th = np.zeros_like(self.dh)
        self.working = self.dh.copy()
        self.hist = History(K, self.H, self.W, rho_dict)
        self.rng = np.random.default_rng(seed)
        self.prev_code = None
        self.prev_filters = f.copy()
        self.code_change = np.inf
        self.dict_change = np.inf

    def step_batch(self, xs):
        """One mini-batch; returns list of (state dict, objective) per sample."""
        xs = np.asarray(xs, dtype=np.float64).reshape(-1, self.H, self.W)
        out = []
        for x in xs:
            st = code_admm(x, self.working, self.beta, self.rho_code, self.max_iters, self.rel_tol)
            out.append((st, objective(x, self.working, st["code"], self.beta)))
        for x, (st, _) in zip(xs, out):
            self.hist.fold(fwd(st["code"]), fwd(x))
        dh, v, th = dict_admm(self.dh, self.v, self.hist, self.J, self.M0, self.M1)
        self.dh, self.v = dh, v
        if th is not None:
            self.th = th
        self.working = fwd(self.v)
        last = out[-1][0]["code"]
        if self.prev_code is not None:
            self.code_change = np.linalg.norm(last - self.prev_code) / max(np.linalg.norm(last), 1e-12)
        self.prev_code = last
        filt = crop(self.v, self.M0, self.M1)
        self.dict_change = np.linalg.norm(filt - self.prev_filters) / max(np.linalg.norm(filt), 1e-12)
        self.prev_filters = filt
        return out

    def converged(self) -> bool:
        return self.code_change < self.stop_tol and self.dict_change < self.stop_tol

    def coding_filters(self):
        return crop(self.v, self.M0, self.M1)

    def final_filters(self):
        return crop(inv(self.dh), self.M0, self.M1)


def train_online(samples, dims, filter_dims, batch_size=1, max_passes=10, **kw):
    """Shuffled passes with the change-metric stop (training.py:178-223).

    Returns dict(filters, records=[(pass, train_obj)], objectives, stopped_early).
    """
    H, W = grid_of(dims)
    samples = np.asarray(samples, dtype=np.float64).reshape(-1, H * W)
    tr = Trainer(dims, filter_dims, **kw)
    report = {"records": [], "objectives": [], "stopped_early": False}
    if samples.shape[0] == 0:
        report["filters"] = tr.coding_filters()
        return report
    for pass_idx in range(1, max_passes + 1):
        order = tr.rng.permutation(samples.shape[0])
        objs, stopped = [], False
        for s in range(0, len(order), batch_size):
            res = tr.step_batch(samples[order[s:s + batch_size]])
            objs.extend(o for _, o in res)
            if tr.converged():
                stopped = True
                break
        report["objectives"].extend(objs)
        report["records"].append((pass_idx, float(np.mean(objs))))
        if stopped:
            report["stopped_early"] = True
            break
    report["filters"] = tr.final_filters()
    report["trainer"] = tr
    return report


# ---------------------------------------------------------- preprocessing --
# preprocessing.py:13-100 (row f4): grayscale, Gaussian LCN, seeded edge taper.  scipy's
# correlate1d(mode="reflect") is restated as np.pad(mode="symmetric") + a sliding dot product
# with the kernel centre at size // 2.

LUMA = (0.299, 0.587, 0.114)


def gray(image):
    a = np.asarray(image, dtype=np.float64)
    return a if a.ndim == 2 else a[..., 0] * LUMA[0] + a[..., 1] * LUMA[1] + a[..., 2] * LUMA[2]


def gauss(size: int, sigma: float):
    xs = np.arange(size) - (size - 1) / 2.0
    k = np.exp(-0.5 * (xs / sigma) ** 2)
    return k / k.sum()


def correlate_reflect(a, k, axis: int):
    """scipy.ndimage.correlate1d(a, k, axis, mode='reflect') (preprocessing.py:53-55)."""
    s = len(k)
    c = s // 2
    pad = [(0, 0)] * a.ndim
    pad[axis] = (c, s - 1 - c)
    p = np.pad(a, pad, mode="symmetric")
    n = a.shape[axis]
    out = np.zeros_like(a)
    for t in range(s):
        out += k[t] * np.take(p, np.arange(t, t + n), axis=axis)
    return out


def separable(a, k):
    return correlate_reflect(correlate_reflect(a, k, 0), k, 1)


def lcn(a, window=9, sigma=3.0, eps=1e-4):
    k = gauss(window, sigma)
    m = separable(a, k)
    v = separable(a * a, k) - m * m
    return (a - m) / np.maximum(np.sqrt(np.maximum(v, 0.0)), eps)


def taper(a, size=11, sigma=2.0):
    b = separable(a, gauss(size, sigma))

    def ramp(n):
        i = np.arange(n) + 0.5
        return np.minimum(np.minimum(i, n - i) / size, 1.0)

    w = np.outer(ramp(a.shape[0]), ramp(a.shape[1]))
    return w * a + (1.0 - w) * b


def preprocess(image, window=9, sigma=3.0, eps=1e-4, size=11, sigma_range=(1.0, 3.0), seed=0):
    s = float(np.random.default_rng(seed).uniform(*sigma_range))
    return taper(lcn(gray(image), window, sigma, eps), size, s)
