"""Layout helpers shared by tests: reference (P, K) columns <-> (K, H, W) planes."""

import numpy as np


def hw(dims):
    dims = tuple(int(d) for d in np.atleast_1d(dims))
    return (1, dims[0]) if len(dims) == 1 else dims


def cols_to_planes(cols, dims):
    H, W = hw(dims)
    cols = np.asarray(cols)
    return cols.T.reshape(cols.shape[1], H, W)


def planes_to_cols(planes):
    planes = np.asarray(planes)
    return planes.reshape(planes.shape[0], -1).T


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(np.asarray(b).ravel()), 1e-300))
