"""ctypes binding of libocsc_b200.so (include/ocsc_b200.h).

The shared library is built in-tree (`python __graft_entry__.py` -> build()).
There is no CPU fallback: importing a compute entry point without the library
or without a CUDA device raises immediately.
"""

from __future__ import annotations

import ctypes
import os

import torch

from .errors import (
    DivergenceError,
    ShapeMismatchError,
    UninitializedHistoryError,
)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libocsc_b200.so")

F32, F64, U8 = 4, 8, 1

_I, _I64, _D, _P, _SZ = ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p, ctypes.c_size_t

# name -> argtypes (restype int unless listed in _RESTYPES); mirrors include/ocsc_b200.h
SIGNATURES = {
    "ocsc_last_error": [],
    "ocsc_abi_version": [],
    "ocsc_kernel_launches": [],
    "ocsc_fft_prepare": [_I, _I, _I, _I],
    "ocsc_rfft2": [_I, _I, _I, _I, _P, _P, _P],
    "ocsc_irfft2": [_I, _I, _I, _I, _P, _P, _P],
    "ocsc_dft_cols": [_I, _I, _I, _I, _P, _I, _P, _I, _P],
    "ocsc_residue_stats": [_I, _I64, _P, _P, _P, _P],
    "ocsc_real_part": [_I, _I64, _P, _D, _P, _P],
    "ocsc_half_to_cols": [_I, _I, _I, _I, _P, _P, _P],
    "ocsc_cols_to_half": [_I, _I, _I, _I, _P, _P, _P],
    "ocsc_hermitian_defect": [_I, _I, _I, _I, _P, _P, _P],
    "ocsc_soft_threshold": [_I, _I64, _P, _D, _P, _P],
    "ocsc_solve_code_rows": [_I, _I, _I, _P, _P, _P, _D, _P, _P],
    "ocsc_code_den": [_I, _I, _I, _P, _D, _P, _P],
    "ocsc_code_workspace_bytes": [_I, _I, _I, _I, _I, _I],
    "ocsc_code_admm": [_I, _I, _I, _I, _I, _P, _P, _P, _D, _D, _I, _D, _P, _P, _P, _P, _P, _P, _I, _P],
    "ocsc_code_fused_cluster": [_I, _I, _I, _I, _I],
    "ocsc_code_fused_info": [_I, _I, _I, _I, _I, _P],
    "ocsc_code_fused_side_info": [_I, _I, _I, _I, _I, _P],
    "ocsc_debug_fused_profile": [_P],
    "ocsc_debug_chol_profile": [_P],
    "ocsc_debug_plane_profile": [_P],
    "ocsc_debug_fused_iterations": [_P],
    "ocsc_debug_fused_timeline": [_P],
    "ocsc_code_fused": [_I, _I, _I, _I, _I, _P, _P, _P, _D, _D, _I, _D, _P, _P, _P, _P, _P, _P, _P, _P],
    "ocsc_code_stream_supported": [_I, _I, _I],
    "ocsc_code_stream_workspace_bytes": [_I, _I, _I, _I, _I],
    "ocsc_code_stream": [_I, _I, _I, _I, _I, _P, _P, _P, _D, _D, _I, _D, _P, _P, _P, _P, _I, _P],
    "ocsc_code_objective": [_I, _I, _I, _I, _I, _P, _P, _P, _D, _P, _P, _P, _P],
    "ocsc_synthesize": [_I, _I, _I, _I, _P, _P, _P, _P],
    "ocsc_history_accumulate": [_I, _I, _I, _I, _I, _P, _I64, _I64, _I64, _P, _I64, _I64, _P, _P, _P],
    "ocsc_history_invert": [_I, _I, _I, _I, _P, _D, _D, _P, _P, _P],
    "ocsc_code_stream_plane_ctas": [_I, _I, _I, _I, _I],
    "ocsc_history_invert_claim": [_I, _I, _I, _I, _P, _D, _D, _P, _P, _P, _I, _P],
    "ocsc_history_woodbury": [_I, _I, _I, _I, _I, _P, _P, _I64, _I64, _I64, _P, _P, _P, _I64, _I64, _P, _P, _P],
    "ocsc_history_woodbury_smem": [_I, _I],
    "ocsc_packed_to_full": [_I, _I, _I, _P, _D, _P, _P],
    "ocsc_history_factor_bytes": [_I, _I, _I],
    "ocsc_history_factor": [_I, _I, _I, _P, _D, _P, _P, _P],
    "ocsc_dict_rowsolve_chol": [_I, _I, _I, _I, _P, _P, _D, _P, _P, _I64, _I64, _P, _P],
    "ocsc_nonfinite": [_I, _I64, _P, _P, _P],
    "ocsc_dict_rowsolve": [_I, _I, _I, _I, _I, _P, _P, _D, _P, _P, _I64, _I64, _P, _P],
    "ocsc_dict_project": [_I, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P],
    "ocsc_crop_irfft": [_I, _I, _I, _I, _I, _I, _P, _P, _P],
    "ocsc_crop_normalize_cols": [_I, _I, _I, _I, _I, _I, _P, _P, _P],
    "ocsc_support_rfft": [_I, _I, _I, _I, _I, _I, _P, _P, _P],
    "ocsc_norms2": [_I, _I64, _P, _P, _P, _P],
    "ocsc_dict_gaps": [_I, _I, _I, _I, _P, _P, _P, _P],
    "ocsc_crop_irfft_rows": [_I, _I, _I, _I, _I, _I, _I, _I, _P, _P, _P, _P],
    "ocsc_normalize_support": [_I, _I, _I, _P, _P, _P],
    "ocsc_support_rfft_rows": [_I, _I, _I, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P],
    "ocsc_preprocess": [_I, _I, _I, _I, _I, _I, _P, _I, _I, _D, _D, _I, _P, _I64, _D, _D, _P, _P],
    "ocsc_taper_sigmas": [_I64, _I, _D, _D, _P],
}
_RESTYPES = {"ocsc_last_error": ctypes.c_char_p, "ocsc_code_workspace_bytes": _SZ,
             "ocsc_code_stream_workspace_bytes": _SZ, "ocsc_history_factor_bytes": _SZ,
             "ocsc_history_woodbury_smem": _SZ,
             "ocsc_kernel_launches": ctypes.c_int64}

_lib = None


class NativeLibraryError(RuntimeError):
    """libocsc_b200.so is missing, stale, or the CUDA device is unusable."""


def load(path: str = LIB_PATH):
    """Load and type the shared library (no device needed)."""
    global _lib
    if _lib is not None and path == LIB_PATH:
        return _lib
    if not os.path.exists(path):
        raise NativeLibraryError(
            f"{path} not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)"
        )
    lib = ctypes.CDLL(path)
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RESTYPES.get(name, ctypes.c_int)
    if lib.ocsc_abi_version() != 1:
        raise NativeLibraryError("libocsc_b200.so ABI version mismatch; rebuild")
    if path == LIB_PATH:
        _lib = lib
    return lib


def device() -> torch.device:
    """The CUDA device the hot path runs on; fails loudly without one."""
    if not torch.cuda.is_available():
        raise NativeLibraryError("the OCSC B200 path needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def stream(dev: torch.device | None = None) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def code(dtype: torch.dtype) -> int:
    if dtype in (torch.float32, torch.complex64):
        return F32
    if dtype in (torch.float64, torch.complex128):
        return F64
    raise ValueError(f"unsupported dtype {dtype}")


def check(rc: int, what: str = "") -> None:
    if rc == 0:
        return
    msg = (_lib.ocsc_last_error() or b"").decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == -1:
        raise ShapeMismatchError(text)
    if rc == -2:
        raise DivergenceError(text)
    if rc == -3:
        raise UninitializedHistoryError(text)
    if rc == -6:
        raise ValueError(text)
    raise NativeLibraryError(text)


def call(name: str, *args) -> None:
    """Invoke an entry point and map its status to the reference exceptions."""
    lib = load()
    check(getattr(lib, name)(*args), name)
