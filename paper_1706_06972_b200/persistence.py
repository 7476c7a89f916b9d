"""State persistence.

* `.dic` / `.smp` envelopes, byte-compatible with the reference (persistence.py:25-141),
  so dictionaries move between this build and the reference CLI (`eval`, `mosaic`):
  8-byte magic, little-endian u32 axis count and extents, (dictionaries: u32 filter
  count), u32 element tag 1 (= little-endian float64), the float64 payload
  (filters filter-major), u32 CRC32 of the payload.
* Trainer checkpoints (new: the reference cannot resume an online run): every piece of
  device state of an `OnlineTrainer` (history sums and count, dictionary spectrum, dual,
  working spectrum, feasible filters, change-metric memory) plus the pass-order RNG,
  in one `.npz`; `load_checkpoint` resumes bit-identically.
"""

from __future__ import annotations

import json
import struct
import zlib

import numpy as np
import torch

from .errors import BadMagicError, ChecksumError, DataFileError, ShapeMismatchError, TruncatedFileError

DICT_MAGIC = b"OCSCDIC1"
SAMPLE_MAGIC = b"OCSCSMP1"
F64_TAG = 1


def _u32(v: int) -> bytes:
    return struct.pack("<I", int(v))


def _write_envelope(path, magic: bytes, extents, extra, values: np.ndarray) -> None:
    body = np.ascontiguousarray(values, dtype="<f8").tobytes()
    head = magic + _u32(len(extents)) + b"".join(_u32(e) for e in extents) + b"".join(_u32(e) for e in extra)
    with open(path, "wb") as fh:
        fh.write(head + _u32(F64_TAG) + body + _u32(zlib.crc32(body) & 0xFFFFFFFF))


def _read_envelope(path, magic: bytes, n_extra: int):
    blob = open(path, "rb").read()
    pos = 0

    def take(n):
        nonlocal pos
        if pos + n > len(blob):
            raise TruncatedFileError(f"{path}: file ends {pos + n - len(blob)} bytes early")
        chunk = blob[pos:pos + n]
        pos += n
        return chunk

    def u32():
        return struct.unpack("<I", take(4))[0]

    tag = take(len(magic))
    if tag != magic:
        raise BadMagicError(f"{path}: expected magic {magic!r}, found {tag!r}")
    naxes = u32()
    if naxes not in (1, 2):
        raise DataFileError(f"{path}: expected 1 or 2 axes, got {naxes}")
    dims = tuple(u32() for _ in range(naxes))
    extra = tuple(u32() for _ in range(n_extra))
    if u32() != F64_TAG:
        raise DataFileError(f"{path}: unknown element type tag")
    count = int(np.prod(dims)) * (extra[0] if extra else 1)
    body = take(8 * count)
    crc = u32()
    if pos != len(blob):
        raise DataFileError(f"{path}: {len(blob) - pos} trailing bytes after checksum")
    if crc != zlib.crc32(body) & 0xFFFFFFFF:
        raise ChecksumError(f"{path}: payload checksum mismatch")
    return dims, extra, np.frombuffer(body, dtype="<f8").astype(np.float64)


def save_dictionary(filters, filter_dims, path) -> None:
    """(M, K) filters -> `.dic` (reference persistence.py:84-97 format)."""
    arr = np.asarray(filters, dtype=np.float64)
    dims = tuple(int(d) for d in filter_dims)
    if arr.ndim != 2 or arr.shape[0] != int(np.prod(dims)):
        raise ShapeMismatchError(f"filters {arr.shape} do not match filter extents {dims}")
    _write_envelope(path, DICT_MAGIC, dims, (arr.shape[1],), arr.T)


def load_dictionary(path):
    """`.dic` -> ((M, K) filters, filter extents)."""
    dims, (k,), flat = _read_envelope(path, DICT_MAGIC, 1)
    return flat.reshape(k, int(np.prod(dims))).T.copy(), dims


def save_sample(signal, dims, path) -> None:
    """One flattened signal -> `.smp` (reference persistence.py:116-127 format)."""
    arr = np.asarray(signal, dtype=np.float64).ravel()
    dims = tuple(int(d) for d in dims)
    if arr.size != int(np.prod(dims)):
        raise ShapeMismatchError(f"signal size {arr.size} does not match dims {dims}")
    _write_envelope(path, SAMPLE_MAGIC, dims, (), arr)


def load_sample(path):
    """`.smp` -> ((P,) signal, extents)."""
    dims, _, flat = _read_envelope(path, SAMPLE_MAGIC, 0)
    return flat, dims


# ------------------------------------------------------------ checkpoints --

_STATE = ("Wh", "den", "Dh", "Th", "alpha", "_prev_alpha")


def save_checkpoint(trainer, path) -> None:
    """Every piece of an OnlineTrainer's state -> one `.npz` (resumable).  A ShardedTrainer writes
    one file per rank (`ShardedTrainer.save_checkpoint`; reload with `ShardedTrainer.load_checkpoint`)."""
    if getattr(trainer, "_collective", False):
        return trainer.save_checkpoint(path)
    h = trainer.history
    arrays = {name: getattr(trainer, name).detach().cpu().numpy() for name in _STATE}
    arrays["hist_S"] = h.S.detach().cpu().numpy()
    arrays["hist_c"] = h.c.detach().cpu().numpy()
    if trainer._prev_code is not None:
        arrays["prev_code"] = trainer._prev_code.detach().cpu().numpy()
    meta = {
        "config": trainer.config.__dict__,
        "dims": trainer.shape.dims,
        "filter_dims": trainer.shape.filter_dims,
        "count": h.count,
        "code_change": trainer.code_change,
        "dict_change": trainer.dict_change,
        "last_objective": trainer.last_objective,
        "rng": trainer.rng.bit_generator.state,
    }
    np.savez(path, meta=np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8), **arrays)


def load_checkpoint(path):
    """`.npz` from save_checkpoint -> an OnlineTrainer positioned exactly where it was saved."""
    from .training import OnlineTrainer, TrainConfig
    from .transforms import SignalShape

    z = np.load(path, allow_pickle=False)
    meta = json.loads(bytes(z["meta"]).decode())
    shape = SignalShape(tuple(meta["dims"]), tuple(meta["filter_dims"]))
    trainer = OnlineTrainer(shape, TrainConfig(**meta["config"]))
    for name in _STATE:
        getattr(trainer, name).copy_(torch.from_numpy(z[name]))
    h = trainer.history
    h.S.copy_(torch.from_numpy(z["hist_S"]))
    h.c.copy_(torch.from_numpy(z["hist_c"]))
    h.count = int(meta["count"])
    h._inv_count = -1
    if "prev_code" in z.files:
        trainer._prev_code = torch.from_numpy(z["prev_code"]).to(trainer.dev)
    trainer.code_change = float(meta["code_change"])
    trainer.dict_change = float(meta["dict_change"])
    trainer.last_objective = float(meta["last_objective"])
    trainer.rng.bit_generator.state = meta["rng"]
    return trainer
