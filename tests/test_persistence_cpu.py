"""File formats: byte compatibility with the reference's .dic / .smp files."""

import os

import numpy as np
import pytest

from paper_1706_06972_b200 import persistence as ps
from paper_1706_06972_b200.errors import BadMagicError, ChecksumError, ShapeMismatchError, TruncatedFileError
from tests.conftest import GOLDEN


def test_reads_reference_dictionary_and_rewrites_identical_bytes(tmp_path):
    src = os.path.join(GOLDEN, "dict_2x3_k3.dic")
    filters, dims = ps.load_dictionary(src)
    assert filters.shape == (6, 3) and dims == (2, 3)
    out = tmp_path / "copy.dic"
    ps.save_dictionary(filters, dims, out)
    assert open(out, "rb").read() == open(src, "rb").read()


def test_reads_reference_sample_and_rewrites_identical_bytes(tmp_path):
    src = os.path.join(GOLDEN, "sample_4x5.smp")
    sig, dims = ps.load_sample(src)
    assert sig.shape == (20,) and dims == (4, 5)
    out = tmp_path / "copy.smp"
    ps.save_sample(sig, dims, out)
    assert open(out, "rb").read() == open(src, "rb").read()


def test_error_contract(tmp_path):
    src = open(os.path.join(GOLDEN, "dict_2x3_k3.dic"), "rb").read()
    bad = tmp_path / "bad.dic"
    bad.write_bytes(b"XXXXXXXX" + src[8:])
    with pytest.raises(BadMagicError):
        ps.load_dictionary(bad)
    bad.write_bytes(src[:-10])
    with pytest.raises(TruncatedFileError):
        ps.load_dictionary(bad)
    corrupt = bytearray(src)
    corrupt[40] ^= 0xFF
    bad.write_bytes(bytes(corrupt))
    with pytest.raises(ChecksumError):
        ps.load_dictionary(bad)
    with pytest.raises(ShapeMismatchError):
        ps.save_dictionary(np.zeros((5, 2)), (2, 3), tmp_path / "x.dic")
