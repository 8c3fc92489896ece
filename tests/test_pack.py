"""Compact column transfer format (csrc/kp_pack.cu): kp_pack_cols (host, OpenMP) writes
column i at bits [i*b, (i+1)*b) of a little-endian 32-bit word stream, b = ceil(log2(n_cols)).
Checked on the CPU against a numpy restatement of the bit layout (no GPU needed); the
device unpacker is checked in tests/test_gpu_pack.py."""
import ctypes

import numpy as np
import pytest

from paper_2403_17017_b200 import _lib


def np_unpack(words: np.ndarray, n: int, b: int) -> np.ndarray:
    bits = np.unpackbits(words.view(np.uint8), bitorder="little")
    idx = np.arange(n, dtype=np.int64)[:, None] * b + np.arange(b)
    return (bits[idx].astype(np.int64) << np.arange(b)).sum(1)


@pytest.mark.parametrize("n_cols", [1, 2, 3, 1000, 1 << 20, (1 << 20) + 1, 10_000_019, 1 << 31])
@pytest.mark.parametrize("n", [0, 1, 31, 32, 33, 1000, 100_003])
def test_pack_matches_bit_layout(n, n_cols):
    L = _lib.load()
    b = L.kp_pack_bits(n_cols)
    assert b == max(1, int(np.ceil(np.log2(n_cols)))) if n_cols > 1 else b == 1
    rng = np.random.default_rng(n + n_cols)
    cols = rng.integers(0, n_cols, n, dtype=np.int64).astype(np.int32)
    if n:
        cols[0], cols[-1] = n_cols - 1, 0
    nbytes = L.kp_pack_cols_bytes(n, n_cols)
    out = np.full(nbytes // 4, 0xDEADBEEF, dtype=np.uint32)
    for threads in (1, 4):
        rc = L.kp_pack_cols(cols.ctypes.data_as(ctypes.c_void_p), n, n_cols, out.ctypes.data_as(ctypes.c_void_p), threads)
        assert rc == _lib.KP_OK
        assert np.array_equal(np_unpack(out, n, b), cols.astype(np.int64))
    assert nbytes <= (n * b + 31) // 32 * 4 + 4


def test_pack_rejects_out_of_range():
    L = _lib.load()
    cols = np.array([0, 5, 7], dtype=np.int32)
    out = np.zeros(L.kp_pack_cols_bytes(3, 7) // 4, dtype=np.uint32)
    rc = L.kp_pack_cols(cols.ctypes.data_as(ctypes.c_void_p), 3, 7, out.ctypes.data_as(ctypes.c_void_p), 1)
    assert rc == _lib.KP_ERANGE
    assert L.kp_pack_cols(None, -1, 7, None, 1) == _lib.KP_EINVAL
