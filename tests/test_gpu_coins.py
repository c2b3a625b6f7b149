"""The coin-word routine every coin producer uses (coins_kernel, the spread
round's in-kernel coins): word w of a stream holds the coins of draws
32w .. 32w + 31, bit b = mix64(key + (32w + b + 1) * gamma) < th
(rng.hpp:40-54).  Checked against numpy SplitMix64 for random thresholds
and for thresholds that tie a draw's high word (the exact-compare path)."""
import ctypes as C

import numpy as np
import pytest
import torch

import paper_2204_06787_b200 as mb  # noqa: F401  (loads the library)
from paper_2204_06787_b200 import _native as N

pytestmark = pytest.mark.gpu
GAMMA = np.uint64(0x9E3779B97F4A7C15)


def mix64(z):
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def draws(key, n):
    with np.errstate(over="ignore"):
        return mix64(np.uint64(key) + (np.arange(n, dtype=np.uint64) + np.uint64(1)) * GAMMA)


def device_words(key, th, n_chunks):
    lib = N.lib()
    f = lib.marsit_debug_coin_words
    f.restype = C.c_int
    f.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, C.c_void_p]
    out = torch.zeros(n_chunks * 64, dtype=torch.int32, device="cuda")
    assert f(key, th, n_chunks, out.data_ptr()) == 0
    return out.cpu().numpy().view(np.uint32)


def expected_words(x, th):
    bits = (x < np.uint64(th)).astype(np.uint64).reshape(-1, 32)
    return (bits << np.arange(32, dtype=np.uint64)).sum(axis=1).astype(np.uint32)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_coin_words_random_thresholds(seed):
    rng = np.random.default_rng(seed)
    key = int(rng.integers(0, 2**63)) * 2 + 1
    n_chunks = 37
    x = draws(key, n_chunks * 2048)
    for p in (0.5, 2 / 3, 7 / 8, 1e-3, 1 - 1e-9):
        th = int(np.ceil(p * 2**53)) << 11  # the plan's threshold form
        assert np.array_equal(device_words(key, th, n_chunks), expected_words(x, th)), p


def test_coin_words_tie_thresholds():
    """Thresholds sharing a draw's high word (down to equality with the draw
    and one above it): the flagged run takes the exact 64-bit compare."""
    key = 0x243F6A8885A308D3
    n_chunks = 5
    x = draws(key, n_chunks * 2048)
    for k in (0, 31, 777, 2048 * 3 + 5):
        xk = int(x[k])
        hi = xk & ~0xFFFFFFFF
        for th in (xk, xk + 1, xk - 1, hi, hi | 0xFFFFF800, (xk ^ (1 << 32)) & ~0x7FF):
            th &= (1 << 64) - 1
            assert np.array_equal(device_words(key, th, n_chunks), expected_words(x, th)), (k, hex(th))
