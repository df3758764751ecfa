"""R-4': the walker-side alias limit lim = ceil(thr * 2^64 / T) (saturated at thr = T) computed
on the device without a 128-bit division, against exact Python integers -- random pairs over
every magnitude plus the boundary cases (thr = 1, thr = T - 1, T = 2^64 - 1, powers of two)."""
from __future__ import annotations

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _lib():
    from paper_2504_10233_b200 import _build
    _build.build()
    L = ctypes.CDLL(_build.TOOLS_LIB)
    L.bt_alias_lim.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_uint64]
    return L


def _ref(thr, T):
    if thr >= T:
        return (1 << 64) - 1
    return -((-(thr << 64)) // T)


def test_alias_lim_exact():
    rng = np.random.default_rng(3)
    pairs = []
    for bits in range(1, 65):
        for _ in range(300):
            T = int(rng.integers(1, 1 << 62, dtype=np.uint64)) >> (62 - min(bits, 62)) if bits <= 62 else \
                int(rng.integers(1 << 62, (1 << 64) - 1, dtype=np.uint64))
            T = max(T, 1)
            thr = int(rng.integers(0, T + 1, dtype=np.uint64)) if T < (1 << 63) else \
                int(rng.integers(0, 1 << 63, dtype=np.uint64)) * 2 % (T + 1)
            pairs.append((thr, T))
    M = (1 << 64) - 1
    for T in (1, 2, 3, 7, 1 << 20, (1 << 32) + 1, 1 << 63, (1 << 63) + 1, M - 1, M):
        for thr in (0, 1, 2, T // 2, T // 3, max(T - 2, 0), T - 1, T):
            if 0 <= thr <= T:
                pairs.append((thr, T))
    thr = np.array([p[0] for p in pairs], dtype=np.uint64)
    T = np.array([p[1] for p in pairs], dtype=np.uint64)
    out = np.zeros_like(thr)
    assert _lib().bt_alias_lim(thr.ctypes.data, T.ctypes.data, out.ctypes.data, len(pairs)) == 0
    bad = [(int(a), int(b), int(c), _ref(int(a), int(b))) for a, b, c in zip(thr, T, out)
           if int(c) != _ref(int(a), int(b))]
    assert not bad, bad[:5]
