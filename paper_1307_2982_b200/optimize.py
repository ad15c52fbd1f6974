"""Correlation-driven substring assignment — host mirror of
/root/reference/proj/include/mih/optimize.hpp.

* ``estimate_correlations(sample)`` (optimize.hpp:47-92): the AND-popcount Gram matrix of the
  bit columns runs on the GPU (libmihg.so, csrc/optimize.cu); the |Pearson| finish reproduces the
  reference's double arithmetic bit for bit.
* ``greedy_assign(corr, m, seed)`` (optimize.hpp:101-172): host logic in libmihg.so (no GPU).

Same names, argument meaning and errors as the reference (``ValueError`` for its
``std::invalid_argument``).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .codes import CodeDatabase, Partition


class CorrelationMatrix:
    """optimize.hpp:22-43: absolute pairwise correlations, diagonal 1, constant-bit flags."""

    def __init__(self, bits: int, values: np.ndarray | None = None, constant: np.ndarray | None = None,
                 counts: np.ndarray | None = None):
        self._bits = int(bits)
        self.values = np.eye(bits, dtype=np.float64) if values is None else np.ascontiguousarray(values, np.float64)
        self.constant = np.zeros(bits, bool) if constant is None else np.asarray(constant, bool)
        self.counts = counts  # exact AND counts (diagonal = ones) when computed on the GPU

    def bits(self) -> int:
        return self._bits

    def at(self, i: int, j: int) -> float:
        return float(self.values[i, j])

    def set(self, i: int, j: int, v: float) -> None:
        self.values[i, j] = self.values[j, i] = v

    def is_constant(self, i: int) -> bool:
        return bool(self.constant[i])

    def set_constant(self, i: int) -> None:
        self.constant[i] = True


def estimate_correlations(sample, device: int = 0, codes_on_device: bool = False) -> CorrelationMatrix:
    """|Pearson| between every pair of bit positions over ``sample`` (a CodeDatabase, or a raw
    device pointer + (n, bits) when ``codes_on_device``: pass ``sample=(ptr, n, bits)``)."""
    if codes_on_device:
        ptr, n, bits = sample
        keep = None
    else:
        if not isinstance(sample, CodeDatabase):
            raise TypeError("estimate_correlations: expected a CodeDatabase")
        n, bits = sample.size(), sample.bits()
        keep = np.ascontiguousarray(sample.raw_words(), np.uint64)
        ptr = keep.ctypes.data if n else None
    if n < 2:
        raise ValueError("estimate_correlations: need at least 2 codes")
    corr = np.zeros((bits, bits), np.float64)
    const = np.zeros(bits, np.uint8)
    counts = np.zeros((bits, bits), np.uint64)
    _lib.check(_lib.lib().mihg_estimate_correlations(
        C.c_void_p(ptr), n, bits, device, 1 if codes_on_device else 0,
        corr.ctypes.data_as(C.POINTER(C.c_double)), const.ctypes.data_as(C.POINTER(C.c_uint8)),
        counts.ctypes.data_as(_lib.u64p)))
    del keep
    return CorrelationMatrix(bits, corr, const.astype(bool), counts)


def greedy_assign(corr: CorrelationMatrix, m: int, seed: int) -> Partition:
    """Greedy min-max-correlation assignment of bit positions to m balanced substrings."""
    bits = corr.bits()
    if m == 0 or m > bits:
        raise ValueError("greedy_assign: need 1 <= m <= bits")
    vals = np.ascontiguousarray(corr.values, np.float64)
    const = np.ascontiguousarray(corr.constant, np.uint8)
    lengths = np.zeros(m, np.uint32)
    pos = np.zeros(bits, np.uint32)
    _lib.check(_lib.lib().mihg_greedy_assign(
        vals.ctypes.data_as(C.POINTER(C.c_double)), const.ctypes.data_as(C.POINTER(C.c_uint8)),
        bits, m, C.c_uint64(seed & (2**64 - 1)), lengths.ctypes.data_as(_lib.u32p), pos.ctypes.data_as(_lib.u32p)))
    subs, at = [], 0
    for L in lengths:
        subs.append([int(x) for x in pos[at:at + int(L)]])
        at += int(L)
    return Partition(bits, subs)
