"""Packed binary codes and partitions — host mirror of /root/reference/proj/include/mih/codes.hpp.

Same names, argument meaning and error behaviour (ValueError where the reference throws
std::invalid_argument). Storage is a numpy (n, ceil(bits/64)) uint64 array: bit i of a code is
word i/64, bit i%64 (LSB first), padding bits zero (codes.hpp:26-33, :87-95).
"""
from __future__ import annotations

import numpy as np

kMaxCodeBits = 4096  # codes.hpp:16


def words_per_code(bits: int) -> int:  # codes.hpp:18
    return (bits + 63) // 64


def last_word_mask(bits: int) -> int:  # codes.hpp:21-24
    used = bits & 63
    return (1 << 64) - 1 if used == 0 else (1 << used) - 1


class BinaryCode:
    """Non-owning view of one code (codes.hpp:28-33)."""

    __slots__ = ("words", "bits")

    def __init__(self, words, bits: int):
        self.words = np.ascontiguousarray(words, dtype=np.uint64).reshape(-1)
        self.bits = int(bits)

    def bit(self, i: int) -> bool:
        return bool((int(self.words[i >> 6]) >> (i & 63)) & 1)


def hamming_distance(a: BinaryCode, b: BinaryCode) -> int:  # codes.hpp:46-51
    if a.bits != b.bits:
        raise ValueError(f"hamming_distance: code widths differ ({a.bits} vs {b.bits})")
    x = np.bitwise_xor(a.words, b.words)
    return int(sum(bin(int(w)).count("1") for w in x))


class CodeDatabase:
    """Flat store of n equal-width codes; a code's id is its position (codes.hpp:54-120)."""

    def __init__(self, bits: int, words: np.ndarray | None = None):
        if bits == 0 or bits > kMaxCodeBits:
            raise ValueError(f"CodeDatabase: code width must be in [1, {kMaxCodeBits}], got {bits}")
        self._bits = int(bits)
        wpc = words_per_code(bits)
        if words is None:
            self._words = np.zeros((0, wpc), np.uint64)
        else:
            w = np.ascontiguousarray(words, dtype=np.uint64).reshape(-1, wpc)
            self._check_count(w.shape[0])
            pad = np.uint64(((1 << 64) - 1) ^ last_word_mask(bits))
            if w.shape[0] and np.any(w[:, -1] & pad):
                raise ValueError("CodeDatabase::append: nonzero padding bits")
            self._words = w

    @staticmethod
    def _check_count(n: int) -> None:
        if n > (1 << 32):  # codes.hpp:111-115
            raise ValueError("CodeDatabase: at most 2^32 codes supported")

    @classmethod
    def zeros(cls, bits: int, n: int) -> "CodeDatabase":
        cls._check_count(n)
        return cls(bits, np.zeros((n, words_per_code(bits)), np.uint64))

    def bits(self) -> int:
        return self._bits

    def size(self) -> int:
        return int(self._words.shape[0])

    def words_per_entry(self) -> int:
        return words_per_code(self._bits)

    def code(self, i: int) -> BinaryCode:
        return BinaryCode(self._words[i], self._bits)

    def append(self, c: BinaryCode) -> None:
        if c.bits != self._bits:
            raise ValueError("CodeDatabase::append: width mismatch")
        self.append_words(c.words)

    def append_words(self, w) -> None:
        w = np.ascontiguousarray(w, dtype=np.uint64).reshape(1, -1)
        self._check_count(self.size() + 1)
        if int(w[0, -1]) & (((1 << 64) - 1) ^ last_word_mask(self._bits)):
            raise ValueError("CodeDatabase::append: nonzero padding bits")
        self._words = np.concatenate([self._words, w], axis=0)

    def raw_words(self) -> np.ndarray:
        """(n, words_per_entry) uint64 view."""
        return self._words

    def set_bit(self, i: int, pos: int, v: bool) -> None:
        m = np.uint64(1 << (pos & 63))
        if v:
            self._words[i, pos >> 6] |= m
        else:
            self._words[i, pos >> 6] &= ~m

    def __eq__(self, o) -> bool:
        return isinstance(o, CodeDatabase) and self._bits == o._bits and np.array_equal(self._words, o._words)


class Partition:
    """Assignment of bit positions {0..bits-1} to m disjoint balanced substrings
    (codes.hpp:124-195)."""

    def __init__(self, bits: int, substrings):
        self._bits = int(bits)
        self._subs = [list(map(int, s)) for s in substrings]
        self._validate()

    def _validate(self) -> None:  # codes.hpp:152-176
        m, bits = len(self._subs), self._bits
        if bits == 0 or bits > kMaxCodeBits:
            raise ValueError("Partition: bad width")
        if m == 0 or m > bits:
            raise ValueError("Partition: substring count must be in [1, bits]")
        seen = [False] * bits
        for sub in self._subs:
            for pos in sub:
                if pos >= bits or pos < 0:
                    raise ValueError(f"Partition: bit position {pos} out of range")
                if seen[pos]:
                    raise ValueError(f"Partition: bit position {pos} assigned twice")
                seen[pos] = True
        if sum(len(s) for s in self._subs) != bits:
            raise ValueError("Partition: positions do not cover the code")
        lens = [len(s) for s in self._subs]
        if max(lens) - min(lens) > 1:
            raise ValueError("Partition: substring sizes differ by more than 1")

    def bits(self) -> int:
        return self._bits

    def m(self) -> int:
        return len(self._subs)

    def length(self, j: int) -> int:
        return len(self._subs[j])

    def positions(self, j: int):
        return list(self._subs[j])

    def substrings(self):
        return [list(s) for s in self._subs]

    def contiguous(self, j: int) -> bool:
        s = self._subs[j]
        return all(s[i] == s[i - 1] + 1 for i in range(1, len(s)))

    def lengths_array(self) -> np.ndarray:
        return np.array([len(s) for s in self._subs], np.uint32)

    def positions_array(self) -> np.ndarray:
        return np.array([p for s in self._subs for p in s], np.uint32)

    def __eq__(self, o) -> bool:
        return isinstance(o, Partition) and self._bits == o._bits and self._subs == o._subs


def consecutive_partition(bits: int, m: int) -> Partition:  # codes.hpp:198-211
    if m == 0 or m > bits:
        raise ValueError(f"consecutive_partition: need 1 <= m <= bits, got m={m}, bits={bits}")
    base, extra = divmod(bits, m)
    subs, pos = [], 0
    for j in range(m):
        ln = base + (1 if j < extra else 0)
        subs.append(list(range(pos, pos + ln)))
        pos += ln
    return Partition(bits, subs)


def extract_substring(code: BinaryCode, p: Partition, j: int) -> int:  # codes.hpp:214-231
    if j >= p.m():
        raise ValueError("extract_substring: substring index out of range")
    if code.bits != p.bits():
        raise ValueError("extract_substring: width mismatch")
    sub = p.positions(j)
    if len(sub) > 64:
        raise ValueError("extract_substring: substring wider than 64 bits")
    v = 0
    for i, pos in enumerate(sub):
        v |= int(code.bit(pos)) << i
    return v
