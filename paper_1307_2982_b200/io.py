"""Codes files and synthetic data — host mirror of the parts of
/root/reference/proj/include/mih/io.hpp the hot path's callers use.

* BMIH codes files (io.hpp:151-171): "BMIH" | u32 version=1 | u32 bits | u64 n | n records of
  ceil(bits/64) u64 words, padding zero. Errors are FormatError with a byte offset (io.hpp:35-44).
* gen_uniform (io.hpp:266-277): std::mt19937_64 words, last word masked — computed natively in
  libmihg.so (mihg_gen_uniform), bit-identical to the reference for every seed.
"""
from __future__ import annotations

import os
import struct

import numpy as np

from . import _lib
from .codes import CodeDatabase, kMaxCodeBits, last_word_mask, words_per_code

_CODES_MAGIC = b"BMIH"
_VERSION = 1


class FormatError(RuntimeError):  # io.hpp:35-44
    def __init__(self, what: str, offset: int):
        super().__init__(f"{what} (byte offset {offset})")
        self.offset = offset


def write_index(idx, path: str) -> None:
    """write_index (io.hpp:335-358): the BMIX file, byte-identical to the reference's."""
    _lib.check(_lib.lib().mihg_index_write(idx._h, path.encode()))


def read_index(path: str, device: int = 0):
    """read_index (io.hpp:360-425): validated load of a BMIX file (FormatError with byte offset);
    the file's tables are loaded onto the GPU as given."""
    import ctypes as C

    from .codes import Partition
    from .index import MihIndex

    h = C.c_void_p()
    _lib.check(_lib.lib().mihg_index_read(path.encode(), device, C.byref(h)))
    # host-side mirror of the codes and partition (db(), partition() accessors)
    with open(path, "rb") as f:
        f.seek(8)
        bits, n = struct.unpack("<IQ", f.read(12))
        wpc = words_per_code(bits)
        words = np.frombuffer(f.read(n * wpc * 8), dtype="<u8").astype(np.uint64).reshape(n, wpc)
        (m,) = struct.unpack("<I", f.read(4))
        subs = []
        for _ in range(m):
            (ln,) = struct.unpack("<I", f.read(4))
            subs.append(list(np.frombuffer(f.read(4 * ln), dtype="<u4")))
    return MihIndex(h, CodeDatabase(bits, words), Partition(bits, subs), bits, n, device, 0)


def gen_uniform(n: int, bits: int, seed: int) -> CodeDatabase:
    if bits == 0 or bits > kMaxCodeBits:
        raise ValueError("gen_uniform: bad width")
    wpc = words_per_code(bits)
    out = np.zeros((max(n, 1), wpc), np.uint64)
    _lib.check(_lib.lib().mihg_gen_uniform(n, bits, seed, out.ctypes.data_as(_lib.u64p)))
    return CodeDatabase(bits, out[:n])


def write_codes(db: CodeDatabase, path: str) -> None:
    with open(path, "wb") as f:
        f.write(_CODES_MAGIC)
        f.write(struct.pack("<IIQ", _VERSION, db.bits(), db.size()))
        f.write(np.ascontiguousarray(db.raw_words(), dtype="<u8").tobytes())


def read_codes(path: str) -> CodeDatabase:
    size = os.path.getsize(path)
    with open(path, "rb") as f:
        data = f.read()

    def need(at, nbytes, what):
        if at + nbytes > size:
            raise FormatError(f"truncated file {path}: reading {what} needs {nbytes} bytes, "
                              f"{size - at} remain", at)

    need(0, 4, "magic")
    if data[:4] != _CODES_MAGIC:
        raise FormatError("not a codes file (bad magic)", 0)
    need(4, 4, "version")
    (version,) = struct.unpack_from("<I", data, 4)
    if version != _VERSION:
        raise FormatError(f"unsupported codes file version {version}", 4)
    need(8, 4, "code width")
    (bits,) = struct.unpack_from("<I", data, 8)
    if bits == 0 or bits > kMaxCodeBits:
        raise FormatError(f"bad code width {bits}", 8)
    need(12, 8, "code count")
    (n,) = struct.unpack_from("<Q", data, 12)
    if n > (1 << 32):
        raise FormatError("code count exceeds 2^32", 12)
    wpc = words_per_code(bits)
    payload = n * wpc * 8
    need(20, payload, "code words")
    words = np.frombuffer(data, dtype="<u8", count=n * wpc, offset=20).astype(np.uint64).reshape(n, wpc)
    pad = np.uint64(((1 << 64) - 1) ^ last_word_mask(bits))
    bad = np.nonzero(words[:, -1] & pad)[0] if n else []
    if len(bad):
        i = int(bad[0])
        raise FormatError(f"nonzero padding bits in record {i}", 20 + (i * wpc + wpc - 1) * 8)
    if 20 + payload != size:
        raise FormatError(f"trailing bytes after codes payload in {path}: expected size "
                          f"{20 + payload}, file has {size}", 20 + payload)
    return CodeDatabase(bits, words)
