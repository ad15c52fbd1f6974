"""TEST INFRASTRUCTURE ONLY — the CPU checker for the CUDA product path.

Two CPU implementations of the reference hot path, both behind ctypes:

* ``port``  — ``oracle/_build/liboracle.so``: the plain-C restatement in ``mih_oracle.c``
  (always buildable with gcc; each function cites the reference file:line it follows).
* ``ref``   — ``oracle/_ref/libmihref.so``: the reference's OWN headers
  (/root/reference/proj/include/mih/*.hpp) compiled by ``oracle/Makefile`` behind the C-ABI
  driver ``ref_driver.cpp``. Built in the dev container (where /root/reference exists); the
  prebuilt .so travels to the GPU box.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package. The product package
``paper_1307_2982_b200`` never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(_HERE, "_build", "liboracle.so")
REF_SO = os.path.join(_HERE, "_ref", "libmihref.so")
REF_INC = "/root/reference/proj/include"

_u64p = C.POINTER(C.c_uint64)
_u32p = C.POINTER(C.c_uint32)


class OracleError(RuntimeError):
    pass


def build(ref: bool = True) -> None:
    """Compile the checker libraries (port always; ref only where the reference exists)."""
    subprocess.run(["make", "-s", "-C", _HERE, "all"], check=True)
    if ref and os.path.isdir(os.path.join(REF_INC, "mih")):
        subprocess.run(["make", "-s", "-C", _HERE, "ref"], check=True)


def _p64(a):
    return a.ctypes.data_as(_u64p) if a is not None else None


def _p32(a):
    return a.ctypes.data_as(_u32p) if a is not None else None


def wpc(bits: int) -> int:
    return (bits + 63) // 64


class _Lib:
    prefix = ""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise OracleError(f"checker library missing: {path} (run oracle.build())")
        self.lib = C.CDLL(path)
        self._err = getattr(self.lib, self.prefix + "last_error")
        self._err.restype = C.c_char_p

    def _check(self, rc):
        if rc == 1:
            raise ValueError(self._err().decode())
        if rc:
            raise OracleError(self._err().decode())

    def estimate_correlations(self, codes, bits):
        """optimize.hpp:47-92 -> (corr[b,b] f64, constant[b] bool, counts[b,b] u64 or None)."""
        codes = np.ascontiguousarray(codes, np.uint64).reshape(-1)
        n = codes.size // wpc(bits)
        corr = np.zeros((bits, bits), np.float64)
        const = np.zeros(bits, np.uint8)
        dp, cp = corr.ctypes.data_as(C.POINTER(C.c_double)), const.ctypes.data_as(C.POINTER(C.c_uint8))
        if self.prefix == "or_":
            counts = np.zeros((bits, bits), np.uint64)
            self._check(self.lib.or_estimate_correlations(_p64(codes), C.c_uint64(n), C.c_uint32(bits),
                                                          dp, cp, _p64(counts)))
        else:
            counts = None
            self._check(self.lib.ref_estimate_correlations(_p64(codes), C.c_uint64(n), C.c_uint32(bits),
                                                           dp, cp))
        return corr, const.astype(bool), counts

    def greedy_assign(self, corr, constant, m, seed):
        """optimize.hpp:101-172 -> list of m sorted position lists."""
        corr = np.ascontiguousarray(corr, np.float64)
        const = np.ascontiguousarray(constant, np.uint8)
        bits = corr.shape[0]
        lengths = np.zeros(max(m, 1), np.uint32)
        pos = np.zeros(bits, np.uint32)
        self._check(getattr(self.lib, self.prefix + "greedy_assign")(
            corr.ctypes.data_as(C.POINTER(C.c_double)), const.ctypes.data_as(C.POINTER(C.c_uint8)),
            C.c_uint32(bits), C.c_uint32(m), C.c_uint64(seed), _p32(lengths), _p32(pos)))
        out, at = [], 0
        for L in lengths[:m]:
            out.append([int(x) for x in pos[at:at + L]])
            at += int(L)
        return out


class Port(_Lib):
    """The C restatement (mih_oracle.c)."""

    prefix = "or_"

    def __init__(self):
        super().__init__(PORT_SO)
        self.lib.or_index_build.argtypes = [_u64p, C.c_uint64, C.c_uint32, C.c_uint32, _u32p, _u32p,
                                            C.POINTER(C.c_void_p)]
        self.lib.or_index_free.argtypes = [C.c_void_p]
        self.lib.or_knn.argtypes = [C.c_void_p, _u64p, C.c_uint64, C.c_uint32, _u32p, _u32p, _u64p]
        self.lib.or_range.argtypes = [C.c_void_p, _u64p, C.c_uint32, _u32p, _u32p, C.c_uint64,
                                      _u64p, _u64p]
        self.lib.or_bucket.argtypes = [C.c_void_p, C.c_uint32, C.c_uint64, _u32p, C.c_uint64, _u64p]
        self.lib.or_scan_knn.argtypes = [_u64p, C.c_uint64, C.c_uint32, _u64p, C.c_uint64,
                                         C.c_uint32, _u32p, _u32p]
        self.lib.or_gen_uniform.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, _u64p]
        self.lib.or_gen_mixture.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32,
                                            C.c_uint32, C.c_uint64, C.c_uint64, _u64p, C.c_int]

    def gen_mixture(self, first, n, bits, dim, comps, model_seed, data_seed, threads=None):
        out = np.zeros(max(n * wpc(bits), 1), np.uint64)
        self._check(self.lib.or_gen_mixture(first, n, bits, dim, comps, model_seed, data_seed,
                                            _p64(out), threads or os.cpu_count() or 1))
        return out[: n * wpc(bits)].reshape(n, wpc(bits))

    def gen_uniform(self, n, bits, seed):
        out = np.zeros(max(n * wpc(bits), 1), np.uint64)
        self._check(self.lib.or_gen_uniform(n, bits, seed, _p64(out)))
        return out[: n * wpc(bits)].reshape(n, wpc(bits))

    def build(self, codes, bits, m, lengths=None, positions=None):
        codes = np.ascontiguousarray(codes, np.uint64).reshape(-1)
        n = codes.size // wpc(bits)
        h = C.c_void_p()
        ln = None if lengths is None else np.ascontiguousarray(lengths, np.uint32)
        ps = None if positions is None else np.ascontiguousarray(positions, np.uint32)
        self._check(self.lib.or_index_build(_p64(codes), n, bits, m, _p32(ln), _p32(ps), C.byref(h)))
        return _Handle(self, h, bits, n)

    def scan_knn(self, codes, bits, queries, k):
        codes = np.ascontiguousarray(codes, np.uint64).reshape(-1)
        queries = np.ascontiguousarray(queries, np.uint64).reshape(-1)
        n, nq = codes.size // wpc(bits), queries.size // wpc(bits)
        ids = np.zeros(max(nq * k, 1), np.uint32)
        dists = np.zeros(max(nq * k, 1), np.uint32)
        self._check(self.lib.or_scan_knn(_p64(codes), n, bits, _p64(queries), nq, k, _p32(ids), _p32(dists)))
        return ids[: nq * k].reshape(nq, k), dists[: nq * k].reshape(nq, k)


class Ref(_Lib):
    """The reference's own headers behind ref_driver.cpp."""

    prefix = "ref_"

    def __init__(self, threads: int | None = None):
        super().__init__(REF_SO)
        L = self.lib
        self.threads = threads or os.cpu_count() or 1
        L.ref_index_build.argtypes = [_u64p, C.c_uint64, C.c_uint32, C.c_uint32, _u32p, _u32p,
                                      C.POINTER(C.c_void_p)]
        L.ref_index_free.argtypes = [C.c_void_p]
        L.ref_index_build_parallel.argtypes = [_u64p, C.c_uint64, C.c_uint32, C.c_uint32,
                                               C.POINTER(C.c_void_p)]
        L.ref_knn.argtypes = [C.c_void_p, _u64p, C.c_uint64, C.c_uint32, _u32p, _u32p, _u64p, C.c_int]
        L.ref_range.argtypes = [C.c_void_p, _u64p, C.c_uint32, _u32p, _u32p, C.c_uint64, _u64p, _u64p]
        L.ref_bucket.argtypes = [C.c_void_p, C.c_uint32, C.c_uint64, _u32p, C.c_uint64, _u64p]
        L.ref_table_stats.argtypes = [C.c_void_p, C.c_uint32, _u64p]
        L.ref_scan_knn.argtypes = [_u64p, C.c_uint64, C.c_uint32, _u64p, C.c_uint64, C.c_uint32,
                                   _u32p, _u32p, C.c_int]
        L.ref_scan_range.argtypes = [_u64p, C.c_uint64, C.c_uint32, _u64p, C.c_uint32, _u32p, _u32p,
                                     C.c_uint64, _u64p]
        L.ref_gen_uniform.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, _u64p]
        L.ref_gen_lsh.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_double,
                                  C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint64, _u64p]
        L.ref_write_codes.argtypes = [_u64p, C.c_uint64, C.c_uint32, C.c_char_p]
        L.ref_write_index.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_read_index.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
        L.ref_knn_timed.argtypes = [C.c_void_p, _u64p, C.c_uint64, C.c_uint32, _u32p, _u32p, _u64p, C.c_int,
                                    C.POINTER(C.c_double)]
        L.ref_index_scan_knn_timed.argtypes = [C.c_void_p, _u64p, C.c_uint64, C.c_uint32, _u32p, _u32p,
                                               C.c_int, C.POINTER(C.c_double)]
        L.ref_db_new.argtypes = [_u64p, C.c_uint64, C.c_uint32, C.POINTER(C.c_void_p)]
        L.ref_db_gen_uniform.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.POINTER(C.c_void_p)]
        L.ref_db_words.argtypes = [C.c_void_p]
        L.ref_db_words.restype = C.c_void_p
        L.ref_db_free.argtypes = [C.c_void_p]
        L.ref_db_scan_knn_timed.argtypes = [C.c_void_p, _u64p, C.c_uint64, C.c_uint32, _u32p, _u32p, C.c_int,
                                            C.POINTER(C.c_double)]

    def gen_uniform(self, n, bits, seed):
        out = np.zeros(max(n * wpc(bits), 1), np.uint64)
        self._check(self.lib.ref_gen_uniform(n, bits, seed, _p64(out)))
        return out[: n * wpc(bits)].reshape(n, wpc(bits))

    def gen_lsh(self, fit_n, enc_n, dim, group, noise, fit_seed, enc_seed, bits, spec_seed):
        out = np.zeros(max(enc_n * wpc(bits), 1), np.uint64)
        self._check(self.lib.ref_gen_lsh(fit_n, enc_n, dim, group, noise, fit_seed, enc_seed, bits,
                                         spec_seed, _p64(out)))
        return out[: enc_n * wpc(bits)].reshape(enc_n, wpc(bits))

    def build(self, codes, bits, m, lengths=None, positions=None):
        codes = np.ascontiguousarray(codes, np.uint64).reshape(-1)
        n = codes.size // wpc(bits)
        h = C.c_void_p()
        ln = None if lengths is None else np.ascontiguousarray(lengths, np.uint32)
        ps = None if positions is None else np.ascontiguousarray(positions, np.uint32)
        self._check(self.lib.ref_index_build(_p64(codes), n, bits, m, _p32(ln), _p32(ps), C.byref(h)))
        return _Handle(self, h, bits, n)

    def build_parallel(self, codes, bits, m):
        """Tables built concurrently through SubstringTable::build + MihIndex::assemble."""
        codes = np.ascontiguousarray(codes, np.uint64).reshape(-1)
        n = codes.size // wpc(bits)
        h = C.c_void_p()
        self._check(self.lib.ref_index_build_parallel(_p64(codes), n, bits, m, C.byref(h)))
        return _Handle(self, h, bits, n)

    def scan_knn(self, codes, bits, queries, k, threads=None):
        codes = np.ascontiguousarray(codes, np.uint64).reshape(-1)
        queries = np.ascontiguousarray(queries, np.uint64).reshape(-1)
        n, nq = codes.size // wpc(bits), queries.size // wpc(bits)
        ids = np.zeros(max(nq * k, 1), np.uint32)
        dists = np.zeros(max(nq * k, 1), np.uint32)
        self._check(self.lib.ref_scan_knn(_p64(codes), n, bits, _p64(queries), nq, k, _p32(ids),
                                          _p32(dists), threads or self.threads))
        return ids[: nq * k].reshape(nq, k), dists[: nq * k].reshape(nq, k)

    def db_new(self, codes, bits):
        codes = np.ascontiguousarray(codes, np.uint64).reshape(-1)
        n = codes.size // wpc(bits)
        h = C.c_void_p()
        self._check(self.lib.ref_db_new(_p64(codes), n, bits, C.byref(h)))
        return RefDb(self, h, bits, n)

    def db_gen_uniform(self, n, bits, seed):
        h = C.c_void_p()
        self._check(self.lib.ref_db_gen_uniform(n, bits, seed, C.byref(h)))
        return RefDb(self, h, bits, n)

    def scan_range(self, codes, bits, q, r):
        codes = np.ascontiguousarray(codes, np.uint64).reshape(-1)
        q = np.ascontiguousarray(q, np.uint64).reshape(-1)
        n = codes.size // wpc(bits)
        cnt = C.c_uint64()
        ids = np.zeros(max(n, 1), np.uint32)
        dists = np.zeros(max(n, 1), np.uint32)
        self._check(self.lib.ref_scan_range(_p64(codes), n, bits, _p64(q), r, _p32(ids), _p32(dists),
                                            n, C.byref(cnt)))
        return ids[: cnt.value], dists[: cnt.value]


def _pd(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_double))


class RefDb:
    """A reference CodeDatabase held in the driver (scan-only baseline, e.g. config 5)."""

    def __init__(self, owner, h, bits, n):
        self.owner, self.h, self.bits, self.n = owner, h, bits, n

    def __del__(self):
        try:
            self.owner.lib.ref_db_free(self.h)
        except Exception:
            pass

    def words(self):
        """numpy view [n, W] of the held codes (valid while this object lives)."""
        W = wpc(self.bits)
        p = self.owner.lib.ref_db_words(self.h)
        buf = (C.c_uint64 * (self.n * W)).from_address(p)
        return np.frombuffer(buf, np.uint64).reshape(self.n, W)

    def scan_knn_timed(self, queries, k, threads=None):
        return _scan_timed(self.owner, self.owner.lib.ref_db_scan_knn_timed, self.h, self.bits, queries, k, threads)


def _scan_timed(owner, fn, h, bits, queries, k, threads):
    queries = np.ascontiguousarray(queries, np.uint64).reshape(-1)
    nq = queries.size // wpc(bits)
    ids = np.zeros(max(nq * k, 1), np.uint32)
    dists = np.zeros(max(nq * k, 1), np.uint32)
    secs = np.zeros(max(nq, 1), np.float64)
    owner._check(fn(h, _p64(queries), nq, k, _p32(ids), _p32(dists), threads or owner.threads, _pd(secs)))
    return ids[: nq * k].reshape(nq, k), dists[: nq * k].reshape(nq, k), secs[:nq]


class _Handle:
    def __init__(self, owner, h, bits, n):
        self.owner, self.h, self.bits, self.n = owner, h, bits, n
        self.p = owner.prefix

    def __del__(self):
        try:
            getattr(self.owner.lib, self.p + "index_free")(self.h)
        except Exception:
            pass

    def knn(self, queries, k, threads=None):
        """Returns (ids[nq,k], dists[nq,k], traces[nq,5]); traces columns are SearchTrace
        {lookups, candidates, unique_candidates, distance_evaluations, final_radius}."""
        queries = np.ascontiguousarray(queries, np.uint64).reshape(-1)
        nq = queries.size // wpc(self.bits)
        ids = np.zeros(max(nq * k, 1), np.uint32)
        dists = np.zeros(max(nq * k, 1), np.uint32)
        tr = np.zeros(max(nq * 5, 1), np.uint64)
        L = self.owner.lib
        if self.p == "ref_":
            rc = L.ref_knn(self.h, _p64(queries), nq, k, _p32(ids), _p32(dists), _p64(tr),
                           threads or self.owner.threads)
        else:
            rc = L.or_knn(self.h, _p64(queries), nq, k, _p32(ids), _p32(dists), _p64(tr))
        self.owner._check(rc)
        return ids[: nq * k].reshape(nq, k), dists[: nq * k].reshape(nq, k), tr[: nq * 5].reshape(nq, 5)

    def knn_timed(self, queries, k, threads=None):
        """ref_knn plus the wall time of every query (seconds): (ids, dists, traces, secs)."""
        queries = np.ascontiguousarray(queries, np.uint64).reshape(-1)
        nq = queries.size // wpc(self.bits)
        ids = np.zeros(max(nq * k, 1), np.uint32)
        dists = np.zeros(max(nq * k, 1), np.uint32)
        tr = np.zeros(max(nq * 5, 1), np.uint64)
        secs = np.zeros(max(nq, 1), np.float64)
        self.owner._check(self.owner.lib.ref_knn_timed(self.h, _p64(queries), nq, k, _p32(ids), _p32(dists),
                                                       _p64(tr), threads or self.owner.threads, _pd(secs)))
        return (ids[: nq * k].reshape(nq, k), dists[: nq * k].reshape(nq, k), tr[: nq * 5].reshape(nq, 5),
                secs[:nq])

    def scan_knn_timed(self, queries, k, threads=None):
        """the reference's scan_knn over this index's own database: (ids, dists, secs)."""
        return _scan_timed(self.owner, self.owner.lib.ref_index_scan_knn_timed, self.h, self.bits, queries, k,
                           threads)

    def range(self, q, r):
        q = np.ascontiguousarray(q, np.uint64).reshape(-1)
        cnt = C.c_uint64()
        ids = np.zeros(max(self.n, 1), np.uint32)
        dists = np.zeros(max(self.n, 1), np.uint32)
        tr = np.zeros(5, np.uint64)
        self.owner._check(getattr(self.owner.lib, self.p + "range")(self.h, _p64(q), r, _p32(ids), _p32(dists),
                                                           self.n, C.byref(cnt), _p64(tr)))
        return ids[: cnt.value], dists[: cnt.value], tr

    def bucket(self, j, value):
        cnt = C.c_uint64()
        out = np.zeros(max(self.n, 1), np.uint32)
        self.owner._check(getattr(self.owner.lib, self.p + "bucket")(self.h, j, value, _p32(out), self.n, C.byref(cnt)))
        return out[: cnt.value]


_port = None
_ref = None


def port() -> Port:
    global _port
    if _port is None:
        _port = Port()
    return _port


def ref(threads: int | None = None) -> Ref:
    global _ref
    if _ref is None:
        _ref = Ref(threads)
    return _ref


def have_ref() -> bool:
    return os.path.exists(REF_SO)
