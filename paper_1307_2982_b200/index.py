"""MihIndex on the GPU — host mirror of mih::MihIndex (/root/reference/proj/include/mih/index.hpp).

The interface keeps the reference's names and contracts:

* ``MihIndex.build(db, partition)``   — index.hpp:101-121 (ValueError where it throws
  std::invalid_argument: width mismatch :102-103, substring > 32 bits :108-112).
* ``idx.knn_search(q, k, trace=None)`` — index.hpp:185-253: the k smallest (dist, id) pairs in
  (dist asc, id asc) order; ``k > n`` raises, ``k == 0`` returns []. ``trace`` (a SearchTrace) is
  overwritten like the reference's out-parameter.
* ``db()``, ``partition()``, ``num_tables()``, ``table(j)`` accessors (index.hpp:143-146).

plus batch entry points that are the actual GPU calls: ``knn_search_batch`` (host arrays in and
out) and ``knn_search_device`` (device tensors, no host copies). Everything runs through the
C ABI of include/mihg.h (libmihg.so); there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np

from . import _lib
from .codes import BinaryCode, CodeDatabase, Partition, words_per_code


class Neighbor(NamedTuple):  # scan.hpp:14-19
    id: int
    dist: int


def neighbor_less(a: Neighbor, b: Neighbor) -> bool:  # scan.hpp:24-26
    return a.dist < b.dist if a.dist != b.dist else a.id < b.id


@dataclass
class SearchTrace:  # index.hpp:45-51
    lookups: int = 0
    candidates: int = 0
    unique_candidates: int = 0
    distance_evaluations: int = 0
    final_radius: int = 0


@dataclass
class TableStats:  # table.hpp:33-47
    non_empty_buckets: int = 0
    max_bucket_size: int = 0
    total_entries: int = 0
    estimated_bytes: int = 0


def _p64(a: np.ndarray):
    return a.ctypes.data_as(_lib.u64p)


def _p32(a: np.ndarray):
    return a.ctypes.data_as(_lib.u32p)


class SubstringTableView:
    """Read-only view of table j (the SubstringTable accessors callers use, table.hpp:161-197)."""

    def __init__(self, owner: "MihIndex", j: int):
        self._owner, self._j = owner, j
        info = _lib.TableInfo()
        _lib.check(_lib.lib().mihg_table_get_info(owner._h, j, C.byref(info)))
        self._info = info

    def s(self) -> int:
        return int(self._info.s)

    def size(self) -> int:
        return int(self._info.total_entries)

    def dense(self) -> bool:
        return bool(self._info.dense)

    def device_bytes(self) -> int:
        return int(self._info.device_bytes)

    def non_empty_buckets(self) -> int:
        return int(self._info.non_empty_buckets)

    def max_bucket_size(self) -> int:
        return int(self._info.max_bucket_size)

    def bucket_lookup(self, value: int) -> np.ndarray:
        """Ids of bucket `value` in insertion (= ascending id) order (table.hpp:169-175)."""
        cnt = C.c_uint64()
        L = _lib.lib()
        _lib.check(L.mihg_bucket_lookup(self._owner._h, self._j, value, None, 0, C.byref(cnt)))
        out = np.zeros(max(cnt.value, 1), np.uint32)
        _lib.check(L.mihg_bucket_lookup(self._owner._h, self._j, value, _p32(out), cnt.value, C.byref(cnt)))
        return out[: cnt.value]

    def stats(self) -> TableStats:
        return TableStats(int(self._info.non_empty_buckets), int(self._info.max_bucket_size),
                          int(self._info.total_entries), int(self._info.estimated_bytes))


class MihIndex:
    """GPU multi-index over m disjoint substrings (index.hpp:98-285)."""

    def __init__(self, h, db: CodeDatabase | None, partition: Partition, bits: int, n: int,
                 device: int, id_base: int):
        self._h = h
        self._db = db
        self._partition = partition
        self._bits = bits
        self._n = n
        self._device = device
        self._id_base = id_base

    # ---- construction -------------------------------------------------------------------
    @staticmethod
    def build(db: CodeDatabase, partition: Partition, device: int = 0, *, id_base: int = 0,
              layout: str = "auto", dense_max_bits: int = 0, keep_host_db: bool = True) -> "MihIndex":
        if partition.bits() != db.bits():
            raise ValueError("MihIndex::build: partition width does not match codes")
        for j in range(partition.m()):
            if partition.length(j) > 32:
                raise ValueError(
                    f"MihIndex::build: substring {j} is {partition.length(j)} bits; direct "
                    f"addressing supports at most 32 (use more substrings)")
        words = np.ascontiguousarray(db.raw_words(), dtype=np.uint64)
        return MihIndex._build_raw(words, db.size(), db.bits(), partition, device, id_base, layout,
                                   dense_max_bits, db if keep_host_db else None, on_device=False)

    @staticmethod
    def build_from_device(codes_ptr: int, n: int, bits: int, partition: Partition, device: int = 0,
                          *, id_base: int = 0, layout: str = "auto", dense_max_bits: int = 0) -> "MihIndex":
        """Build from codes already resident on `device` (e.g. a torch CUDA tensor's data_ptr)."""
        return MihIndex._build_raw(codes_ptr, n, bits, partition, device, id_base, layout,
                                   dense_max_bits, None, on_device=True)

    @staticmethod
    def _build_raw(words, n, bits, partition, device, id_base, layout, dense_max_bits, db, on_device):
        L = _lib.lib()
        lengths = partition.lengths_array()
        positions = partition.positions_array()
        p = _lib.BuildParams()
        p.codes = C.cast(C.c_void_p(words), _lib.u64p) if on_device else _p64(words)
        p.n = n
        p.bits = bits
        p.m = partition.m()
        p.lengths = _p32(lengths)
        p.positions = _p32(positions)
        p.device = device
        p.codes_on_device = 1 if on_device else 0
        p.id_base = id_base
        p.dense_max_bits = dense_max_bits
        p.layout = {"auto": 0, "dense": 1, "sparse": 2}[layout]
        h = C.c_void_p()
        _lib.check(L.mihg_index_build_ex(C.byref(p), C.byref(h)))
        return MihIndex(h, db, partition, bits, n, device, id_base)

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.lib().mihg_index_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- accessors (index.hpp:143-146) ----------------------------------------------------
    def db(self) -> CodeDatabase:
        if self._db is None:
            raise ValueError("MihIndex: host copy of the database was not kept")
        return self._db

    def partition(self) -> Partition:
        return self._partition

    def num_tables(self) -> int:
        return self._partition.m()

    def table(self, j: int) -> SubstringTableView:
        return SubstringTableView(self, j)

    def size(self) -> int:
        return self._n

    def bits(self) -> int:
        return self._bits

    def device(self) -> int:
        return self._device

    def device_bytes(self) -> int:
        info = _lib.IndexInfo()
        _lib.check(_lib.lib().mihg_index_get_info(self._h, C.byref(info)))
        return int(info.device_bytes)

    def codes_device_ptr(self) -> int:
        p = C.c_void_p()
        _lib.check(_lib.lib().mihg_index_codes(self._h, C.byref(p)))
        return int(p.value or 0)

    # ---- queries --------------------------------------------------------------------------
    def _queries(self, queries) -> np.ndarray:
        q = np.ascontiguousarray(queries, dtype=np.uint64)
        wpc = words_per_code(self._bits)
        if q.size % wpc:
            raise ValueError("knn_search: query width mismatch")
        return q.reshape(-1, wpc)

    def knn_search(self, q: BinaryCode, k: int, trace: SearchTrace | None = None, scratch=None):
        """index.hpp:185-253. `scratch` is accepted for signature parity (the GPU workspace is
        per index)."""
        if q.bits != self._bits:
            raise ValueError("knn_search: query width mismatch")
        if k > self._n:
            raise ValueError("knn_search: k exceeds database size")
        res = self.knn_search_batch(q.words.reshape(1, -1), k, with_trace=trace is not None)
        ids, dists = res[0], res[1]
        if trace is not None:
            t = res[2][0]
            trace.lookups, trace.candidates = int(t.lookups), int(t.candidates)
            trace.unique_candidates = int(t.unique_candidates)
            trace.distance_evaluations = int(t.distance_evaluations)
            trace.final_radius = int(t.final_radius)
        return [Neighbor(int(i), int(d)) for i, d in zip(ids[0], dists[0])]

    def knn_search_batch(self, queries, k: int, with_trace: bool = False):
        """Returns ids[nq, k], dists[nq, k] (uint32) and, if requested, a ctypes Trace array."""
        q = self._queries(queries)
        nq = q.shape[0]
        if k > self._n:
            raise ValueError("knn_search: k exceeds database size")
        ids = np.zeros((nq, k), np.uint32)
        dists = np.zeros((nq, k), np.uint32)
        tr = (_lib.Trace * max(nq, 1))() if with_trace else None
        _lib.check(_lib.lib().mihg_knn_batch(self._h, _p64(q), nq, k, _p32(ids), _p32(dists), tr))
        return (ids, dists, tr) if with_trace else (ids, dists)

    def knn_search_device(self, d_queries, nq: int, k: int, d_ids, d_dists, d_traces=None,
                          stream: int = 0, partition=None) -> None:
        """Device-pointer batch (ints from torch .data_ptr()); ordered on `stream`.

        partition=(count, rank, allreduce) runs the probe-space partitioned search of one rank:
        ``allreduce(dev_ptr, n, dtype, stream)`` sums n device elements (dtype 0 u32, 1 u64) in
        place across ranks; the outputs are this rank's local top-k (merge across ranks).
        partition=(count, rank, allreduce, True[, k_stop]) is the id-range-shard layout with global
        stopping instead (this index holds one shard, built with id_base); k_stop is the global k
        of the stopping rule when this shard's k is clamped below it (default: k)."""
        L = _lib.lib()
        sp = C.c_void_p(stream) if stream else None
        tr = C.c_void_p(d_traces) if d_traces else None
        if partition is None:
            _lib.check(L.mihg_knn_batch_device(self._h, C.c_void_p(d_queries), nq, k, C.c_void_p(d_ids),
                                               C.c_void_p(d_dists), tr, sp))
            return
        count, rank, fn = partition[:3]
        id_shards = bool(partition[3]) if len(partition) > 3 else False
        k_stop = int(partition[4]) if len(partition) > 4 else 0
        errors = []

        def _cb(user, ptr, n, dtype, strm):
            try:
                fn(int(ptr), int(n), int(dtype), int(strm or 0))
                return 0
            except Exception as e:  # surfaced after the call returns
                errors.append(e)
                return 1

        cb = _lib.ALLREDUCE_FN(_cb)
        part = _lib.Partition(count, rank, cb, None, 1 if id_shards else 0, k_stop)
        rc = L.mihg_knn_batch_device_part(self._h, C.c_void_p(d_queries), nq, k, C.c_void_p(d_ids),
                                          C.c_void_p(d_dists), tr, C.byref(part), sp)
        if errors:
            raise errors[0]
        _lib.check(rc)

    def range_search(self, q: BinaryCode, r: int, trace: SearchTrace | None = None, scratch=None):
        """index.hpp:149-176: exactly {(i, d_i) : d_i <= r}, sorted by (distance, id)."""
        if q.bits != self._bits:
            raise ValueError("range_search: query width mismatch")
        offs, ids, dists, tr = self.range_search_batch(q.words.reshape(1, -1), r, with_trace=trace is not None)
        if trace is not None:
            t = tr[0]
            trace.lookups, trace.candidates = int(t.lookups), int(t.candidates)
            trace.unique_candidates = int(t.unique_candidates)
            trace.distance_evaluations = int(t.distance_evaluations)
            trace.final_radius = int(t.final_radius)
        return [Neighbor(int(i), int(d)) for i, d in zip(ids, dists)]

    def range_search_batch(self, queries, r: int, with_trace: bool = False):
        """Returns (offsets[nq+1], ids, dists, traces|None): query i's neighbours are
        ids[offsets[i]:offsets[i+1]] in (dist, id) order."""
        q = self._queries(queries)
        nq = q.shape[0]
        if r > self._bits:
            raise ValueError("range_search: radius exceeds code width")
        offs = np.zeros(nq + 1, np.uint64)
        tr = (_lib.Trace * max(nq, 1))() if with_trace else None
        L = _lib.lib()
        cap = min(self._n * nq, 1 << 22)
        while True:
            ids = np.zeros(max(cap, 1), np.uint32)
            dists = np.zeros(max(cap, 1), np.uint32)
            _lib.check(L.mihg_range_batch(self._h, _p64(q), nq, r, _p64(offs), _p32(ids), _p32(dists), cap, tr))
            total = int(offs[nq])
            if total <= cap:
                return offs, ids[:total], dists[:total], tr
            cap = total

    def scan_knn_batch(self, queries, k: int):
        """Exhaustive GPU comparator over the index's codes (scan.hpp:43-68 semantics)."""
        q = self._queries(queries)
        nq = q.shape[0]
        if k > self._n:
            raise ValueError("scan_knn: k exceeds database size")
        ids = np.zeros((nq, k), np.uint32)
        dists = np.zeros((nq, k), np.uint32)
        _lib.check(_lib.lib().mihg_scan_knn_batch(self._h, _p64(q), nq, k, _p32(ids), _p32(dists)))
        return ids, dists

    def scan_knn_device(self, d_queries, nq: int, k: int, d_ids, d_dists, stream: int = 0) -> None:
        _lib.check(_lib.lib().mihg_scan_knn_batch_device(self._h, C.c_void_p(d_queries), nq, k,
                                                         C.c_void_p(d_ids), C.c_void_p(d_dists),
                                                         C.c_void_p(stream) if stream else None))


def build_index(db: CodeDatabase, partition: Partition, device: int = 0) -> MihIndex:  # index.hpp:287
    return MihIndex.build(db, partition, device)


def scan_knn(db: CodeDatabase, q: BinaryCode, k: int, device: int = 0):
    """scan_knn (scan.hpp:43-68) on the GPU for a single query."""
    if q.bits != db.bits():
        raise ValueError("scan_knn: query width mismatch")
    if k > db.size():
        raise ValueError("scan_knn: k exceeds database size")
    if k == 0:
        return []
    import torch  # device memory plumbing only

    dev = torch.device("cuda", device)
    codes = torch.from_numpy(np.ascontiguousarray(db.raw_words()).view(np.int64)).to(dev)
    qq = torch.from_numpy(np.ascontiguousarray(q.words).view(np.int64)).to(dev)
    ids = torch.empty(k, dtype=torch.int32, device=dev)
    dists = torch.empty(k, dtype=torch.int32, device=dev)
    _lib.check(_lib.lib().mihg_scan_knn_raw_device(C.c_void_p(codes.data_ptr()), db.size(), db.bits(), 0,
                                                   C.c_void_p(qq.data_ptr()), 1, k,
                                                   C.c_void_p(ids.data_ptr()), C.c_void_p(dists.data_ptr()),
                                                   None))
    torch.cuda.synchronize(dev)
    i = ids.cpu().numpy().view(np.uint32)
    d = dists.cpu().numpy().view(np.uint32)
    return [Neighbor(int(a), int(b)) for a, b in zip(i, d)]
