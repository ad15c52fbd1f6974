"""ctypes binding of the C ABI in include/mihg.h (libmihg.so, built in-tree for sm_100a).

There is no CPU fallback: if the shared library is missing, importing the package's compute API
raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MIHG_LIB_PATH") or os.path.join(_HERE, "libmihg.so")  # override: A/B builds

MIHG_OK, MIHG_EINVAL, MIHG_EINTERNAL, MIHG_ENOMEM, MIHG_ECUDA, MIHG_ENCCL, MIHG_EFORMAT, MIHG_EIO = range(8)

u64p = C.POINTER(C.c_uint64)
u32p = C.POINTER(C.c_uint32)


class MihgError(RuntimeError):
    """A failing mihg C-ABI call (CUDA, internal)."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"mihg error {code}: {msg}")
        self.code = code


class Trace(C.Structure):
    """mihg_trace == mih::SearchTrace (index.hpp:45-51)."""

    _fields_ = [("lookups", C.c_uint64), ("candidates", C.c_uint64),
                ("unique_candidates", C.c_uint64), ("distance_evaluations", C.c_uint64),
                ("final_radius", C.c_uint32), ("reserved", C.c_uint32)]


class BuildParams(C.Structure):
    _fields_ = [("codes", u64p), ("n", C.c_uint64), ("bits", C.c_uint32), ("m", C.c_uint32),
                ("lengths", u32p), ("positions", u32p), ("device", C.c_int),
                ("codes_on_device", C.c_int), ("id_base", C.c_uint32),
                ("dense_max_bits", C.c_uint32), ("layout", C.c_int)]


class IndexInfo(C.Structure):
    _fields_ = [("n", C.c_uint64), ("bits", C.c_uint32), ("m", C.c_uint32),
                ("id_base", C.c_uint32), ("device", C.c_int), ("device_bytes", C.c_uint64)]


class TableInfo(C.Structure):
    _fields_ = [("s", C.c_uint32), ("dense", C.c_uint32), ("non_empty_buckets", C.c_uint64),
                ("max_bucket_size", C.c_uint64), ("total_entries", C.c_uint64),
                ("estimated_bytes", C.c_uint64), ("device_bytes", C.c_uint64),
                ("escaped_blocks", C.c_uint64)]


ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_void_p)


class Partition(C.Structure):
    """mihg_partition: probe-space partition of a multi-GPU kNN call."""

    _fields_ = [("count", C.c_uint32), ("rank", C.c_uint32), ("allreduce", ALLREDUCE_FN),
                ("user", C.c_void_p), ("id_shards", C.c_uint32), ("k_stop", C.c_uint32),
                ("comm", C.c_void_p)]


class Profile(C.Structure):
    _fields_ = [("kernel_launches", C.c_uint64), ("probe_ms", C.c_double),
                ("probe_launches", C.c_uint64), ("scan_ms", C.c_double),
                ("scan_launches", C.c_uint64), ("switched_queries", C.c_uint64),
                ("rerun_queries", C.c_uint64), ("rerun_ms", C.c_double)]


# every symbol include/mihg.h declares: (name, restype, argtypes)
SYMBOLS = [
    ("mihg_last_error", C.c_char_p, []),
    ("mihg_abi_version", C.c_int, []),
    ("mihg_device_count", C.c_int, [C.POINTER(C.c_int)]),
    ("mihg_index_build", C.c_int, [u64p, C.c_uint64, C.c_uint32, C.c_uint32, u32p, u32p, C.c_int,
                                   C.POINTER(C.c_void_p)]),
    ("mihg_index_build_ex", C.c_int, [C.POINTER(BuildParams), C.POINTER(C.c_void_p)]),
    ("mihg_index_free", None, [C.c_void_p]),
    ("mihg_index_get_info", C.c_int, [C.c_void_p, C.POINTER(IndexInfo)]),
    ("mihg_table_get_info", C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(TableInfo)]),
    ("mihg_bucket_lookup", C.c_int, [C.c_void_p, C.c_uint32, C.c_uint64, u32p, C.c_uint64, u64p]),
    ("mihg_index_write", C.c_int, [C.c_void_p, C.c_char_p]),
    ("mihg_index_read", C.c_int, [C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]),
    ("mihg_index_codes", C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    ("mihg_knn_batch", C.c_int, [C.c_void_p, u64p, C.c_uint64, C.c_uint32, u32p, u32p,
                                 C.POINTER(Trace)]),
    ("mihg_knn_batch_device", C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_void_p,
                                        C.c_void_p, C.c_void_p, C.c_void_p]),
    ("mihg_range_batch", C.c_int, [C.c_void_p, u64p, C.c_uint64, C.c_uint32, u64p, u32p, u32p,
                                   C.c_uint64, C.POINTER(Trace)]),
    ("mihg_knn_batch_device_part", C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32,
                                             C.c_void_p, C.c_void_p, C.c_void_p,
                                             C.POINTER(Partition), C.c_void_p]),
    ("mihg_comm_unique_id", C.c_int, [C.POINTER(C.c_uint8)]),
    ("mihg_comm_init", C.c_int, [C.POINTER(C.c_uint8), C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    ("mihg_comm_free", None, [C.c_void_p]),
    ("mihg_nccl_version", C.c_int, [C.POINTER(C.c_int)]),
    ("mihg_knn_sharded_device", C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_uint64, C.c_void_p,
                                          C.c_uint64, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.c_void_p]),
    ("mihg_scan_knn_batch", C.c_int, [C.c_void_p, u64p, C.c_uint64, C.c_uint32, u32p, u32p]),
    ("mihg_scan_knn_batch_device", C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32,
                                             C.c_void_p, C.c_void_p, C.c_void_p]),
    ("mihg_scan_knn_raw_device", C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32,
                                           C.c_void_p, C.c_uint64, C.c_uint32, C.c_void_p,
                                           C.c_void_p, C.c_void_p]),
    ("mihg_scan_kernel_for", C.c_int, [C.c_uint32]),
    ("mihg_tc_distances_device", C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, C.c_void_p, C.c_uint64,
                                           C.c_void_p, C.c_void_p]),
    ("mihg_merge_topk_device", C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint64,
                                         C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p,
                                         C.c_void_p]),
    ("mihg_gen_uniform", C.c_int, [C.c_uint64, C.c_uint32, C.c_uint64, u64p]),
    ("mihg_mt64_create", C.c_int, [C.c_uint64, C.POINTER(C.c_void_p)]),
    ("mihg_mt64_next_codes", C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, u64p]),
    ("mihg_mt64_free", None, [C.c_void_p]),
    ("mihg_gen_uniform_range", C.c_int, [C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint64, u64p]),
    ("mihg_gen_mixture_device", C.c_int, [C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32,
                                          C.c_uint32, C.c_uint64, C.c_uint64, C.c_void_p,
                                          C.c_void_p]),
    ("mihg_estimate_correlations", C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, C.c_int, C.c_int,
                                             C.POINTER(C.c_double), C.POINTER(C.c_uint8), u64p]),
    ("mihg_greedy_assign", C.c_int, [C.POINTER(C.c_double), C.POINTER(C.c_uint8), C.c_uint32,
                                     C.c_uint32, C.c_uint64, u32p, u32p]),
    ("mihg_profile_enable", C.c_int, [C.c_int]),
    ("mihg_profile_reset", None, []),
    ("mihg_profile_read", C.c_int, [C.POINTER(Profile)]),
    ("mihg_calibrate_random_lookups", C.c_int, [C.c_int, C.c_uint64, C.c_uint64, C.c_uint32,
                                                C.POINTER(C.c_double)]),
]

_lib = None


def lib():
    """Load libmihg.so once. Raises if the CUDA extension has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"CUDA extension missing: {LIB_PATH}. Build it with `python -c 'import "
                f"__graft_entry__ as g; g.build()'` (no CPU fallback exists).")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SYMBOLS:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == MIHG_OK:
        return
    msg = lib().mihg_last_error().decode(errors="replace")
    if rc == MIHG_EINVAL:
        raise ValueError(msg)  # the reference throws std::invalid_argument
    if rc == MIHG_ENOMEM:
        raise MemoryError(msg)  # std::bad_alloc
    if rc == MIHG_EFORMAT:
        import re

        from .io import FormatError

        m = re.search(r"\(byte offset (\d+)\)$", msg)
        raise FormatError(msg[: m.start()].rstrip() if m else msg, int(m.group(1)) if m else 0)
    if rc == MIHG_EIO:
        raise OSError(msg)
    raise MihgError(rc, msg)
