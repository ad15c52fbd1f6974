"""Id-range sharded exact kNN over the ranks of a torch.distributed group.

Rank r owns ids [r*ceil(n/G), (r+1)*ceil(n/G)) and an index over them built with
``id_base = first id`` (global id = local id + id_base). A query batch is answered by every rank
with its exact local top-k (k clamped to the shard size, padded with dist 0xFFFFFFFF), the
per-rank lists are exchanged in ONE collective (all-gather over NCCL/NVLink), and an exact k-way
merge keeps the k smallest packed keys (dist << 32 | id). Exact by construction: the global
top-k under the reference's (dist, id) order (scan.hpp:24-26) lies in the union of the local
top-k sets, and the id offsets preserve order within and across shards.

The local search and the merge are injectable so the host logic can be exercised on CPU with the
gloo backend; the defaults are the GPU kernels (``MihIndex.knn_search_device`` and
``mihg_merge_topk_device``) — there is no CPU fallback in the product path.
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, Optional

PAD = 0xFFFFFFFF


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    per = (n + world - 1) // world
    lo = min(n, rank * per)
    return lo, min(n, lo + per)


class _CudaArray:
    """Zero-copy view of raw device memory for torch (``__cuda_array_interface__``)."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def nccl_allreduce(group=None):
    """Callback for MihIndex.knn_search_device(partition=...): in-place SUM over the group of a
    device buffer (u32 counts as int32, u64 as int64), ordered on the library's stream."""
    import torch
    import torch.distributed as dist

    def fn(ptr: int, n: int, dtype: int, stream: int):
        t = torch.as_tensor(_CudaArray(ptr, n, "<i4" if dtype == 0 else "<i8"), device="cuda")
        with torch.cuda.stream(torch.cuda.ExternalStream(stream)) if stream else _nullctx():
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)

    return fn


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


class NcclComm:
    """The library's own NCCL communicator (mihg_comm_init) over the ranks of a torch.distributed
    group: rank 0 draws the unique id, the group broadcasts it once (the only host-side step),
    and from then on every collective of the sharded search is enqueued by libmihg itself."""

    def __init__(self, device: int, group=None):
        import torch
        import torch.distributed as dist

        from . import _lib

        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        uid = (C.c_uint8 * 128)()
        if self.rank == 0:
            _lib.check(_lib.lib().mihg_comm_unique_id(uid))
        on = torch.device("cuda", device) if dist.get_backend(group) == "nccl" else "cpu"
        t = torch.tensor(list(bytes(uid)), dtype=torch.uint8, device=on)
        dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        uid = (C.c_uint8 * 128)(*t.cpu().tolist())
        h = C.c_void_p()
        _lib.check(_lib.lib().mihg_comm_init(uid, self.world, self.rank, device, C.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    def close(self):
        from . import _lib

        if self._h:
            _lib.lib().mihg_comm_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def native_sharded_search(index, comm: NcclComm, layout: str, n_total: int, queries, k: int, traces=None,
                          stream: int = 0):
    """Exact global top-k on every rank in ONE library call (mihg_knn_sharded_device): local search
    with the per-round NCCL histogram all-reduce, NCCL all-gather of the local lists, device merge.
    layout: "probe" (replicated index, probe-space partition) or "id" (id-range shards)."""
    import torch

    from . import _lib

    nq = queries.shape[0]
    ids = torch.empty((nq, k), dtype=torch.int32, device=queries.device)
    d = torch.empty_like(ids)
    stream = stream or torch.cuda.current_stream(queries.device).cuda_stream
    _lib.check(_lib.lib().mihg_knn_sharded_device(index._h, comm.handle, 0 if layout == "probe" else 1, n_total,
                                                  C.c_void_p(queries.data_ptr()), nq, k, C.c_void_p(ids.data_ptr()),
                                                  C.c_void_p(d.data_ptr()),
                                                  C.c_void_p(traces.data_ptr()) if traces is not None else None,
                                                  C.c_void_p(stream)))
    return ids, d


def gpu_merge(all_ids, all_dists, k: int):
    """Exact k-way merge on the GPU: all_* are int32 CUDA tensors [G, nq, k_in]."""
    import torch

    from . import _lib

    G, nq, k_in = all_ids.shape
    out_ids = torch.empty((nq, k), dtype=torch.int32, device=all_ids.device)
    out_d = torch.empty((nq, k), dtype=torch.int32, device=all_ids.device)
    stream = torch.cuda.current_stream(all_ids.device).cuda_stream
    _lib.check(_lib.lib().mihg_merge_topk_device(C.c_void_p(all_ids.data_ptr()), C.c_void_p(all_dists.data_ptr()),
                                                 G, nq, k_in, k, C.c_void_p(out_ids.data_ptr()),
                                                 C.c_void_p(out_d.data_ptr()), C.c_void_p(stream)))
    return out_ids, out_d


class ShardedKnn:
    """One rank's view of an id-range sharded index.

    ``local_search(queries, k_local, k_global, collective)`` returns the rank's exact local top
    ``k_local`` as int32 [nq, k_local] (global ids). With ``collective`` it runs the per-round
    histogram all-reduce of global stopping, so every rank of the group must call it together."""

    def __init__(self, local_search: Callable, n_local: int, group=None,
                 merge: Optional[Callable] = None, global_stopping: bool = False):
        import torch.distributed as dist

        self.local_search = local_search
        self.n_local = n_local
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.merge = merge or gpu_merge
        self.global_stopping = global_stopping and self.world > 1
        self._min_local = None

    @classmethod
    def probe_partitioned(cls, index, group=None):
        """Every rank holds the full index and probes only its slice of the substring key
        space (rank = top log2(G) key bits); per-round histograms are all-reduced over NCCL so
        all ranks stop together, and the local top-k lists merge exactly. Divides probe and
        verification work by G (id-range shards cannot: SURVEY.md §7 hard part 5)."""
        import torch
        import torch.distributed as dist

        world, rank = dist.get_world_size(group), dist.get_rank(group)
        ar = nccl_allreduce(group)

        def local(queries, k, k_global=None, collective=True):
            nq = queries.shape[0]
            ids = torch.empty((nq, k), dtype=torch.int32, device=queries.device)
            d = torch.empty((nq, k), dtype=torch.int32, device=queries.device)
            index.knn_search_device(queries.data_ptr(), nq, k, ids.data_ptr(), d.data_ptr(),
                                    stream=torch.cuda.current_stream(queries.device).cuda_stream,
                                    partition=(world, rank, ar) if world > 1 else None)
            return ids, d

        return cls(local, index.size(), group)

    @classmethod
    def from_index(cls, index, group=None, global_stopping: bool = True):
        """Wrap a local ``MihIndex`` (built with id_base = shard start) whose queries live on the GPU.
        With ``global_stopping`` (SURVEY §8e refinement 1) the per-round histograms are summed
        over the group so every shard stops at the global d_k, not its larger local d_k."""
        import torch
        import torch.distributed as dist

        world, rank = dist.get_world_size(group), dist.get_rank(group)
        ar = nccl_allreduce(group) if (global_stopping and world > 1) else None

        def local(queries, k, k_global=None, collective=False):
            nq = queries.shape[0]
            ids = torch.empty((nq, k), dtype=torch.int32, device=queries.device)
            d = torch.empty((nq, k), dtype=torch.int32, device=queries.device)
            # the stopping rule of global stopping uses the caller's global k (a shard smaller
            # than k searches its whole local k = n_local but stops with the others)
            part = (world, rank, ar, True, k_global or k) if collective else None
            index.knn_search_device(queries.data_ptr(), nq, k, ids.data_ptr(), d.data_ptr(),
                                    stream=torch.cuda.current_stream(queries.device).cuda_stream,
                                    partition=part)
            return ids, d

        return cls(local, index.size(), group, global_stopping=ar is not None)

    def _smallest_shard(self, device):
        """min over ranks of the shard sizes (identical on every rank; one collective, cached)."""
        import torch
        import torch.distributed as dist

        if self._min_local is None:
            on = device if dist.get_backend(self.group) == "nccl" else "cpu"
            t = torch.tensor([self.n_local], dtype=torch.int64, device=on)
            dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.group)
            self._min_local = int(t.item())
        return self._min_local

    def search(self, queries, k: int):
        """Exact global top-k for every query (all ranks return the same result)."""
        import torch
        import torch.distributed as dist

        nq = queries.shape[0]
        kk = min(k, self.n_local)
        # global stopping needs every rank in every round: an empty shard cannot search, so then
        # all ranks (same decision everywhere) stop on their local counts instead (also exact)
        collective = self.global_stopping and self._smallest_shard(queries.device) > 0
        if kk > 0:
            ids, d = self.local_search(queries, kk, k, collective)
        else:
            ids = torch.empty((nq, 0), dtype=torch.int32, device=queries.device)
            d = torch.empty((nq, 0), dtype=torch.int32, device=queries.device)
        if kk < k:  # shard smaller than k: pad (dist 0xFFFFFFFF sorts last, never selected first)
            pad = torch.full((nq, k - kk), -1, dtype=torch.int32, device=queries.device)
            ids = torch.cat([ids, pad], 1)
            d = torch.cat([d, pad], 1)
        ids, d = ids.contiguous(), d.contiguous()
        all_ids = torch.empty((self.world, nq, k), dtype=torch.int32, device=queries.device)
        all_d = torch.empty_like(all_ids)
        if dist.get_backend(self.group) == "nccl":
            dist.all_gather_into_tensor(all_ids, ids, group=self.group)
            dist.all_gather_into_tensor(all_d, d, group=self.group)
        else:
            dist.all_gather(list(all_ids.unbind(0)), ids, group=self.group)
            dist.all_gather(list(all_d.unbind(0)), d, group=self.group)
        return self.merge(all_ids, all_d, k)
