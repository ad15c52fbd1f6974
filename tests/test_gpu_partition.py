"""GPU: probe-space partitioned kNN (the multi-GPU algorithm) emulated with G host threads on one
GPU. Each "rank" has its own index handle and stream; the per-round all-reduce is a host barrier
that sums the ranks' device buffers (no kernel ever waits on another). The merged local top-k
lists must equal the single-index result, and the all-reduced traces the single-index traces."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run_partitioned(mg, db, part, qs, k, G, traced):
    import torch

    from paper_1307_2982_b200.shard import _CudaArray

    nq = qs.shape[0]
    idxs = [mg.MihIndex.build(db, part) for _ in range(G)]
    dq = torch.from_numpy(np.ascontiguousarray(qs).view(np.int64)).cuda()
    barrier = threading.Barrier(G)
    slots = [None] * G
    outs = [None] * G
    errs = []

    def make_ar(rank):
        def ar(ptr, n, dtype, stream):
            t = torch.as_tensor(_CudaArray(ptr, n, "<i4" if dtype == 0 else "<i8"), device="cuda")
            s = torch.cuda.ExternalStream(stream)
            s.synchronize()
            slots[rank] = t.cpu()
            barrier.wait()
            total = sum(slots[1:], slots[0].clone())
            barrier.wait()
            with torch.cuda.stream(s):
                t.copy_(total.cuda())
            s.synchronize()
        return ar

    def worker(rank):
        try:
            st = torch.cuda.Stream()
            ids = torch.empty((nq, k), dtype=torch.int32, device="cuda")
            d = torch.empty((nq, k), dtype=torch.int32, device="cuda")
            tr = torch.empty((nq, 5), dtype=torch.int64, device="cuda") if traced else None
            idxs[rank].knn_search_device(dq.data_ptr(), nq, k, ids.data_ptr(), d.data_ptr(),
                                         tr.data_ptr() if traced else None, stream=st.cuda_stream,
                                         partition=(G, rank, make_ar(rank)))
            st.synchronize()
            outs[rank] = (ids.cpu(), d.cpu(), tr.cpu() if traced else None)
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)
            barrier.abort()

    th = [threading.Thread(target=worker, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    if errs:
        raise errs[0]
    from _helpers import numpy_merge

    all_i = torch.stack([o[0] for o in outs])
    all_d = torch.stack([o[1] for o in outs])
    mi, md = numpy_merge(all_i, all_d, k)
    return mi.numpy().view(np.uint32), md.numpy().view(np.uint32), (outs[0][2].numpy() if traced else None)


@pytest.mark.parametrize("G", [2, 4])
@pytest.mark.parametrize("bits,m,n", [(64, 2, 300000), (64, 4, 200000), (128, 6, 100000)])
def test_partitioned_equals_single_index(cuda_ok, bits, m, n, G):
    import paper_1307_2982_b200 as mg

    db = mg.gen_uniform(n, bits, 700 + bits + m)
    qs = mg.gen_uniform(32, bits, 800 + bits + m).raw_words()
    part = mg.consecutive_partition(bits, m)
    single = mg.MihIndex.build(db, part)
    for k in (10, 100):
        si, sd, st = single.knn_search_batch(qs, k, with_trace=True)
        for traced in (True, False):
            pi, pd, pt = _run_partitioned(mg, db, part, qs, k, G, traced)
            assert np.array_equal(pi, si) and np.array_equal(pd, sd), (G, k, traced)
            if traced:
                want = np.array([[t.lookups, t.candidates, t.unique_candidates, t.distance_evaluations,
                                  t.final_radius] for t in st], np.int64)
                assert np.array_equal(pt, want), (G, k)


def test_nccl_allreduce_callback_plumbing(cuda_ok):
    """shard.nccl_allreduce wraps raw device memory (__cuda_array_interface__) and all-reduces it
    on the library's stream through torch.distributed/NCCL (1-rank group here)."""
    import os
    import socket

    import torch
    import torch.distributed as dist

    from paper_1307_2982_b200.shard import nccl_allreduce

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        fn = nccl_allreduce()
        st = torch.cuda.Stream()
        a = torch.arange(1000, dtype=torch.int32, device="cuda")
        b = torch.arange(1000, dtype=torch.int64, device="cuda") * (1 << 33)
        fn(a.data_ptr(), a.numel(), 0, st.cuda_stream)
        fn(b.data_ptr(), b.numel(), 1, st.cuda_stream)
        st.synchronize()
        assert torch.equal(a.cpu(), torch.arange(1000, dtype=torch.int32))
        assert torch.equal(b.cpu(), torch.arange(1000, dtype=torch.int64) * (1 << 33))
    finally:
        dist.destroy_process_group()


def _run_id_shards(mg, db, part, qs, k, G, traced):
    """G id-range shards (own index over ids [lo, hi) with id_base = lo) with global stopping; the
    all-reduce is a host barrier sum. Returns merged ids/dists and every shard's traces."""
    import torch

    from paper_1307_2982_b200.shard import _CudaArray, shard_range

    n, nq = db.size(), qs.shape[0]
    words = db.raw_words()
    idxs = []
    for r in range(G):
        lo, hi = shard_range(n, r, G)
        idxs.append(mg.MihIndex.build(mg.CodeDatabase(db.bits(), words[lo:hi]), part, id_base=lo))
    dq = torch.from_numpy(np.ascontiguousarray(qs).view(np.int64)).cuda()
    barrier = threading.Barrier(G)
    slots = [None] * G
    outs = [None] * G
    errs = []

    def make_ar(rank):
        def ar(ptr, cnt, dtype, stream):
            t = torch.as_tensor(_CudaArray(ptr, cnt, "<i4" if dtype == 0 else "<i8"), device="cuda")
            s = torch.cuda.ExternalStream(stream)
            s.synchronize()
            slots[rank] = t.cpu()
            barrier.wait()
            total = sum(slots[1:], slots[0].clone())
            barrier.wait()
            with torch.cuda.stream(s):
                t.copy_(total.cuda())
            s.synchronize()
        return ar

    def worker(rank):
        try:
            st = torch.cuda.Stream()
            kk = min(k, idxs[rank].size())
            ids = torch.full((nq, k), -1, dtype=torch.int32, device="cuda")
            d = torch.full((nq, k), -1, dtype=torch.int32, device="cuda")
            li = torch.empty((nq, kk), dtype=torch.int32, device="cuda")
            ld = torch.empty((nq, kk), dtype=torch.int32, device="cuda")
            tr = torch.empty((nq, 5), dtype=torch.int64, device="cuda") if traced else None
            idxs[rank].knn_search_device(dq.data_ptr(), nq, kk, li.data_ptr(), ld.data_ptr(),
                                         tr.data_ptr() if traced else None, stream=st.cuda_stream,
                                         partition=(G, rank, make_ar(rank), True))
            st.synchronize()
            ids[:, :kk] = li
            d[:, :kk] = ld
            outs[rank] = (ids.cpu(), d.cpu(), tr.cpu() if traced else None)
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)
            barrier.abort()

    th = [threading.Thread(target=worker, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    if errs:
        raise errs[0]
    from _helpers import numpy_merge

    mi, md = numpy_merge(torch.stack([o[0] for o in outs]), torch.stack([o[1] for o in outs]), k)
    return mi.numpy().view(np.uint32), md.numpy().view(np.uint32), [o[2] for o in outs]


@pytest.mark.parametrize("G", [2, 3, 4])
@pytest.mark.parametrize("bits,m,n", [(64, 2, 300000), (64, 4, 200000), (128, 6, 100000)])
def test_id_shards_global_stopping_equal_single_index(cuda_ok, bits, m, n, G):
    """§8e refinement 1: id-range shards whose per-round histograms are summed stop at the global
    d_k; merged results equal the single index, and the summed candidate/unique counts, every
    shard's lookups and final radius equal the single-index trace."""
    import paper_1307_2982_b200 as mg

    db = mg.gen_uniform(n, bits, 900 + bits + m)
    qs = mg.gen_uniform(32, bits, 901 + bits + m).raw_words()
    part = mg.consecutive_partition(bits, m)
    single = mg.MihIndex.build(db, part)
    for k in (10, 100):
        si, sd, st = single.knn_search_batch(qs, k, with_trace=True)
        want = np.array([[t.lookups, t.candidates, t.unique_candidates, t.distance_evaluations,
                          t.final_radius] for t in st], np.int64)
        for traced in (True, False):
            pi, pd, trs = _run_id_shards(mg, db, part, qs, k, G, traced)
            assert np.array_equal(pi, si) and np.array_equal(pd, sd), (G, k, traced)
            if traced:
                for t in trs:
                    assert np.array_equal(t.numpy(), want), (G, k)
