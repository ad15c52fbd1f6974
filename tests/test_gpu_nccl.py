"""GPU: the library-owned NCCL path of the multi-GPU layouts: mihg_comm_* and
mihg_knn_sharded_device, where the per-round histogram all-reduce, the all-gather of the local
top-k lists and the exact merge all run inside libmihg (no host language in the round loop).

One GPU is visible on the test boxes, so the collective path runs on a one-rank NCCL group (the
all-reduce and all-gather are real NCCL calls on the index stream); the two-process test runs
when two GPUs are visible and is skipped otherwise. Results and traces must equal the single
index (ids, dists, SearchTrace)."""
import ctypes as C
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _one_rank_comm(_lib):
    uid = (C.c_uint8 * 128)()
    _lib.check(_lib.lib().mihg_comm_unique_id(uid))
    h = C.c_void_p()
    _lib.check(_lib.lib().mihg_comm_init(uid, 1, 0, 0, C.byref(h)))
    return h


def _sharded(_lib, idx, comm, layout, n_total, dq, k, traced):
    import torch

    nq = dq.shape[0]
    ids = torch.empty((nq, k), dtype=torch.int32, device="cuda")
    d = torch.empty_like(ids)
    tr = torch.zeros((nq, 5), dtype=torch.int64, device="cuda") if traced else None
    st = torch.cuda.Stream()
    _lib.check(_lib.lib().mihg_knn_sharded_device(idx._h, comm, layout, n_total, C.c_void_p(dq.data_ptr()), nq, k,
                                                  C.c_void_p(ids.data_ptr()), C.c_void_p(d.data_ptr()),
                                                  C.c_void_p(tr.data_ptr()) if traced else None,
                                                  C.c_void_p(st.cuda_stream)))
    st.synchronize()
    return ids.cpu().numpy().view(np.uint32), d.cpu().numpy().view(np.uint32), (tr.cpu().numpy() if traced else None)


@pytest.mark.parametrize("n,bits,m,k", [(20000, 64, 4, 10), (5000, 128, 6, 100), (300, 64, 2, 300)])
def test_one_rank_nccl_sharded_equals_single_index(cuda_ok, n, bits, m, k):
    import torch

    import paper_1307_2982_b200 as mg
    from paper_1307_2982_b200 import _lib

    v = C.c_int()
    _lib.check(_lib.lib().mihg_nccl_version(C.byref(v)))
    assert v.value >= 21800
    db = mg.gen_uniform(n, bits, 31 + bits)
    qs = mg.gen_uniform(40, bits, 32 + bits).raw_words()
    idx = mg.MihIndex.build(db, mg.consecutive_partition(bits, m))
    want_i, want_d, want_tr = idx.knn_search_batch(qs, k, with_trace=True)
    want_t = np.array([[t.lookups, t.candidates, t.unique_candidates, t.distance_evaluations, t.final_radius]
                       for t in want_tr], np.int64)
    dq = torch.from_numpy(np.ascontiguousarray(qs).view(np.int64)).cuda()
    comm = _one_rank_comm(_lib)
    try:
        for layout in (0, 1):
            for traced in (False, True):
                i, d, t = _sharded(_lib, idx, comm, layout, n, dq, k, traced)
                assert np.array_equal(i, want_i) and np.array_equal(d, want_d), (layout, traced)
                if traced:
                    assert np.array_equal(t, want_t), layout
        # contract errors: wrong n_total for the layout, k > n_total
        with pytest.raises(ValueError):
            _sharded(_lib, idx, comm, 0, n + 1, dq, k, False)
        with pytest.raises(ValueError):
            _sharded(_lib, idx, comm, 1, n, dq, n + 1, False)
    finally:
        _lib.lib().mihg_comm_free(comm)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _two_rank_worker(rank, world, port, q):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        import paper_1307_2982_b200 as mg
        from paper_1307_2982_b200.shard import NcclComm, native_sharded_search, shard_range

        n, bits, m, k = 30001, 64, 4, 50
        db = mg.gen_uniform(n, bits, 5)
        qs = mg.gen_uniform(64, bits, 6).raw_words()
        dq = torch.from_numpy(np.ascontiguousarray(qs).view(np.int64)).cuda()
        comm = NcclComm(rank)
        full = mg.MihIndex.build(db, mg.consecutive_partition(bits, m), device=rank)
        want_i, want_d = full.knn_search_batch(qs, k)
        ok = True
        i, d = native_sharded_search(full, comm, "probe", n, dq, k)
        ok &= np.array_equal(i.cpu().numpy().view(np.uint32), want_i) and np.array_equal(d.cpu().numpy().view(np.uint32), want_d)
        lo, hi = shard_range(n, rank, world)
        w = db.raw_words()[lo:hi]
        shard = mg.MihIndex.build_from_device(torch.from_numpy(np.ascontiguousarray(w).view(np.int64)).cuda().data_ptr(),
                                              hi - lo, bits, mg.consecutive_partition(bits, m), rank, id_base=lo)
        i, d = native_sharded_search(shard, comm, "id", n, dq, k)
        ok &= np.array_equal(i.cpu().numpy().view(np.uint32), want_i) and np.array_equal(d.cpu().numpy().view(np.uint32), want_d)
        comm.close()
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_two_process_nccl_sharded(cuda_ok):
    import torch
    import torch.multiprocessing as mp

    if torch.cuda.device_count() < 2:
        pytest.skip("needs two visible GPUs (the gloo world-2 test covers the host logic)")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_two_rank_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    assert dict(q.get(timeout=10) for _ in range(2)) == {0: True, 1: True}
