"""CPU, world_size 2, gloo: the id-range sharding + exchange + exact-merge logic of
paper_1307_2982_b200/shard.py. The per-shard search is the C oracle on that shard (ids offset by
the shard start) and the merge is a numpy restatement here, so the test isolates the host logic;
the GPU merge kernel is covered in tests/test_gpu_merge.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

from _helpers import numpy_merge  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, bits, m, k, result_q):
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_1307_2982_b200.shard import ShardedKnn, shard_range

        P = oracle.port()
        db = P.gen_uniform(n, bits, 77)
        qs = P.gen_uniform(25, bits, 78)
        lo, hi = shard_range(n, rank, world)
        h = P.build(db[lo:hi], bits, m) if hi > lo else None

        calls = []

        def local(queries, kk, k_global=None, collective=False):
            calls.append((kk, k_global, collective))
            ids, d, _ = h.knn(queries.numpy().view(np.uint64), kk)
            return (torch.from_numpy((ids.astype(np.uint64) + lo).astype(np.uint32).view(np.int32)),
                    torch.from_numpy(d.view(np.int32)))

        sk = ShardedKnn(local, hi - lo, merge=numpy_merge, global_stopping=True)
        ids, d = sk.search(torch.from_numpy(qs.view(np.int64)), k)
        want_i, want_d = P.scan_knn(db, bits, qs, k)
        ok = np.array_equal(ids.numpy().view(np.uint32), want_i) and np.array_equal(d.numpy().view(np.uint32), want_d)
        # global stopping: the stopping k is the caller's k on every rank, and the collective
        # local search runs on every rank or on none (an empty shard turns it off everywhere)
        if hi > lo:
            ok = ok and calls == [(min(k, hi - lo), k, n >= world)]
        else:
            ok = ok and calls == []
        result_q.put((rank, bool(ok), [c[2] for c in calls]))
    finally:
        dist.destroy_process_group()


# (150, k=100): shards of 75 < k; (1, k=1): rank 1's shard is empty, so global stopping is off
@pytest.mark.parametrize("n,bits,m,k", [(5000, 64, 4, 10), (3001, 70, 4, 100), (150, 64, 4, 100), (1, 64, 4, 1)])
def test_sharded_knn_equals_single_index(n, bits, m, k):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, bits, m, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    res = {}
    for _ in range(world):
        r, ok, coll = q.get(timeout=10)
        res[r] = ok
    assert res == {0: True, 1: True}


def test_shard_ranges_cover_ids_exactly_once():
    from paper_1307_2982_b200.shard import shard_range

    for n in (0, 1, 7, 1000, 10**9):
        for world in (1, 2, 3, 4, 8):
            rs = [shard_range(n, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            for (a, b), (c, d) in zip(rs, rs[1:]):
                assert b == c and a <= b
