"""GPU: the tensor-core exhaustive scan (K7, csrc/tcscan.cu) — every distance equals the
reference's hamming_words (codes.hpp:38-42), and its top-k equals scan_knn (scan.hpp:43-68) through
the oracle and through the POPC-pipe scan (K6) on the same inputs, ties included."""
import ctypes as C
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["single", "pair"], autouse=True)
def tc_geometry(request):
    """Every K7 test runs in both geometries: one CTA per 128-query x 256-code tile, and CTA pairs
    (cta_group::2, M = 256) that split each code tile between two SMs (MIHG_TC_PAIR=1)."""
    os.environ["MIHG_TC_PAIR"] = "1" if request.param == "pair" else "0"
    yield request.param
    os.environ.pop("MIHG_TC_PAIR", None)


def _popc_dist(q, x):
    """[nq, n] Hamming distances of packed u64 rows (numpy restatement of hamming_words)."""
    d = np.zeros((q.shape[0], x.shape[0]), np.int64)
    for w in range(q.shape[1]):
        v = np.bitwise_xor(q[:, w][:, None], x[:, w][None, :])
        d += np.unpackbits(v.view(np.uint8).reshape(v.shape + (8,)), axis=-1).sum(-1).astype(np.int64)
    return d


@pytest.mark.parametrize("bits,n,nq", [(64, 3000, 200), (128, 2500, 130), (192, 1000, 70),
                                       (256, 1300, 129), (70, 777, 5), (17, 600, 40)])
def test_tc_distances_exact(cuda_ok, bits, n, nq):
    import torch

    from paper_1307_2982_b200 import _lib
    import paper_1307_2982_b200 as mg

    L = _lib.lib()
    db = mg.gen_uniform(n, bits, 100 + bits).raw_words()
    qs = mg.gen_uniform(nq, bits, 200 + bits).raw_words()
    dd = torch.from_numpy(db.view(np.int64)).cuda()
    dq = torch.from_numpy(qs.view(np.int64)).cuda()
    out = torch.full((nq, n), -7, dtype=torch.int32, device="cuda")
    _lib.check(L.mihg_tc_distances_device(C.c_void_p(dd.data_ptr()), n, bits, C.c_void_p(dq.data_ptr()), nq,
                                          C.c_void_p(out.data_ptr()), None))
    torch.cuda.synchronize()
    want = _popc_dist(qs, db)
    got = out.cpu().numpy()
    assert np.array_equal(got, want), f"bits={bits}: {np.argwhere(got != want)[:5]}"


def _scan(idx, qs, k, kernel):
    os.environ["MIHG_SCAN_KERNEL"] = kernel
    try:
        return idx.scan_knn_batch(qs, k)
    finally:
        os.environ.pop("MIHG_SCAN_KERNEL", None)


@pytest.mark.parametrize("bits,n,nq,k", [(64, 50000, 300, 10), (64, 200000, 1000, 100), (128, 60000, 257, 33),
                                         (256, 40000, 140, 100), (192, 30000, 64, 1), (40, 30000, 50, 500)])
def test_tc_scan_matches_oracle_and_popc(cuda_ok, port, bits, n, nq, k):
    import paper_1307_2982_b200 as mg

    db = mg.gen_uniform(n, bits, 7 + bits)
    qs = mg.gen_uniform(nq, bits, 8 + bits).raw_words()
    idx = mg.MihIndex.build(db, mg.consecutive_partition(bits, max(1, -(-bits // 32))), device=0)
    ti, td = _scan(idx, qs, k, "tc")
    pi, pd = _scan(idx, qs, k, "popc")
    assert np.array_equal(ti, pi) and np.array_equal(td, pd)
    if n * nq <= 2e7:
        oi, od = port.scan_knn(db.raw_words(), bits, qs, k)
        assert np.array_equal(ti, oi) and np.array_equal(td, od)


def test_tc_scan_heavy_ties(cuda_ok):
    """Few distinct codes: thousands of exact ties at every distance; the smaller id must win."""
    import paper_1307_2982_b200 as mg

    rng = np.random.default_rng(5)
    centres = rng.integers(0, 2**63, size=(6, 2), dtype=np.int64).view(np.uint64)
    pick = rng.integers(0, 6, size=70000)
    codes = centres[pick].copy()
    flip = rng.random(70000) < 0.1
    codes[flip, 0] ^= np.uint64(1) << rng.integers(0, 64, size=flip.sum()).astype(np.uint64)
    db = mg.CodeDatabase(128, codes)
    qs = np.concatenate([centres, codes[:60]])
    idx = mg.MihIndex.build(db, mg.consecutive_partition(128, 4), device=0)
    for k in (1, 100, 3000):
        ti, td = _scan(idx, qs, k, "tc")
        pi, pd = _scan(idx, qs, k, "popc")
        assert np.array_equal(ti, pi) and np.array_equal(td, pd), k


@pytest.mark.parametrize("bits,first,n", [(64, 1, 5001), (192, 3, 4099), (64, 0, 129), (128, 5, 77)])
def test_tc_scan_misaligned_and_ragged(cuda_ok, port, bits, first, n):
    """Raw device scan over codes starting at an arbitrary row (8-byte aligned only: the TMA bulk
    copies take the 16-byte-aligned interior, plain loads the head and tail) and ragged sizes."""
    import torch

    from paper_1307_2982_b200 import _lib
    import paper_1307_2982_b200 as mg

    L = _lib.lib()
    W = (bits + 63) // 64
    allc = mg.gen_uniform(first + n, bits, 40 + bits).raw_words()
    qs = mg.gen_uniform(130, bits, 41 + bits).raw_words()
    k = min(50, n)
    d_all = torch.from_numpy(allc.view(np.int64)).cuda()
    dq = torch.from_numpy(qs.view(np.int64)).cuda()
    ids = torch.empty((130, k), dtype=torch.int32, device="cuda")
    ds = torch.empty((130, k), dtype=torch.int32, device="cuda")
    os.environ["MIHG_SCAN_KERNEL"] = "tc"
    try:
        _lib.check(L.mihg_scan_knn_raw_device(C.c_void_p(d_all.data_ptr() + first * W * 8), n, bits, 1000,
                                              C.c_void_p(dq.data_ptr()), 130, k, C.c_void_p(ids.data_ptr()),
                                              C.c_void_p(ds.data_ptr()), None))
        torch.cuda.synchronize()
    finally:
        os.environ.pop("MIHG_SCAN_KERNEL", None)
    oi, od = port.scan_knn(allc[first:], bits, qs, k)
    assert np.array_equal(ids.cpu().numpy().view(np.uint32), oi + 1000)
    assert np.array_equal(ds.cpu().numpy().view(np.uint32), od)


@pytest.mark.parametrize("bits,k", [(64, 3), (256, 10), (128, 1)])
def test_tc_scan_seeded_bound(cuda_ok, port, bits, k):
    """The K7 lists start from a bound seeded by the exact k-th distance over the first codes of the
    database (an upper bound on the true k-th distance; ties kept): same answer as the oracle,
    also when the sample's k-th distance ties with many later codes (duplicated database rows)."""
    import paper_1307_2982_b200 as mg

    n = 40000
    base = mg.gen_uniform(n, bits, 60 + bits).raw_words()
    base[n // 2:] = base[: n - n // 2]  # every code twice: the sample's k-th distance recurs later
    db = mg.CodeDatabase(bits, base)
    qs = mg.gen_uniform(150, bits, 61 + bits).raw_words()
    idx = mg.MihIndex.build(db, mg.consecutive_partition(bits, max(1, -(-bits // 32))), device=0)
    want = port.scan_knn(base, bits, qs, k)
    for seed in ("0", "256", "512"):
        os.environ["MIHG_TC_SEED"] = seed
        try:
            got = _scan(idx, qs, k, "tc")
        finally:
            os.environ.pop("MIHG_TC_SEED", None)
        assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1]), seed
