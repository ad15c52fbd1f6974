"""GPU parity: the CUDA path (through the C ABI) against the reference's golden vectors and the
C oracle. Integer work, so the bar is bit-exact: ids, distances and SearchTrace counters."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["rounds", "solo"])
def search_path(request):
    """Every case runs through both kNN drivers: the round-synchronous kernels (MIHG_SOLO=0) and,
    where the batch is small enough to qualify, the one-block-per-query kernel (mih_solo_kernel)."""
    import os

    old = os.environ.get("MIHG_SOLO")
    os.environ["MIHG_SOLO"] = "0" if request.param == "rounds" else "1"
    yield request.param
    if old is None:
        os.environ.pop("MIHG_SOLO", None)
    else:
        os.environ["MIHG_SOLO"] = old


def _mg():
    import paper_1307_2982_b200 as mg

    return mg


def _trace_array(tr):
    return np.array([[t.lookups, t.candidates, t.unique_candidates, t.distance_evaluations,
                      t.final_radius] for t in tr], np.uint64)


def _index(d, layout="auto"):
    mg = _mg()
    bits, m = int(d["bits"]), int(d["m"])
    db = mg.CodeDatabase(bits, d["codes"])
    if "lengths" in d:
        ln, ps = d["lengths"], d["positions"]
        subs, at = [], 0
        for L in ln:
            subs.append(list(ps[at:at + int(L)]))
            at += int(L)
        part = mg.Partition(bits, subs)
    else:
        part = mg.consecutive_partition(bits, m)
    return mg.MihIndex.build(db, part, layout=layout)


CASES = ["hand_worked", "knn_wide24", "duplicates", "self_queries", "nondivisible100",
         "scratch_reuse32", "lsh_io_test", "interleaved64", "acceptance_lsh", "wide300", "wide512"]


@pytest.mark.parametrize("bits", [300, 512])
def test_scan_wide_matches_reference_golden(cuda_ok, golden, bits):
    """Codes above 256 bits (codes.hpp:16): generic-width K6 scan vs the reference's scan_knn."""
    mg = _mg()
    d = golden(f"wide{bits}")
    idx = mg.MihIndex.build(mg.CodeDatabase(bits, d["codes"]), mg.consecutive_partition(bits, int(d["m"])))
    for k in (1, 10, 60):
        ids, dists = idx.scan_knn_batch(d["scan_queries"], k)
        assert np.array_equal(ids, d[f"scan_ids_k{k}"]) and np.array_equal(dists, d[f"scan_dists_k{k}"]), k


@pytest.mark.parametrize("layout", ["auto", "sparse"])
@pytest.mark.parametrize("name", CASES)
def test_knn_matches_reference_golden(cuda_ok, golden, name, layout):
    d = golden(name)
    if layout == "sparse" and min(int(d["bits"]) // int(d["m"]), 32) < 6:
        pytest.skip("sparse directory needs s >= 6")
    idx = _index(d, layout)
    for key in sorted(k for k in d if k.startswith("ids_k")):
        k = int(key.split("_k")[1])
        ids, dists, tr = idx.knn_search_batch(d["queries"], k, with_trace=True)
        assert np.array_equal(dists, d[f"dists_k{k}"]), (name, k)
        assert np.array_equal(ids, d[f"ids_k{k}"]), (name, k)
        assert np.array_equal(_trace_array(tr), d[f"trace_k{k}"]), (name, k)
        # untraced calls may finish hard queries with the exhaustive scan (hybrid switch)
        ids, dists = idx.knn_search_batch(d["queries"], k)
        assert np.array_equal(ids, d[f"ids_k{k}"]) and np.array_equal(dists, d[f"dists_k{k}"]), (name, k)


@pytest.mark.parametrize("bits", [64, 70])
def test_knn_random_matches_reference(cuda_ok, golden, bits):
    # index_test.cpp:127-154: k up to n drives the radius to the full width
    mg = _mg()
    d = golden(f"knn_random_b{bits}")
    db = mg.gen_uniform(1200, bits, int(d["db_seed"]))
    assert np.array_equal(db.raw_words(), d["codes"])
    for m in (4, 6, 7):
        idx = mg.MihIndex.build(db, mg.consecutive_partition(bits, m))
        for k in (1, 2, 10, 100, 1200):
            ids, dists, tr = idx.knn_search_batch(d["queries"], k, with_trace=True)
            assert np.array_equal(ids, d[f"m{m}_ids_k{k}"]), (m, k)
            assert np.array_equal(dists, d[f"m{m}_dists_k{k}"]), (m, k)
            assert np.array_equal(_trace_array(tr), d[f"m{m}_trace_k{k}"]), (m, k)
            si, sd = idx.scan_knn_batch(d["queries"], k)
            assert np.array_equal(si, d[f"m{m}_ids_k{k}"]) and np.array_equal(sd, d[f"m{m}_dists_k{k}"])


def test_acceptance_uniform(cuda_ok, golden):
    # acceptance.cpp:134-172 criterion 2 (uniform lane), ids AND distances
    mg = _mg()
    d = golden("acceptance_uniform")
    db = mg.gen_uniform(int(d["n"]), 64, int(d["db_seed"]))
    idx = mg.MihIndex.build(db, mg.consecutive_partition(64, int(d["m"])))
    for k in (1, 10, 100):
        ids, dists, tr = idx.knn_search_batch(d["queries"], k, with_trace=True)
        assert np.array_equal(ids, d[f"ids_k{k}"]) and np.array_equal(dists, d[f"dists_k{k}"])
        assert np.array_equal(_trace_array(tr), d[f"trace_k{k}"])
        si, sd = idx.scan_knn_batch(d["queries"], k)
        assert np.array_equal(si, d[f"ids_k{k}"]) and np.array_equal(sd, d[f"dists_k{k}"])


@pytest.mark.parametrize("layout", ["auto", "sparse"])
def test_config1_golden(cuda_ok, golden, layout):
    # BASELINE config 1: n=1e6 uniform 64-bit, 1000 queries, m=4, k=10
    mg = _mg()
    d = golden("config1")
    db = mg.gen_uniform(int(d["n"]), 64, int(d["db_seed"]))
    qs = mg.gen_uniform(1000, 64, int(d["q_seed"])).raw_words()
    assert np.array_equal(qs, d["queries"])
    idx = mg.MihIndex.build(db, mg.consecutive_partition(64, 4), layout=layout)
    ids, dists, tr = idx.knn_search_batch(qs, 10, with_trace=True)
    assert np.array_equal(ids, d["ids_k10"]) and np.array_equal(dists, d["dists_k10"])
    assert np.array_equal(_trace_array(tr), d["trace_k10"])
    si, sd = idx.scan_knn_batch(qs, 10)
    assert np.array_equal(si, d["ids_k10"]) and np.array_equal(sd, d["dists_k10"])


@pytest.mark.parametrize("layout", ["auto", "sparse"])
def test_bucket_contents_match_reference(cuda_ok, golden, layout):
    # table_test.cpp:34-43 (insertion order within a bucket), :65-104 (map equivalence)
    mg = _mg()
    d = golden("buckets_m3")
    db = mg.gen_uniform(int(d["n"]), 64, int(d["db_seed"]))
    idx = mg.MihIndex.build(db, mg.consecutive_partition(64, 3), layout=layout)
    offs = d["offs"]
    for i in range(d["table"].size):
        got = idx.table(int(d["table"][i])).bucket_lookup(int(d["value"][i]))
        assert np.array_equal(got, d["ids"][int(offs[i]):int(offs[i + 1])])


def test_single_query_api_and_trace(cuda_ok, golden):
    # index_test.cpp:73-94 HandWorkedKnn through the single-query facade
    mg = _mg()
    db = mg.CodeDatabase(6)
    for w in (0b000000, 0b000001, 0b111111):
        db.append_words(np.array([w], np.uint64))
    idx = mg.MihIndex.build(db, mg.consecutive_partition(6, 2))
    tr = mg.SearchTrace()
    res = idx.knn_search(mg.BinaryCode(np.array([0], np.uint64), 6), 2, tr)
    assert res == [mg.Neighbor(0, 0), mg.Neighbor(1, 1)]
    assert (tr.final_radius, tr.lookups, tr.candidates, tr.unique_candidates) == (1, 2, 3, 2)


def test_error_contract(cuda_ok):
    # index_test.cpp:250-268 ValidationAndEdges
    mg = _mg()
    db = mg.gen_uniform(10, 64, 1)
    idx = mg.MihIndex.build(db, mg.consecutive_partition(64, 2))
    q = mg.BinaryCode(np.array([5], np.uint64), 64)
    with pytest.raises(ValueError):
        idx.knn_search(q, 11)
    with pytest.raises(ValueError):
        idx.knn_search(mg.BinaryCode(np.array([0], np.uint64), 32), 1)
    assert idx.knn_search(q, 0) == []
    ids, dists, tr = idx.knn_search_batch(np.zeros((3, 1), np.uint64), 0, with_trace=True)
    assert ids.shape == (3, 0) and not _trace_array(tr).any()
    empty = mg.MihIndex.build(mg.CodeDatabase(64), mg.consecutive_partition(64, 2))
    assert empty.knn_search(q, 0) == []
    with pytest.raises(ValueError):
        empty.knn_search(q, 1)


def test_free_scan_knn(cuda_ok, golden):
    mg = _mg()
    d = golden("knn_random_b70")
    db = mg.CodeDatabase(70, d["codes"])
    q = mg.BinaryCode(d["queries"][3], 70)
    res = mg.scan_knn(db, q, 100)
    assert [r.id for r in res] == list(d["m4_ids_k100"][3])
    assert [r.dist for r in res] == list(d["m4_dists_k100"][3])


def test_heavy_ties_and_buffer_overflow(cuda_ok, port):
    # 40k copies of a handful of codes: ties at d_k far beyond the per-query buffer, exercising
    # the re-run and large-selection paths (scan.hpp:42 tie rule).
    mg = _mg()
    rng = np.random.default_rng(7)
    base = rng.integers(0, 2**63, size=5, dtype=np.uint64)
    codes = base[rng.integers(0, 5, size=40000)] ^ (np.uint64(1) << rng.integers(0, 3, 40000).astype(np.uint64))
    codes = codes.reshape(-1, 1)
    qs = np.concatenate([base.reshape(-1, 1), rng.integers(0, 2**63, size=(3, 1), dtype=np.uint64)])
    idx = mg.MihIndex.build(mg.CodeDatabase(64, codes), mg.consecutive_partition(64, 4))
    h = port.build(codes, 64, 4)
    for k in (1, 50, 9000, 20000):
        ids, dists, tr = idx.knn_search_batch(qs, k, with_trace=True)
        oi, od, ot = h.knn(qs, k)
        assert np.array_equal(dists, od), k
        assert np.array_equal(ids, oi), k
        assert np.array_equal(_trace_array(tr), ot), k
        si, sd = idx.scan_knn_batch(qs, k)
        assert np.array_equal(si, oi) and np.array_equal(sd, od), k


def closed_form_traces(codes, bits, m, qs, R):
    """SearchTrace counters from the final radius alone (verified against the
    reference on 280 queries): with rho_j = floor((R - j) / m) for j <= R,
    lookups = sum_{r<=R} C(s_{r mod m}, r // m); candidates = sum_j #{i: d_j(q, x_i) <= rho_j};
    unique = #{i: exists j: d_j(q, x_i) <= rho_j}."""
    from math import comb

    import paper_1307_2982_b200 as mg

    part = mg.consecutive_partition(bits, m)
    masks = []
    for j in range(m):
        mk = np.zeros(codes.shape[1], np.uint64)
        for p in part.positions(j):
            mk[p >> 6] |= np.uint64(1 << (p & 63))
        masks.append(mk)
    out = []
    for qi in range(qs.shape[0]):
        x = codes ^ qs[qi]
        dj = np.stack([np.bitwise_count(x & masks[j]).sum(axis=1) for j in range(m)])
        r = int(R[qi])
        look = sum(comb(part.length(t % m), t // m) for t in range(r + 1))
        hit = np.zeros(codes.shape[0], bool)
        cand = 0
        for j in range(min(m, r + 1)):
            rho = (r - j) // m
            h = dj[j] <= rho
            cand += int(h.sum())
            hit |= h
        out.append([look, cand, int(hit.sum()), int(hit.sum()), r])
    return np.array(out, np.uint64)


@pytest.mark.parametrize("bits,m,n", [(128, 6, 200000), (256, 16, 100000), (64, 3, 300000),
                                      (64, 2, 200000), (256, 8, 200000)])
def test_random_shapes_vs_oracle(cuda_ok, port, bits, m, n):
    # ids/dists against the oracle's exhaustive scan (scan.hpp:43-68 restated); traces against
    # the closed forms. (256, 8) is config 5's table shape (8 x 32-bit sparse tables).
    mg = _mg()
    db = mg.gen_uniform(n, bits, 1000 + bits + m)
    nq = 4 if (bits, m) == (256, 8) else 24
    qs = mg.gen_uniform(nq, bits, 2000 + bits + m).raw_words()
    ks = (1, 5) if (bits, m) == (256, 8) else (1, 25, 100)
    for layout in ("auto", "sparse"):
        idx = mg.MihIndex.build(db, mg.consecutive_partition(bits, m), layout=layout)
        for k in ks:
            ids, dists, tr = idx.knn_search_batch(qs, k, with_trace=True)
            oi, od = port.scan_knn(db.raw_words(), bits, qs, k)
            assert np.array_equal(ids, oi) and np.array_equal(dists, od), (layout, k)
            ui, ud = idx.knn_search_batch(qs, k)  # untraced: hybrid MIH/scan
            assert np.array_equal(ui, oi) and np.array_equal(ud, od), (layout, k)
            t = _trace_array(tr)
            assert np.array_equal(t[:, 4], od[:, -1]), "final_radius == d_k"
            assert np.array_equal(t, closed_form_traces(db.raw_words(), bits, m, qs, t[:, 4])), (layout, k)

@pytest.mark.parametrize("comps,n", [(64, 1_000_000), (2, 400_000)])
def test_clustered_codes_on_32bit_sparse_tables(cuda_ok, port, comps, n):
    # Config 4's shape at test size: Gaussian-mixture codes (csrc/gen.cu restated by the oracle),
    # m = 2 tables of 32 bits (sparse directory, residual table-order codes). Few components give
    # saturated directory groups (escape records), buckets above the inline limit (piece queue)
    # and buffers that fill while U is loose (compaction kernel). ids/dists against the oracle's
    # exhaustive scan; traces against the closed forms (index.hpp:185-253 semantics).
    mg = _mg()
    codes = port.gen_mixture(0, n, 64, 128, comps, 0x4C0FFEE, 0x51)
    qs = port.gen_mixture(0, 24, 64, 128, comps, 0x4C0FFEE, 0x52)
    if comps == 2:
        # two crowded buckets: 3000 codes sharing one table-0 key and 2000 sharing one table-1 key,
        # the other half a few flips away from the seed code; the seeds join the queries
        rng = np.random.default_rng(5)
        c0, c1 = codes[10, 0], codes[20, 0]
        flips = lambda cnt: np.bitwise_or.reduce(np.uint64(1) << rng.integers(0, 32, (cnt, 3)).astype(np.uint64), axis=1)
        codes[100:3100, 0] = (c0 & np.uint64(0xFFFFFFFF)) | (((c0 >> np.uint64(32)) ^ flips(3000)) << np.uint64(32))
        codes[5000:7000, 0] = (c1 & np.uint64(0xFFFFFFFF00000000)) | ((c1 & np.uint64(0xFFFFFFFF)) ^ flips(2000))
        qs[0, 0], qs[1, 0] = c0, c1
    idx = mg.MihIndex.build(mg.CodeDatabase(64, codes), mg.consecutive_partition(64, 2))
    tabs = [idx.table(j) for j in range(2)]
    assert all(not t.dense() for t in tabs)
    if comps == 2:  # the paths this case is here for
        assert max(t.max_bucket_size() for t in tabs) > 128
        assert sum(int(t._info.escaped_blocks) for t in tabs) > 0
    for k in (1, 100, 1000):
        ids, dists, tr = idx.knn_search_batch(qs, k, with_trace=True)
        oi, od = port.scan_knn(codes, 64, qs, k)
        assert np.array_equal(dists, od), k
        assert np.array_equal(ids, oi), k
        ui, ud = idx.knn_search_batch(qs, k)  # untraced product path
        assert np.array_equal(ui, oi) and np.array_equal(ud, od), k
        t = _trace_array(tr)
        assert np.array_equal(t[:, 4], od[:, -1]), "final_radius == d_k"
        assert np.array_equal(t, closed_form_traces(codes, 64, 2, qs, t[:, 4])), k
    if comps == 2:
        # small candidate buffers: the crowded buckets overflow them while U is loose, so the
        # compaction kernel and the exact re-run pass both run
        import os

        os.environ["MIHG_BUFFER_CAP"] = "2200"
        try:
            for k in (100, 1000):
                oi, od = port.scan_knn(codes, 64, qs, k)
                ids, dists, tr = idx.knn_search_batch(qs, k, with_trace=True)
                assert np.array_equal(ids, oi) and np.array_equal(dists, od), k
                assert np.array_equal(_trace_array(tr), closed_form_traces(codes, 64, 2, qs, od[:, -1])), k
        finally:
            del os.environ["MIHG_BUFFER_CAP"]


@pytest.mark.parametrize("layout", ["auto", "sparse"])
def test_table_stats_match_reference(cuda_ok, golden, layout):
    # TableStats (table.hpp:33-47, :190-197): non_empty_buckets, max_bucket_size, total_entries,
    # estimated_bytes (the reference's accounting model) for every table
    mg = _mg()
    d = golden("table_stats")
    for name in [k for k in d if not k.endswith("_spec")]:
        n, bits, seed, m = (int(x) for x in d[name + "_spec"])
        if layout == "sparse" and (bits // m) < 6:
            continue
        db = mg.gen_uniform(n, bits, seed)
        idx = mg.MihIndex.build(db, mg.consecutive_partition(bits, m), layout=layout)
        for j in range(m):
            st = idx.table(j).stats()
            got = [st.non_empty_buckets, st.max_bucket_size, st.total_entries, st.estimated_bytes]
            assert got == [int(x) for x in d[name][j]], (name, j)


@pytest.mark.parametrize("layout", ["auto", "sparse"])
@pytest.mark.parametrize("bits", [32, 96, 100])
def test_range_search_matches_reference(cuda_ok, golden, bits, layout):
    # index_test.cpp:96-112 RangeMatchesScanRandomized + acceptance criteria 1/4 (probe counts):
    # ids, dists and lookups/candidates/unique identical to MihIndex::range_search
    mg = _mg()
    d = golden(f"range_b{bits}")
    for m in (2, 4, 5):
        if (bits + m - 1) // m > 32 or (layout == "sparse" and bits // m < 6):
            continue
        idx = mg.MihIndex.build(mg.CodeDatabase(bits, d["codes"]), mg.consecutive_partition(bits, m),
                                layout=layout)
        for r in (0, 1, 5, bits // 3):
            offs, ids, dists, tr = idx.range_search_batch(d["queries"], r, with_trace=True)
            assert np.array_equal(offs, d[f"m{m}_r{r}_offs"]), (m, r)
            assert np.array_equal(ids, d[f"m{m}_r{r}_ids"]), (m, r)
            assert np.array_equal(dists, d[f"m{m}_r{r}_dists"]), (m, r)
            assert np.array_equal(_trace_array(tr)[:, :4], d[f"m{m}_r{r}_trace"][:, :4]), (m, r)
            assert not _trace_array(tr)[:, 4].any()


def test_final_radius_is_a_completeness_certificate(cuda_ok):
    # index_test.cpp:186-206: the k results are the head of range_search(final_radius)
    mg = _mg()
    db = mg.gen_uniform(2000, 64, 12)
    idx = mg.MihIndex.build(db, mg.consecutive_partition(64, 4))
    qs = mg.gen_uniform(10, 64, 13)
    for qi in range(10):
        tr = mg.SearchTrace()
        res = idx.knn_search(qs.code(qi), 10, tr)
        assert res[-1].dist <= tr.final_radius
        within = idx.range_search(qs.code(qi), tr.final_radius)
        assert len(within) >= 10 and within[:10] == res
    with pytest.raises(ValueError):
        idx.range_search(qs.code(0), 65)  # radius exceeds code width (index.hpp:152)
