"""GPU: BMIX index persistence parity (io.hpp:335-425). Files written by the reference's own
write_index load onto the GPU and answer knn/range exactly like the reference (results and
probe counts: io_test.cpp:141-176, acceptance criterion 11); our write_index reproduces the
reference's bytes; corrupted files raise FormatError like io_test.cpp:178-192."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _trace(tr):
    return np.array([[t.lookups, t.candidates, t.unique_candidates, t.distance_evaluations,
                      t.final_radius] for t in tr], np.uint64)


def test_reference_bmix_files_load_and_search(cuda_ok, golden, tmp_path):
    import paper_1307_2982_b200 as mg

    d = golden("bmix_files")
    for c in range(5):
        p = f"c{c}_"
        bits, m, n = (int(x) for x in d[p + "spec"])
        path = str(tmp_path / f"ref{c}.bin")
        d[p + "bmix"].tofile(path)
        idx = mg.read_index(path)
        assert idx.num_tables() == m and idx.size() == n and idx.partition() == mg.consecutive_partition(bits, m)
        qs = d[p + "queries"]
        ids, dists, tr = idx.knn_search_batch(qs, 5, with_trace=True)
        assert np.array_equal(ids, d[p + "knn_ids"]) and np.array_equal(dists, d[p + "knn_dists"])
        assert np.array_equal(_trace(tr), d[p + "knn_trace"])
        offs, rids, rd, rtr = idx.range_search_batch(qs, int(d[p + "range_r"][0]), with_trace=True)
        assert np.array_equal(offs, d[p + "range_offs"]) and np.array_equal(rids, d[p + "range_ids"])
        assert np.array_equal(rd, d[p + "range_dists"])
        assert np.array_equal(_trace(rtr)[:, :2], d[p + "range_trace"][:, :2])
        # export: byte-identical to the reference's write_index of the same index
        out = str(tmp_path / f"ours{c}.bin")
        mg.write_index(idx, out)
        assert open(out, "rb").read() == d[p + "bmix"].tobytes()
        built = mg.MihIndex.build(idx.db(), idx.partition(), layout="sparse" if bits // m >= 6 else "auto")
        mg.write_index(built, out)
        assert open(out, "rb").read() == d[p + "bmix"].tobytes()


def test_bmix_corruption_raises_format_error(cuda_ok, golden, tmp_path):
    import paper_1307_2982_b200 as mg

    blob = golden("bmix_files")["c0_bmix"].tobytes()
    path = str(tmp_path / "x.bin")
    open(path, "wb").write(b"BMIH" + blob[4:])  # codes-file magic is not an index file
    with pytest.raises(mg.FormatError) as e:
        mg.read_index(path)
    assert e.value.offset == 0
    open(path, "wb").write(blob[:-5])  # truncated table area
    with pytest.raises(mg.FormatError):
        mg.read_index(path)
    open(path, "wb").write(blob + b"\0")  # trailing bytes
    with pytest.raises(mg.FormatError):
        mg.read_index(path)
    with pytest.raises(OSError):
        mg.read_index(str(tmp_path / "missing.bin"))


def _first_table_groups(blob):
    """Offsets of the first table's groups in a BMIX file (io.hpp:335-358 layout):
    [(gid_at, mask, starts_at, ids_at, c, e), ...]."""
    import struct

    bits, n = struct.unpack_from("<IQ", blob, 8)
    at = 8 + 12 + n * ((bits + 63) // 64) * 8
    (m,) = struct.unpack_from("<I", blob, at)
    at += 4
    for _ in range(m):
        (ln,) = struct.unpack_from("<I", blob, at)
        at += 4 + 4 * ln
    s, entries, groups = struct.unpack_from("<IQQ", blob, at)
    at += 20
    out = []
    for _ in range(groups):
        gid, mask = struct.unpack_from("<QI", blob, at)
        c = bin(mask).count("1")
        starts_at = at + 12
        e = struct.unpack_from("<I", blob, starts_at + 4 * c)[0]
        out.append((at, mask, starts_at, starts_at + 4 * (c + 1), c, e))
        at = starts_at + 4 * (c + 1 + e)
    return s, out


def test_bmix_inconsistent_tables_rejected(cuda_ok, tmp_path):
    """Structurally valid files whose entries break the table invariant the kNN dedup relies on
    (every id exactly once per table, under its own substring key) are rejected with FormatError;
    so are buckets at keys >= 2^s of a narrow table."""
    import struct

    import paper_1307_2982_b200 as mg

    db = mg.gen_uniform(3000, 64, 7)
    idx = mg.MihIndex.build(db, mg.consecutive_partition(64, 4))
    good = str(tmp_path / "good.bin")
    mg.write_index(idx, good)
    blob = bytearray(open(good, "rb").read())
    s, groups = _first_table_groups(blob)
    # a group with two buckets: move the first entry of bucket 0 into bucket 1's key (swap ids
    # across buckets keeps the permutation but files both ids under the wrong key)
    g = next(x for x in groups if x[4] >= 2 and x[5] >= 2)
    _, _, starts_at, ids_at, c, e = g
    st = struct.unpack_from(f"<{c + 1}I", blob, starts_at)
    a, b = ids_at, ids_at + 4 * st[1]
    bad = bytearray(blob)
    bad[a:a + 4], bad[b:b + 4] = blob[b:b + 4], blob[a:a + 4]
    path = str(tmp_path / "swap.bin")
    open(path, "wb").write(bytes(bad))
    with pytest.raises(mg.FormatError) as ex:
        mg.read_index(path)
    assert "inconsistent index" in str(ex.value)
    # a repeated id (the second entry of the group duplicates the first)
    bad = bytearray(blob)
    bad[ids_at + 4:ids_at + 8] = blob[ids_at:ids_at + 4]
    open(path, "wb").write(bytes(bad))
    with pytest.raises(mg.FormatError) as ex:
        mg.read_index(path)
    assert "more than once" in str(ex.value)
    # the untouched file still loads and answers like the built index
    back = mg.read_index(good)
    qs = mg.gen_uniform(16, 64, 8).raw_words()
    assert all(np.array_equal(x, y) for x, y in zip(back.knn_search_batch(qs, 5), idx.knn_search_batch(qs, 5)))

    # s = 4 (a 16-bit code in 4 substrings): a mask bit at bucket 16..31 is past 2^s
    db4 = mg.gen_uniform(200, 16, 9)
    i4 = mg.MihIndex.build(db4, mg.consecutive_partition(16, 4))
    p4 = str(tmp_path / "s4.bin")
    mg.write_index(i4, p4)
    b4 = bytearray(open(p4, "rb").read())
    s4, g4 = _first_table_groups(b4)
    assert s4 == 4 and len(g4) == 1
    gid_at, mask = g4[0][0], g4[0][1]
    hi = 1 << 31  # bucket 31: same popcount if we move the top set bit there
    top = 1 << (mask.bit_length() - 1)
    struct.pack_into("<I", b4, gid_at + 8, (mask & ~top) | hi)
    open(p4, "wb").write(bytes(b4))
    with pytest.raises(mg.FormatError) as ex:
        mg.read_index(p4)
    assert ">= 2^s" in str(ex.value)
