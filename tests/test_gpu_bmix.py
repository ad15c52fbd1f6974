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
