"""CPU: pin the C restatement (oracle/mih_oracle.c) against the golden vectors produced by the
reference itself (tests/golden/make_golden.py via oracle/_ref)."""
import numpy as np
import pytest

KNN_CASES = [
    ("hand_worked", None),
    ("knn_wide24", None),
    ("duplicates", None),
    ("self_queries", None),
    ("nondivisible100", None),
    ("scratch_reuse32", None),
    ("lsh_io_test", None),
    ("interleaved64", None),
    ("acceptance_lsh", None),
    ("wide300", None),
    ("wide512", None),
]


def _ks(d):
    return sorted(int(k.split("_k")[1]) for k in d if k.startswith("ids_k"))


@pytest.mark.parametrize("name", [c[0] for c in KNN_CASES])
def test_port_knn_matches_reference_golden(port, golden, name):
    d = golden(name)
    bits, m = int(d["bits"]), int(d["m"])
    h = port.build(d["codes"], bits, m, d.get("lengths"), d.get("positions"))
    for k in _ks(d):
        ids, dists, tr = h.knn(d["queries"], k)
        assert np.array_equal(ids, d[f"ids_k{k}"]), (name, k)
        assert np.array_equal(dists, d[f"dists_k{k}"]), (name, k)
        assert np.array_equal(tr, d[f"trace_k{k}"]), (name, k)


@pytest.mark.parametrize("bits", [64, 70])
def test_port_knn_random_matches_reference(port, golden, bits):
    # index_test.cpp:127-154
    d = golden(f"knn_random_b{bits}")
    codes = port.gen_uniform(1200, bits, int(d["db_seed"]))
    assert np.array_equal(codes, d["codes"])
    for m in (4, 6, 7):
        h = port.build(codes, bits, m)
        for k in (1, 2, 10, 100, 1200):
            ids, dists, tr = h.knn(d["queries"], k)
            assert np.array_equal(ids, d[f"m{m}_ids_k{k}"])
            assert np.array_equal(dists, d[f"m{m}_dists_k{k}"])
            assert np.array_equal(tr, d[f"m{m}_trace_k{k}"])


@pytest.mark.parametrize("bits", [300, 512])
def test_port_scan_wide_matches_reference(port, golden, bits):
    d = golden(f"wide{bits}")
    for k in (1, 10, 60):
        ids, dists = port.scan_knn(d["codes"], bits, d["scan_queries"], k)
        assert np.array_equal(ids, d[f"scan_ids_k{k}"]) and np.array_equal(dists, d[f"scan_dists_k{k}"])


def test_port_scan_matches_reference(port, golden):
    d = golden("knn_random_b64")
    for k in (1, 10, 100, 1200):
        ids, dists = port.scan_knn(d["codes"], 64, d["queries"], k)
        # scan_knn == knn_search (index.hpp:178 contract); golden is the reference's knn output
        assert np.array_equal(ids, d[f"m4_ids_k{k}"])
        assert np.array_equal(dists, d[f"m4_dists_k{k}"])


def test_port_gen_uniform_pins(port, golden):
    d = golden("gen_uniform_pins")
    for key, want in d.items():
        _, n, bits, seed = key.split("_")
        assert np.array_equal(port.gen_uniform(int(n), int(bits), int(seed)), want), key


def test_port_acceptance_uniform(port, golden):
    import hashlib

    d = golden("acceptance_uniform")
    codes = port.gen_uniform(int(d["n"]), 64, int(d["db_seed"]))
    assert hashlib.sha256(codes.tobytes()).hexdigest() == str(d["codes_sha256"])
    h = port.build(codes, 64, int(d["m"]))
    qs = d["queries"][:60]
    for k in (1, 10, 100):
        ids, dists, tr = h.knn(qs, k)
        assert np.array_equal(ids, d[f"ids_k{k}"][:60])
        assert np.array_equal(dists, d[f"dists_k{k}"][:60])
        assert np.array_equal(tr, d[f"trace_k{k}"][:60])


@pytest.mark.parametrize("bits", [32, 96, 100])
def test_port_range_matches_reference(port, golden, bits):
    d = golden(f"range_b{bits}")
    for m in (2, 4, 5):
        if (bits + m - 1) // m > 32:
            continue
        h = port.build(d["codes"], bits, m)
        for r in (0, 1, 5, bits // 3):
            offs = d[f"m{m}_r{r}_offs"]
            for qi in range(d["queries"].shape[0]):
                ids, dists, tr = h.range(d["queries"][qi], r)
                lo, hi = int(offs[qi]), int(offs[qi + 1])
                assert np.array_equal(ids, d[f"m{m}_r{r}_ids"][lo:hi])
                assert np.array_equal(dists, d[f"m{m}_r{r}_dists"][lo:hi])
                assert np.array_equal(tr[:4], d[f"m{m}_r{r}_trace"][qi][:4])


def test_port_buckets_match_reference(port, golden):
    d = golden("buckets_m3")
    codes = port.gen_uniform(int(d["n"]), 64, int(d["db_seed"]))
    h = port.build(codes, 64, 3)
    offs = d["offs"]
    for i in range(d["table"].size):
        got = h.bucket(int(d["table"][i]), int(d["value"][i]))
        assert np.array_equal(got, d["ids"][int(offs[i]):int(offs[i + 1])])


def test_port_error_contract(port):
    codes = port.gen_uniform(10, 64, 1)
    with pytest.raises(ValueError):
        port.build(codes, 64, 1)  # 64-bit substring (index_test.cpp:250-256)
    h = port.build(codes, 64, 2)
    with pytest.raises(ValueError):
        h.knn(codes[:1], 11)  # k > n (index.hpp:188)
    ids, dists, tr = h.knn(codes[:1], 0)  # k == 0 -> empty (index.hpp:189-194)
    assert ids.size == 0 and not tr.any()
