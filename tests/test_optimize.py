"""CPU: substring optimisation (optimize.hpp). The C oracle's
estimate_correlations / greedy_assign against the reference's golden outputs (bitwise), the
product library's host-side greedy_assign (mihg_greedy_assign, no GPU needed) against the same
fixtures, and the reference's error contracts."""
import ctypes as C

import numpy as np
import pytest

from _optimize_cases import HAND, SPEC, codes_for, corr_matches, parts_for, subs_of


@pytest.fixture(scope="module")
def g(golden):
    return golden("optimize")


@pytest.mark.parametrize("name", HAND + SPEC)
def test_oracle_estimate_correlations_matches_reference(g, port, name):
    codes, bits = codes_for(g, name)
    corr, const, counts = port.estimate_correlations(codes, bits)
    assert corr_matches(g, name, corr), name
    assert np.array_equal(const.astype(np.uint8), g[name + "_const"])
    if codes.shape[0] <= 5000 and bits <= 256:  # AND counts against a direct numpy count
        bitm = np.unpackbits(codes.view(np.uint8).reshape(codes.shape[0], -1), axis=1,
                             bitorder="little")[:, :bits].astype(np.int64)
        assert np.array_equal(counts.astype(np.int64), bitm.T @ bitm)


@pytest.mark.parametrize("name", HAND + SPEC)
def test_oracle_greedy_assign_matches_reference(g, port, name):
    codes, bits = codes_for(g, name)
    corr, const, _ = port.estimate_correlations(codes, bits)
    for m, seed in parts_for(g, name):
        want = subs_of(g, f"{name}_part_m{m}_s{seed}", f"{name}_lens_m{m}_s{seed}")
        assert port.greedy_assign(corr, const, m, seed) == want, (name, m, seed)


@pytest.mark.parametrize("name", HAND + SPEC)
def test_library_greedy_assign_matches_reference(g, port, name):
    import paper_1307_2982_b200 as mg

    codes, bits = codes_for(g, name)
    corr, const, _ = port.estimate_correlations(codes, bits)  # bitwise the reference's (above)
    cm = mg.CorrelationMatrix(bits, corr, const)
    for m, seed in parts_for(g, name):
        want = subs_of(g, f"{name}_part_m{m}_s{seed}", f"{name}_lens_m{m}_s{seed}")
        p = mg.greedy_assign(cm, m, seed)
        assert p.substrings() == want, (name, m, seed)


def test_library_greedy_assign_random_trials(g, port):
    """optimize_test.cpp:104-120 ProducesValidBalancedPartitions, outputs pinned to the reference."""
    import paper_1307_2982_b200 as mg

    for t, (bits, m, seed) in enumerate(g["trials"].tolist()):
        codes = mg.gen_uniform(200, bits, 1000 + t).raw_words()
        corr, const, _ = port.estimate_correlations(codes, bits)
        p = mg.greedy_assign(mg.CorrelationMatrix(bits, corr, const), m, seed)
        assert p.substrings() == subs_of(g, f"trial{t}_part", f"trial{t}_lens"), t
        assert all(p.length(j) in (bits // m, bits // m + 1) for j in range(m))


def test_reference_expectations_on_hand_cases(port):
    """optimize_test.cpp:16-62: identical columns 1, independent 0, complement 1, constants 0."""
    hand = np.array([[0b000], [0b011], [0b100], [0b111]], np.uint64)
    c, const, _ = port.estimate_correlations(hand, 3)
    assert c[0, 0] == 1.0 and c[0, 1] == 1.0 and c[1, 0] == 1.0 and c[0, 2] == 0.0 and c[1, 2] == 0.0
    anti = np.array([[0b01], [0b10], [0b01], [0b10]], np.uint64)
    assert port.estimate_correlations(anti, 2)[0][0, 1] == 1.0
    cb = np.array([[0b001 | ((i % 2 == 0) << 1)] for i in range(5)], np.uint64)
    c, const, _ = port.estimate_correlations(cb, 3)
    assert list(const) == [True, False, True] and c[0, 1] == 0.0 and c[0, 2] == 0.0


def test_duplicated_pairs_are_separated(g):
    """optimize_test.cpp:87-102: no substring holds both bits of a duplicated pair."""
    for seed in (0, 1, 77):
        subs = subs_of(g, f"dup16_part_m4_s{seed}", f"dup16_lens_m4_s{seed}")
        for sub in subs:
            assert len(sub) == 4 and len({x // 2 for x in sub}) == 4


def test_error_contracts():
    import paper_1307_2982_b200 as mg
    from paper_1307_2982_b200 import _lib

    cm = mg.CorrelationMatrix(8)
    with pytest.raises(ValueError):
        mg.greedy_assign(cm, 0, 1)
    with pytest.raises(ValueError):
        mg.greedy_assign(cm, 9, 1)
    with pytest.raises(ValueError):  # CodeDatabase::zeros(3, 1): one code is not enough
        mg.estimate_correlations(mg.CodeDatabase(3, np.zeros((1, 1), np.uint64)))
    # the C ABI itself rejects m out of range and n < 2 before touching a device
    L = _lib.lib()
    lens = np.zeros(4, np.uint32)
    pos = np.zeros(8, np.uint32)
    corr = np.eye(8)
    const = np.zeros(8, np.uint8)
    rc = L.mihg_greedy_assign(corr.ctypes.data_as(C.POINTER(C.c_double)), const.ctypes.data_as(C.POINTER(C.c_uint8)),
                              8, 0, 1, lens.ctypes.data_as(_lib.u32p), pos.ctypes.data_as(_lib.u32p))
    assert rc == _lib.MIHG_EINVAL
    one = np.zeros(1, np.uint64)
    rc = L.mihg_estimate_correlations(C.c_void_p(one.ctypes.data), 1, 3, 0, 0,
                                      corr.ctypes.data_as(C.POINTER(C.c_double)),
                                      const.ctypes.data_as(C.POINTER(C.c_uint8)), None)
    assert rc == _lib.MIHG_EINVAL
