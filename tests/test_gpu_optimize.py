"""GPU: estimate_correlations' AND-popcount Gram kernel (csrc/optimize.cu) — exact integer
counts and bitwise-identical correlations against the reference's golden outputs, greedy
partitions from the GPU matrix identical to the reference's, host and device inputs, chunk
boundaries; and the effect the reference asserts (optimize_test.cpp:145-170, acceptance
criterion 10) measured through the GPU index."""
import numpy as np
import pytest

from _optimize_cases import HAND, SPEC, codes_for, corr_matches, parts_for, subs_of

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g(golden):
    return golden("optimize")


@pytest.mark.parametrize("name", HAND + SPEC)
def test_gpu_correlations_and_partitions_match_reference(cuda_ok, g, port, name):
    import paper_1307_2982_b200 as mg

    codes, bits = codes_for(g, name)
    cm = mg.estimate_correlations(mg.CodeDatabase(bits, codes))
    assert corr_matches(g, name, cm.values), name
    assert np.array_equal(cm.constant.astype(np.uint8), g[name + "_const"])
    if codes.shape[0] * bits <= 5000 * 256:
        _, _, counts = port.estimate_correlations(codes, bits)
        assert np.array_equal(cm.counts, counts)
    for m, seed in parts_for(g, name):
        want = subs_of(g, f"{name}_part_m{m}_s{seed}", f"{name}_lens_m{m}_s{seed}")
        assert mg.greedy_assign(cm, m, seed).substrings() == want, (name, m, seed)


@pytest.mark.parametrize("bits,n", [(64, (1 << 22) + 12345), (130, 70001), (4096, 300)])
def test_gpu_counts_host_and_device_inputs(cuda_ok, port, bits, n):
    """Exact counts against the C oracle across the 2^22-code chunk boundary, a 3-word width with
    a partial last word, and the maximum width; device-pointer input equals host input."""
    import torch

    import paper_1307_2982_b200 as mg

    db = mg.gen_uniform(n, bits, 4242 + bits)
    codes = db.raw_words()
    host = mg.estimate_correlations(db)
    dev = torch.from_numpy(np.ascontiguousarray(codes).view(np.int64)).cuda()
    on_dev = mg.estimate_correlations((dev.data_ptr(), n, bits), codes_on_device=True)
    assert np.array_equal(host.counts, on_dev.counts)
    assert np.array_equal(host.values.view(np.uint64), on_dev.values.view(np.uint64))
    corr, const, counts = port.estimate_correlations(codes, bits)
    assert np.array_equal(host.counts, counts)
    assert np.array_equal(host.values.view(np.uint64), corr.view(np.uint64))
    assert np.array_equal(host.constant, const)


def test_gpu_tuned_partition_spreads_blocks(cuda_ok):
    """optimize_test.cpp:145-170: on block-duplicated 32-bit codes, consecutive 8-bit substrings
    see 4 values (max bucket >= 4000) while the tuned partition behaves like 8 independent bits
    (max bucket <= 600). Bucket loads read from the GPU index's tables."""
    import paper_1307_2982_b200 as mg
    from paper_1307_2982_b200.cli import gen_duplicated_bits

    db = gen_duplicated_bits(20000, 32, 4, 31)
    tuned = mg.greedy_assign(mg.estimate_correlations(db), 4, 7)

    def max_load(p):
        idx = mg.MihIndex.build(db, p)
        return max(idx.table(j).max_bucket_size() for j in range(4))

    assert max_load(mg.consecutive_partition(32, 4)) >= 4000
    assert max_load(tuned) <= 600


def test_gpu_acceptance_criterion_10(cuda_ok):
    """acceptance.cpp:462-490: n=1e5 128-bit block-correlated codes, m=8, k=10, 1000 queries:
    mean unique candidates with the greedy partition <= with the consecutive one."""
    import paper_1307_2982_b200 as mg
    from paper_1307_2982_b200.cli import gen_duplicated_bits

    db = gen_duplicated_bits(100000, 128, 4, 0xD00D0001)
    qs = gen_duplicated_bits(1000, 128, 4, 0xD00D0002).raw_words()
    tuned = mg.greedy_assign(mg.estimate_correlations(db), 8, 0xD00D0003)

    def mean_unique(p):
        idx = mg.MihIndex.build(db, p)
        _, _, tr = idx.knn_search_batch(qs, 10, with_trace=True)
        return np.mean([t.unique_candidates for t in tr])

    cons, opt = mean_unique(mg.consecutive_partition(128, 8)), mean_unique(tuned)
    assert opt <= cons, (cons, opt)
