"""CPU: pin the Gaussian-mixture sign-projection generator (csrc/gen.cu) with an independent
numpy restatement of its definition; the C restatement (oracle) must agree bit-for-bit, and the
GPU kernel is checked against the C one in tests/test_gpu_merge_datagen.py."""
import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x):
    x = (x + np.uint64(0x9E3779B97F4A7C15)) & M64
    x = ((x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & M64
    x = ((x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & M64
    return x ^ (x >> np.uint64(31))


def hseed(seed, s):
    return splitmix64(np.uint64(seed) ^ ((np.uint64(s) * np.uint64(0xD6E8FEB86659FD93)) & M64))


def g(u, width):
    mask = np.uint64((1 << width) - 1)
    tot = sum(((u >> np.uint64(width * t)) & mask).astype(np.int64) for t in range(4))
    return tot - (2 * ((1 << width) - 1))


def numpy_mixture(first, n, bits, dim, comps, model_seed, data_seed):
    with np.errstate(over="ignore"):
        t = np.arange(bits * dim, dtype=np.uint64)
        W = g(splitmix64(hseed(model_seed, 1) ^ t), 6).reshape(bits, dim)
        t = np.arange(comps * dim, dtype=np.uint64)
        mu = g(splitmix64(hseed(model_seed, 2) ^ t), 5).reshape(comps, dim)
        i = np.arange(first, first + n, dtype=np.uint64)
        c = (splitmix64(hseed(data_seed, 3) ^ i) % np.uint64(comps)).astype(np.int64)
        per = (dim + 2) // 3
        d = np.arange(dim)
        u = splitmix64(hseed(data_seed, 4) ^ (i[:, None] * np.uint64(per) + (d // 3).astype(np.uint64)[None, :]))
        noise = g(u >> (np.uint64(20) * (d % 3).astype(np.uint64))[None, :], 5)
        x = mu[c] + noise
    assert np.abs(x).max() <= 124
    dots = x @ W.T  # [n, bits]
    wpc = (bits + 63) // 64
    out = np.zeros((n, wpc), np.uint64)
    for j in range(bits):
        out[:, j // 64] |= (dots[:, j] >= 0).astype(np.uint64) << np.uint64(j % 64)
    return out


def test_c_generator_matches_numpy_definition(port):
    for bits, first, n in ((64, 0, 3000), (128, 987654321, 1000), (256, 3, 500), (70, 11, 700)):
        want = numpy_mixture(first, n, bits, 128, 64, 0x4C0FFEE, 0x4D0001)
        got = port.gen_mixture(first, n, bits, 128, 64, 0x4C0FFEE, 0x4D0001)
        assert np.array_equal(got, want), bits


def test_generator_is_clustered_but_not_degenerate(port):
    codes = port.gen_mixture(0, 20000, 64, 128, 64, 0x4C0FFEE, 0x4D0001)[:, 0]
    assert len(np.unique(codes)) > 19000  # few exact duplicates at sigma_rel = 1
    bits = ((codes[:, None] >> np.arange(64, dtype=np.uint64)) & np.uint64(1)).mean(0)
    assert 0.2 < bits.min() and bits.max() < 0.8
