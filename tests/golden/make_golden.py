"""Regenerate the golden fixtures in tests/golden/ from the REFERENCE ITSELF.

Run in the dev container (needs /root/reference and oracle/_ref/libmihref.so, built by
``make -C oracle ref``):

    python tests/golden/make_golden.py

Every expected output below comes from the unmodified reference headers (MihIndex::knn_search,
range_search, scan_knn, SubstringTable::bucket_lookup, gen_uniform, lsh_encode) through
oracle/ref_driver.cpp. The cases mirror the reference's own tests (file:line relative to
/root/reference/proj); inputs that the GPU box cannot regenerate without the reference
(std::normal_distribution-based LSH codes) are stored verbatim.
"""
from __future__ import annotations

import hashlib
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402


def knn_case(R, codes, bits, m, queries, ks, lengths=None, positions=None):
    h = R.build(codes, bits, m, lengths, positions)
    out = {}
    for k in ks:
        ids, dists, tr = h.knn(queries, k)
        out[f"ids_k{k}"] = ids
        out[f"dists_k{k}"] = dists
        out[f"trace_k{k}"] = tr
    return out


def clustered_codes(n, bits, centers, flips, seed):
    """Codes within a few bit flips of random centres (numpy PCG64, stored in the fixture): exact
    kNN radii stay small at any width, so the reference MIH answers wide codes quickly."""
    rng = np.random.default_rng(seed)
    W = (bits + 63) // 64
    cen = rng.integers(0, 2**64, size=(centers, W), dtype=np.uint64)
    out = cen[rng.integers(0, centers, size=n)].copy()
    for i in range(n):
        for pos in rng.choice(bits, size=int(rng.integers(0, flips + 1)), replace=False):
            out[i, pos // 64] ^= np.uint64(1) << np.uint64(pos % 64)
    if bits % 64:
        out[:, -1] &= np.uint64((1 << (bits % 64)) - 1)
    return out


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def optimize_codes(spec):
    """Regenerate an optimize-case input from its spec (kind, n, bits, block, seed): 'dup' =
    gen_duplicated_bits (io.hpp:281-297), 'uni' = gen_uniform (io.hpp:266-277). Both
    regenerators are pinned against the reference elsewhere (test_cli / gen_uniform_pins)."""
    from paper_1307_2982_b200 import gen_uniform
    from paper_1307_2982_b200.cli import gen_duplicated_bits

    kind, n, bits, block, seed = spec
    if kind == "dup":
        return gen_duplicated_bits(n, bits, block, seed).raw_words()
    return gen_uniform(n, bits, seed).raw_words()


# (name, spec or None for stored codes, [(m, seed), ...], store the full matrix?)
OPTIMIZE_CASES = [
    ("dup16", ("dup", 3000, 16, 2, 21), [(4, 0), (4, 1), (4, 77)], True),       # optimize_test.cpp:87-102
    ("dup32", ("dup", 2000, 32, 4, 9), [(4, 123)], True),                      # :122-130
    ("dup32_load", ("dup", 20000, 32, 4, 31), [(4, 7)], True),                 # :145-170
    ("uni24", ("uni", 400, 24, 0, 3), [(1, 0), (3, 5), (24, 9)], True),        # :64-82
    ("accept10", ("dup", 100000, 128, 4, 0xD00D0001), [(8, 0xD00D0003)], True),  # acceptance.cpp:462-490
    ("dup100", ("dup", 777, 100, 4, 6), [(3, 1), (7, 2)], True),
    ("dup256", ("dup", 5000, 256, 8, 7), [(8, 3), (16, 4)], False),
    ("dup1000", ("dup", 3000, 1000, 8, 11), [(32, 5)], False),
]


def optimize_fixture(R):
    """estimate_correlations + greedy_assign from the reference (optimize.hpp) on the cases of
    optimize_test.cpp and acceptance criterion 10, plus multi-word widths for the GPU kernel."""
    out = {}

    def put(name, codes, bits, parts, full):
        corr, const, _ = R.estimate_correlations(codes, bits)
        out[name + "_const"] = const.astype(np.uint8)
        if full:
            out[name + "_corr"] = corr
        out[name + "_corr_sha256"] = np.frombuffer(bytes.fromhex(digest(corr)), np.uint8)
        for m, seed in parts:
            subs = R.greedy_assign(corr, const, m, seed)
            out[f"{name}_part_m{m}_s{seed}"] = np.array([x for sub in subs for x in sub], np.uint32)
            out[f"{name}_lens_m{m}_s{seed}"] = np.array([len(sub) for sub in subs], np.uint32)

    # hand-built inputs (optimize_test.cpp:16-62): codes stored verbatim
    hand = np.array([[0b000], [0b011], [0b100], [0b111]], np.uint64)
    anti = np.array([[0b01], [0b10], [0b01], [0b10]], np.uint64)
    cbits = np.array([[0b001 | ((i % 2 == 0) << 1)] for i in range(5)], np.uint64)
    rng = np.random.default_rng(14)  # HandlesConstantBits (:132-143): 4 random bits of 8
    c8 = np.array([[int(rng.integers(0, 16))] for _ in range(100)], np.uint64)
    for name, codes, bits, parts in (("hand", hand, 3, [(1, 0), (3, 0)]), ("anti", anti, 2, [(2, 0)]),
                                     ("constbits", cbits, 3, [(2, 0), (3, 1)]), ("const8", c8, 8, [(4, 5)])):
        out[name + "_codes"] = codes
        out[name + "_bits"] = np.array([bits], np.uint32)
        out[name + "_parts"] = np.array(parts, np.uint64)
        put(name, codes, bits, parts, True)
    for name, spec, parts, full in OPTIMIZE_CASES:
        codes = optimize_codes(spec)
        out[name + "_spec"] = np.array([0 if spec[0] == "dup" else 1] + list(spec[1:]), np.uint64)
        out[name + "_parts"] = np.array(parts, np.uint64)
        put(name, codes, spec[2], parts, full)
    # ProducesValidBalancedPartitions (:104-120): random widths / table counts
    rng = np.random.default_rng(8)
    trials = []
    for t in range(30):
        bits = int(4 + rng.integers(0, 60))
        m = int(1 + rng.integers(0, min(bits, 9)))
        seed = int(rng.integers(0, 1 << 62))
        trials.append((bits, m, seed))
        codes = optimize_codes(("uni", 200, bits, 0, 1000 + t))
        corr, const, _ = R.estimate_correlations(codes, bits)
        subs = R.greedy_assign(corr, const, m, seed)
        out[f"trial{t}_part"] = np.array([x for sub in subs for x in sub], np.uint32)
        out[f"trial{t}_lens"] = np.array([len(sub) for sub in subs], np.uint32)
    out["trials"] = np.array(trials, np.uint64)
    return out


def main(only=None):
    R = oracle.ref()
    files = {}
    files["optimize"] = optimize_fixture(R)
    if only == "optimize":
        files = {"optimize": files["optimize"]}
        return save(files)
    if only == "wide":
        files = {}

    # index_test.cpp:73-94 HandWorkedKnn (and scan_test.cpp:14-19 tiny_db)
    codes = np.array([[0], [1], [63]], np.uint64)
    files["hand_worked"] = dict(codes=codes, bits=6, m=2, queries=np.array([[0]], np.uint64),
                                **knn_case(R, codes, 6, 2, np.array([[0]], np.uint64), [1, 2, 3]))

    # index_test.cpp:127-154 KnnMatchesScanRandomized: b in {64,70}, n=1200, seeds 111+b / 222+b
    for bits in (64, 70):
        codes = R.gen_uniform(1200, bits, 111 + bits)
        qs = R.gen_uniform(15, bits, 222 + bits)
        d = dict(bits=bits, n=1200, db_seed=111 + bits, q_seed=222 + bits, codes=codes, queries=qs)
        for m in (4, 6, 7):
            for key, v in knn_case(R, codes, bits, m, qs, [1, 2, 10, 100, 1200]).items():
                d[f"m{m}_{key}"] = v
        files[f"knn_random_b{bits}"] = d

    # index_test.cpp:143-153: wide substrings, 24-bit, n=800, seeds 501/502, m=2
    codes = R.gen_uniform(800, 24, 501)
    qs = R.gen_uniform(10, 24, 502)
    files["knn_wide24"] = dict(bits=24, m=2, codes=codes, queries=qs,
                               **knn_case(R, codes, 24, 2, qs, [1, 10, 800]))

    # index_test.cpp:169-184 DuplicateCodesAllReported
    codes = np.array([[0x00FF]] * 5 + [[0x0F0F]], np.uint64)
    qs = np.array([[0x00FF]], np.uint64)
    files["duplicates"] = dict(bits=16, m=2, codes=codes, queries=qs,
                               **knn_case(R, codes, 16, 2, qs, [1, 5, 6]))

    # index_test.cpp:156-167 KnnOnDatabaseQueriesFindsSelf (n=600, seed 33, m=4, first 50 codes)
    codes = R.gen_uniform(600, 64, 33)
    files["self_queries"] = dict(bits=64, m=4, codes=codes, queries=codes[:50].copy(),
                                 **knn_case(R, codes, 64, 4, codes[:50], [1, 3]))

    # index_test.cpp:283-295 NonDivisibleWidthUsesUnevenSubstrings: 100 bits, m=8, n=800
    codes = R.gen_uniform(800, 100, 60)
    qs = R.gen_uniform(6, 100, 61)
    files["nondivisible100"] = dict(bits=100, m=8, codes=codes, queries=qs,
                                    **knn_case(R, codes, 100, 8, qs, [25]))

    # index_test.cpp:270-281 ScratchReuseIsClean: 32-bit, n=400, m=4, 40 queries, k=5
    codes = R.gen_uniform(400, 32, 50)
    qs = R.gen_uniform(40, 32, 51)
    files["scratch_reuse32"] = dict(bits=32, m=4, codes=codes, queries=qs,
                                    **knn_case(R, codes, 32, 4, qs, [5]))

    # Non-contiguous partition (codes.hpp:124-195 allows any balanced disjoint cover):
    # interleaved 64-bit partition, m=4, substring j owns bits {j, j+4, j+8, ...}.
    codes = R.gen_uniform(3000, 64, 4242)
    qs = R.gen_uniform(20, 64, 4343)
    lengths = np.full(4, 16, np.uint32)
    positions = np.array([j + 4 * i for j in range(4) for i in range(16)], np.uint32)
    files["interleaved64"] = dict(bits=64, m=4, codes=codes, queries=qs, lengths=lengths,
                                  positions=positions,
                                  **knn_case(R, codes, 64, 4, qs, [1, 10, 50], lengths, positions))

    # io_test.cpp:286-303 LshCodesStillAnswerExactQueries (non-uniform codes, stored verbatim)
    codes = R.gen_lsh(2000, 2000, 16, 4, 0.3, 88, 88, 64, 5)
    qs = R.gen_lsh(2000, 20, 16, 4, 0.3, 88, 89, 64, 5)
    files["lsh_io_test"] = dict(bits=64, m=4, codes=codes, queries=qs,
                                **knn_case(R, codes, 64, 4, qs, [10]))

    # acceptance.cpp:134-172 criterion 2: n=1e5, 64-bit, m=choose_num_tables(64,1e5)=4,
    # k in {1,10,100}; uniform lane (seeds 0xC0DE0001 / 0xC0DE0003) and the angular-embedding
    # lane (gen_correlated_vectors(1e5,32,4,0.3,0x5EED0001), queries 0x5EED0002, spec 0x5EED0003).
    # First 300 of the 1000 queries are pinned.
    m = int(round(64 / math.log2(1e5)))
    codes = R.gen_uniform(100000, 64, 0xC0DE0001)
    qs = R.gen_uniform(1000, 64, 0xC0DE0003)[:300]
    files["acceptance_uniform"] = dict(bits=64, m=m, db_seed=0xC0DE0001, q_seed=0xC0DE0003,
                                       n=100000, queries=qs, codes_sha256=digest(codes),
                                       **knn_case(R, codes, 64, m, qs, [1, 10, 100]))
    codes = R.gen_lsh(100000, 100000, 32, 4, 0.3, 0x5EED0001, 0x5EED0001, 64, 0x5EED0003)
    qs = R.gen_lsh(100000, 1000, 32, 4, 0.3, 0x5EED0001, 0x5EED0002, 64, 0x5EED0003)[:300]
    files["acceptance_lsh"] = dict(bits=64, m=m, codes=codes, queries=qs,
                                   **knn_case(R, codes, 64, m, qs, [1, 10, 100]))

    # BASELINE config 1: n=1e6 uniform 64-bit (seed 1), 1000 queries (seed 2), m=4, k=10.
    codes = R.gen_uniform(1000000, 64, 1)
    qs = R.gen_uniform(1000, 64, 2)
    files["config1"] = dict(bits=64, m=4, n=1000000, db_seed=1, q_seed=2, queries=qs,
                            codes_sha256=digest(codes), **knn_case(R, codes, 64, 4, qs, [10]))

    # index_test.cpp:96-112 RangeMatchesScanRandomized (range_search, next row §8f(1))
    for bits in (32, 96, 100):
        codes = R.gen_uniform(1500, bits, 8000 + bits)
        qs = R.gen_uniform(12, bits, 9000 + bits)
        d = dict(bits=bits, codes=codes, queries=qs)
        for m in (2, 4, 5):
            if (bits + m - 1) // m > 32:
                continue
            h = R.build(codes, bits, m)
            for r in (0, 1, 5, bits // 3):
                allids, alld, offs, trs = [], [], [0], []
                for qi in range(qs.shape[0]):
                    ids, dists, tr = h.range(qs[qi], r)
                    allids.append(ids)
                    alld.append(dists)
                    offs.append(offs[-1] + ids.size)
                    trs.append(tr)
                d[f"m{m}_r{r}_ids"] = np.concatenate(allids).astype(np.uint32)
                d[f"m{m}_r{r}_dists"] = np.concatenate(alld).astype(np.uint32)
                d[f"m{m}_r{r}_offs"] = np.array(offs, np.uint64)
                d[f"m{m}_r{r}_trace"] = np.stack(trs)
        files[f"range_b{bits}"] = d

    # table_test.cpp:34-43 / :65-104 semantics through MihIndex tables: bucket contents (ids in
    # insertion order) for sampled buckets of a 2e4 x 64-bit, m=3 (22/21/21) index.
    codes = R.gen_uniform(20000, 64, 777)
    h = R.build(codes, 64, 3)
    rng = np.random.default_rng(5)
    recs_j, recs_v, recs_ids, recs_off = [], [], [], [0]
    for j, s in enumerate((22, 21, 21)):
        occupied = [(int(codes[i, 0]) >> (0 if j == 0 else 22 + 21 * (j - 1))) & ((1 << s) - 1)
                    for i in rng.integers(0, 20000, 40)]
        for v in occupied + [int(x) for x in rng.integers(0, 1 << s, 20)]:
            ids = h.bucket(j, v)
            recs_j.append(j)
            recs_v.append(v)
            recs_ids.append(ids)
            recs_off.append(recs_off[-1] + ids.size)
    files["buckets_m3"] = dict(bits=64, m=3, db_seed=777, n=20000,
                               table=np.array(recs_j, np.uint32), value=np.array(recs_v, np.uint64),
                               ids=np.concatenate(recs_ids).astype(np.uint32),
                               offs=np.array(recs_off, np.uint64))

    # TableStats (table.hpp:190-197) of every table: non_empty_buckets, max_bucket_size,
    # total_entries, estimated_bytes.
    import ctypes as C
    stats = {}
    for name, n, bits, seed, m in (("b64m4", 1200, 64, 175, 4), ("b64m3", 20000, 64, 777, 3),
                                   ("b100m8", 800, 100, 60, 8), ("b64m2", 50000, 64, 31, 2)):
        codes = R.gen_uniform(n, bits, seed)
        h = R.build(codes, bits, m)
        rows = []
        for j in range(m):
            out = np.zeros(4, np.uint64)
            assert R.lib.ref_table_stats(h.h, j, out.ctypes.data_as(C.POINTER(C.c_uint64))) == 0
            rows.append(out)
        stats[name] = np.stack(rows)
        stats[name + "_spec"] = np.array([n, bits, seed, m], np.uint64)
    files["table_stats"] = stats

    # BMIX index files written by the reference's write_index (io.hpp:335-358), io_test.cpp:141-176
    # style shapes, plus its knn (k=5) and range (r = bits/4) answers on 10 queries each.
    import tempfile
    rng = np.random.default_rng(2)
    bm = {}
    case = 0
    while case < 5:
        bits = int(16 + rng.integers(0, 100))
        m = int(2 + rng.integers(0, 6))
        if (bits + m - 1) // m > 32:
            continue
        n = int(300 + rng.integers(0, 500))
        codes = R.gen_uniform(n, bits, int(rng.integers(1, 1 << 40)))
        qs = R.gen_uniform(10, bits, int(rng.integers(1, 1 << 40)))
        h = R.build(codes, bits, m)
        with tempfile.TemporaryDirectory() as td:
            fp = os.path.join(td, "idx.bin")
            assert R.lib.ref_write_index(h.h, fp.encode()) == 0
            blob = np.frombuffer(open(fp, "rb").read(), np.uint8).copy()
        ids, dists, tr = h.knn(qs, 5)
        rr = bits // 4
        roffs, rids, rd, rtr = [0], [], [], []
        for qi in range(10):
            a, b, t = h.range(qs[qi], rr)
            rids.append(a); rd.append(b); rtr.append(t); roffs.append(roffs[-1] + a.size)
        p_ = f"c{case}_"
        bm.update({p_ + "bmix": blob, p_ + "spec": np.array([bits, m, n], np.uint64), p_ + "queries": qs,
                   p_ + "knn_ids": ids, p_ + "knn_dists": dists, p_ + "knn_trace": tr,
                   p_ + "range_r": np.array([rr], np.uint64), p_ + "range_offs": np.array(roffs, np.uint64),
                   p_ + "range_ids": np.concatenate(rids).astype(np.uint32),
                   p_ + "range_dists": np.concatenate(rd).astype(np.uint32), p_ + "range_trace": np.stack(rtr)})
        case += 1
    files["bmix_files"] = bm

    # Codes wider than 256 bits (codes.hpp:16 allows up to 4096): the GPU's generic-width paths.
    # 300 bits (W = 5, a partial last word), m = 10 x 30-bit substrings; 512 bits (W = 8), m = 16
    # x 32-bit substrings (sparse tables). Clustered codes, queries near the centres; the
    # reference's MIH (ids, dists, traces) and scan_knn (scan.hpp:43-68) answers.
    for bits, m, seed in ((300, 10, 300), (512, 16, 512)):
        codes = clustered_codes(2000, bits, 40, 12, seed)
        qs = clustered_codes(12, bits, 40, 12, seed)  # same centres (same seed), other flips
        qs = np.concatenate([qs, R.gen_uniform(2, bits, seed + 1)])  # and two far-away queries
        d = dict(bits=bits, m=m, codes=codes, queries=qs[:12], scan_queries=qs,
                 **knn_case(R, codes, bits, m, qs[:12], [1, 10, 40]))
        for k in (1, 10, 60):
            si, sd = R.scan_knn(codes, bits, qs, k)
            d[f"scan_ids_k{k}"], d[f"scan_dists_k{k}"] = si, sd
        files[f"wide{bits}"] = d

    # gen_uniform pins (io.hpp:266-277): several widths and seeds.
    pins = {}
    for n, bits, seed in ((5, 64, 1), (7, 70, 181), (3, 256, 42), (4, 24, 501), (2, 130, 9)):
        pins[f"gen_{n}_{bits}_{seed}"] = R.gen_uniform(n, bits, seed)
    files["gen_uniform_pins"] = pins

    if only == "wide":
        files = {k: v for k, v in files.items() if k.startswith("wide")}
    save(files)


def save(files):
    for name, d in files.items():
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **{k: np.asarray(v) for k, v in d.items()})
        print(f"{path}: {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else None)
