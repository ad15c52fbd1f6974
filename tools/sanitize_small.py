"""Small end-to-end cases for compute-sanitizer (memcheck / racecheck / synccheck): MIH kNN on both
table layouts (dense offsets, sparse directory) incl. the piece queue and the exact re-run pass,
the K7 tensor-core scan in both geometries (single CTA, CTA pair), the K6 POPC scan, the large-
segment selection path, range search and the id-shard merge. Exits non-zero on any result
mismatch against the oracle (so the sanitizer log is also a correctness run).

  compute-sanitizer --tool memcheck python tools/sanitize_small.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import oracle
    import paper_1307_2982_b200 as mg

    P = oracle.port()
    bad = 0
    for bits, m, n, k, layout in ((64, 4, 6000, 10, "auto"), (64, 2, 5000, 50, "sparse"), (128, 6, 3000, 20, "auto"),
                                  (256, 8, 2000, 10, "sparse")):
        db = mg.gen_uniform(n, bits, 7 + bits)
        qs = mg.gen_uniform(37, bits, 8 + bits).raw_words()
        idx = mg.MihIndex.build(db, mg.consecutive_partition(bits, m), layout=layout)
        wi, wd = P.scan_knn(db.raw_words(), bits, qs, k)
        for traced in (False, True):
            r = idx.knn_search_batch(qs, k, with_trace=traced)
            bad += not (np.array_equal(r[0], wi) and np.array_equal(r[1], wd))
        for pair in ("0", "1"):
            os.environ["MIHG_TC_PAIR"] = pair
            for kern in ("tc", "popc"):
                os.environ["MIHG_SCAN_KERNEL"] = kern
                si, sd = idx.scan_knn_batch(qs, k)
                bad += not (np.array_equal(si, wi) and np.array_equal(sd, wd))
        os.environ.pop("MIHG_SCAN_KERNEL", None)
        os.environ.pop("MIHG_TC_PAIR", None)
        offs, ri, rd, _ = idx.range_search_batch(qs[:5], bits // 8)
        bad += int(offs[-1] != len(ri))
    # heavy ties: large segments through the radix selection path and the re-run pass
    centres = mg.gen_uniform(3, 64, 99).raw_words()
    rng = np.random.default_rng(5)
    codes = centres[rng.integers(0, 3, 6000)].copy()
    codes[:, 0] ^= np.uint64(1) << rng.integers(0, 64, 6000).astype(np.uint64)
    db = mg.CodeDatabase(64, codes)
    idx = mg.MihIndex.build(db, mg.consecutive_partition(64, 4))
    qs = codes[:9].copy()
    os.environ["MIHG_BUFFER_CAP"] = "300"  # force overflow -> exact re-run pass
    for k in (5, 4500):
        gi, gd = idx.knn_search_batch(qs, k)
        wi, wd = P.scan_knn(codes, 64, qs, k)
        bad += not (np.array_equal(gi, wi) and np.array_equal(gd, wd))
    os.environ.pop("MIHG_BUFFER_CAP", None)
    print("sanitize_small:", "OK" if bad == 0 else f"{bad} MISMATCHES")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
