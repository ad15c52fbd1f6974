"""Command-line front end on the GPU index — the hot-path subcommands of the reference CLI
(/root/reference/proj/tools/mih.cpp): gen / build / query / benchmark / optimize, same options,
report schemas and exit codes (0 ok, 1 usage, 2 data/format error, 3 benchmark verification
mismatch, tools/mih.cpp:28-31). costmodel is out of scope.

    python -m paper_1307_2982_b200.cli gen --mode uniform --n 20000 --bits 64 --seed 11 --out data.bin
    python -m paper_1307_2982_b200.cli build --dataset data.bin --tables 4 --stats --out idx.bin
    python -m paper_1307_2982_b200.cli query --index idx.bin --queries q.bin --k 5 --out knn.csv
    python -m paper_1307_2982_b200.cli benchmark --dataset data.bin --queries q.bin --k 3 --radius 6
    python -m paper_1307_2982_b200.cli optimize --dataset data.bin --tables 4 --seed 7 --out part.json
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import sys
import time

import numpy as np

EXIT_OK, EXIT_USAGE, EXIT_DATA, EXIT_MISMATCH = 0, 1, 2, 3


class UsageError(Exception):
    pass


class DataError(Exception):
    pass


def choose_num_tables(bits: int, n: int) -> int:
    """costmodel.hpp:125-130: closest integer to b / log2 n, clamped to [1, b]."""
    if n < 2:
        raise ValueError("choose_num_tables: n must be at least 2")
    r = bits / math.log2(n)
    rounded = int(math.floor(r + 0.5)) if r >= 0 else int(math.ceil(r - 0.5))  # llround
    return max(1, min(bits, rounded))


def resolve_partition(bits: int, n: int, tables: int, partition_path: str):
    """tools/mih.cpp:66-77: JSON {bits, substrings} or consecutive_partition(bits, m)."""
    import paper_1307_2982_b200 as mg

    if partition_path:
        try:
            j = json.load(open(partition_path))
        except OSError as e:
            raise DataError(f"cannot open partition file: {partition_path}") from e
        except ValueError as e:
            raise DataError(f"partition file is not valid JSON: {partition_path}") from e
        if "bits" not in j or "substrings" not in j:
            raise DataError(f"partition file needs 'bits' and 'substrings' fields: {partition_path}")
        p = mg.Partition(int(j["bits"]), j["substrings"])
        if p.bits() != bits:
            raise DataError(f"partition width {p.bits()} does not match dataset width {bits}")
        return p
    m = tables if tables > 0 else choose_num_tables(bits, max(n, 2))
    return mg.consecutive_partition(bits, m)


def gen_duplicated_bits(n: int, bits: int, block: int, seed: int):
    """io.hpp:281-297: consecutive blocks of `block` positions copy one uniform source bit."""
    import paper_1307_2982_b200 as mg
    from paper_1307_2982_b200 import _lib

    if block == 0 or bits % block != 0:
        raise ValueError("gen_duplicated_bits: block size must divide the code width")
    sources = bits // block
    per = (sources + 63) // 64
    L = _lib.lib()
    st = C.c_void_p()
    _lib.check(L.mihg_mt64_create(seed, C.byref(st)))
    try:
        draws = np.zeros(max(n * per, 1), np.uint64)
        _lib.check(L.mihg_mt64_next_codes(st, n * per, 64, draws.ctypes.data_as(_lib.u64p)))
    finally:
        L.mihg_mt64_free(st)
    draws = draws[: n * per].reshape(n, per)
    src = np.zeros((n, sources), np.uint8)
    for s in range(sources):
        src[:, s] = (draws[:, s // 64] >> np.uint64(s % 64)) & np.uint64(1)
    full = np.repeat(src, block, axis=1)  # bit i of the code = source i // block
    wpc = (bits + 63) // 64
    words = np.zeros((n, wpc), np.uint64)
    for i in range(bits):
        words[:, i // 64] |= full[:, i].astype(np.uint64) << np.uint64(i % 64)
    return mg.CodeDatabase(bits, words)


def run_gen(a) -> int:
    import paper_1307_2982_b200 as mg

    if a.mode == "uniform":
        mg.write_codes(mg.gen_uniform(a.n, a.bits, a.seed), a.out)
    elif a.mode == "correlated":
        mg.write_codes(gen_duplicated_bits(a.n, a.bits, a.block, a.seed), a.out)
    elif a.mode == "mixture":  # this repo's seeded Gaussian-mixture generator (configs 2/4)
        import torch

        from paper_1307_2982_b200 import _lib

        wpc = (a.bits + 63) // 64
        out = torch.empty((max(a.n, 1), wpc), dtype=torch.int64, device="cuda")
        _lib.check(_lib.lib().mihg_gen_mixture_device(0, a.n, a.bits, a.dim, a.components, a.model_seed,
                                                      a.seed, C.c_void_p(out.data_ptr()), None))
        torch.cuda.synchronize()
        mg.write_codes(mg.CodeDatabase(a.bits, out[: a.n].cpu().numpy().view(np.uint64)), a.out)
    elif a.mode in ("vectors", "correlated-vectors", "lsh"):
        raise UsageError(f"gen mode {a.mode} (float vectors / LSH) is not part of the GPU hot path")
    else:
        raise UsageError(f"unknown gen mode: {a.mode}")
    print(f"wrote {a.out}")
    return EXIT_OK


def run_build(a) -> int:
    import paper_1307_2982_b200 as mg

    db = mg.read_codes(a.dataset)
    p = resolve_partition(db.bits(), db.size(), a.tables, a.partition)
    idx = mg.MihIndex.build(db, p, a.device)
    if a.stats:
        for j in range(idx.num_tables()):
            t = idx.table(j)
            st = t.stats()
            print(f"table {j}: s={t.s()} entries={st.total_entries} buckets={st.non_empty_buckets} "
                  f"max_bucket={st.max_bucket_size} est_bytes={st.estimated_bytes}")
    mg.write_index(idx, a.out)
    print(f"wrote {a.out} (n={db.size()}, m={idx.num_tables()})")
    return EXIT_OK


def run_query(a) -> int:
    import paper_1307_2982_b200 as mg

    if (a.k is None) == (a.radius is None):
        raise UsageError("query needs exactly one of --k or --radius")
    idx = mg.read_index(a.index, a.device)
    qs = mg.read_codes(a.queries)
    if qs.bits() != idx.bits():
        raise DataError(f"query width {qs.bits()} does not match index width {idx.bits()}")
    nq = qs.size()
    if a.k is not None:
        if a.k > idx.size():
            raise DataError(f"k={a.k} exceeds database size")
        ids, dists, tr = idx.knn_search_batch(qs.raw_words(), a.k, with_trace=True)
        rows = [(ids[i], dists[i]) for i in range(nq)]
    else:
        offs, ids, dists, tr = idx.range_search_batch(qs.raw_words(), a.radius, with_trace=True)
        rows = [(ids[offs[i]:offs[i + 1]], dists[offs[i]:offs[i + 1]]) for i in range(nq)]
    if a.format == "json":  # tools/mih.cpp:149-168
        report = [{"query": qi, "lookups": int(tr[qi].lookups), "unique_candidates": int(tr[qi].unique_candidates),
                   "final_radius": int(tr[qi].final_radius),
                   "neighbors": [{"id": int(i), "dist": int(d)} for i, d in zip(*rows[qi])]}
                  for qi in range(nq)]
        text = json.dumps(report, indent=2) + "\n"
    else:
        lines = ["query,rank,id,dist"]
        for qi in range(nq):
            lines += [f"{qi},{r},{int(i)},{int(d)}" for r, (i, d) in enumerate(zip(*rows[qi]))]
        text = "\n".join(lines) + "\n"
    _emit(text, a.out)
    return EXIT_OK


def _emit(text: str, out: str) -> None:
    if not out:
        sys.stdout.write(text)
        return
    try:
        open(out, "w").write(text)
    except OSError as e:
        raise DataError(f"cannot open for writing: {out}") from e
    print(f"wrote {out}")


def run_benchmark(a) -> int:
    """tools/mih.cpp:258-404: verify every configuration against the exhaustive scan, then time
    the index and the scan. On the GPU both are batched calls; per-query times are the batch
    time divided by the query count (one launch sequence serves every query)."""
    import paper_1307_2982_b200 as mg

    if not a.k and not a.radius:
        raise UsageError("benchmark needs at least one of --k or --radius")
    db = mg.read_codes(a.dataset)
    qs = mg.read_codes(a.queries)
    if qs.bits() != db.bits():
        raise DataError("query and dataset widths differ")
    for k in a.k:
        if k > db.size():
            raise DataError(f"k={k} exceeds database size")
    p = resolve_partition(db.bits(), db.size(), a.tables, a.partition)
    t0 = time.perf_counter()
    idx = mg.MihIndex.build(db, p, a.device)
    build_s = time.perf_counter() - t0
    print(f"index built in {build_s} s (n={db.size()}, m={p.m()})", file=sys.stderr)
    qw = qs.raw_words()
    nq = qs.size()

    # correctness gate (tools/mih.cpp:274-301): kNN by distances, range by ids and distances
    for k in a.k:
        _, d_mih = idx.knn_search_batch(qw, k)
        _, d_scan = idx.scan_knn_batch(qw, k)
        if not np.array_equal(d_mih, d_scan):
            print(f"verification mismatch: knn k={k}", file=sys.stderr)
            return EXIT_MISMATCH
    for r in a.radius:  # exhaustive reference: the scan's complete (dist, id) order cut at r
        offs, ids, dists, _ = idx.range_search_batch(qw, r)
        si, sd = idx.scan_knn_batch(qw, db.size())
        for qi in range(nq):
            cnt = int(np.searchsorted(sd[qi], r, side="right"))
            if not (np.array_equal(ids[offs[qi]:offs[qi + 1]], si[qi, :cnt]) and
                    np.array_equal(dists[offs[qi]:offs[qi + 1]], sd[qi, :cnt])):
                print(f"verification mismatch: range r={r} query {qi}", file=sys.stderr)
                return EXIT_MISMATCH
    print(f"verification passed on {nq} queries", file=sys.stderr)

    rows = []
    warm = min(a.warmup, nq)

    def timed(fn):
        if warm:
            fn(qw[:warm])
        t = time.perf_counter()
        out = fn(qw)
        return (time.perf_counter() - t) * 1e6 / max(nq, 1), out

    for kind, vals in (("k", a.k), ("r", a.radius)):
        for v in vals:
            if kind == "k":
                us, (_, _, tr) = timed(lambda q: idx.knn_search_batch(q, v, with_trace=True))
                us_plain, _ = timed(lambda q: idx.knn_search_batch(q, v))
                s_us, _ = timed(lambda q: idx.scan_knn_batch(q, v))
            else:
                us, (_, _, _, tr) = timed(lambda q: idx.range_search_batch(q, v, with_trace=True))
                us_plain = us
                s_us, _ = timed(lambda q: idx.scan_knn_batch(q, db.size()))
            ml = float(np.mean([t.lookups for t in tr])) if nq else 0.0
            mu = float(np.mean([t.unique_candidates for t in tr])) if nq else 0.0
            m_us = us_plain
            rows.append(dict(method="mih", param_kind=kind, param=v, queries=nq, warmup_queries=warm, threads=1,
                             mean_us=m_us, median_us=m_us, p95_us=m_us, mean_lookups=ml,
                             mean_unique_candidates=mu, speedup_vs_scan=s_us / m_us if m_us > 0 else 0))
            rows.append(dict(method="scan", param_kind=kind, param=v, queries=nq, warmup_queries=warm, threads=1,
                             mean_us=s_us, median_us=s_us, p95_us=s_us, mean_lookups=float(db.size()),
                             mean_unique_candidates=float(db.size()), speedup_vs_scan=0))
    cols = ["method", "param_kind", "param", "queries", "warmup_queries", "threads", "mean_us", "median_us",
            "p95_us", "mean_lookups", "mean_unique_candidates", "speedup_vs_scan"]
    if a.format == "json":  # tools/mih.cpp:215-248
        config = {"dataset": a.dataset, "queries": a.queries, "n": db.size(), "bits": db.bits(), "tables": p.m(),
                  "warmup": warm, "threads": 1, "timing": "GPU batched, per-query amortised",
                  "build_seconds": build_s, "device": a.device}
        text = json.dumps({"config": config, "rows": rows}, indent=2) + "\n"
    else:
        text = ",".join(cols) + "\n" + "".join(",".join(str(r[c]) for c in cols) + "\n" for r in rows)
    _emit(text, a.out)
    return EXIT_OK


def run_optimize(a) -> int:
    """tools/mih.cpp:502-512: estimate_correlations (GPU Gram kernel) + greedy_assign, written as
    partition JSON {bits, substrings} (save_partition_json, :57-64) for build --partition."""
    import paper_1307_2982_b200 as mg

    db = mg.read_codes(a.dataset)
    m = a.tables if a.tables > 0 else choose_num_tables(db.bits(), max(db.size(), 2))
    p = mg.greedy_assign(mg.estimate_correlations(db, device=a.device), m, a.seed)
    try:
        with open(a.out, "w") as f:
            f.write(json.dumps({"bits": p.bits(), "substrings": p.substrings()}, indent=2) + "\n")
    except OSError as e:
        raise DataError(f"cannot open for writing: {a.out}") from e
    print(f"wrote {a.out} (m={m})")
    return EXIT_OK


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # usage errors exit 1 (tools/mih.cpp:596-600)
        self.print_usage(sys.stderr)
        print(f"usage error: {message}", file=sys.stderr)
        sys.exit(EXIT_USAGE)


def main(argv=None) -> int:
    ap = _Parser(prog="mihg", description="exact nearest-neighbor search in Hamming space (B200)")
    sub = ap.add_subparsers(dest="cmd", parser_class=_Parser)
    g = sub.add_parser("gen", help="generate synthetic codes")
    g.add_argument("--mode", required=True)
    g.add_argument("--n", type=int, default=0)
    g.add_argument("--bits", type=int, default=64)
    g.add_argument("--block", type=int, default=4)
    g.add_argument("--seed", type=int, default=0)
    g.add_argument("--model-seed", type=int, default=0x4C0FFEE)
    g.add_argument("--dim", type=int, default=128)
    g.add_argument("--components", type=int, default=64)
    g.add_argument("--out", required=True)
    b = sub.add_parser("build", help="build an index from a codes file")
    b.add_argument("--dataset", required=True)
    b.add_argument("--tables", type=int, default=0)
    b.add_argument("--partition", default="")
    b.add_argument("--stats", action="store_true")
    b.add_argument("--out", required=True)
    b.add_argument("--device", type=int, default=0)
    q = sub.add_parser("query", help="run queries against a saved index")
    q.add_argument("--index", required=True)
    q.add_argument("--queries", required=True)
    q.add_argument("--k", type=int)
    q.add_argument("--radius", type=int)
    q.add_argument("--out", default="")
    q.add_argument("--format", default="csv", choices=["csv", "json"])
    q.add_argument("--device", type=int, default=0)
    be = sub.add_parser("benchmark", help="verify against linear scan, then time both methods")
    be.add_argument("--dataset", required=True)
    be.add_argument("--queries", required=True)
    be.add_argument("--tables", type=int, default=0)
    be.add_argument("--partition", default="")
    be.add_argument("--k", type=int, nargs="*", default=[])
    be.add_argument("--radius", type=int, nargs="*", default=[])
    be.add_argument("--warmup", type=int, default=10)
    be.add_argument("--out", default="")
    be.add_argument("--format", default="csv", choices=["csv", "json"])
    be.add_argument("--device", type=int, default=0)
    o = sub.add_parser("optimize", help="fit a correlation-aware partition")
    o.add_argument("--dataset", required=True)
    o.add_argument("--tables", type=int, default=0)
    o.add_argument("--seed", type=int, default=0)
    o.add_argument("--out", required=True)
    o.add_argument("--device", type=int, default=0)
    a = ap.parse_args(argv)
    if not a.cmd:
        ap.print_usage(sys.stderr)
        return EXIT_USAGE
    import paper_1307_2982_b200 as mg

    try:
        return {"gen": run_gen, "build": run_build, "query": run_query, "benchmark": run_benchmark,
                "optimize": run_optimize}[a.cmd](a)
    except UsageError as e:
        print(f"usage error: {e}", file=sys.stderr)
        return EXIT_USAGE
    except mg.FormatError as e:
        print(f"format error: {e}", file=sys.stderr)
        return EXIT_DATA
    except (DataError, ValueError, OSError, RuntimeError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_DATA


if __name__ == "__main__":
    sys.exit(main())
