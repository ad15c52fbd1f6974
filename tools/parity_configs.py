#!/usr/bin/env python
"""Full-size parity of the GPU kNN path against the reference itself, BASELINE configs 2-5.

For each (config, k): the GPU answers the whole query batch through MihIndex.knn_search_device
(the product path: device index, untraced, hybrid switch allowed), plus one traced run for the
SearchTrace counters; then the reference (oracle/_ref: the reference's own headers, unmodified)
answers a stated query subset on the same codes on the host:
  configs 2, 3 : MihIndex::knn_search (index.hpp:185-253) on all 10,000 queries, traces included;
  config 4     : MihIndex::knn_search on the first 2,000 (k=1, 100) / 500 (k=1000) queries
                 against the full n=1e9 reference index, traces included;
  config 5     : scan_knn (scan.hpp:43-68) on the first 128 queries (the reference MIH index,
                 ~106 GB plus minutes per query, does not fit the box: SURVEY.md §8c).
ids and distances must be identical row for row (the reference's (dist, id) order), and the
traces (lookups, candidates, unique_candidates, final_radius) identical where both exist.
Writes one JSON per case under the output directory and exits 3 on any mismatch.

  python tools/parity_configs.py [--out profiles/r02/parity] [--cases 2:10,4:100,...]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

CASES = [(2, 1, 10000), (2, 10, 10000), (2, 100, 10000), (3, 100, 10000), (4, 1, 2000), (4, 100, 2000),
         (4, 1000, 500), (5, 100, 128)]


def log(msg):
    print(f"[parity {time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)


def gpu_answers(cfg, ks, torch, L, mg, with_trace):
    """GPU index over the config's codes; per k: (ids, dists, traces) for the whole batch."""
    dev = torch.device("cuda", 0)
    nq, bits = cfg["nq"], cfg["bits"]
    codes = bench.make_codes_device(cfg, 0, cfg["n"], cfg["db_seed"], torch, dev, L)
    queries = bench.make_codes_device(cfg, 0, nq, cfg["q_seed"], torch, dev, L)
    t0 = time.time()
    idx = mg.MihIndex.build_from_device(codes.data_ptr(), cfg["n"], bits, mg.consecutive_partition(bits, cfg["m"]), 0)
    torch.cuda.synchronize()
    build_s = time.time() - t0
    db_host = None if cfg["data"] == "uniform" else codes.cpu().numpy().view(np.uint64)
    del codes
    torch.cuda.empty_cache()
    stream = torch.cuda.Stream(dev)
    res = {}
    for k in ks:
        ids = torch.empty((nq, k), dtype=torch.int32, device=dev)
        d = torch.empty_like(ids)
        t0 = time.time()
        idx.knn_search_device(queries.data_ptr(), nq, k, ids.data_ptr(), d.data_ptr(), stream=stream.cuda_stream)
        torch.cuda.synchronize()
        run_s = time.time() - t0
        tr = None
        if with_trace:
            tt = torch.empty((nq, 5), dtype=torch.int64, device=dev)
            ti = torch.empty_like(ids)
            td = torch.empty_like(ids)
            idx.knn_search_device(queries.data_ptr(), nq, k, ti.data_ptr(), td.data_ptr(), tt.data_ptr(),
                                  stream=stream.cuda_stream)
            torch.cuda.synchronize()
            tr = tt.cpu().numpy()
            # the traced run (pure MIH) must give the product run's answer (hybrid allowed)
            assert torch.equal(ti, ids) and torch.equal(td, d), "traced and untraced GPU runs differ"
        res[k] = (ids.cpu().numpy().view(np.uint32), d.cpu().numpy().view(np.uint32), tr, run_s)
        del ids, d
    qh = queries.cpu().numpy().view(np.uint64)
    idx.close()
    del queries
    torch.cuda.empty_cache()
    return res, qh, db_host, build_s


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02", "parity"))
    ap.add_argument("--cases", default="", help="comma list config:k:queries (default: all of CASES)")
    a = ap.parse_args()
    cases = CASES if not a.cases else [tuple(int(x) for x in c.split(":")) for c in a.cases.split(",")]
    os.makedirs(a.out, exist_ok=True)
    import torch

    import oracle
    import paper_1307_2982_b200 as mg
    from paper_1307_2982_b200 import _lib

    L = _lib.lib()
    R = oracle.ref()
    threads = os.cpu_count() or 1
    torch.cuda.set_device(0)
    failed = 0
    summary = []
    for config_id in sorted({c[0] for c in cases}):
        cc = [c for c in cases if c[0] == config_id]
        cfg = dict(bench.CONFIGS[config_id])
        mih_ok = bench.REF_MIH_FEASIBLE[config_id]
        log(f"config {config_id}: GPU, k in {[c[1] for c in cc]}")
        res, qh, db_host, build_s = gpu_answers(cfg, [c[1] for c in cc], torch, L, mg, with_trace=mih_ok)
        log(f"config {config_id}: GPU build {build_s:.1f}s, runs " +
            ", ".join(f"k={k}: {v[3]:.2f}s" for k, v in res.items()) + "; reference")
        t0 = time.time()
        if db_host is None:  # uniform configs: the reference's own gen_uniform (io.hpp:266-277)
            held = R.db_gen_uniform(cfg["n"], cfg["bits"], cfg["db_seed"])
        else:
            held = R.db_new(db_host, cfg["bits"])
            del db_host
        gen_s = time.time() - t0
        ref_index, ref_build_s = None, 0.0
        if mih_ok:
            t0 = time.time()
            ref_index = R.build_parallel(held.words(), cfg["bits"], cfg["m"])
            ref_build_s = time.time() - t0
            del held
            held = None
        log(f"config {config_id}: reference data {gen_s:.0f}s, index build {ref_build_s:.0f}s")
        for _, k, nref in cc:
            gi, gd, gt, run_s = res[k]
            q = qh[:nref]
            t0 = time.time()
            if mih_ok:
                ri, rd, rt, secs = ref_index.knn_timed(q, k, threads=threads)
                leg = {"mih": {"ids": ri, "dists": rd, "traces": rt}}
            else:
                ri, rd, secs = held.scan_knn_timed(q, k, threads=threads)
                leg = {"scan": {"ids": ri, "dists": rd}}
            ref_s = time.time() - t0
            par = bench.parity_check(leg, gi, gd, gt)
            rec = {"config": config_id, "k": k, "n": cfg["n"], "bits": cfg["bits"], "m": cfg["m"],
                   "data": cfg["data"], "gpu_queries": cfg["nq"], "gpu_knn_s": run_s, "gpu_build_s": build_s,
                   "reference": ("MihIndex::knn_search (index.hpp:185-253), traces included" if mih_ok
                                 else "scan_knn (scan.hpp:43-68)"),
                   "reference_queries": nref, "reference_threads": threads, "reference_s": ref_s,
                   "reference_build_s": ref_build_s, "reference_data_s": gen_s, "cpu_model": bench.cpu_model(),
                   "parity": par,
                   "mean_trace_gpu": (gt[:nref].mean(0).tolist() if gt is not None else None)}
            path = os.path.join(a.out, f"c{config_id}_k{k}.json")
            json.dump(rec, open(path, "w"), indent=1)
            log(f"config {config_id} k={k}: {par['queries']} queries vs reference ({ref_s:.0f}s), "
                f"mismatches {par['mismatches']} -> {path}")
            summary.append({"config": config_id, "k": k, "queries": par["queries"],
                            "mismatches": par["mismatches"], "vs": par["vs"]})
            failed += par["mismatches"] != 0
        del ref_index, held, res
    json.dump(summary, open(os.path.join(a.out, "summary.json"), "w"), indent=1)
    print(json.dumps(summary))
    sys.exit(3 if failed else 0)


if __name__ == "__main__":
    main()
