"""One untraced MIH kNN step of a bench config (for ncu traffic captures), or with --traced the
algorithmic bytes of that step (SURVEY.md §8d accounting) printed as JSON."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--nq", type=int, default=0)
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--traced", action="store_true")
    ap.add_argument("--profile-search", action="store_true",
                    help="bracket only the search with cudaProfilerStart/Stop (ncu --profile-from-start off)")
    a = ap.parse_args()
    import torch

    import paper_1307_2982_b200 as mg
    from paper_1307_2982_b200 import _lib

    cfg = dict(bench.CONFIGS[a.config])
    if a.nq:
        cfg["nq"] = a.nq
    if a.k:
        cfg["k"] = a.k
    dev = torch.device("cuda", 0)
    L = _lib.lib()
    codes = bench.make_codes_device(cfg, 0, cfg["n"], cfg["db_seed"], torch, dev, L)
    qs = bench.make_codes_device(cfg, 0, cfg["nq"], cfg["q_seed"], torch, dev, L)
    idx = mg.MihIndex.build_from_device(codes.data_ptr(), cfg["n"], cfg["bits"],
                                        mg.consecutive_partition(cfg["bits"], cfg["m"]), 0)
    del codes
    nq, k = cfg["nq"], cfg["k"]
    ids = torch.empty((nq, k), dtype=torch.int32, device=dev)
    d = torch.empty((nq, k), dtype=torch.int32, device=dev)
    tr = torch.empty((nq, 5), dtype=torch.int64, device=dev) if a.traced else None
    if a.profile_search:  # warm-up search outside the profiled range
        idx.knn_search_device(qs.data_ptr(), nq, k, ids.data_ptr(), d.data_ptr(), None)
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
    idx.knn_search_device(qs.data_ptr(), nq, k, ids.data_ptr(), d.data_ptr(), tr.data_ptr() if a.traced else None)
    torch.cuda.synchronize()
    if a.profile_search:
        torch.cuda.profiler.stop()
    if a.traced:
        t = tr.cpu().numpy().astype(np.float64)
        alg = float((8 * t[:, 0] + 4 * t[:, 1] + (cfg["bits"] / 8) * t[:, 2]).sum())
        print(json.dumps({"config": a.config, "nq": nq, "alg_bytes_per_step": alg}))


if __name__ == "__main__":
    main()
