"""Bucket statistics SEEN BY THE PROBES of a 2 x 32-bit config (default: config 4): for a sample
of queries, every bucket the MIH search probes (rings 0..final radius of both tables), looked up
in the sorted key array with torch. Prints, per table: empty fraction, bucket-size histogram,
entries per aligned bucket group (16/32/64 buckets) at the probed positions, and how many
distinct groups / sector-sized directory runs the probes of one query touch. Layout planning
input for the sparse directory."""
import argparse
import itertools
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def masks_upto(s, z):
    out = []
    for zz in range(z + 1):
        for c in itertools.combinations(range(s), zz):
            v = 0
            for b in c:
                v |= 1 << b
            out.append((v, zz))
    a = np.array(out, dtype=np.int64)
    return a[:, 0], a[:, 1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--sample", type=int, default=256)
    a = ap.parse_args()
    import torch

    import paper_1307_2982_b200 as mg
    from paper_1307_2982_b200 import _lib

    cfg = dict(bench.CONFIGS[a.config])
    dev = torch.device("cuda", 0)
    L = _lib.lib()
    codes = bench.make_codes_device(cfg, 0, cfg["n"], cfg["db_seed"], torch, dev, L)
    qs = bench.make_codes_device(cfg, 0, cfg["nq"], cfg["q_seed"], torch, dev, L)
    idx = mg.MihIndex.build_from_device(codes.data_ptr(), cfg["n"], cfg["bits"],
                                        mg.consecutive_partition(cfg["bits"], cfg["m"]), 0)
    nq, k = a.sample, cfg["k"]
    ids = torch.empty((nq, k), dtype=torch.int32, device=dev)
    d = torch.empty((nq, k), dtype=torch.int32, device=dev)
    tr = torch.empty((nq, 5), dtype=torch.int64, device=dev)
    idx.knn_search_device(qs.data_ptr(), nq, k, ids.data_ptr(), d.data_ptr(), tr.data_ptr())
    torch.cuda.synchronize()
    final_r = tr[:, 4].cpu().numpy()
    del idx
    torch.cuda.empty_cache()
    mv, mz = masks_upto(32, 4)
    mv_t = torch.from_numpy(mv).to(dev)
    mz_t = torch.from_numpy(mz).to(dev)
    out = {"config": a.config, "sample": nq, "mean_final_radius": float(final_r.mean())}
    cw = codes.view(-1)
    for j in range(2):
        keys = ((cw >> (32 * j)) & 0xFFFFFFFF).to(torch.int64)
        keys, _ = torch.sort(keys)
        uk, cnt = torch.unique_consecutive(keys, return_counts=True)
        del keys
        st = {"nonempty_buckets": int(uk.numel()), "max_bucket": int(cnt.max())}
        qk = ((qs.view(-1)[:nq] >> (32 * j)) & 0xFFFFFFFF).to(torch.int64)
        # step r probes ring r // 2 of table r % 2; a query with final radius R runs steps 0..R
        rr_max = torch.from_numpy(np.where(final_r >= j, (final_r - j) // 2, -1)).to(dev)
        probes, sizes = [], []
        tot_lookups = 0
        grp_touch = {16: 0, 32: 0, 64: 0, 128: 0}
        for qi in range(nq):
            sel = mz_t <= rr_max[qi]
            v = qk[qi] ^ mv_t[sel]
            tot_lookups += int(v.numel())
            pos = torch.searchsorted(uk, v)
            pos_c = pos.clamp(max=uk.numel() - 1)
            hit = uk[pos_c] == v
            c = torch.where(hit, cnt[pos_c], torch.zeros_like(pos_c))
            probes.append(v)
            sizes.append(c)
            for g in grp_touch:
                grp_touch[g] += int(torch.unique(v // g).numel())
        v = torch.cat(probes)
        c = torch.cat(sizes)
        st["lookups_per_query"] = tot_lookups / nq
        st["candidates_per_query"] = float(c.sum()) / nq
        st["empty_frac"] = float((c == 0).float().mean())
        edges = [0, 1, 2, 3, 4, 5, 6, 7, 8, 12, 16, 24, 32, 64, 128, 256, 1024, 1 << 30]
        hist, cand_share = {}, {}
        for lo, hi in zip(edges[:-1], edges[1:]):
            m = (c >= lo) & (c < hi)
            hist[f"{lo}-{hi - 1}"] = float(m.float().mean())
            cand_share[f"{lo}-{hi - 1}"] = float(c[m].sum()) / max(1.0, float(c.sum()))
        st["bucket_size_hist_over_probes"] = hist
        st["candidate_share_by_bucket_size"] = cand_share
        st["distinct_groups_per_lookup"] = {g: grp_touch[g] / tot_lookups for g in grp_touch}
        # entries of the aligned group around each probed NON-EMPTY bucket
        csum = torch.cat([torch.zeros(1, dtype=torch.int64, device=dev), torch.cumsum(cnt, 0)])
        ne = c > 0
        vn = v[ne]
        for g in (8, 16, 32, 64):
            lo = torch.searchsorted(uk, (vn // g) * g)
            hi = torch.searchsorted(uk, (vn // g) * g + g)
            tot = csum[hi] - csum[lo]
            qs_ = torch.tensor([0.25, 0.5, 0.75, 0.9, 0.99], device=dev, dtype=torch.float64)
            samp = tot[torch.randint(0, tot.numel(), (min(tot.numel(), 4_000_000),), device=dev)].double()
            st[f"group{g}_entries_at_nonempty_probes"] = {
                "mean": float(tot.double().mean()),
                "quantiles_25_50_75_90_99": [float(x) for x in torch.quantile(samp, qs_)],
                "frac_le": {str(t): float((tot <= t).float().mean()) for t in (4, 6, 8, 10, 12, 14, 16, 24, 28, 32, 48, 56, 64)},
            }
        out[f"table{j}"] = st
        del uk, cnt, csum
        torch.cuda.empty_cache()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
