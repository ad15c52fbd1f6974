#!/usr/bin/env python
"""Exact Hamming kNN throughput on B200 (BASELINE.json metric: exact kNN queries/s, n=1B, k=100).

Default workload = BASELINE config 4: n = 1e9 64-bit Gaussian-mixture sign-projection codes,
10k queries from the same generator, k = 100, m = 2 sparse tables of 32-bit substrings, id-range
sharded over the ranks (one process per GPU, NCCL all-gather + exact k-way merge for N > 1).

One step = one pass of the MIH kNN hot path over the whole 10k-query batch.
  value : queries/s with queries and results resident in HBM (device-pointer C ABI call),
          whole job (all ranks), timed with CUDA events, max over ranks.
  e2e   : the same through the host-pointer C ABI (mihg_knn_batch): pinned host queries in,
          host results out, copies inside the timed region.
  roofline : the MIH probe kernel's algorithmic bytes (8*lookups + 4*candidates
          + (b/8)*unique, from the reference-identical SearchTrace counters) over its CUDA-event
          time, against MEASURED_PEAKS.json hbm_gbs.
  cpu_baseline : the reference's own MihIndex::knn_search (oracle/_ref, built from the reference
          headers) on the host cores, on a bounded sample of this workload's queries.

`--impl reference` times only that CPU reference arm (rank 0; other ranks exit 0).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    1: dict(n=1_000_000, bits=64, m=4, k=10, nq=1000, data="uniform", db_seed=1, q_seed=2),
    2: dict(n=10_000_000, bits=128, m=6, k=10, nq=10000, data="mixture", model_seed=0x2C0FFEE,
            db_seed=0x2D0001, q_seed=0x2D0002),
    3: dict(n=100_000_000, bits=64, m=3, k=100, nq=10000, data="uniform", db_seed=3, q_seed=4),
    4: dict(n=1_000_000_000, bits=64, m=2, k=100, nq=10000, data="mixture", model_seed=0x4C0FFEE,
            db_seed=0x4D0001, q_seed=0x4D0002),
    5: dict(n=1_000_000_000, bits=256, m=8, k=100, nq=10000, data="uniform", db_seed=5, q_seed=6),
}
MIX_DIM, MIX_COMPS = 128, 64


_REAL_STDOUT = None


def claim_stdout():
    """Keep stdout for the ONE JSON line: everything else written to fd 1 from here on (NCCL's
    version banner, library chatter) goes to stderr."""
    global _REAL_STDOUT
    if _REAL_STDOUT is None:
        sys.stdout.flush()
        _REAL_STDOUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)


def emit(obj):
    out = _REAL_STDOUT or sys.stdout
    print(json.dumps(obj), file=out, flush=True)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=0, help="override database size (testing only)")
    ap.add_argument("--nq", type=int, default=0)
    ap.add_argument("--single-layout", action="store_true",
                    help="torchrun: skip the second multi-GPU layout's line (other_layout)")
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--cpu-sample", type=int, default=0, help="queries per CPU-reference step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shard", default="probe", choices=["probe", "id"],
                    help="N>1: probe = every rank holds the index and probes 1/N of the substring key "
                         "space (work divides by N); id = id-range shards (north_star's layout)")
    ap.add_argument("--method", default="mih", choices=["mih", "scan"],
                    help="mih: MihIndex::knn_search path (default); scan: the exhaustive K6 comparator")
    return ap.parse_args()


def workload(args):
    cfg = dict(CONFIGS[args.config])
    if args.n:
        cfg["n"] = args.n
    if args.nq:
        cfg["nq"] = args.nq
    if args.k:
        cfg["k"] = args.k
    return cfg


def wpc(bits):
    return (bits + 63) // 64


def shard_range(n, rank, world):
    per = (n + world - 1) // world
    lo = min(n, rank * per)
    return lo, min(n, lo + per)


# ---------------------------------------------------------------------------------------------
# clocks sampled during the timed region (B200_PROFILING.md clocks line)
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.dev = device_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.thread.join(timeout=2)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sms, mx, reasons = [], None, set()
        for r in self.rows:
            try:
                sms.append(float(r[1]))
                mx = float(r[2])
            except ValueError:
                continue
            for nm, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sms) if sms else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sms)}


# ---------------------------------------------------------------------------------------------
def make_codes_device(cfg, lo, hi, seed, torch, dev, lib):
    """Codes [lo, hi) of the workload's generator, resident on `dev` as int64 words."""
    W = wpc(cfg["bits"])
    n = hi - lo
    out = torch.empty((max(n, 1), W), dtype=torch.int64, device=dev)
    if cfg["data"] == "mixture":
        from paper_1307_2982_b200 import _lib
        _lib.check(lib.mihg_gen_mixture_device(lo, n, cfg["bits"], MIX_DIM, MIX_COMPS, cfg["model_seed"],
                                               seed, C.c_void_p(out.data_ptr()), None))
        torch.cuda.synchronize(dev)
    else:  # mt19937_64 stream (gen_uniform), generated and uploaded in chunks
        from paper_1307_2982_b200 import _lib
        st = C.c_void_p()
        _lib.check(lib.mihg_mt64_create(seed, C.byref(st)))
        try:
            _lib.check(lib.mihg_mt64_next_codes(st, lo, cfg["bits"], None))  # skip [0, lo)
            chunk = 1 << 25
            host = torch.empty((min(chunk, max(n, 1)), W), dtype=torch.int64).pin_memory()
            for c0 in range(0, n, chunk):
                cn = min(chunk, n - c0)
                hv = host[:cn]
                _lib.check(lib.mihg_mt64_next_codes(st, cn, cfg["bits"], C.cast(C.c_void_p(hv.data_ptr()), _lib.u64p)))
                out[c0:c0 + cn].copy_(hv)
        finally:
            lib.mihg_mt64_free(st)
    return out


def make_codes_host_cpu(cfg, lo, hi, seed):
    """The same codes generated on the host only (CPU reference arm: no GPU code involved)."""
    import oracle

    if cfg["data"] == "mixture":
        return oracle.port().gen_mixture(lo, hi - lo, cfg["bits"], MIX_DIM, MIX_COMPS, cfg["model_seed"], seed)
    R = oracle.ref()
    if lo == 0:
        return R.gen_uniform(hi, cfg["bits"], seed)
    return R.gen_uniform(hi, cfg["bits"], seed)[lo:]


def config_desc(cfg, args, world):
    d = {"workload": f"BASELINE config {args.config}: exact {cfg['k']}-NN over n={cfg['n']:.0e} "
                     f"{cfg['bits']}-bit {cfg['data']} codes, {cfg['nq']} queries, MIH m={cfg['m']}",
         "n": cfg["n"], "bits": cfg["bits"], "m": cfg["m"], "k": cfg["k"], "queries": cfg["nq"],
         "data_generator": cfg["data"],
         "parallelism": (f"probe-space partition x{world} (replicated index, rank g probes the ring values whose "
                         f"top log2({world}) key bits equal g; per-round NCCL histogram all-reduce, NCCL all-gather "
                         f"of local top-k + device merge, all inside libmihg)" if world > 1 and args.shard == "probe"
                         else (f"id-range shards x{world} (north_star layout: rank g indexes ids [g*ceil(n/{world}), ...); "
                               f"global stopping via per-round NCCL histogram all-reduce; NCCL all-gather + device "
                               f"merge, all inside libmihg)" if world > 1 else "single GPU")),
         "allgather_bytes_per_step": int(world * cfg["nq"] * cfg["k"] * 8) if world > 1 else 0,
         "l2_policy": "inputs larger than L2 (index >> 126 MB); no flush"}
    if cfg["data"] == "mixture":
        d.update({"mixture": {"dim": MIX_DIM, "components": MIX_COMPS, "sigma_rel": 1.0,
                              "model_seed": cfg["model_seed"], "db_seed": cfg["db_seed"],
                              "q_seed": cfg["q_seed"], "arith": "exact int8 (csrc/gen.cu)"}})
    else:
        d.update({"db_seed": cfg["db_seed"], "q_seed": cfg["q_seed"], "generator": "gen_uniform (mt19937_64)"})
    return d


# ---------------------------------------------------------------------------------------------
# The reference's CPU implementation (oracle/_ref = the reference's own headers, unmodified):
# MihIndex::knn_search and scan_knn timed on the host cores, and their answers kept as the parity
# oracle of the GPU rows for the same queries (the verify-before-report gate of
# tools/mih.cpp:274-301, against the reference itself).
REF_MIH_FEASIBLE = {1: True, 2: True, 3: True, 4: True, 5: False}  # config 5: ~106 GB index
MIH_SAMPLE = {1: 1000, 2: 1024, 3: 1024, 4: 1024, 5: 0}            # queries timed with all threads
SCAN_SAMPLE = {1: 64, 2: 32, 3: 16, 4: 16, 5: 64}                 # scan_knn queries, all threads


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def _stats(secs):
    secs = sorted(float(x) for x in secs)
    if not secs:
        return None
    p95 = secs[min(len(secs) - 1, int(round(0.95 * (len(secs) - 1))))]
    return {"mean_ms": 1e3 * statistics.mean(secs), "median_ms": 1e3 * statistics.median(secs),
            "p95_ms": 1e3 * p95, "queries": len(secs)}


def reference_leg(cfg, config_id, queries_host, db_words=None, mih_sample=None, scan_sample=None,
                  single_sample=None, steps=1, warmup=0, log=None):
    """Run the reference on the host. db_words: [n, W] host codes, or None for gen_uniform inside
    the reference (uniform configs). Returns a dict with timings and the reference's answers:
      mih: {qps, threads, per_query (all-thread), single_thread stats, ids, dists, traces, q0, nq}
      scan: {qps, threads, per_query, ids, dists, q0, nq}
    Queries are the first rows of the batch (q0 = 0)."""
    import oracle

    R = oracle.ref()
    threads = os.cpu_count() or 1
    bits, k = cfg["bits"], cfg["k"]
    out = {"cpu_model": cpu_model(), "cores": threads}
    t0 = time.time()
    held = None
    if db_words is None:
        held = R.db_gen_uniform(cfg["n"], bits, cfg["db_seed"])
        db_words = held.words()
    out["gen_s"] = time.time() - t0
    ms = MIH_SAMPLE[config_id] if mih_sample is None else mih_sample
    ss = SCAN_SAMPLE[config_id] if scan_sample is None else scan_sample
    ms, ss = min(ms, queries_host.shape[0]), min(ss, queries_host.shape[0])
    scan_owner = held
    if REF_MIH_FEASIBLE[config_id] and ms > 0:
        t0 = time.time()
        h = R.build_parallel(db_words, bits, cfg["m"])
        out["index_build_s"] = time.time() - t0
        if held is not None:  # the index holds its own copy now
            del db_words
            held = None
        scan_owner = h
        q = queries_host[:ms]
        best = None
        for s in range(warmup + steps):  # best of `steps` (tools/mih.cpp:308-314), warm-up untimed
            t = time.perf_counter()
            ids, dists, tr, secs = h.knn_timed(q, k, threads=threads)
            dt = time.perf_counter() - t
            if s >= warmup and (best is None or dt < best):
                best = dt
        ns = min(single_sample or 32, ms)
        _, _, _, secs1 = h.knn_timed(queries_host[:ns], k, threads=1)
        out["mih"] = {"qps": ms / best, "threads": threads, "queries": ms, "wall_s": best,
                      "per_query_under_load": _stats(secs), "single_thread": _stats(secs1),
                      "ids": ids, "dists": dists, "traces": tr}
        if log:
            log(f"reference MIH: {ms} queries, {ms / best:.1f} q/s on {threads} threads")
    if ss > 0:
        q = queries_host[:ss]
        t = time.perf_counter()
        ids, dists, secs = scan_owner.scan_knn_timed(q, k, threads=threads)
        dt = time.perf_counter() - t
        ns = min(4, ss)
        _, _, secs1 = scan_owner.scan_knn_timed(queries_host[:ns], k, threads=1)
        out["scan"] = {"qps": ss / dt, "threads": threads, "queries": ss, "wall_s": dt,
                       "per_query_under_load": _stats(secs), "single_thread": _stats(secs1),
                       "ids": ids, "dists": dists}
        if log:
            log(f"reference scan_knn: {ss} queries, {ss / dt:.2f} q/s on {threads} threads")
    return out


def reference_baseline_json(leg, config_id):
    """The cpu_baseline object (value = the reference MIH's all-thread q/s, or its scan where the
    reference MIH cannot run)."""
    mih, scan = leg.get("mih"), leg.get("scan")
    strip = lambda d: None if d is None else {k: v for k, v in d.items() if k not in ("ids", "dists", "traces")}
    head = mih or scan
    what = "MihIndex::knn_search" if mih else "scan_knn (reference MIH index does not fit host memory)"
    sample = (f"{head['queries']} queries (first rows of the batch), {what}, {head['threads']} threads, "
              f"best of steps; full-size reference index/database; "
              f"index build {leg.get('index_build_s', 0):.0f}s and data gen {leg.get('gen_s', 0):.0f}s excluded")
    return {"value": head["qps"], "unit": "queries/s", "cores": leg["cores"], "kind": "reference",
            "sample": sample, "cpu_model": leg["cpu_model"], "mih": strip(mih), "scan": strip(scan)}


def parity_check(leg, gpu_ids, gpu_dists, gpu_traces=None):
    """Compare GPU rows with the reference's answers for the same queries (ids and distances
    exactly; traces where both exist). Returns the parity object of the JSON line."""
    res = {"vs": [], "queries": 0, "mismatches": 0}
    def cmp(name, ids, dists, tr=None):
        n = ids.shape[0]
        gi = np.asarray(gpu_ids[:n]).view(np.uint32).reshape(n, -1)
        gd = np.asarray(gpu_dists[:n]).view(np.uint32).reshape(n, -1)
        bad = int((~((gi == ids).all(1) & (gd == dists).all(1))).sum())
        res["vs"].append(f"oracle/_ref {name}")
        res["queries"] = max(res["queries"], n)
        res["mismatches"] += bad
        res[name] = {"queries": n, "mismatches": bad}
        if tr is not None and gpu_traces is not None:
            gt = np.asarray(gpu_traces[:n])
            tb = int((~(gt[:, [0, 1, 2, 4]] == tr[:, [0, 1, 2, 4]]).all(1)).sum())
            res[name]["trace_mismatches"] = tb
            res["mismatches"] += tb
    if leg.get("mih"):
        m = leg["mih"]
        cmp("MihIndex::knn_search", m["ids"], m["dists"], m["traces"])
    if leg.get("scan"):
        cmp("scan_knn", leg["scan"]["ids"], leg["scan"]["dists"])
    return res


def run_reference_arm(args):
    cfg = workload(args)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    import oracle

    if not oracle.have_ref():
        emit({"impl": "reference", "unavailable": "oracle/_ref/libmihref.so not built"})
        return
    t0 = time.time()
    db = None if cfg["data"] == "uniform" else make_codes_host_cpu(cfg, 0, cfg["n"], cfg["db_seed"])
    queries = make_codes_host_cpu(cfg, 0, cfg["nq"], cfg["q_seed"])
    gen_s = time.time() - t0
    leg = reference_leg(cfg, args.config, queries, db, mih_sample=args.cpu_sample or None,
                        steps=args.steps, warmup=args.warmup)
    cpu = reference_baseline_json(leg, args.config)
    head = leg.get("mih") or leg.get("scan")
    line = {
        "metric": "exact kNN queries/s", "value": cpu["value"], "unit": "queries/s", "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * head["wall_s"], "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": config_desc(cfg, args, 1),
        "cpu_baseline": cpu,
        "e2e": {"value": cpu["value"], "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "setup": {"gen_s": gen_s + leg.get("gen_s", 0), "index_build_s": leg.get("index_build_s")},
    }
    emit(line)


# ---------------------------------------------------------------------------------------------
def main():
    args = parse()
    claim_stdout()
    if args.impl == "reference":
        run_reference_arm(args)
        return
    import torch

    from paper_1307_2982_b200 import _lib
    import paper_1307_2982_b200 as mg

    cfg = workload(args)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    use_dist = world > 1 or "TORCHELASTIC_RUN_ID" in os.environ  # torchrun: exchange path even at N=1
    if use_dist:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    L = _lib.lib()
    bits, m, k, nq, W = cfg["bits"], cfg["m"], cfg["k"], cfg["nq"], wpc(cfg["bits"])
    probe_part = world > 1 and args.shard == "probe" and args.method == "mih"
    lo, hi = (0, cfg["n"]) if probe_part else shard_range(cfg["n"], rank, world)

    # ---- data + index (setup, untimed) ----
    t0 = time.time()
    codes = make_codes_device(cfg, lo, hi, cfg["db_seed"], torch, dev, L)
    queries = make_codes_device(cfg, 0, nq, cfg["q_seed"], torch, dev, L)
    if os.environ.get("MIHG_BENCH_SORTQ") == "1":  # experiment: batch order by code value
        qn = queries.cpu().numpy().view(np.uint64)
        order = np.lexsort(qn.T[::-1])
        queries = torch.from_numpy(np.ascontiguousarray(qn[order]).view(np.int64)).to(dev)
    gen_s = time.time() - t0
    t0 = time.time()
    idx = mg.MihIndex.build_from_device(codes.data_ptr(), hi - lo, bits, mg.consecutive_partition(bits, m),
                                        local_rank, id_base=lo)
    torch.cuda.synchronize(dev)
    build_s = time.time() - t0
    del codes  # the index holds its own copy
    torch.cuda.empty_cache()

    kk = min(k, hi - lo)  # shard-local k (exact: global top-k is inside the union of local top-k)
    ids = torch.empty((nq, kk), dtype=torch.int32, device=dev)
    dists = torch.empty((nq, kk), dtype=torch.int32, device=dev)
    if use_dist:
        all_ids = torch.empty((world, nq, kk), dtype=torch.int32, device=dev)
        all_d = torch.empty((world, nq, kk), dtype=torch.int32, device=dev)
        out_ids = torch.empty((nq, k), dtype=torch.int32, device=dev)
        out_d = torch.empty((nq, k), dtype=torch.int32, device=dev)
    # a dedicated (non-default) stream: the library's stream-ordered workspace allocations are then
    # reused within the stream instead of going through the legacy default stream
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)

    # N > 1, MIH: one library call per rank and step (mihg_knn_sharded_device): the per-round NCCL
    # histogram all-reduce, the NCCL all-gather of the local top-k lists and the exact device merge
    # all run inside libmihg on its own NCCL communicator (no host language in the round loop)
    comm = None
    layout = 0 if probe_part else 1
    if use_dist and args.method == "mih":
        from paper_1307_2982_b200.shard import NcclComm

        comm = NcclComm(local_rank)

    def sharded(qptr, nqq, out_i, out_dd, trp=None):
        _lib.check(L.mihg_knn_sharded_device(idx._h, comm.handle, layout, cfg["n"], C.c_void_p(qptr), nqq, k,
                                             C.c_void_p(out_i.data_ptr()), C.c_void_p(out_dd.data_ptr()),
                                             C.c_void_p(trp) if trp else None, C.c_void_p(stream.cuda_stream)))

    def step(qptr=None):
        qptr = qptr or queries.data_ptr()
        if comm is not None:
            sharded(qptr, nq, out_ids, out_d)
            return
        if args.method == "scan":
            idx.scan_knn_device(qptr, nq, kk, ids.data_ptr(), dists.data_ptr(), stream=stream.cuda_stream)
        else:
            idx.knn_search_device(qptr, nq, kk, ids.data_ptr(), dists.data_ptr(), stream=stream.cuda_stream)
        if use_dist:
            dist.all_gather_into_tensor(all_ids, ids)
            dist.all_gather_into_tensor(all_d, dists)
            _lib.check(L.mihg_merge_topk_device(C.c_void_p(all_ids.data_ptr()), C.c_void_p(all_d.data_ptr()),
                                                world, nq, kk, k, C.c_void_p(out_ids.data_ptr()),
                                                C.c_void_p(out_d.data_ptr()), C.c_void_p(stream.cuda_stream)))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)

    # ---- timed region: device-resident inputs ----
    prof0 = _lib.Profile()
    L.mihg_profile_reset()
    L.mihg_profile_enable(1)
    L.mihg_profile_read(C.byref(prof0))
    clocks = ClockSampler(local_rank)
    clocks.start()
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    clk = clocks.stop()
    prof1 = _lib.Profile()
    L.mihg_profile_read(C.byref(prof1))
    L.mihg_profile_enable(0)
    ms = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    value = nq * args.steps / (ms / 1000.0)
    launches = int(prof1.kernel_launches - prof0.kernel_launches)
    probe_ms = prof1.probe_ms / args.steps
    probe_launches = prof1.probe_launches / args.steps

    # the timed path's own answer (last timed step), kept for the gates below
    if use_dist:
        res_ids, res_d = out_ids.clone(), out_d.clone()
    else:
        res_ids, res_d = ids.clone(), dists.clone()

    # ---- verify before reporting (tools/mih.cpp:274-301 pattern): the timed step's rows == the
    # exhaustive scan (K7/K6) of the same queries; N > 1: every rank scans its own id range (or,
    # probe partition, the full index) and the merged scans must equal the merged timed output ----
    nv = min(nq, 64)
    si = torch.empty((nv, kk if not probe_part else k), dtype=torch.int32, device=dev)
    sd = torch.empty_like(si)
    if probe_part:  # replicated index: one full scan is the answer
        idx.scan_knn_device(queries.data_ptr(), nv, k, si.data_ptr(), sd.data_ptr(), stream=stream.cuda_stream)
        torch.cuda.synchronize(dev)
        verified = bool(torch.equal(res_ids[:nv], si) and torch.equal(res_d[:nv], sd))
    elif use_dist:  # id-range shards: merge of the per-shard scans
        idx.scan_knn_device(queries.data_ptr(), nv, kk, si.data_ptr(), sd.data_ptr(), stream=stream.cuda_stream)
        gi = torch.empty((world, nv, kk), dtype=torch.int32, device=dev)
        gd = torch.empty_like(gi)
        dist.all_gather_into_tensor(gi, si)
        dist.all_gather_into_tensor(gd, sd)
        mi = torch.empty((nv, k), dtype=torch.int32, device=dev)
        md = torch.empty_like(mi)
        _lib.check(L.mihg_merge_topk_device(C.c_void_p(gi.data_ptr()), C.c_void_p(gd.data_ptr()), world, nv, kk, k,
                                            C.c_void_p(mi.data_ptr()), C.c_void_p(md.data_ptr()),
                                            C.c_void_p(stream.cuda_stream)))
        torch.cuda.synchronize(dev)
        verified = bool(torch.equal(res_ids[:nv], mi) and torch.equal(res_d[:nv], md))
    else:
        idx.scan_knn_device(queries.data_ptr(), nv, kk, si.data_ptr(), sd.data_ptr(), stream=stream.cuda_stream)
        torch.cuda.synchronize(dev)
        verified = bool(torch.equal(res_ids[:nv], si) and torch.equal(res_d[:nv], sd))
    if use_dist:  # every rank checks; all must pass
        vt = torch.tensor([1 if verified else 0], device=dev)
        dist.all_reduce(vt, op=dist.ReduceOp.MIN)
        verified = bool(vt.item())
    if not verified:
        emit({"error": "verification failed: the timed kNN result differs from the exhaustive scan"})
        sys.exit(3)

    # ---- algorithmic bytes from the reference-identical traces (untimed run) ----
    # (traced calls run pure MIH; at 256 bits that is ~50 q/s, so a 256-query sample is traced and
    # scaled: its numbers only feed the HBM roofline, which the hybrid's tensor-core line replaces)
    nq_tr = nq if bits <= 128 else min(nq, 256)
    tr = torch.empty((nq_tr, 5), dtype=torch.int64, device=dev)
    if comm is not None:  # global traces (candidates / unique summed over ranks)
        sharded(queries.data_ptr(), nq_tr, torch.empty_like(out_ids), torch.empty_like(out_d), tr.data_ptr())
    else:
        idx.knn_search_device(queries.data_ptr(), nq_tr, kk, ids.data_ptr(), dists.data_ptr(), tr.data_ptr(),
                              stream=stream.cuda_stream)
    torch.cuda.synchronize(dev)
    t = tr.cpu().numpy()
    lookups, cands, uniq, radius = (t[:, 0].astype(np.float64), t[:, 1].astype(np.float64),
                                    t[:, 2].astype(np.float64), t[:, 4].astype(np.float64))
    alg_bytes = float((8 * lookups + 4 * cands + (bits / 8) * uniq).sum()) * nq / nq_tr
    popc64 = float(uniq.sum() * W) * nq / nq_tr

    # ---- e2e through the host-pointer C ABI ----
    hq = torch.from_numpy(np.ascontiguousarray(queries.cpu().numpy())).pin_memory()
    hid = torch.empty((nq, k), dtype=torch.int32).pin_memory()
    hd = torch.empty((nq, k), dtype=torch.int32).pin_memory()
    if not use_dist:
        def e2e_step():
            qp = C.cast(C.c_void_p(hq.data_ptr()), _lib.u64p)
            ip = C.cast(C.c_void_p(hid.data_ptr()), _lib.u32p)
            dp = C.cast(C.c_void_p(hd.data_ptr()), _lib.u32p)
            if args.method == "scan":
                _lib.check(L.mihg_scan_knn_batch(idx._h, qp, nq, k, ip, dp))
            else:
                _lib.check(L.mihg_knn_batch(idx._h, qp, nq, k, ip, dp, None))
    else:
        dq = torch.empty_like(queries)

        def e2e_step():
            dq.copy_(hq, non_blocking=True)
            step(dq.data_ptr())
            hid.copy_(out_ids, non_blocking=True)
            hd.copy_(out_d, non_blocking=True)
            torch.cuda.synchronize(dev)

    for _ in range(max(args.warmup, 3)):
        e2e_step()
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0.record(stream)
    for _ in range(args.steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    e2e_ms = e0.elapsed_time(e1)
    if dist:
        tt = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    e2e_value = nq * args.steps / (e2e_ms / 1000.0)

    # ---- roofline ----
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    # DRAM traffic of the probe kernels per step, from a committed ncu capture of the same
    # config (tools/ncu_traffic.sh; traffic is a profiler measurement, never taken live)
    traffic = None
    tp = next((t for t in (os.path.join(ROOT, "profiles", r, f"traffic_c{args.config}.json") for r in ("r02", "r01"))
               if os.path.exists(t)), "")
    if (os.path.exists(tp) and world == 1 and cfg["n"] == CONFIGS[args.config]["n"]
            and cfg["nq"] == CONFIGS[args.config]["nq"] and cfg["k"] == CONFIGS[args.config]["k"]):
        tj = json.load(open(tp))
        traffic = {"dram_bytes_per_step": tj["dram_bytes_per_step"], "over_alg_bytes": tj["traffic_over_alg"],
                   "source": os.path.relpath(tp, ROOT)}
    # per GPU: a probe-partitioned rank moves 1/N of the step's algorithmic bytes
    achieved = alg_bytes / (world if probe_part else 1) / (probe_ms / 1000.0) / 1e9 if probe_ms > 0 else 0.0
    switched = (prof1.switched_queries - prof0.switched_queries) / args.steps
    scan_ms_step = (prof1.scan_ms - prof0.scan_ms) / args.steps
    scanned_q = nq if args.method == "scan" else switched
    if (args.method == "scan" or switched >= 0.5 * nq) and L.mihg_scan_kernel_for(bits) == 1:
        # K7 (tcgen05 kind::i8): one useful MAC per code bit per (query, code) pair; the peak is the
        # dense int8 rate = 2x the measured cuBLAS bf16 burst (MEASURED_PEAKS.json), else 2x fallback
        bf16 = float(peaks.get("bf16_tflops", 0) or 0)
        i8_peak = 2.0 * (bf16 if bf16 > 0 else 1590.0)
        t_s = (scan_ms_step if scan_ms_step > 0 else ms_per_step) / 1000.0
        ops = 2.0 * scanned_q * (hi - lo) * bits
        roofline = {"bound": "tensor", "achieved": ops / t_s / 1e12, "peak": i8_peak, "unit": "TOPS",
                    "frac": ops / t_s / 1e12 / i8_peak, "traffic": None, "kernel": "tc_scan_kernel",
                    "peak_source": ("2x MEASURED_PEAKS.json bf16_tflops (dense int8 = 2x bf16)" if bf16 > 0
                                    else "2x fallback 1590 TF/s bf16"),
                    "scan_kernel_ms_per_step": scan_ms_step,
                    "scanned_queries_per_step": scanned_q,
                    "note": ("exhaustive K7 path" if args.method == "scan" else
                             "hybrid: %d of %d queries per step finished by the tensor-core scan" % (switched, nq))}
    elif args.method == "scan" or switched >= 0.5 * nq:
        # K6 is POPC-bound: n*W popc64 = 2*n*W POPC32 per query; peak = 16 POPC/clk/SM measured
        # 4.56e12/s at 1.925 GHz (tools/probe/ubench.cu), scaled to the sampled SM clock.
        pc_peak = 4.56e12 * ((clk.get("sm_mhz") or 1925.0) / 1925.0)
        pc_ach = 2.0 * (hi - lo) * W * nq / (ms_per_step / 1000.0)
        roofline = {"bound": "popc", "achieved": pc_ach / 1e12, "peak": pc_peak / 1e12, "unit": "TPOPC32/s",
                    "frac": pc_ach / pc_peak, "traffic": None, "kernel": "scan_kernel",
                    "peak_source": "tools/probe/ubench.cu POPC microbenchmark (16/clk/SM)",
                    "note": ("hybrid: %d of %d queries per step finished by the exhaustive scan; frac "
                             "counts the scan's popcounts over the whole step" % (switched, nq))
                    if args.method != "scan" else "exhaustive K6 path"}
    else:
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak if peak else None, "traffic": traffic,
                    "kernel": "mih_probe_kernel", "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6650",
                    "alg_bytes_per_step": alg_bytes, "probe_ms_per_step": probe_ms,
                    "probe_launches_per_step": probe_launches,
                "hybrid_scan_queries_per_step": (prof1.switched_queries - prof0.switched_queries) / args.steps,
                    "rerun_queries_per_step": (prof1.rerun_queries - prof0.rerun_queries) / args.steps,
                    "rerun_ms_per_step": (prof1.rerun_ms - prof0.rerun_ms) / args.steps,
                    "step_frac_of_roofline": (alg_bytes / (ms_per_step / 1000.0) / 1e9) / peak,
                    "popc64_per_step": popc64,
                    "mean_trace": {"lookups": float(lookups.mean()), "candidates": float(cands.mean()),
                                   "unique": float(uniq.mean()), "final_radius": float(radius.mean())}}

        # Sparse (32-bit substring) tables: the probe kernel is bound by the GPU's random-access
        # rate, not by streaming bandwidth. Measure that rate here for one
        # lookup's access pattern — a directory group in a 128 MB key slice, then for 29% of the
        # lookups (tools/probe_stats_c4.py) a candidate code in the slice's share of the
        # table-order codes — and report the kernel's own lookup rate beside it.
        s_bits = bits // cfg["m"]
        if rank == 0 and probe_ms > 0 and s_bits >= 27 and (1 << s_bits) > max(1 << 24, 2 * (hi - lo)):
            dir_total = (1 << (s_bits - 5)) * 16
            dir_slice = min(dir_total, 128 << 20)
            code_bytes = (hi - lo) * (4 if (W == 1 and cfg["m"] == 2) else 8 * W)
            codes_slice = max(1 << 20, int(code_bytes * dir_slice / dir_total))
            rate = C.c_double(0.0)
            _lib.check(L.mihg_calibrate_random_lookups(dev.index or 0, dir_slice, codes_slice, 29, C.byref(rate)))
            ach = float(lookups.sum()) * nq / nq_tr / (world if probe_part else 1) / (probe_ms / 1000.0)
            roofline["random_access"] = {
                "achieved_lookups_per_s": ach, "device_lookups_per_s": rate.value,
                "frac": ach / rate.value if rate.value else None,
                "model": "mihg_calibrate_random_lookups: 16 B at a random place of a %d MB directory slice, then "
                         "for 29%% of the lookups 4 B at a random place of %d MB of table-order codes; 4 lookups "
                         "in flight per lane, 6 x 256 threads per SM" % (dir_slice >> 20, codes_slice >> 20)}

    # ---- CPU baseline + parity against the reference itself (rank 0, N = 1 only) ----
    cpu, parity = None, None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle

        if oracle.have_ref():
            qh = queries.cpu().numpy().view(np.uint64)
            if cfg["data"] == "uniform":
                db_host = None  # the reference generates it (gen_uniform, io.hpp:266-277)
            else:
                db_host = make_codes_device(cfg, 0, cfg["n"], cfg["db_seed"], torch, dev, L).cpu().numpy().view(np.uint64)
                torch.cuda.empty_cache()
            leg = reference_leg(cfg, args.config, qh, db_host, mih_sample=args.cpu_sample or None,
                                log=lambda msg: print(msg, file=sys.stderr))
            del db_host
            cpu = reference_baseline_json(leg, args.config)
            parity = parity_check(leg, res_ids.cpu().numpy(), res_d.cpu().numpy(), t)
            if parity["mismatches"]:
                emit({"error": "parity failed: GPU rows differ from the reference", "parity": parity})
                sys.exit(3)
        else:
            cpu = {"value": None, "unavailable": "oracle/_ref not built"}

    # ---- N > 1 (torchrun): the OTHER multi-GPU layout beside the headline one, same workload,
    # same timing rules, checked against the headline layout's answer (both are exact) ----
    index_bytes = idx.device_bytes()
    other_layout = None
    if comm is not None and not args.single_layout:
        pp2 = not probe_part
        idx.close()
        torch.cuda.empty_cache()
        lo2, hi2 = (0, cfg["n"]) if pp2 else shard_range(cfg["n"], rank, world)
        codes2 = make_codes_device(cfg, lo2, hi2, cfg["db_seed"], torch, dev, L)
        idx = mg.MihIndex.build_from_device(codes2.data_ptr(), hi2 - lo2, bits, mg.consecutive_partition(bits, m),
                                            local_rank, id_base=lo2)
        del codes2
        torch.cuda.empty_cache()
        o_ids, o_d = torch.empty_like(out_ids), torch.empty_like(out_d)

        def step2():
            _lib.check(L.mihg_knn_sharded_device(idx._h, comm.handle, 0 if pp2 else 1, cfg["n"],
                                                 C.c_void_p(queries.data_ptr()), nq, k, C.c_void_p(o_ids.data_ptr()),
                                                 C.c_void_p(o_d.data_ptr()), None, C.c_void_p(stream.cuda_stream)))

        for _ in range(max(args.warmup, 3)):
            step2()
        dist.barrier()
        torch.cuda.synchronize(dev)
        e0.record(stream)
        for _ in range(args.steps):
            step2()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        tt = torch.tensor([e0.elapsed_time(e1)], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms2 = float(tt.item())
        same = torch.tensor([1 if (torch.equal(o_ids, res_ids) and torch.equal(o_d, res_d)) else 0], device=dev)
        dist.all_reduce(same, op=dist.ReduceOp.MIN)
        other_layout = {"parallelism": ("probe-space partition x%d (replicated index)" if pp2
                                        else "id-range shards x%d (north_star layout)") % world,
                        "value": nq * args.steps / (ms2 / 1000.0), "unit": "queries/s",
                        "ms_per_step": ms2 / args.steps, "same_answer_as_headline_layout": bool(same.item())}

    if rank == 0:
        line = {
            "metric": "exact kNN queries/s", "value": value, "unit": "queries/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic", "config": config_desc(cfg, args, world),
            "e2e": {"value": e2e_value, "unit": "queries/s", "h2d_bytes_per_step": int(nq * W * 8),
                    "d2h_bytes_per_step": int(nq * k * 8)},
            "gpu_launches": launches, "verified_vs_scan": verified, "parity": parity, "roofline": roofline,
            "cpu_baseline": cpu, "clocks": clk, "other_layout": other_layout,
            "setup": {"gen_s": gen_s, "index_build_s": build_s, "index_device_bytes": index_bytes},
        }
        emit(line)
    idx.close()
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
