"""A/B of the exhaustive scan kernels on one GPU: K6 (POPC pipe) vs K7 (tcgen05 int8 tensor cores).

Random device-resident codes (torch.randint; timing only — parity lives in tests/test_gpu_tcscan.py),
CUDA events around mihg_scan_knn_raw_device, results compared between the kernels.
usage: python tools/bench_tcscan.py [n] [bits] [nq] [k] [kernels]
"""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1307_2982_b200 import _lib  # noqa: E402


def main():
    n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
    bits = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    nq = int(sys.argv[3]) if len(sys.argv) > 3 else 10000
    k = int(sys.argv[4]) if len(sys.argv) > 4 else 100
    kernels = sys.argv[5].split(",") if len(sys.argv) > 5 else ["tc", "popc"]
    W = (bits + 63) // 64
    L = _lib.lib()
    g = torch.Generator(device="cuda").manual_seed(1)
    codes = torch.randint(-2**63, 2**63 - 1, (n, W), dtype=torch.int64, device="cuda", generator=g)
    qs = torch.randint(-2**63, 2**63 - 1, (nq, W), dtype=torch.int64, device="cuda", generator=g)
    if bits % 64:
        mask = (1 << (bits % 64)) - 1
        codes[:, -1] &= mask
        qs[:, -1] &= mask
    res = {}
    for kern in kernels:
        os.environ["MIHG_SCAN_KERNEL"] = kern
        ids = torch.empty((nq, k), dtype=torch.int32, device="cuda")
        d = torch.empty((nq, k), dtype=torch.int32, device="cuda")

        def run():
            _lib.check(L.mihg_scan_knn_raw_device(C.c_void_p(codes.data_ptr()), n, bits, 0,
                                                  C.c_void_p(qs.data_ptr()), nq, k, C.c_void_p(ids.data_ptr()),
                                                  C.c_void_p(d.data_ptr()), None))

        run()
        torch.cuda.synchronize()
        prof0 = _lib.Profile()
        L.mihg_profile_reset()
        L.mihg_profile_enable(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 3
        e0.record()
        for _ in range(reps):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        prof = _lib.Profile()
        L.mihg_profile_read(C.byref(prof))
        L.mihg_profile_enable(0)
        scan_ms = prof.scan_ms / reps
        pairs = n * nq
        res[kern] = {"ms": ms, "scan_kernel_ms": scan_ms, "qps": nq / (ms / 1e3), "pairs_per_s": pairs / (ms / 1e3),
                     "int8_tops_useful": 2 * pairs * bits / (ms / 1e3) / 1e12}
        res[kern + "_out"] = (ids.cpu(), d.cpu())
    same = None
    if "tc" in kernels and "popc" in kernels:
        same = bool(torch.equal(res["tc_out"][0], res["popc_out"][0]) and torch.equal(res["tc_out"][1], res["popc_out"][1]))
    out = {"n": n, "bits": bits, "nq": nq, "k": k, "identical": same}
    out.update({kk: v for kk, v in res.items() if not kk.endswith("_out")})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
