"""Time estimate_correlations' GPU Gram path (device-resident codes) and, for scale, the
reference's CPU implementation (oracle/_ref) on a bounded sample. Prints one JSON line per shape."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_2982_b200 as mg  # noqa: E402
from paper_1307_2982_b200 import _lib  # noqa: E402


def main():
    for n, bits in ((100_000_000, 64), (20_000_000, 256), (1_000_000, 1024)):
        W = (bits + 63) // 64
        d = torch.empty(n * W, dtype=torch.int64, device="cuda")
        _lib.check(_lib.lib().mihg_gen_mixture_device(0, n, bits, 128, 64, 1, 2, d.data_ptr(), None)) if bits <= 256 else \
            d.random_()
        torch.cuda.synchronize()
        mg.estimate_correlations((d.data_ptr(), n, bits), codes_on_device=True)  # warm-up
        reps = 3
        t0 = time.perf_counter()
        for _ in range(reps):
            mg.estimate_correlations((d.data_ptr(), n, bits), codes_on_device=True)
        dt = (time.perf_counter() - t0) / reps
        wp = (bits + 63) // 64 * 64
        popc = (wp // 64) * ((wp // 64) + 1) // 2 * 64 * 64 * (n / 32)  # u32 AND-popcounts issued
        line = {"shape": f"n={n} bits={bits}", "gpu_s": dt, "codes_GBps": n * W * 8 / dt / 1e9,
                "popc32_per_s": popc / dt}
        try:
            import oracle

            R = oracle.ref()
            ns = min(n, 200_000)
            codes = d[: ns * W].cpu().numpy().view(np.uint64).reshape(ns, W)
            t0 = time.perf_counter()
            R.estimate_correlations(codes, bits)
            line["ref_cpu_s_per_code"] = (time.perf_counter() - t0) / ns
            line["ref_cpu_sample"] = ns
            line["speedup_vs_ref_1thread"] = line["ref_cpu_s_per_code"] * n / dt
        except Exception as e:  # reference library absent
            line["ref_cpu"] = f"unavailable: {e}"
        print(json.dumps(line), flush=True)
        del d
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
