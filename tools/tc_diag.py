"""Diagnose the K7 distance matrix: which (query, code) entries differ and where their values come from."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1307_2982_b200 import _lib  # noqa: E402


def popc_dist(q, x):
    d = np.zeros((q.shape[0], x.shape[0]), np.int64)
    for w in range(q.shape[1]):
        v = np.bitwise_xor(q[:, w][:, None], x[:, w][None, :])
        d += np.unpackbits(v.view(np.uint8).reshape(v.shape + (8,)), axis=-1).sum(-1).astype(np.int64)
    return d


L = _lib.lib()
rng = np.random.default_rng(0)
for bits, n, nq in ((64, 3000, 200), (64, 5000, 128), (256, 3000, 128)):
    W = bits // 64
    db = rng.integers(0, 2**63, size=(n, W), dtype=np.int64).view(np.uint64)
    qs = rng.integers(0, 2**63, size=(nq, W), dtype=np.int64).view(np.uint64)
    want = popc_dist(qs, db)
    dd = torch.from_numpy(db.view(np.int64)).cuda()
    dq = torch.from_numpy(qs.view(np.int64)).cuda()
    out = torch.full((nq, n), -7, dtype=torch.int32, device="cuda")
    rc = L.mihg_tc_distances_device(C.c_void_p(dd.data_ptr()), n, bits, C.c_void_p(dq.data_ptr()), nq,
                                    C.c_void_p(out.data_ptr()), None)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    bad = got != want
    print(f"bits={bits} n={n} rc={rc} mismatches={bad.sum()} of {got.size}", flush=True)
    if bad.any():
        cols = np.where(bad.any(0))[0]
        rows = np.where(bad.any(1))[0]
        print(" bad columns:", len(cols), cols[:40], "tiles:", np.unique(cols // 128)[:40])
        print(" bad rows:", len(rows), rows[:20])
        c = cols[0]
        src = [c2 for c2 in range(n) if np.array_equal(got[:, c], want[:, c2])]
        print(f" column {c} equals want column(s) {src[:5]}; got==-7: {(got[:, c] == -7).sum()}")
