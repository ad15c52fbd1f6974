"""K7 precision probe: query 0 (all +1) and query all-ones (all -1) against codes with the first j
bits set (j = 0..bits): the dot products are +j and -j exactly."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1307_2982_b200 import _lib  # noqa: E402

L = _lib.lib()
bits = int(sys.argv[1]) if len(sys.argv) > 1 else 64
W = bits // 64
codes = np.zeros((bits + 1, W), np.uint64)
for j in range(bits + 1):
    for i in range(j):
        codes[j, i // 64] |= np.uint64(1) << np.uint64(i % 64)
qs = np.zeros((3, W), np.uint64)
qs[1, :] = np.uint64(0xFFFFFFFFFFFFFFFF)
qs[2, :] = np.uint64(0x5555555555555555)
d = torch.from_numpy(codes.view(np.int64)).cuda()
q = torch.from_numpy(qs.view(np.int64)).cuda()
out = torch.full((3, bits + 1), -7, dtype=torch.int32, device="cuda")
L.mihg_tc_distances_device(C.c_void_p(d.data_ptr()), bits + 1, bits, C.c_void_p(q.data_ptr()), 3,
                           C.c_void_p(out.data_ptr()), None)
torch.cuda.synchronize()
g = out.cpu().numpy()
pq = np.array([0, bits, bits // 2])
j = np.arange(bits + 1)
want = np.array([j, bits - j, [abs(((np.arange(bits) % 2 == 0) & (np.arange(bits) < jj)).sum() - 0) for jj in j]])
print("dot q0 (want +j):", (g[0] - pq[0]).tolist())
print("dot q1 (want -j):", (g[1] - pq[1]).tolist())
