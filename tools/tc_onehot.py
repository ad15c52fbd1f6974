"""K7 layout probe: one-hot queries x one-hot codes (64-bit). With the +-1 query encoding the
distance matrix is 2 - 2*[i == j]; any other pattern shows which query element the MMA pairs with
which code element."""
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
eye = np.zeros((bits, W), np.uint64)
for i in range(bits):
    eye[i, i // 64] = np.uint64(1) << np.uint64(i % 64)
d = torch.from_numpy(eye.view(np.int64)).cuda()
out = torch.full((bits, bits), -7, dtype=torch.int32, device="cuda")
rc = L.mihg_tc_distances_device(C.c_void_p(d.data_ptr()), bits, bits, C.c_void_p(d.data_ptr()), bits,
                                C.c_void_p(out.data_ptr()), None)
torch.cuda.synchronize()
g = out.cpu().numpy()
print("rc", rc, "exact:", np.array_equal(g, 2 - 2 * np.eye(bits, dtype=np.int64)))
v = g - 1  # = dot = px - 2*pairs = 1 - 2*[paired]
pairs = np.argwhere(v < 0)
print("paired (query bit -> code bit):", [tuple(x) for x in pairs[:80]])
print("value histogram:", dict(zip(*np.unique(g, return_counts=True))))
np.save("gpurun_out/onehot_%d.npy" % bits, g)
