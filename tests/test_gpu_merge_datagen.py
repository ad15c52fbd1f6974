"""GPU: the exact k-way shard merge kernel (K9) and the mixture generator (configs 2/4)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_merge_topk_matches_numpy(cuda_ok):
    import torch

    from paper_1307_2982_b200.shard import gpu_merge
    from _helpers import numpy_merge

    rng = np.random.default_rng(3)
    for G, nq, k_in, k in ((2, 50, 10, 10), (8, 300, 100, 100), (4, 7, 5, 17), (3, 20, 64, 1)):
        d = np.sort(rng.integers(0, 40, size=(G, nq, k_in)), axis=2).astype(np.uint32)
        ids = np.zeros((G, nq, k_in), np.uint32)
        for g in range(G):  # disjoint id ranges per shard, ascending within equal distances
            ids[g] = g * 1000 + rng.permutation(1000)[:k_in][None, :]
            for q in range(nq):
                order = np.lexsort((ids[g, q], d[g, q]))
                ids[g, q], d[g, q] = ids[g, q][order], d[g, q][order]
        d[0, :, -1] = 0xFFFFFFFF  # padding from a short shard
        ti = torch.from_numpy(ids.view(np.int32)).cuda()
        td = torch.from_numpy(d.view(np.int32)).cuda()
        kk = min(k, G * k_in)
        gi, gd = gpu_merge(ti, td, kk)
        wi, wd = numpy_merge(torch.from_numpy(ids.view(np.int32)), torch.from_numpy(d.view(np.int32)), kk)
        assert np.array_equal(gi.cpu().numpy(), wi.numpy()) and np.array_equal(gd.cpu().numpy(), wd.numpy())


def test_gpu_mixture_generator_matches_c_restatement(cuda_ok, port):
    import torch

    from paper_1307_2982_b200 import _lib

    L = _lib.lib()
    for bits, first, n in ((64, 0, 50000), (128, 123456789, 20000), (256, 7, 3000), (70, 5, 1000)):
        W = (bits + 63) // 64
        out = torch.empty((n, W), dtype=torch.int64, device="cuda")
        _lib.check(L.mihg_gen_mixture_device(first, n, bits, 128, 64, 0x4C0FFEE, 0x4D0001,
                                             C.c_void_p(out.data_ptr()), None))
        torch.cuda.synchronize()
        want = port.gen_mixture(first, n, bits, 128, 64, 0x4C0FFEE, 0x4D0001)
        assert np.array_equal(out.cpu().numpy().view(np.uint64), want), bits
