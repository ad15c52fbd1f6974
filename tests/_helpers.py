"""Shared test helpers (numpy restatements used as checkers)."""
import numpy as np
import torch


def numpy_merge(all_ids, all_d, k):
    """Smallest k packed keys (dist << 32 | id) per query; padding dist 0xFFFFFFFF sorts last."""
    ids = all_ids.numpy().view(np.uint32).astype(np.uint64)
    d = all_d.numpy().view(np.uint32).astype(np.uint64)
    keys = (d << np.uint64(32)) | ids  # [G, nq, k]
    keys = np.sort(np.concatenate(list(keys), axis=1), axis=1)[:, :k]
    out_d = (keys >> np.uint64(32)).astype(np.uint32)
    out_i = (keys & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    return torch.from_numpy(out_i.view(np.int32)), torch.from_numpy(out_d.view(np.int32))
