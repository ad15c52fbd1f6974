"""GPU: the device-pointer entry points are ordered on the caller's stream (the library runs on the
index's own stream, joined to the caller's with events): work enqueued on the caller's stream
before the call is visible to it, and work enqueued after it sees its results — no host sync."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_knn_device_orders_with_caller_stream(cuda_ok, port):
    import torch

    import paper_1307_2982_b200 as mg

    db = mg.gen_uniform(60000, 64, 71)
    qs = mg.gen_uniform(500, 64, 72).raw_words()
    idx = mg.MihIndex.build(db, mg.consecutive_partition(64, 4), device=0)
    k = 10
    s = torch.cuda.Stream()
    host_q = torch.from_numpy(qs.view(np.int64)).pin_memory()
    with torch.cuda.stream(s):
        dq = torch.zeros((500, 1), dtype=torch.int64, device="cuda")
        torch.cuda._sleep(20_000_000)  # keep the stream busy: the copy below lands late
        dq.copy_(host_q, non_blocking=True)
        ids = torch.full((500, k), -1, dtype=torch.int32, device="cuda")
        dists = torch.full((500, k), -1, dtype=torch.int32, device="cuda")
        idx.knn_search_device(dq.data_ptr(), 500, k, ids.data_ptr(), dists.data_ptr(), stream=s.cuda_stream)
        got_i = ids.clone()  # enqueued after the call on the same stream
        got_d = dists.clone()
    s.synchronize()
    oi, od = port.scan_knn(db.raw_words(), 64, qs, k)
    assert np.array_equal(got_i.cpu().numpy().view(np.uint32), oi)
    assert np.array_equal(got_d.cpu().numpy().view(np.uint32), od)


def test_calibrate_random_lookups(cuda_ok):
    """The calibration entry point (bench.py's random-access reference) returns a positive rate and
    rejects bad arguments."""
    import ctypes as C

    from paper_1307_2982_b200 import _lib

    L = _lib.lib()
    rate = C.c_double(0.0)
    _lib.check(L.mihg_calibrate_random_lookups(0, 8 << 20, 16 << 20, 29, C.byref(rate)))
    assert rate.value > 1e8
    assert L.mihg_calibrate_random_lookups(0, 8, 16 << 20, 29, C.byref(rate)) != 0
    assert L.mihg_calibrate_random_lookups(0, 8 << 20, 16 << 20, 101, C.byref(rate)) != 0
