import sys, torch
sys.path.insert(0, "/root/repo")
import bench, paper_1307_2982_b200 as mg
from paper_1307_2982_b200 import _lib
import ctypes as C
cfg = dict(bench.CONFIGS[4]); dev = torch.device("cuda", 0); L = _lib.lib()
codes = bench.make_codes_device(cfg, 0, cfg["n"], cfg["db_seed"], torch, dev, L)
idx = mg.MihIndex.build_from_device(codes.data_ptr(), cfg["n"], cfg["bits"], mg.consecutive_partition(64, 2), 0)
for j in range(2):
    info = _lib.TableInfo(); _lib.check(L.mihg_table_get_info(idx._h, j, C.byref(info)))
    print(j, "s", info.s, "dense", info.dense, "nonempty", info.non_empty_buckets, "maxb", info.max_bucket_size,
          "escaped_blocks", info.escaped_blocks, "of", 2**(info.s-6), "frac", info.escaped_blocks / 2**(info.s-6),
          "dev GB", info.device_bytes/1e9)
