import sys; sys.path.insert(0, '/root/repo')
import numpy as np, paper_1307_2982_b200 as mg
db = mg.gen_uniform(2000, 64, 1); qs = mg.gen_uniform(5, 64, 2).raw_words()
idx = mg.MihIndex.build(db, mg.consecutive_partition(64, 4))
print(idx.scan_knn_batch(qs, 10)[1][0])
