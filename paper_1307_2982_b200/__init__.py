"""paper_1307_2982_b200 — B200-native exact Hamming k-NN (multi-index hashing, arXiv 1307.2982).

Drop-in for the reference's hot path (mih::MihIndex::build + knn_search). The compute runs in
hand-written sm_100a kernels behind the C ABI of include/mihg.h (libmihg.so); this package is
the host-side mirror of the reference interface (names, argument meaning, error behaviour).
"""
from .codes import (BinaryCode, CodeDatabase, Partition, consecutive_partition, extract_substring,
                    hamming_distance, kMaxCodeBits, words_per_code)
from .index import (MihIndex, Neighbor, SearchTrace, TableStats, build_index, neighbor_less,
                    scan_knn)
from .io import FormatError, gen_uniform, read_codes, read_index, write_codes, write_index
from .optimize import CorrelationMatrix, estimate_correlations, greedy_assign

__all__ = [
    "BinaryCode", "CodeDatabase", "Partition", "consecutive_partition", "extract_substring",
    "hamming_distance", "kMaxCodeBits", "words_per_code", "MihIndex", "Neighbor", "SearchTrace",
    "TableStats", "build_index", "neighbor_less", "scan_knn", "FormatError", "gen_uniform",
    "read_codes", "write_codes", "read_index", "write_index", "CorrelationMatrix",
    "estimate_correlations", "greedy_assign",
]
