/*
 * mihg — B200-native exact Hamming k-NN (multi-index hashing), C ABI.
 *
 * This is the drop-in boundary for the reference's hot path, the C++ interface in
 * /root/reference/proj/include/mih (no C ABI exists there). Every entry point is
 * extern "C", takes plain pointers and sizes, never throws, and returns a status code:
 *
 *   MIHG_OK       0
 *   MIHG_EINVAL   1  <-> std::invalid_argument in the reference (index.hpp:102-112, :187-188,
 *                       codes.hpp:152-176, table.hpp:273-277)
 *   MIHG_EINTERNAL 2
 *   MIHG_ENOMEM   3  <-> std::bad_alloc (table.hpp:59)
 *   MIHG_ECUDA    4  CUDA runtime / kernel failure
 *   MIHG_ENCCL    5  (reserved for the multi-GPU layer; the C++/Python hosts raise it)
 *   MIHG_EFORMAT  6  <-> FormatError (io.hpp:35-44), message carries the byte offset
 *   MIHG_EIO      7  file open / read / write failure
 *
 * mihg_last_error() returns a thread-local message for the last failing call on this thread.
 *
 * Code layout (codes.hpp:26-33, :54-120): n records of ceil(bits/64) little-endian u64 words,
 * bit i at word i/64 bit i%64, padding bits zero; a code's id is its row index.
 * Result layout: row-major [nq][k] ids and distances ordered by (distance asc, id asc), the
 * reference's neighbor_less (scan.hpp:24-26) and tie rule (scan.hpp:42, index.hpp:243).
 *
 * Threading: an index is immutable after build; calls on one index are serialised internally
 * (the device workspace is per index). Different indexes may be used concurrently.
 */
#ifndef MIHG_H
#define MIHG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MIHG_OK 0
#define MIHG_EINVAL 1
#define MIHG_EINTERNAL 2
#define MIHG_ENOMEM 3
#define MIHG_ECUDA 4
#define MIHG_ENCCL 5
#define MIHG_EFORMAT 6  /* <-> FormatError (io.hpp:35-44); message ends "(byte offset N)" */
#define MIHG_EIO 7      /* cannot open / read / write a file (std::runtime_error in io.hpp) */

#define MIHG_ABI_VERSION 1

typedef struct mihg_index mihg_index;

/* mih::SearchTrace (index.hpp:45-51). */
typedef struct mihg_trace {
  uint64_t lookups;              /* buckets probed */
  uint64_t candidates;           /* ids retrieved before duplicate suppression */
  uint64_t unique_candidates;    /* distinct ids retrieved */
  uint64_t distance_evaluations; /* always equals unique_candidates */
  uint32_t final_radius;         /* kNN: completed guarantee radius */
  uint32_t reserved;
} mihg_trace;

/* Extended build parameters (mihg_index_build covers the common case). */
typedef struct mihg_build_params {
  const uint64_t* codes;      /* n * ceil(bits/64) words (host, or device if codes_on_device) */
  uint64_t n;
  uint32_t bits;
  uint32_t m;                 /* number of substrings / tables */
  const uint32_t* lengths;    /* NULL: consecutive_partition(bits, m) (codes.hpp:198-211) */
  const uint32_t* positions;  /* concatenated bit positions of substring 0, 1, ... */
  int device;                 /* CUDA device ordinal */
  int codes_on_device;        /* 1: `codes` is a device pointer on `device` */
  uint32_t id_base;           /* global id of local id 0 (id-range shard); 0 for a whole DB */
  uint32_t dense_max_bits;    /* 0 = default (24): tables with 2^s <= max(2^this, 2n) are dense */
  int layout;                 /* 0 auto, 1 force dense offsets, 2 force sparse directory */
} mihg_build_params;

typedef struct mihg_index_info {
  uint64_t n;
  uint32_t bits;
  uint32_t m;
  uint32_t id_base;
  int device;
  uint64_t device_bytes;      /* codes + all tables */
} mihg_index_info;

/* mih::TableStats (table.hpp:33-47) plus the GPU layout. */
typedef struct mihg_table_info {
  uint32_t s;
  uint32_t dense;             /* 1: offsets[2^s+1]; 0: blocked-count directory */
  uint64_t non_empty_buckets;
  uint64_t max_bucket_size;
  uint64_t total_entries;
  uint64_t estimated_bytes;   /* the reference's accounting model, TableStats::estimate_bytes */
  uint64_t device_bytes;      /* this table's actual HBM footprint */
  uint64_t escaped_blocks;
} mihg_table_info;

const char* mihg_last_error(void);
int mihg_abi_version(void);
int mihg_device_count(int* count);

/* MihIndex::build(CodeDatabase db, Partition partition) — index.hpp:101-121 (and build_index,
 * index.hpp:287-289). Host codes; lengths/positions NULL -> consecutive_partition(bits, m). */
int mihg_index_build(const uint64_t* codes, uint64_t n, uint32_t bits, uint32_t m,
                     const uint32_t* lengths, const uint32_t* positions, int device,
                     mihg_index** out);
int mihg_index_build_ex(const mihg_build_params* params, mihg_index** out);
void mihg_index_free(mihg_index* idx);

/* MihIndex::num_tables / table(j).stats() — index.hpp:145-146, table.hpp:190-197. */
int mihg_index_get_info(const mihg_index* idx, mihg_index_info* out);
int mihg_table_get_info(const mihg_index* idx, uint32_t j, mihg_table_info* out);

/* SubstringTable::bucket_lookup — table.hpp:169-175: ids of bucket `value` of table j in
 * insertion (ascending id) order; writes min(count, cap) ids (global ids). */
int mihg_bucket_lookup(const mihg_index* idx, uint32_t j, uint64_t value, uint32_t* out_ids,
                       uint64_t cap, uint64_t* count);

/* write_index(idx, path) — io.hpp:335-358: the BMIX index file, byte-identical to the
 * reference's output for the same codes and partition. */
int mihg_index_write(mihg_index* idx, const char* path);
/* read_index(path) — io.hpp:360-425: parses and validates a BMIX file (reference checks and
 * messages, MIHG_EFORMAT with byte offset) and loads the file's tables onto `device` as given. */
int mihg_index_read(const char* path, int device, mihg_index** out);

/* Device pointer to the index's codes (n * ceil(bits/64) words). */
int mihg_index_codes(const mihg_index* idx, const uint64_t** d_codes);

/* MihIndex::knn_search(BinaryCode q, uint32_t k, SearchTrace*, SearchScratch*) — index.hpp:185-253,
 * batched over nq queries. k > n -> MIHG_EINVAL; k == 0 -> no output, zero traces.
 * Host pointers: queries nq*ceil(bits/64) words; out_ids/out_dists nq*k; traces nq or NULL. */
int mihg_knn_batch(mihg_index* idx, const uint64_t* queries, uint64_t nq, uint32_t k,
                   uint32_t* out_ids, uint32_t* out_dists, mihg_trace* traces);
/* Same, all pointers on the index's device, ordered on `stream` (cudaStream_t, NULL = legacy). */
int mihg_knn_batch_device(mihg_index* idx, const uint64_t* d_queries, uint64_t nq, uint32_t k,
                          uint32_t* d_ids, uint32_t* d_dists, mihg_trace* d_traces, void* stream);

/* MihIndex::range_search(BinaryCode q, uint32_t r, SearchTrace*, SearchScratch*) — index.hpp:149-176
 * (paper Alg. 2), batched, host pointers. Every (id, dist) with dist <= r per query in (dist, id)
 * order, query-major. out_offsets[nq+1] is always written (out_offsets[nq] = total); ids/dists
 * (capacity entries each) are written only when total <= capacity — otherwise call again with
 * larger buffers. r > bits -> MIHG_EINVAL. traces: nq or NULL (final_radius = 0 as the
 * reference's range_search leaves it). */
int mihg_range_batch(mihg_index* idx, const uint64_t* queries, uint64_t nq, uint32_t r,
                     uint64_t* out_offsets, uint32_t* out_ids, uint32_t* out_dists, uint64_t capacity,
                     mihg_trace* traces);

/* Probe-space partitioned kNN for multi-GPU (SURVEY.md §8e remedy (iii)): every rank holds the
 * same index; rank `rank` of `count` (power of two) probes only ring values whose top
 * log2(count) substring bits equal `rank`, so probe AND verification work divide by count.
 * `allreduce(user, dev_ptr, n, dtype, stream)` must sum n device elements (dtype 0: u32,
 * 1: u64) in place across ranks, ordered on `stream`, and return 0 (e.g. an NCCL all-reduce);
 * it is called once per radius round with the per-query histograms, so all ranks apply the
 * reference's stopping rule to the global counts. Outputs are the rank's LOCAL top-k (padded
 * with 0xFFFFFFFF): all-gather them and merge with mihg_merge_topk_device. Traces are global.
 *
 * id_shards = 1 selects the id-range layout instead (refinement 1 "global
 * stopping"): each rank's index holds only its own id range (built with id_base), every rank
 * probes every ring, and the same per-round histogram all-reduce makes all shards stop at the
 * GLOBAL d_k instead of their larger local d_k. count may be any value >= 1; the hybrid
 * scan switch is off (ranks' shard sizes may differ, the decision must be collective).
 * Traces: candidates/unique are summed over shards (= the single-index trace), lookups and
 * final_radius are every shard's own (= the single-index values). */
typedef int (*mihg_allreduce_fn)(void* user, void* dev_ptr, uint64_t count, int dtype, void* stream);
typedef struct mihg_comm mihg_comm;
typedef struct mihg_partition {
  uint32_t count;
  uint32_t rank;
  mihg_allreduce_fn allreduce;
  void* user;
  uint32_t id_shards; /* 0: probe-space partition of a replicated index; 1: id-range shards */
  uint32_t k_stop;    /* k of the GLOBAL stopping rule (id_shards: the caller's k, which may exceed
                         a small shard's local k); 0 -> the call's k. Must be equal on all ranks. */
  mihg_comm* comm;    /* non-NULL: the per-round all-reduce is an NCCL all-reduce on this library
                         communicator (allreduce/user ignored); count/rank must match it */
} mihg_partition;
int mihg_knn_batch_device_part(mihg_index* idx, const uint64_t* d_queries, uint64_t nq, uint32_t k,
                               uint32_t* d_ids, uint32_t* d_dists, mihg_trace* d_traces,
                               const mihg_partition* part, void* stream);

/* NCCL communicator owned by the library (SURVEY.md §8e exchange steps). NCCL is loaded at run
 * time (the copy already in the process if any, else MIHG_NCCL_LIBRARY, else libnccl.so.2);
 * failures -> MIHG_ENCCL. Rank 0 calls mihg_comm_unique_id, ships the 128 bytes to every rank
 * (any out-of-band channel), and every rank calls mihg_comm_init with its device. */
int mihg_comm_unique_id(uint8_t out_id[128]);
int mihg_comm_init(const uint8_t id[128], int nranks, int rank, int device, mihg_comm** out);
void mihg_comm_free(mihg_comm* comm);
int mihg_nccl_version(int* version);

/* Multi-GPU exact kNN in one call per rank, every collective inside the library (NCCL on the
 * index stream, joined to `stream`): the rank's local search with the per-round histogram
 * all-reduce, then an all-gather of the local top-k lists and the exact k-way merge on the device.
 * Every rank passes the same queries and k and receives the GLOBAL top-k in d_ids/d_dists [nq][k].
 *   layout 0: probe-space partition — every rank's index holds all n_total codes; rank g probes
 *             the ring values whose top log2(G) key bits equal g (G a power of two).
 *   layout 1: id-range shards (north_star's layout) — rank g's index holds ids
 *             [g*ceil(n_total/G), ...) built with that id_base; global stopping on the summed
 *             histograms (local stopping when some shard is empty).
 * d_traces: nq global traces or NULL (candidates/unique summed over ranks). */
int mihg_knn_sharded_device(mihg_index* idx, mihg_comm* comm, int layout, uint64_t n_total,
                            const uint64_t* d_queries, uint64_t nq, uint32_t k, uint32_t* d_ids,
                            uint32_t* d_dists, mihg_trace* d_traces, void* stream);

/* scan_knn(db, q, k) — scan.hpp:43-68, batched, over the index's device codes. */
int mihg_scan_knn_batch(mihg_index* idx, const uint64_t* queries, uint64_t nq, uint32_t k,
                        uint32_t* out_ids, uint32_t* out_dists);
int mihg_scan_knn_batch_device(mihg_index* idx, const uint64_t* d_queries, uint64_t nq, uint32_t k,
                               uint32_t* d_ids, uint32_t* d_dists, void* stream);
/* scan_knn over raw device codes (no index). */
int mihg_scan_knn_raw_device(const uint64_t* d_codes, uint64_t n, uint32_t bits, uint32_t id_base,
                             const uint64_t* d_queries, uint64_t nq, uint32_t k, uint32_t* d_ids,
                             uint32_t* d_dists, void* stream);

/* Exhaustive kernel behind the scan entry points: K7 (tcgen05 int8 tensor-core scan, codes of at
 * most 256 bits; the default there) or K6 (POPC pipe). Results are identical. Environment
 * MIHG_SCAN_KERNEL=popc|tc overrides the choice. Returns 0 = K6, 1 = K7 for a code width. */
int mihg_scan_kernel_for(uint32_t bits);
/* Test hook: every K7 distance of nq queries x n codes (device int32 [nq][n]), n*nq small. */
int mihg_tc_distances_device(const uint64_t* d_codes, uint64_t n, uint32_t bits,
                             const uint64_t* d_queries, uint64_t nq, int32_t* d_out, void* stream);

/* Exact k-way merge of G per-shard top-k lists: inputs [G][nq][k_in] device
 * arrays (dist 0xFFFFFFFF = padding), output the k_out smallest (dist, id) per query. */
int mihg_merge_topk_device(const uint32_t* d_ids, const uint32_t* d_dists, uint32_t G, uint64_t nq,
                           uint32_t k_in, uint32_t k_out, uint32_t* d_out_ids,
                           uint32_t* d_out_dists, void* stream);

/* gen_uniform(n, bits, seed) — io.hpp:266-277 (std::mt19937_64, standard-specified). Host. */
int mihg_gen_uniform(uint64_t n, uint32_t bits, uint64_t seed, uint64_t* out);
/* Codes [first, first + n) of gen_uniform(., bits, seed) — an id-range shard of the same stream. */
int mihg_gen_uniform_range(uint64_t first, uint64_t n, uint32_t bits, uint64_t seed, uint64_t* out);

/* Streaming gen_uniform: the same mt19937_64 sequence produced chunk by chunk (out == NULL
 * skips codes), so large databases are generated without holding them on the host. */
typedef struct mihg_mt64 mihg_mt64;
int mihg_mt64_create(uint64_t seed, mihg_mt64** out);
int mihg_mt64_next_codes(mihg_mt64* state, uint64_t n, uint32_t bits, uint64_t* out);
void mihg_mt64_free(mihg_mt64* state);

/* Live profiling: kernel launch count of this library (process-wide), and CUDA-event time of the
 * MIH probe kernel launches (recorded on their own stream) while enabled. */
typedef struct mihg_profile {
  uint64_t kernel_launches;
  double probe_ms;
  uint64_t probe_launches;
  double scan_ms;
  uint64_t scan_launches;
  uint64_t switched_queries; /* untraced kNN queries finished by the exhaustive scan (hybrid) */
  uint64_t rerun_queries;    /* queries whose candidate buffer overflowed (exact re-run pass) */
  double rerun_ms;           /* host wall time spent in re-run passes (synchronous) */
} mihg_profile;
int mihg_profile_enable(int on);
void mihg_profile_reset(void);
int mihg_profile_read(mihg_profile* out);

/* Calibration (no reference counterpart): the rate at which THIS GPU serves the dependent random
 * access pattern of one MIH lookup on a sparse table — a 16-byte directory group read at a random
 * place of a `dir_bytes` slice, followed for `nonempty_pct` percent of the lookups by a 4-byte
 * candidate read at a random place of a `codes_bytes` range — in lookups per second. Uses a
 * scratch allocation of dir_bytes + codes_bytes on `device`. bench.py reports it next to the MIH
 * probe kernel's own lookup rate (the probe kernel is bound by this
 * random-access rate, not by streaming HBM bandwidth). */
int mihg_calibrate_random_lookups(int device, uint64_t dir_bytes, uint64_t codes_bytes,
                                  uint32_t nonempty_pct, double* lookups_per_s);

/* Seeded Gaussian-mixture sign-projection codes (BASELINE configs 2 and 4; not in the reference,
 * which has gen_correlated_vectors + lsh_encode, io.hpp:245-262, :312-331). Exact integer
 * arithmetic, defined in paper_1307_2982_b200/csrc/gen.cu. Writes codes [first, first + n) as
 * n * ceil(bits/64) words to device memory. bits <= 256, dim % 4 == 0 and dim <= 256, comps <= 256. */
int mihg_gen_mixture_device(uint64_t first, uint64_t n, uint32_t bits, uint32_t dim, uint32_t comps,
                            uint64_t model_seed, uint64_t data_seed, uint64_t* d_out, void* stream);

/* ---- substring optimisation ---- */

/* estimate_correlations (optimize.hpp:47-92; replaces mih::estimate_correlations): |Pearson|
 * between every pair of bit positions over n >= 2 codes (n * ceil(bits/64) words, host memory,
 * or device memory on `device` when codes_on_device). The AND-popcount Gram matrix runs on the
 * GPU; out_corr receives bits*bits doubles row-major (diagonal 1; 0 against constant bits),
 * out_constant bits flags (CorrelationMatrix::is_constant), out_counts (nullable) the exact
 * integer counts #(bit_i AND bit_j) (diagonal = ones). n < 2 -> MIHG_EINVAL (the reference's
 * std::invalid_argument). Values are bitwise the reference's as built by its CMake on an FMA host. */
int mihg_estimate_correlations(const uint64_t* codes, uint64_t n, uint32_t bits, int device,
                               int codes_on_device, double* out_corr, uint8_t* out_constant,
                               uint64_t* out_counts);

/* greedy_assign (optimize.hpp:101-172; replaces mih::greedy_assign): host-only (no GPU needed).
 * corr/constant as produced above; writes out_lengths[m] and the m sorted position lists
 * concatenated into out_positions[bits] (the Partition's substrings). m == 0 or m > bits ->
 * MIHG_EINVAL. Same std::mt19937_64 + std::uniform_int_distribution draw as the reference. */
int mihg_greedy_assign(const double* corr, const uint8_t* constant, uint32_t bits, uint32_t m,
                       uint64_t seed, uint32_t* out_lengths, uint32_t* out_positions);

#ifdef __cplusplus
}
#endif

#endif /* MIHG_H */
