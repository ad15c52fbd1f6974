#pragma once
#include "index.cuh"

namespace mihg {

// Mirrors mih::SearchTrace (index.hpp:45-51); layout shared with include/mihg.h mihg_trace.
struct Trace {
  uint64_t lookups, candidates, unique_candidates, distance_evaluations;
  uint32_t final_radius, reserved;
};
static_assert(sizeof(Trace) == 40, "mihg_trace ABI");

// Probe-space partition across ranks (multi-GPU): rank `rank` of `count` (a power of two) probes
// only the ring values whose top log2(count) key bits equal `rank`; the per-query histograms are
// summed across ranks every round through `allreduce` (in place on device memory, ordered on
// `stream`; dtype 0 = u32, 1 = u64) so all ranks share the reference's stopping rule. The call
// then returns the rank's LOCAL top-k candidates; the caller all-gathers and merges them.
struct Comm;  // NCCL communicator (comm.cu)
struct NcclError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Partition {
  uint32_t count = 1, rank = 0;
  int (*allreduce)(void* user, void* dev_ptr, uint64_t count, int dtype, void* stream) = nullptr;
  void* user = nullptr;
  bool id_shards = false;  // id-range shards with global stopping (no probe split)
  uint32_t k_stop = 0;     // k of the global stopping rule (0: the call's k)
  Comm* comm = nullptr;    // library-owned NCCL communicator: used instead of `allreduce`
};

// NCCL (comm.cu; loaded at run time). Collectives are enqueued on `st`, no host synchronisation.
void comm_unique_id(uint8_t* out128);
Comm* comm_init(const uint8_t* id128, int nranks, int rank, int device);
void comm_free(Comm* c);
int comm_size(const Comm* c);
int comm_rank(const Comm* c);
int nccl_version();
void comm_allreduce_sum(Comm* c, void* ptr, uint64_t n, int dtype, cudaStream_t st);
void comm_allgather(Comm* c, const void* send, void* recv, uint64_t bytes, cudaStream_t st);

struct KnnOptions {
  // per-query candidate buffer (u64 keys) in the main pass: 32768 keys (256 KB per query, 4 GB
  // per 16384-query chunk) keep clustered data out of the exact re-run pass (config 4: +4.7%)
  uint32_t buffer_cap = 32768;
  uint32_t query_chunk = 16384; // queries per workspace pass
  const Partition* part = nullptr;
};

// Batched MihIndex::knn_search (index.hpp:185-253). All pointers are device pointers on
// idx.device; results ordered by (dist, id) with global ids (local + idx.id_base).
void knn_device(Index& idx, const uint64_t* d_queries, uint64_t nq, uint32_t k, uint32_t* d_ids,
                uint32_t* d_dists, Trace* d_traces, cudaStream_t st, const KnnOptions& opt = {});

// Batched MihIndex::range_search (index.hpp:149-176) with host buffers: offsets[nq+1] always
// written; ids/dists (capacity entries) written when offsets[nq] <= capacity.
void range_host(Index& idx, const uint64_t* h_queries, uint64_t nq, uint32_t r, uint64_t* h_offsets,
                uint32_t* h_ids, uint32_t* h_dists, uint64_t capacity, Trace* h_traces, cudaStream_t st,
                const KnnOptions& opt = {});

// Batched scan_knn (scan.hpp:43-68) over the index's device-resident codes.
void scan_knn_device(const uint64_t* d_codes, uint64_t n, uint32_t bits, uint32_t id_base,
                     const uint64_t* d_queries, uint64_t nq, uint32_t k, uint32_t* d_ids,
                     uint32_t* d_dists, cudaStream_t st);

// K6 itself (POPC pipe), any width.
void popc_scan_knn_device(const uint64_t* d_codes, uint64_t n, uint32_t bits, uint32_t id_base,
                          const uint64_t* d_queries, uint64_t nq, uint32_t k, uint32_t* d_ids,
                          uint32_t* d_dists, cudaStream_t st);

// K7: the same exhaustive k-NN on the tensor cores (tcscan.cu), codes of 1..256 bits. d_dump
// (tests only, nullable): every distance, nq x n row-major.
bool tc_scan_supported(uint32_t bits);
void tc_scan_knn_device(const uint64_t* d_codes, uint64_t n, uint32_t bits, uint32_t id_base,
                        const uint64_t* d_queries, uint64_t nq, uint32_t k, uint32_t* d_ids,
                        uint32_t* d_dists, cudaStream_t st, int32_t* d_dump);
enum class ScanKernel { Popc, Tensor };
ScanKernel scan_kernel_for(uint32_t bits);

// k-way merge of G per-shard sorted (dist, id) lists per query (exact: smallest keys win).
void merge_topk_device(const uint32_t* d_ids, const uint32_t* d_dists, uint32_t G, uint64_t nq,
                       uint32_t k_in, uint32_t k_out, uint32_t* d_out_ids, uint32_t* d_out_dists,
                       cudaStream_t st);

// Per-query top-k selection of packed keys (dist << 32 | id) held in segments of a buffer.
// Used by the MIH, scan and merge paths.
struct SegmentSelect {
  const uint64_t* keys;
  const uint64_t* seg_base;  // per slot
  const uint32_t* seg_count; // per slot (entries already filtered to the candidate set)
};

}  // namespace mihg
