// Device-resident multi-index: the GPU counterpart of mih::MihIndex (index.hpp:98-285).
#pragma once
#include <memory>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "sort.cuh"

namespace mihg {

// Owning storage of one substring table (replaces SubstringTable, table.hpp:85-290).
struct TableStorage {
  uint32_t s = 0;
  bool dense = true;
  DeviceBuffer<uint32_t> ids;      // n, sorted by (key, id)
  DeviceBuffer<uint32_t> offsets;  // dense: 2^s + 1
  DeviceBuffer<DirGroup> dir;      // sparse: 2^(s-5) groups of 16 bytes
  DeviceBuffer<uint32_t> esc;      // sparse: 33 per escaped group
  DeviceBuffer<uint64_t> tcodes;   // optional: codes in table order (bucket = contiguous run)
  DeviceBuffer<uint32_t> occ;      // sparse: occupancy bitmap, 1 bit per bucket
  DeviceBuffer<uint32_t> rcodes;   // optional: 32-bit residual codes in table order (see DevTable)
  uint32_t rshift = 0;
  uint64_t escaped_blocks = 0;
  uint64_t non_empty_buckets = 0;
  uint64_t non_empty_groups = 0;  // 32-bucket groups (the reference's accounting unit)
  uint64_t max_bucket = 0;
  DevTable view() const {
    return DevTable{ids.get(), offsets.get(), dir.get(), esc.get(), tcodes.get(), occ.get(), s,
                    dense ? 1u : 0u, rcodes.get(), rshift, uint32_t(ids.size()), uint32_t(escaped_blocks)};
  }
  // frees every device buffer (stream-ordered on the index stream, before that stream goes away)
  void release() {
    ids.reset();
    offsets.reset();
    dir.reset();
    esc.reset();
    tcodes.reset();
    occ.reset();
    rcodes.reset();
  }
  uint64_t bytes() const {
    return ids.size() * 4 + offsets.size() * 4 + dir.size() * sizeof(DirGroup) + esc.size() * 4 +
           tcodes.size() * 8 + occ.size() * 4 + rcodes.size() * 4;
  }
};

// A table given in final (key, id) order, e.g. loaded from a BMIX index file.
struct PreTable {
  std::vector<uint32_t> keys, ids;
};

struct BuildOptions {
  // Dense direct-address offsets when 2^s <= max(2^dense_max_bits, dense_ratio * n);
  // otherwise the blocked-count sparse directory. (north_star: 32-bit substrings -> sparse.)
  uint32_t dense_max_bits = 24;
  uint32_t dense_ratio = 2;
  int force = 0;  // 0 auto, 1 dense, 2 sparse
  // Codes stored inline in table order so a bucket's candidates are one contiguous read:
  // -1 auto (when all tables' inline codes fit in 40% of free HBM), 0 off, 1 on.
  int inline_codes = -1;
  // 64-bit codes with two 32-bit substrings: 4-byte residual table-order codes (MIHG_RESIDUAL=0 off)
  bool residual_codes = true;
  // Sparse tables: 1-bit-per-bucket occupancy bitmap in front of the directory, so a probe of
  // an empty bucket is one 4-byte (L2-resident per key slice) read instead of a DRAM sector.
  bool occupancy = false;
  // measured: occupancy on, config 4 703K -> 674K q/s (a dependent L2 read per probe)
  const std::vector<PreTable>* pre = nullptr;  // use these tables instead of sorting
};

// A loaded table (BuildOptions::pre) whose entries are not a permutation of [0, n) filed under
// their own substring key: the stateless first-discovery dedup of the kNN kernels relies on it.
struct InconsistentTable : std::runtime_error {
  uint32_t table;
  InconsistentTable(uint32_t j, const std::string& what) : std::runtime_error(what), table(j) {}
};

struct Index {
  int device = 0;
  cudaStream_t stream = nullptr;
  uint32_t bits = 0, W = 0, m = 0;
  uint64_t n = 0;
  uint32_t id_base = 0;  // global id of local id 0 (id-range shards)
  std::vector<uint32_t> lengths, positions;
  std::vector<DevSubstring> subs;
  DeviceBuffer<uint64_t> codes;      // n * W words, bit i at word i/64 bit i%64
  DeviceBuffer<uint32_t> d_positions;
  DeviceBuffer<DevSubstring> d_subs;
  DeviceBuffer<uint64_t> d_submask;  // m * W: bit mask of the positions owned by substring j
  bool inline_codes = false;
  std::vector<std::unique_ptr<TableStorage>> tables;
  DeviceBuffer<DevTable> d_tables;
  std::mutex mu;  // one host call at a time per index (workspace is shared)
  struct Workspace* ws = nullptr;
  // grow-only device staging of the host-pointer entry points (queries in, results out), reused
  // across calls so a host call allocates nothing once warm
  DeviceBuffer<uint64_t> stage_q;
  DeviceBuffer<uint32_t> stage_ids, stage_dists;
  DeviceBuffer<unsigned char> stage_tr;
  template <typename T>
  static T* grow(DeviceBuffer<T>& b, uint64_t n, cudaStream_t st) {
    if (b.size() < n) b = DeviceBuffer<T>(n, st);
    return b.get();
  }
  ~Index();
};

// Validates like Partition::validate (codes.hpp:152-176) and MihIndex::build (index.hpp:101-112);
// throws InvalidArgument with the reference's wording.
void validate_partition(uint32_t bits, uint32_t m, const uint32_t* lengths,
                        const uint32_t* positions);

// d_codes: n*W words already on `device` (copied into the index unless `adopt`).
Index* build_index(const uint64_t* codes, bool codes_on_device, uint64_t n, uint32_t bits,
                   uint32_t m, const uint32_t* lengths, const uint32_t* positions, int device,
                   uint32_t id_base, const BuildOptions& opt);

// Device key extraction for a batch of codes: keys[i*m + j] = substring j of code i.
void extract_all_keys(const Index& idx, const uint64_t* d_codes, uint64_t count, uint32_t* d_keys,
                      cudaStream_t st);

}  // namespace mihg
