#pragma once
#include "sort.cuh"

namespace mihg {

constexpr uint32_t kSmemKeys = 4096;  // bitonic sort capacity of the one-CTA path (32 KB)

// Segment `seg` holds seg_count[seg] packed keys (dist << 32 | local id) starting at
// seg_base(seg); only keys with dist <= seg_maxd[seg] (when given) are candidates. The k
// smallest candidates go to out row out_row[seg] (or seg), ids offset by id_base. Rows with
// fewer than k candidates are padded with 0xFFFFFFFF.
struct SelectArgs {
  const uint64_t* keys = nullptr;
  const uint64_t* seg_base_arr = nullptr;  // explicit per-segment base, or
  uint64_t seg_stride = 0;                 //   base = seg * stride
  const uint32_t* seg_count = nullptr;
  const uint32_t* seg_maxd = nullptr;
  const uint64_t* out_row = nullptr;
  uint32_t k = 0;
  uint32_t id_base = 0;
  uint32_t max_dist = 4096;  // an upper bound on every key's distance (the code width): sizes the histogram
  uint32_t* out_ids = nullptr;
  uint32_t* out_dists = nullptr;
  // filled by select_topk
  uint32_t* filtered_count = nullptr;
  uint32_t* large_list = nullptr;
  uint32_t* large_count = nullptr;

  __device__ __forceinline__ uint64_t seg_base(uint32_t seg) const {
    return seg_base_arr ? seg_base_arr[seg] : uint64_t(seg) * seg_stride;
  }
};

void select_topk(SelectArgs a, uint32_t nseg, cudaStream_t st);

}  // namespace mihg
