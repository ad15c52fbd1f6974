// Exact per-query top-k selection of packed keys (dist << 32 | id).
//
// Packing makes the numeric key order equal the reference's result order: neighbor_less
// (scan.hpp:24-26) = (dist asc, id asc), i.e. ties at the cut go to smaller ids (scan.hpp:42,
// index.hpp:243). Small segments (<= kSmemKeys after filtering) are sorted by one CTA in shared
// memory (bitonic); larger ones (large k, heavy ties) go through a device radix sort of
// (segment << 45 | key) composite keys.
#include <algorithm>
#include <vector>

#include "select.cuh"

namespace mihg {

namespace {

constexpr int kSelThreads = 512;
constexpr uint32_t kSelHistBins = 4097;  // distances 0..4096 (codes.hpp:16)

__device__ __forceinline__ bool keep_key(uint64_t key, uint32_t maxd) {
  return uint32_t(key >> 32) <= maxd;
}

__global__ void __launch_bounds__(kSelThreads) select_small_kernel(SelectArgs a) {
  extern __shared__ uint64_t sk[];
  __shared__ uint32_t s_cnt;
  const uint32_t seg = blockIdx.x;
  const uint64_t base = a.seg_base(seg);
  const uint32_t cnt = a.seg_count[seg];
  const uint32_t maxd = a.seg_maxd ? a.seg_maxd[seg] : 0xFFFFFFFFu;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  // one pass: filtered keys go straight to shared memory while they fit; the count decides
  // afterwards whether the segment belongs to the large path (oversized: nothing was lost, the
  // large path re-reads the segment)
  // (one shared-memory atomic per warp: every thread bumping the same counter serialised the
  // whole block — the kernel's length at config 4)
  const uint32_t lane = threadIdx.x & 31, ltm = (1u << lane) - 1u;
  for (uint32_t i0 = 0; i0 < cnt; i0 += blockDim.x) {
    const uint32_t i = i0 + threadIdx.x;
    const uint64_t key = i < cnt ? a.keys[base + i] : ~0ull;
    const bool keep = i < cnt && keep_key(key, maxd);
    const uint32_t bal = __ballot_sync(~0u, keep);
    uint32_t wbase = 0;
    if (lane == 0 && bal) wbase = atomicAdd(&s_cnt, uint32_t(__popc(bal)));
    wbase = __shfl_sync(~0u, wbase, 0);
    if (keep) {
      const uint32_t at = wbase + __popc(bal & ltm);
      if (at < kSmemKeys) sk[at] = key;
    }
  }
  __syncthreads();
  const uint32_t total = s_cnt;
  if (a.filtered_count) a.filtered_count[seg] = total;
  if (total > kSmemKeys) {
    if (threadIdx.x == 0) a.large_list[atomicAdd(a.large_count, 1u)] = seg;
    return;
  }
  uint32_t m = total;  // keys still in play, sk[0, m)
  if (total > 2 * a.k && total > 256) {
    // Pre-selection: the k-th smallest distance D from a distance histogram, then only the keys
    // with d <= D are sorted (the top k by (dist, id) lies among them; ties at D keep every
    // key so the smallest ids win in the sort).
    __shared__ uint32_t s_dmax, s_D, s_m;
    uint32_t* hist = reinterpret_cast<uint32_t*>(sk + kSmemKeys);
    if (threadIdx.x == 0) {
      s_dmax = 0;
      s_m = 0;
    }
    __syncthreads();
    uint32_t dm = 0;
    for (uint32_t i = threadIdx.x; i < total; i += blockDim.x) dm = max(dm, uint32_t(sk[i] >> 32));
    atomicMax(&s_dmax, dm);
    __syncthreads();
    const uint32_t dmax = min(s_dmax, min(a.max_dist, kSelHistBins - 1));
    for (uint32_t d = threadIdx.x; d <= dmax; d += blockDim.x) hist[d] = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < total; i += blockDim.x) atomicAdd(&hist[min(uint32_t(sk[i] >> 32), dmax)], 1u);
    __syncthreads();
    if (threadIdx.x < 32) {  // warp 0: running prefix, 32 bins per step
      const uint32_t lane = threadIdx.x;
      uint32_t run = 0, D = dmax;
      for (uint32_t d0 = 0; d0 <= dmax; d0 += 32) {
        uint32_t x = d0 + lane <= dmax ? hist[d0 + lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(~0u, x, o);
          if (lane >= uint32_t(o)) x += y;
        }
        const uint32_t ok = __ballot_sync(~0u, d0 + lane <= dmax && run + x >= a.k);
        if (ok) {
          D = d0 + __ffs(ok) - 1;
          break;
        }
        run += __shfl_sync(~0u, x, 31);
      }
      if (lane == 0) s_D = D;
    }
    __syncthreads();
    const uint32_t D = s_D;
    uint64_t mine[kSmemKeys / kSelThreads];
#pragma unroll
    for (uint32_t j = 0; j < kSmemKeys / kSelThreads; ++j) {
      const uint32_t i = threadIdx.x + j * blockDim.x;
      mine[j] = i < total ? sk[i] : ~0ull;
    }
    __syncthreads();
#pragma unroll
    for (uint32_t j = 0; j < kSmemKeys / kSelThreads; ++j) {
      const bool keep = mine[j] != ~0ull && uint32_t(mine[j] >> 32) <= D;
      const uint32_t bal = __ballot_sync(~0u, keep);
      uint32_t wbase = 0;
      if (lane == 0 && bal) wbase = atomicAdd(&s_m, uint32_t(__popc(bal)));
      wbase = __shfl_sync(~0u, wbase, 0);
      if (keep) sk[wbase + __popc(bal & ltm)] = mine[j];
    }
    __syncthreads();
    m = s_m;
  }
  uint32_t N = 32;
  while (N < m) N <<= 1;
  __syncthreads();
  for (uint32_t i = m + threadIdx.x; i < N; i += blockDim.x) sk[i] = ~0ull;
  __syncthreads();
  for (uint32_t k2 = 2; k2 <= N; k2 <<= 1) {
    for (uint32_t j = k2 >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) {
        const uint32_t ixj = i ^ j;
        if (ixj > i) {
          const uint64_t x = sk[i], y = sk[ixj];
          const bool asc = (i & k2) == 0;
          if ((x > y) == asc) {
            sk[i] = y;
            sk[ixj] = x;
          }
        }
      }
      __syncthreads();
    }
  }
  const uint64_t row = a.out_row ? a.out_row[seg] : seg;
  const uint32_t kk = min(a.k, m);
  for (uint32_t i = threadIdx.x; i < a.k; i += blockDim.x) {
    const bool ok = i < kk;
    const uint64_t key = ok ? sk[i] : ~0ull;
    a.out_ids[row * a.k + i] = ok ? uint32_t(key) + a.id_base : 0xFFFFFFFFu;
    a.out_dists[row * a.k + i] = ok ? uint32_t(key >> 32) : 0xFFFFFFFFu;
  }
}

// Large path: copy filtered entries of segment list[l] as (l << 45 | key) to dst[dbase[l]...].
__global__ void compose_kernel(SelectArgs a, const uint32_t* __restrict__ list,
                               const uint64_t* __restrict__ dbase, uint64_t* __restrict__ dst) {
  __shared__ uint32_t s_at;
  const uint32_t l = blockIdx.x;
  const uint32_t seg = list[l];
  const uint64_t base = a.seg_base(seg);
  const uint32_t cnt = a.seg_count[seg];
  const uint32_t maxd = a.seg_maxd ? a.seg_maxd[seg] : 0xFFFFFFFFu;
  if (threadIdx.x == 0) s_at = 0;
  __syncthreads();
  const uint64_t tag = uint64_t(l) << 45;
  for (uint32_t i0 = 0; i0 < cnt; i0 += blockDim.x) {
    const uint32_t i = i0 + threadIdx.x;
    const uint64_t key = i < cnt ? a.keys[base + i] : ~0ull;
    const bool keep = i < cnt && keep_key(key, maxd);
    if (keep) dst[dbase[l] + atomicAdd(&s_at, 1u)] = tag | key;
  }
}

__global__ void emit_large_kernel(SelectArgs a, const uint32_t* __restrict__ list,
                                  const uint64_t* __restrict__ dbase,
                                  const uint32_t* __restrict__ fcount,
                                  const uint64_t* __restrict__ sorted) {
  const uint32_t l = blockIdx.x;
  const uint32_t seg = list[l];
  const uint64_t row = a.out_row ? a.out_row[seg] : seg;
  const uint32_t kk = min(a.k, fcount[seg]);
  const uint64_t mask45 = (uint64_t(1) << 45) - 1;
  for (uint32_t i = threadIdx.x; i < a.k; i += blockDim.x) {
    const bool ok = i < kk;
    const uint64_t key = ok ? (sorted[dbase[l] + i] & mask45) : ~0ull;
    a.out_ids[row * a.k + i] = ok ? uint32_t(key) + a.id_base : 0xFFFFFFFFu;
    a.out_dists[row * a.k + i] = ok ? uint32_t(key >> 32) : 0xFFFFFFFFu;
  }
}

}  // namespace

void select_topk(SelectArgs a, uint32_t nseg, cudaStream_t st) {
  if (nseg == 0 || a.k == 0) return;
  DeviceBuffer<uint32_t> fcount(nseg, st), list(nseg, st), lcount(1, st);
  MIHG_CUDA(cudaMemsetAsync(lcount.get(), 0, 4, st));
  a.filtered_count = fcount.get();
  a.large_list = list.get();
  a.large_count = lcount.get();
  const size_t smem = size_t(kSmemKeys) * 8 + size_t(std::min(a.max_dist + 1, kSelHistBins)) * 4;
  // per call (cheap), so every device the process uses gets the attribute
  MIHG_CUDA(cudaFuncSetAttribute(select_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  select_small_kernel<<<nseg, kSelThreads, smem, st>>>(a);
  MIHG_LAUNCH();
  uint32_t L = 0;
  MIHG_CUDA(cudaMemcpyAsync(&L, lcount.get(), 4, cudaMemcpyDeviceToHost, st));
  MIHG_CUDA(cudaStreamSynchronize(st));
  if (L == 0) return;
  if (L >= (1u << 19)) throw CudaError("select_topk: too many oversized segments in one pass");
  std::vector<uint32_t> hlist(L), hcnt(nseg);
  MIHG_CUDA(cudaMemcpyAsync(hlist.data(), list.get(), L * 4, cudaMemcpyDeviceToHost, st));
  MIHG_CUDA(cudaMemcpyAsync(hcnt.data(), fcount.get(), nseg * 4, cudaMemcpyDeviceToHost, st));
  MIHG_CUDA(cudaStreamSynchronize(st));
  std::vector<uint64_t> hbase(L);
  uint64_t total = 0;
  for (uint32_t l = 0; l < L; ++l) {
    hbase[l] = total;
    total += hcnt[hlist[l]];
  }
  DeviceBuffer<uint64_t> dbase(L, st), comp(std::max<uint64_t>(total, 1), st);
  MIHG_CUDA(cudaMemcpyAsync(dbase.get(), hbase.data(), L * 8, cudaMemcpyHostToDevice, st));
  compose_kernel<<<L, 256, 0, st>>>(a, list.get(), dbase.get(), comp.get());
  MIHG_LAUNCH();
  uint32_t lbits = 0;
  while ((1u << lbits) < L) ++lbits;
  radix_sort_keys_u64(comp.get(), total, 45 + lbits, st);
  emit_large_kernel<<<L, 256, 0, st>>>(a, list.get(), dbase.get(), fcount.get(), comp.get());
  MIHG_LAUNCH();
  MIHG_CUDA(cudaStreamSynchronize(st));
}

}  // namespace mihg
