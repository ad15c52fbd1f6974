// Device primitives for the index build: exclusive scan and a stable LSD radix sort.
//
// The reference builds each substring table with std::stable_sort of (key, id) pairs
// (table.hpp:98-99); ids within a bucket therefore stay in insertion (= ascending id) order.
// The GPU build reproduces that order with a stable least-significant-digit radix sort over the
// s key bits (8-bit digits): per pass a tile histogram, a device-wide exclusive scan of the
// digit-major histogram matrix, and a stable scatter whose in-tile ranks come from warp
// __match_any_sync groups processed in item order.
#include "sort.cuh"

namespace mihg {

namespace {

constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T u = __shfl_up_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) >= o) v += u;
  }
  return v;
}

// Block-wide exclusive scan of a 4096-element tile; writes the tile total to sums[block].
template <typename T>
__global__ void __launch_bounds__(kScanThreads) scan_tiles_kernel(const T* __restrict__ in,
                                                                  T* __restrict__ out, uint64_t n,
                                                                  T* __restrict__ sums) {
  __shared__ T warp_tot[32];
  const uint64_t base = uint64_t(blockIdx.x) * kScanTile + uint64_t(threadIdx.x) * kScanItems;
  T v[kScanItems];
  T run = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = base + i < n ? in[base + i] : T(0);
    run += v[i];
  }
  const T incl = warp_inclusive_scan(run);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    T w = warp_tot[lane];
    const T wi = warp_inclusive_scan(w);
    warp_tot[lane] = wi - w;
    if (lane == 31 && sums) sums[blockIdx.x] = wi;
  }
  __syncthreads();
  T acc = warp_tot[warp] + incl - run;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < n) out[base + i] = acc;
    acc += v[i];
  }
}

template <typename T>
__global__ void add_tile_offsets_kernel(T* __restrict__ out, uint64_t n, const T* __restrict__ sums) {
  const T add = sums[blockIdx.x];
  const uint64_t base = uint64_t(blockIdx.x) * kScanTile;
  for (uint32_t i = threadIdx.x; i < kScanTile; i += blockDim.x)
    if (base + i < n) out[base + i] += add;
}

}  // namespace

template <typename T>
void exclusive_scan(const T* in, T* out, uint64_t n, cudaStream_t st) {
  if (n == 0) return;
  const uint64_t tiles = (n + kScanTile - 1) / kScanTile;
  if (tiles == 1) {
    scan_tiles_kernel<T><<<1, kScanThreads, 0, st>>>(in, out, n, nullptr);
    MIHG_LAUNCH();
    return;
  }
  DeviceBuffer<T> sums(tiles, st);
  scan_tiles_kernel<T><<<tiles, kScanThreads, 0, st>>>(in, out, n, sums.get());
  MIHG_LAUNCH();
  exclusive_scan<T>(sums.get(), sums.get(), tiles, st);
  add_tile_offsets_kernel<T><<<tiles, 256, 0, st>>>(out, n, sums.get());
  MIHG_LAUNCH();
}

template void exclusive_scan<uint32_t>(const uint32_t*, uint32_t*, uint64_t, cudaStream_t);
template void exclusive_scan<uint64_t>(const uint64_t*, uint64_t*, uint64_t, cudaStream_t);

namespace {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortIpt = 16;  // items per thread
constexpr int kSortTile = kSortThreads * kSortIpt;
constexpr int kRadix = 256;

template <typename K>
__device__ __forceinline__ uint32_t digit_of(K k, uint32_t shift) {
  return uint32_t(k >> shift) & (kRadix - 1);
}

// Per-tile digit histogram, written digit-major: hist[d * ntiles + tile].
template <typename K>
__global__ void __launch_bounds__(kSortThreads) radix_hist_kernel(const K* __restrict__ keys,
                                                                  uint64_t n, uint32_t shift,
                                                                  uint32_t* __restrict__ hist,
                                                                  uint32_t ntiles) {
  __shared__ uint32_t h[kSortWarps][kRadix];
  for (int i = threadIdx.x; i < kSortWarps * kRadix; i += kSortThreads) (&h[0][0])[i] = 0;
  __syncthreads();
  const uint64_t base = uint64_t(blockIdx.x) * kSortTile;
  const int warp = threadIdx.x >> 5;
#pragma unroll 4
  for (int i = 0; i < kSortIpt; ++i) {
    const uint64_t idx = base + uint64_t(i) * kSortThreads + threadIdx.x;
    if (idx < n) atomicAdd(&h[warp][digit_of(keys[idx], shift)], 1u);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < kRadix; d += kSortThreads) {
    uint32_t s = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) s += h[w][d];
    hist[uint64_t(d) * ntiles + blockIdx.x] = s;
  }
}

// Stable scatter. Warp w owns the contiguous sub-tile [w*32*IPT, (w+1)*32*IPT); iteration i
// covers 32 consecutive items, so (warp, iteration, lane) order equals item order and the
// __match_any_sync rank is a stable in-tile rank.
template <typename K, bool kVals>
__global__ void __launch_bounds__(kSortThreads) radix_scatter_kernel(
    const K* __restrict__ kin, const uint32_t* __restrict__ vin, K* __restrict__ kout,
    uint32_t* __restrict__ vout, uint64_t n, uint32_t shift, const uint32_t* __restrict__ offs,
    uint32_t ntiles) {
  __shared__ uint32_t wcnt[kSortWarps][kRadix];
  for (int i = threadIdx.x; i < kSortWarps * kRadix; i += kSortThreads) (&wcnt[0][0])[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t base = uint64_t(blockIdx.x) * kSortTile + uint64_t(warp) * 32 * kSortIpt;
  const uint32_t lt = lanemask_lt();
  K k[kSortIpt];
  uint32_t v[kSortIpt];
  uint32_t rank[kSortIpt];
#pragma unroll
  for (int i = 0; i < kSortIpt; ++i) {
    const uint64_t idx = base + uint64_t(i) * 32 + lane;
    const bool ok = idx < n;
    k[i] = ok ? kin[idx] : K(0);
    if constexpr (kVals) v[i] = ok ? vin[idx] : 0u;
    const uint32_t d = ok ? digit_of(k[i], shift) : uint32_t(kRadix);
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    const uint32_t before = ok ? wcnt[warp][d] : 0u;
    rank[i] = before + __popc(peers & lt);
    __syncwarp();
    if (ok && (peers & lt) == 0) wcnt[warp][d] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // wcnt[w][d] <- global start of (tile, warp w, digit d)
  for (int d = threadIdx.x; d < kRadix; d += kSortThreads) {
    uint32_t off = offs[uint64_t(d) * ntiles + blockIdx.x];
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) {
      const uint32_t c = wcnt[w][d];
      wcnt[w][d] = off;
      off += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kSortIpt; ++i) {
    const uint64_t idx = base + uint64_t(i) * 32 + lane;
    if (idx < n) {
      const uint32_t dst = wcnt[warp][digit_of(k[i], shift)] + rank[i];
      kout[dst] = k[i];
      if constexpr (kVals) vout[dst] = v[i];
    }
  }
}

template <typename K, bool kVals>
void radix_sort_impl(K* keys, uint32_t* vals, uint64_t n, uint32_t key_bits, cudaStream_t st) {
  if (n <= 1 || key_bits == 0) return;
  if (n > 0xFFFFFFFFull) throw InvalidArgument("radix sort: more than 2^32-1 items");
  const uint32_t ntiles = ceil_div_u32(n, kSortTile);
  DeviceBuffer<K> kalt(n, st);
  DeviceBuffer<uint32_t> valt(kVals ? n : 0, st);
  DeviceBuffer<uint32_t> hist(uint64_t(kRadix) * ntiles, st);
  K* ka = keys;
  K* kb = kalt.get();
  uint32_t* va = vals;
  uint32_t* vb = valt.get();
  const uint32_t passes = (key_bits + 7) / 8;
  for (uint32_t p = 0; p < passes; ++p) {
    const uint32_t shift = 8 * p;
    radix_hist_kernel<K><<<ntiles, kSortThreads, 0, st>>>(ka, n, shift, hist.get(), ntiles);
    MIHG_LAUNCH();
    exclusive_scan<uint32_t>(hist.get(), hist.get(), uint64_t(kRadix) * ntiles, st);
    radix_scatter_kernel<K, kVals><<<ntiles, kSortThreads, 0, st>>>(ka, va, kb, vb, n, shift,
                                                                     hist.get(), ntiles);
    MIHG_LAUNCH();
    std::swap(ka, kb);
    std::swap(va, vb);
  }
  if (ka != keys) {
    MIHG_CUDA(cudaMemcpyAsync(keys, ka, n * sizeof(K), cudaMemcpyDeviceToDevice, st));
    if constexpr (kVals)
      MIHG_CUDA(cudaMemcpyAsync(vals, va, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
  }
}

}  // namespace

void radix_sort_pairs_u32(uint32_t* keys, uint32_t* vals, uint64_t n, uint32_t key_bits,
                          cudaStream_t st) {
  radix_sort_impl<uint32_t, true>(keys, vals, n, key_bits, st);
}

void radix_sort_keys_u64(uint64_t* keys, uint64_t n, uint32_t key_bits, cudaStream_t st) {
  radix_sort_impl<uint64_t, false>(keys, nullptr, n, key_bits, st);
}

}  // namespace mihg
