// Substring optimisation.
//
// estimate_correlations (/root/reference/proj/include/mih/optimize.hpp:47-92) is a b x b
// AND-popcount Gram matrix over the transposed bit columns plus a scalar finish. The Gram
// matrix runs on the GPU in two kernels per chunk of codes:
//   * bit_transpose_kernel — one warp per 32 codes: 64 ballots per code word turn the rows
//     into column words, stored group-major cols[group][position] so every warp writes
//     contiguous 128 B lines (the reference's column bitsets, optimize.hpp:51-57, transposed
//     to suit coalescing);
//   * and_gram_kernel — 64 x 64 position tiles of the upper triangle, 32 groups (1024 codes)
//     per shared-memory stage, a 4 x 4 register micro-tile of LOP3+POPC per thread, split-K
//     over groups with one u64 atomic per (pair, block) at the end.
// Integer counts are exact; the floating-point finish (finish_correlations) reproduces the
// reference's expressions in the same order on the host.
//
// greedy_assign (optimize.hpp:101-172) is O(b^2 m) sequential host logic over the matrix and
// stays on the host (b <= 4096).
#include <algorithm>
#include <cmath>
#include <random>
#include <vector>

#include "common.cuh"
#include "optimize.cuh"
#include "sort.cuh"

namespace mihg {
namespace {

constexpr uint32_t kTile = 64;        // positions per tile side
constexpr uint32_t kStage = 32;       // groups (of 32 codes) per shared-memory stage
constexpr uint64_t kChunk = 1u << 22;  // codes per transpose/gram pass

__global__ void __launch_bounds__(256) bit_transpose_kernel(const uint64_t* __restrict__ codes,
                                                            uint64_t nc, uint32_t W, uint32_t stride,
                                                            uint32_t* __restrict__ cols) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t groups = (nc + 31) / 32;
  const uint64_t nwarps = uint64_t(gridDim.x) * (blockDim.x / 32);
  for (uint64_t g = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) / 32; g < groups; g += nwarps) {
    const uint64_t row = g * 32 + lane;
    uint32_t* out = cols + g * stride;
    for (uint32_t w = 0; w < W; ++w) {
      const uint64_t x = row < nc ? codes[row * W + w] : 0;
      uint32_t lo = 0, hi = 0;
#pragma unroll
      for (uint32_t t = 0; t < 32; ++t) {
        const uint32_t b0 = __ballot_sync(0xffffffffu, (x >> t) & 1);
        const uint32_t b1 = __ballot_sync(0xffffffffu, (x >> (t + 32)) & 1);
        if (lane == t) {
          lo = b0;
          hi = b1;
        }
      }
      out[64 * w + lane] = lo;
      out[64 * w + 32 + lane] = hi;
    }
  }
}

__global__ void __launch_bounds__(256) and_gram_kernel(const uint32_t* __restrict__ cols, uint64_t groups,
                                                       uint32_t stride, uint32_t bits, uint32_t ntiles,
                                                       uint64_t per_split, unsigned long long* counts) {
  __shared__ __align__(16) uint32_t As[kStage][kTile];
  __shared__ __align__(16) uint32_t Bs[kStage][kTile];
  uint32_t rem = blockIdx.x, ti = 0;
  while (rem >= ntiles - ti) {
    rem -= ntiles - ti;
    ++ti;
  }
  const uint32_t tj = ti + rem;
  const uint64_t g0 = blockIdx.y * per_split, g1 = min(groups, g0 + per_split);
  const uint32_t t = threadIdx.x, ty = t / 16, tx = t % 16;
  uint32_t acc[4][4] = {};
  for (uint64_t gs = g0; gs < g1; gs += kStage) {
#pragma unroll
    for (uint32_t q = 0; q < kStage * kTile / 256; ++q) {
      const uint32_t e = t + 256 * q, r = e / kTile, c = e % kTile;
      const bool ok = gs + r < g1;
      As[r][c] = ok ? cols[(gs + r) * stride + ti * kTile + c] : 0u;
      Bs[r][c] = ok ? cols[(gs + r) * stride + tj * kTile + c] : 0u;
    }
    __syncthreads();
#pragma unroll 8
    for (uint32_t kk = 0; kk < kStage; ++kk) {
      const uint4 a = *reinterpret_cast<const uint4*>(&As[kk][ty * 4]);
      const uint4 b = *reinterpret_cast<const uint4*>(&Bs[kk][tx * 4]);
      const uint32_t av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] += __popc(av[i] & bv[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t pi = ti * kTile + ty * 4 + i, pj = tj * kTile + tx * 4 + j;
      if (pi < bits && pj < bits && acc[i][j])
        atomicAdd(&counts[uint64_t(pi) * bits + pj], (unsigned long long)acc[i][j]);
    }
}

}  // namespace

void and_count_gram(const uint64_t* codes, uint64_t n, uint32_t bits, bool on_device,
                    uint64_t* d_counts, cudaStream_t st) {
  const uint32_t W = (bits + 63) / 64, stride = W * 64, ntiles = (bits + kTile - 1) / kTile;
  const uint32_t tiles = ntiles * (ntiles + 1) / 2;
  const uint64_t chunk = std::min<uint64_t>(kChunk, std::max<uint64_t>(n, 1));
  DeviceBuffer<uint64_t> staging(on_device ? 0 : chunk * W, st);
  DeviceBuffer<uint32_t> cols((chunk + 31) / 32 * stride, st);
  const int sms = device_sm_count();
  for (uint64_t at = 0; at < n; at += chunk) {
    const uint64_t nc = std::min(chunk, n - at);
    const uint64_t* src = codes + at * W;
    if (!on_device) {
      MIHG_CUDA(cudaMemcpyAsync(staging.get(), src, nc * W * 8, cudaMemcpyHostToDevice, st));
      src = staging.get();
    }
    const uint64_t groups = (nc + 31) / 32;
    bit_transpose_kernel<<<unsigned(std::min<uint64_t>((groups + 7) / 8, uint64_t(sms) * 16)), 256, 0, st>>>(
        src, nc, W, stride, cols.get());
    MIHG_LAUNCH();
    const uint64_t stages = (groups + kStage - 1) / kStage;
    const uint64_t want = std::max<uint64_t>(1, (uint64_t(sms) * 8 + tiles - 1) / tiles);
    const uint64_t splits = std::min<uint64_t>(std::min<uint64_t>(want, stages), 65535);
    const uint64_t per_split = (stages + splits - 1) / splits * kStage;
    const dim3 grid(tiles, unsigned((groups + per_split - 1) / per_split));
    and_gram_kernel<<<grid, 256, 0, st>>>(cols.get(), groups, stride, bits, ntiles, per_split,
                                          reinterpret_cast<unsigned long long*>(d_counts));
    MIHG_LAUNCH();
  }
}

void finish_correlations(const uint64_t* counts, uint64_t n, uint32_t bits, double* corr,
                         uint8_t* constant) {
  // optimize.hpp:72-91 in the same evaluation order. The reference's CMake build
  // (-O3 -march=native) lets g++ contract `pij - pi * pj` into one fused multiply-add on any
  // FMA host; std::fma states that explicitly so the result is bitwise the reference's.
  std::vector<double> var(bits);
  for (uint32_t i = 0; i < bits; ++i) {
    const uint64_t ones = counts[uint64_t(i) * bits + i];
    const double p = static_cast<double>(ones) / n;
    var[i] = p * (1.0 - p);
    constant[i] = (ones == 0 || ones == n) ? 1 : 0;
  }
  for (uint64_t e = 0; e < uint64_t(bits) * bits; ++e) corr[e] = 0.0;
  for (uint32_t i = 0; i < bits; ++i) corr[uint64_t(i) * bits + i] = 1.0;
  for (uint32_t i = 0; i < bits; ++i) {
    for (uint32_t j = i + 1; j < bits; ++j) {
      if (var[i] == 0.0 || var[j] == 0.0) continue;
      const double pi = static_cast<double>(counts[uint64_t(i) * bits + i]) / n;
      const double pj = static_cast<double>(counts[uint64_t(j) * bits + j]) / n;
      const double pij = static_cast<double>(counts[uint64_t(i) * bits + j]) / n;
      const double c = std::fabs(std::fma(-pi, pj, pij)) / std::sqrt(var[i] * var[j]);
      corr[uint64_t(i) * bits + j] = corr[uint64_t(j) * bits + i] = std::min(c, 1.0);
    }
  }
}

// greedy_assign (optimize.hpp:101-172), restated as incremental arg-min/arg-max scans. Per
// substring j the table near[j][c] holds max over j's members o of |corr(c, o)|, raised by one row of
// the matrix whenever j takes a bit, so a visit is a single pass over the free bits (O(b)) instead
// of re-reducing over the members. Selection rules are the reference's: strict comparisons over
// ascending bit index (ties to the lowest index), the chain opening through mt19937_64 +
// uniform_int_distribution over the free non-constant bits, balanced capacities with the extras
// on the lowest substrings, constant bits dealt round-robin last, members sorted.
void greedy_assign(const double* corr, const uint8_t* constant, uint32_t bits, uint32_t m,
                   uint64_t seed, uint32_t* lengths, uint32_t* positions) {
  if (m == 0 || m > bits) throw InvalidArgument("greedy_assign: need 1 <= m <= bits");
  const auto row = [&](uint32_t i) { return corr + uint64_t(i) * bits; };
  std::vector<uint32_t> capacity(m);
  for (uint32_t j = 0; j < m; ++j) capacity[j] = bits / m + (j < bits % m ? 1u : 0u);
  std::vector<std::vector<uint32_t>> members(m);
  std::vector<uint8_t> open(bits);  // 1: non-constant and not yet assigned
  uint32_t n_open = 0;
  for (uint32_t i = 0; i < bits; ++i) n_open += (open[i] = constant[i] ? 0 : 1);
  std::vector<double> near(uint64_t(m) * bits, 0.0);
  const auto assign = [&](uint32_t j, uint32_t bit) {
    members[j].push_back(bit);
    open[bit] = 0;
    --n_open;
    double* nj = near.data() + uint64_t(j) * bits;
    const double* r = row(bit);
    for (uint32_t c = 0; c < bits; ++c) nj[c] = std::max(nj[c], r[c]);
  };

  if (n_open) {
    // the opener: the (draw)-th free bit in ascending order
    std::mt19937_64 rng(seed);
    size_t draw = std::uniform_int_distribution<size_t>(0, n_open - 1)(rng);
    uint32_t opener = 0;
    for (uint32_t c = 0; c < bits; ++c)
      if (open[c] && draw-- == 0) {
        opener = c;
        break;
      }
    assign(0, opener);
    // substring j opens with the free bit most correlated with substring j-1's opener
    for (uint32_t j = 1; j < m && n_open; ++j) {
      const double* r = row(members[j - 1].empty() ? opener : members[j - 1].front());
      uint32_t pick = bits;
      for (uint32_t c = 0; c < bits; ++c)
        if (open[c] && (pick == bits || r[c] > r[pick])) pick = c;
      assign(j, pick);
    }
  }
  // rounds: each substring with room takes the free bit of smallest max-correlation to it
  while (n_open) {
    bool took = false;
    for (uint32_t j = 0; j < m && n_open; ++j) {
      if (members[j].size() >= capacity[j]) continue;
      const double* nj = near.data() + uint64_t(j) * bits;
      uint32_t pick = bits;
      for (uint32_t c = 0; c < bits; ++c)
        if (open[c] && (pick == bits || nj[c] < nj[pick])) pick = c;
      assign(j, pick);
      took = true;
    }
    if (!took) break;  // no room left (cannot happen with balanced capacities)
  }
  // constant bits: dealt round-robin over the remaining room
  for (uint32_t c = 0, j = 0; c < bits; ++c) {
    if (!constant[c]) continue;
    while (members[j].size() >= capacity[j]) j = (j + 1) % m;
    members[j].push_back(c);
    j = (j + 1) % m;
  }
  for (uint32_t j = 0, at = 0; j < m; ++j) {
    std::sort(members[j].begin(), members[j].end());
    lengths[j] = uint32_t(members[j].size());
    for (uint32_t v : members[j]) positions[at++] = v;
  }
}

}  // namespace mihg
