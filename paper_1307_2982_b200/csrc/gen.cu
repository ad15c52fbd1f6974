// Seeded Gaussian-mixture sign-projection code generator (BASELINE configs 2 and 4).
//
// The configs name "sign(W x), W a seeded Gaussian matrix, x from a 64-component isotropic
// Gaussian mixture in R^128" without fixing parameters or arithmetic. Floating-point dot
// products make sign bits implementation-dependent near 0, so this generator is defined in exact
// integer arithmetic and is therefore bit-identical on any device or host (the numpy
// restatement in tests/test_datagen.py pins it):
//
//   h(seed, s, i)  = splitmix64(splitmix64(seed ^ s * 0xD6E8FEB86659FD93) ^ i)
//   g5(u) = sum_{t<4} ((u >> 5t) & 31) - 62          Irwin-Hall(4) ~ N(0, 18.5^2), |g5| <= 62
//   g6(u) = sum_{t<4} ((u >> 6t) & 63) - 126         Irwin-Hall(4) ~ N(0, 36.9^2), |g6| <= 126
//   W[j][d]  = g6(h(model_seed, 1, j*dim + d))        projection rows
//   mu[c][d] = g5(h(model_seed, 2, c*dim + d))        component means ("N(0, I)")
//   c(i)     = h(data_seed, 3, i) mod comps           uniform component choice
//   x_i[d]   = mu[c(i)][d] + g5(h(data_seed, 4, i*ceil(dim/3) + d/3) >> 20*(d%3))   unit noise
//   bit j of code i = [sum_d W[j][d] * x_i[d] >= 0]   (io.hpp:258: dot >= 0 -> bit 1)
//
// Means and noise have equal scale (sigma = 1 relative), i.e. an isotropic mixture with unit
// covariance around N(0, I) means. |x| <= 124 fits int8, so the dot product is __dp4a.
#include <algorithm>

#include "../../include/mihg.h"
#include "common.cuh"

namespace mihg {

namespace {

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__host__ __device__ __forceinline__ uint64_t hseed(uint64_t seed, uint64_t s) {
  return splitmix64(seed ^ (s * 0xD6E8FEB86659FD93ull));
}
__host__ __device__ __forceinline__ int g5(uint64_t u) {
  return int(u & 31) + int((u >> 5) & 31) + int((u >> 10) & 31) + int((u >> 15) & 31) - 62;
}
__host__ __device__ __forceinline__ int g6(uint64_t u) {
  return int(u & 63) + int((u >> 6) & 63) + int((u >> 12) & 63) + int((u >> 18) & 63) - 126;
}

constexpr int kGenThreads = 256;

// smem: W as int8 [bits][dim], mu as int8 [comps][dim]. kDW = dim/4 when compile-time (x in
// registers), 0 for the generic path.
template <int kDW>
__global__ void __launch_bounds__(kGenThreads) gen_mixture_kernel(uint64_t n, uint32_t bits,
                                                                  uint32_t dim, uint32_t comps,
                                                                  uint64_t model_seed,
                                                                  uint64_t data_seed, uint64_t first,
                                                                  uint64_t* __restrict__ out) {
  extern __shared__ uint32_t sm[];
  const uint32_t dw = kDW ? kDW : dim / 4;
  uint32_t* sW = sm;                    // bits * dw words
  uint32_t* sMu = sm + bits * dw;       // comps * dw words
  const uint64_t hW = hseed(model_seed, 1), hMu = hseed(model_seed, 2);
  for (uint32_t t = threadIdx.x; t < bits * dw; t += blockDim.x) {
    uint32_t packed = 0;
    for (int b = 0; b < 4; ++b) {
      const int v = g6(splitmix64(hW ^ (uint64_t(t) * 4 + b)));
      packed |= uint32_t(uint8_t(int8_t(v))) << (8 * b);
    }
    sW[t] = packed;
  }
  for (uint32_t t = threadIdx.x; t < comps * dw; t += blockDim.x) {
    uint32_t packed = 0;
    for (int b = 0; b < 4; ++b) {
      const int v = g5(splitmix64(hMu ^ (uint64_t(t) * 4 + b)));
      packed |= uint32_t(uint8_t(int8_t(v))) << (8 * b);
    }
    sMu[t] = packed;
  }
  __syncthreads();
  const uint64_t hC = hseed(data_seed, 3), hX = hseed(data_seed, 4);
  const uint32_t per = (dim + 2) / 3;
  const uint32_t W = (bits + 63) / 64;
  for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < n;
       r += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t i = first + r;  // global code index (shards generate their own id range)
    const uint32_t c = uint32_t(splitmix64(hC ^ i) % comps);
    uint32_t x[kDW ? kDW : 64];  // dim <= 256
    uint64_t u = 0;
#pragma unroll
    for (uint32_t w = 0; w < dw; ++w) {
      const uint32_t mu = sMu[c * dw + w];
      uint32_t packed = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const uint32_t d = w * 4 + b;
        if (d % 3 == 0) u = splitmix64(hX ^ (i * per + d / 3));
        const int v = int(int8_t(uint8_t(mu >> (8 * b)))) + g5(u >> (20 * (d % 3)));
        packed |= uint32_t(uint8_t(int8_t(v))) << (8 * b);
      }
      x[w] = packed;
    }
    for (uint32_t w64 = 0; w64 < W; ++w64) {
      uint64_t word = 0;
      const uint32_t jend = min(bits, (w64 + 1) * 64);
      for (uint32_t j = w64 * 64; j < jend; ++j) {
        int acc = 0;
        const uint32_t* wr = sW + j * dw;
#pragma unroll
        for (uint32_t w = 0; w < dw; ++w) acc = __dp4a(int(wr[w]), int(x[w]), acc);
        if (acc >= 0) word |= uint64_t(1) << (j - w64 * 64);
      }
      out[r * W + w64] = word;
    }
  }
}

}  // namespace

void gen_mixture_device(uint64_t first, uint64_t n, uint32_t bits, uint32_t dim, uint32_t comps,
                        uint64_t model_seed, uint64_t data_seed, uint64_t* d_out, cudaStream_t st) {
  if (bits == 0 || bits > 256) throw InvalidArgument("gen_mixture: bits must be in [1, 256]");
  if (dim == 0 || dim % 4 || dim > 256) throw InvalidArgument("gen_mixture: dim must be a multiple of 4 in [4, 256]");
  if (comps == 0 || comps > 256) throw InvalidArgument("gen_mixture: comps must be in [1, 256]");
  if (n == 0) return;
  const size_t smem = size_t(bits + comps) * dim;
  const uint64_t blocks = std::min<uint64_t>((n + kGenThreads - 1) / kGenThreads, uint64_t(device_sm_count()) * 8);
  if (dim == 128) {
    MIHG_CUDA(cudaFuncSetAttribute(gen_mixture_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    gen_mixture_kernel<32><<<unsigned(blocks), kGenThreads, smem, st>>>(n, bits, dim, comps, model_seed,
                                                                        data_seed, first, d_out);
  } else {
    MIHG_CUDA(cudaFuncSetAttribute(gen_mixture_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    gen_mixture_kernel<0><<<unsigned(blocks), kGenThreads, smem, st>>>(n, bits, dim, comps, model_seed,
                                                                       data_seed, first, d_out);
  }
  MIHG_LAUNCH();
}

}  // namespace mihg

extern "C" int mihg_gen_mixture_device(uint64_t first, uint64_t n, uint32_t bits, uint32_t dim,
                                       uint32_t comps, uint64_t model_seed, uint64_t data_seed,
                                       uint64_t* d_out, void* stream) {
  try {
    mihg::gen_mixture_device(first, n, bits, dim, comps, model_seed, data_seed, d_out,
                             static_cast<cudaStream_t>(stream));
    return MIHG_OK;
  } catch (const std::invalid_argument& e) {
    mihg::set_last_error(e.what());
    return MIHG_EINVAL;
  } catch (const std::exception& e) {
    mihg::set_last_error(e.what());
    return MIHG_ECUDA;
  }
}
