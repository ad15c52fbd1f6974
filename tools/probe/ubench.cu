// Microbenchmarks for design decisions: POPC/LOP3 issue rate and random 32B-sector gather rate.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__global__ void popc_kernel(const uint64_t* __restrict__ in, uint32_t* out, int iters) {
  uint64_t a = in[threadIdx.x & 31] + blockIdx.x, b = in[(threadIdx.x + 7) & 31], c = in[(threadIdx.x+3)&31], d = in[(threadIdx.x+11)&31];
  uint32_t s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  for (int i = 0; i < iters; ++i) {
    #pragma unroll
    for (int u = 0; u < 8; ++u) {
      s0 += __popcll(a ^ b); s1 += __popcll(c ^ d); s2 += __popcll(a ^ d); s3 += __popcll(b ^ c);
      a += 0x9E3779B97F4A7C15ull; c ^= a;
    }
  }
  if (s0 + s1 + s2 + s3 == 0x12345) out[0] = s0;
}

__global__ void gather_kernel(const uint32_t* __restrict__ tab, uint64_t nwords, uint64_t nprobe, uint32_t* out, uint64_t seed) {
  uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint32_t acc = 0;
  for (uint64_t i = tid; i < nprobe; i += stride * 4) {
    uint32_t v[4];
    #pragma unroll
    for (int u = 0; u < 4; ++u) {
      uint64_t x = (i + u * stride) * 0x9E3779B97F4A7C15ull + seed; x ^= x >> 29; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 32;
      v[u] = __ldg(tab + (x % nwords));
    }
    acc += v[0] + v[1] + v[2] + v[3];
  }
  if (acc == 0x12345) out[0] = acc;
}

int main() {
  uint64_t *din; uint32_t* dout;
  CK(cudaMalloc(&din, 256)); CK(cudaMemset(din, 0x5a, 256)); CK(cudaMalloc(&dout, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d clock %d kHz\n", nsm, clk);
  for (int rep = 0; rep < 3; ++rep) {
    int iters = 4000; int blocks = nsm * 8, threads = 256;
    cudaEventRecord(e0); popc_kernel<<<blocks, threads>>>(din, dout, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double popc64 = (double)blocks * threads * iters * 8 * 4;
    printf("popc64 %.3e/s (= %.3e popc32/s), %.1f ms\n", popc64 / ms * 1e3, 2 * popc64 / ms * 1e3, ms);
  }
  size_t bytes = (size_t)16 << 30; uint32_t* tab; CK(cudaMalloc(&tab, bytes)); CK(cudaMemset(tab, 1, bytes));
  for (int rep = 0; rep < 3; ++rep) {
    uint64_t nprobe = 1ull << 30;
    cudaEventRecord(e0); gather_kernel<<<nsm * 16, 256>>>(tab, bytes / 4, nprobe, dout, rep); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("random 4B gathers over 16GB: %.3e/s  (x32B sectors = %.1f GB/s), %.1f ms\n", nprobe / ms * 1e3, nprobe * 32.0 / ms / 1e6, ms);
  }
  for (int rep = 0; rep < 2; ++rep) {
    uint64_t nprobe = 1ull << 30; size_t small = 64 << 20;
    cudaEventRecord(e0); gather_kernel<<<nsm * 16, 256>>>(tab, small / 4, nprobe, dout, rep); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("random 4B gathers over 64MB (L2): %.3e/s, %.1f ms\n", nprobe / ms * 1e3, ms);
  }
  return 0;
}
