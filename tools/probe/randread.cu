// Random-access DRAM read ceiling on B200: each lane issues independent loads of `gran` bytes at
// hashed addresses inside a `span`-byte buffer (>> L2), `unroll` loads in flight per lane.
// Prints useful GB/s and requests/s per granularity. nvcc -O3 -arch=sm_100a randread.cu -o randread
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33; return x;
}
template <int GRAN, int UNROLL>
__global__ void rr(const uint8_t* __restrict__ buf, uint64_t nslots, uint64_t per_thread, uint64_t seed, uint32_t* sink) {
  const uint64_t tid = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  uint32_t acc = 0;
  for (uint64_t i = 0; i < per_thread; i += UNROLL) {
    uint32_t v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const uint64_t s = mix(seed + tid * per_thread + i + u) % nslots;
      const uint8_t* p = buf + s * GRAN;
      if (GRAN == 4) v[u] = __ldg((const uint32_t*)p);
      else if (GRAN == 16) { uint4 t = __ldg((const uint4*)p); v[u] = t.x ^ t.w; }
      else if (GRAN == 32) { uint4 t = __ldg((const uint4*)p); uint4 t2 = __ldg((const uint4*)(p + 16)); v[u] = t.x ^ t2.w; }
      else if (GRAN == 64) { uint4 t = __ldg((const uint4*)p); uint4 t2 = __ldg((const uint4*)(p + 32)); v[u] = t.x ^ t2.w; }
      else { uint4 t = __ldg((const uint4*)p); uint4 t2 = __ldg((const uint4*)(p + 32)); uint4 t3 = __ldg((const uint4*)(p + 64)); uint4 t4 = __ldg((const uint4*)(p + 96)); v[u] = t.x ^ t2.w ^ t3.y ^ t4.z; }
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) acc ^= v[u];
  }
  if (acc == 0x12345) *sink = acc;
}
template <int GRAN, int UNROLL>
void run(const uint8_t* buf, uint64_t span, uint32_t* sink, int blocks_per_sm) {
  const uint64_t nslots = span / GRAN;
  const int threads = 256, blocks = 148 * blocks_per_sm;
  const uint64_t per_thread = 512;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  rr<GRAN, UNROLL><<<blocks, threads>>>(buf, nslots, per_thread, 1, sink);
  cudaEventRecord(a);
  rr<GRAN, UNROLL><<<blocks, threads>>>(buf, nslots, per_thread, 77, sink);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double req = double(blocks) * threads * per_thread;
  const int sect = GRAN <= 32 ? 1 : GRAN / 32;
  printf("gran %3d B unroll %d blocks/SM %d: %.3f ms  %.3e req/s  sectors %.3e/s  sector-bytes %.0f GB/s  (cudaErr %d)\n", GRAN, UNROLL,
         blocks_per_sm, ms, req / ms * 1e3, req * sect / ms * 1e3, req * sect * 32 / ms / 1e6, int(cudaGetLastError()));
}
int main(int argc, char** argv) {
  // argv[1] = "async": the buffer comes from the stream-ordered pool (cudaMallocAsync) instead of
  // cudaMalloc — the library's index arrays do; does the mapping differ (page size / TLB reach)?
  const bool async = argc > 1 && argv[1][0] == 'a';
  const uint64_t cap = 8ull << 30;
  uint8_t* buf; uint32_t* sink;
  if (async) cudaMallocAsync((void**)&buf, cap, 0); else cudaMalloc(&buf, cap);
  cudaMalloc(&sink, 4); cudaMemset(buf, 1, cap);
  printf("allocation: %s\n", async ? "cudaMallocAsync (default pool)" : "cudaMalloc");
  for (uint64_t span : {128ull << 20, 256ull << 20, 384ull << 20, 512ull << 20, 1ull << 30, 2ull << 30, 8ull << 30}) {
    printf("-- span %llu MB\n", (unsigned long long)(span >> 20));
    run<4, 4>(buf, span, sink, 8); run<128, 4>(buf, span, sink, 8);
  }
  return 0;
}
