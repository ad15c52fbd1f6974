// Access-pattern model of one MIH lookup on a 32-bit sparse table (config 4), to compare table
// layouts before building them. OLD: 16 B directory read (random in a DIR-byte slice), then for
// 29% of the lookups a dependent 4 B read at a random place of an RC-byte range. NEW (packed group
// records): 4 B offset read (random in an OFF-byte slice, L2-resident), for PG of the lookups a
// dependent 16 B header read at a random place of a REC-byte range, and for 29% a 4 B read 16-80 B
// behind the header (same 128 B line). Prints lookups/s.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33; return x;
}
constexpr int U = 4;
__global__ void old_layout(const uint8_t* __restrict__ dir, uint64_t dir_bytes, const uint8_t* __restrict__ rc, uint64_t rc_bytes,
                           uint64_t per_thread, uint64_t seed, uint32_t* sink) {
  const uint64_t tid = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  uint32_t acc = 0;
  for (uint64_t i = 0; i < per_thread; i += U) {
    uint4 g[U]; uint64_t h[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { h[u] = mix(seed + tid * per_thread + i + u); g[u] = __ldg((const uint4*)(dir + ((h[u] % dir_bytes) & ~15ull))); }
    uint32_t r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool ne = ((h[u] >> 40) % 100) < 29;
      const uint64_t pos = ((h[u] >> 8) + g[u].x) % rc_bytes & ~3ull;
      r[u] = ne ? __ldg((const uint32_t*)(rc + pos)) : g[u].y;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= r[u];
  }
  if (acc == 0x12345) *sink = acc;
}
__global__ void new_layout(const uint8_t* __restrict__ off, uint64_t off_bytes, const uint8_t* __restrict__ rec, uint64_t rec_bytes,
                           uint32_t pg, uint64_t per_thread, uint64_t seed, uint32_t* sink) {
  const uint64_t tid = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  uint32_t acc = 0;
  for (uint64_t i = 0; i < per_thread; i += U) {
    uint32_t o[U]; uint64_t h[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { h[u] = mix(seed + tid * per_thread + i + u); o[u] = __ldg((const uint32_t*)(off + ((h[u] % off_bytes) & ~3ull))); }
    uint4 g[U]; uint64_t pos[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool gne = ((h[u] >> 48) % 100) < pg;
      pos[u] = (((h[u] >> 8) + o[u]) % rec_bytes) & ~15ull;
      g[u] = gne ? __ldg((const uint4*)(rec + pos[u])) : make_uint4(o[u], 0, 0, 0);
    }
    uint32_t r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool ne = ((h[u] >> 40) % 100) < 29;
      const uint64_t p2 = pos[u] + 16 + ((g[u].x + (h[u] >> 20)) & 63ull & ~3ull);
      r[u] = ne ? __ldg((const uint32_t*)(rec + (p2 < rec_bytes ? p2 : 0))) : g[u].y;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= r[u];
  }
  if (acc == 0x12345) *sink = acc;
}
int main() {
  const uint64_t cap = 6ull << 30;
  uint8_t* buf; uint32_t* sink;
  cudaMalloc(&buf, cap); cudaMalloc(&sink, 4); cudaMemset(buf, 0, cap);
  const int blocks = 148 * 6, threads = 256; const uint64_t per_thread = 1024;
  const double lookups = double(blocks) * threads * per_thread;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  for (int rep = 0; rep < 2; ++rep) {
    for (uint64_t scale : {1ull, 2ull, 4ull}) {  // slice sizes: 128/256 MB x scale
      const uint64_t dirb = (128ull << 20) / scale * 1, rcb = (256ull << 20) / scale;
      cudaEventRecord(a); old_layout<<<blocks, threads>>>(buf, dirb, buf + (2ull << 30), rcb, per_thread, 7 + rep, sink); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("OLD dir %4llu MB rcodes %4llu MB: %.3e lookups/s\n", (unsigned long long)(dirb >> 20), (unsigned long long)(rcb >> 20), lookups / ms * 1e3);
      for (uint32_t pg : {50u, 65u, 80u}) {
        const uint64_t offb = (32ull << 20) / scale, recb = (384ull << 20) / scale;
        cudaEventRecord(a); new_layout<<<blocks, threads>>>(buf, offb, buf + (2ull << 30), recb, pg, per_thread, 7 + rep, sink); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        if (rep) printf("NEW off %4llu MB records %4llu MB, P(group non-empty) %u%%: %.3e lookups/s\n", (unsigned long long)(offb >> 20), (unsigned long long)(recb >> 20), pg, lookups / ms * 1e3);
      }
    }
  }
  printf("cudaErr %d\n", int(cudaGetLastError()));
  return 0;
}
