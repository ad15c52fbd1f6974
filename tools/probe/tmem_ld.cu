// Probe (tools only, not product code): semantics and throughput of tcgen05.ld shapes on B200.
//  1) 32x32b.x32.pack::16b: which TMEM columns land in which register halves.
//  2) TMEM -> register throughput per SM for 32x32b.x32 vs .x32.pack::16b (16 warps, 4 per
//     subpartition, each re-reading 64 columns of its lanes), in bytes of TMEM columns per clock.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe/tmem_ld tools/probe/tmem_ld.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

#define R8(i) "=r"(v[i]), "=r"(v[i + 1]), "=r"(v[i + 2]), "=r"(v[i + 3]), "=r"(v[i + 4]), "=r"(v[i + 5]), "=r"(v[i + 6]), "=r"(v[i + 7])
__device__ __forceinline__ void ld32(uint32_t ta, uint32_t (&v)[32]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
               : R8(0), R8(8), R8(16), R8(24) : "r"(ta));
}
__device__ __forceinline__ void ld32p(uint32_t ta, uint32_t (&v)[32]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
               : R8(0), R8(8), R8(16), R8(24) : "r"(ta));
}
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__global__ void __launch_bounds__(512, 1) probe(uint32_t* out, int mode, int iters, unsigned long long* cyc) {
  __shared__ uint32_t slot;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  const uint32_t quad = warp & 3, row = quad * 32 + lane;
  if (warp < 4) {  // column c of lane row = row * 1000 + c (c < 256), 16 columns per store
    for (uint32_t c0 = 0; c0 < 256; c0 += 16) {
      uint32_t w[16];
      for (int i = 0; i < 16; ++i) w[i] = row * 1000 + c0 + i;
      asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                   ::"r"(tmem + ((quad * 32) << 16) + c0), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]),
                   "r"(w[6]), "r"(w[7]), "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (mode == 0) {  // semantics: lane 0 of warp 0, first packed load of columns from 0
    if (warp == 0) {
      uint32_t v[32];
      ld32p(tmem, v);
      wait_ld();
      if (lane == 0)
        for (int i = 0; i < 32; ++i) out[i] = v[i];
      ld32(tmem, v);
      wait_ld();
      if (lane == 0)
        for (int i = 0; i < 32; ++i) out[32 + i] = v[i];
    }
  } else {  // throughput: every warp reads its quadrant's columns [64 g, 64 g + 64) repeatedly
    const uint32_t g = warp >> 2;
    uint32_t acc = 0;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      uint32_t v[32], u[32];
      const uint32_t ta = tmem + ((quad * 32) << 16) + (g * 64) % 256;
      if (mode == 1) {  // two plain loads of 32 columns = 64 columns
        ld32(ta, v);
        ld32(ta + 32, u);
        wait_ld();
        for (int i = 0; i < 32; ++i) acc += v[i] ^ u[i];
      } else {  // one packed load (columns per register per the semantics probe)
        ld32p(ta, v);
        wait_ld();
        for (int i = 0; i < 32; ++i) acc += v[i];
      }
    }
    __syncthreads();
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) *cyc = t1 - t0;
    if (acc == 0x12345678) out[0] = acc;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  uint32_t* d;
  unsigned long long* dc;
  cudaMalloc(&d, 64 * 4);
  cudaMalloc(&dc, 8);
  probe<<<1, 512>>>(d, 0, 0, dc);
  uint32_t h[64];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("packed x32 (lane 0 = row 0, column c holds c):\n");
  for (int i = 0; i < 32; ++i) printf("  r%-2d lo %5u hi %5u\n", i, h[i] & 0xFFFF, h[i] >> 16);
  printf("plain x32: r0 %u r1 %u r31 %u\n", h[32], h[33], h[63]);
  const int iters = 20000;
  for (int mode = 1; mode <= 2; ++mode) {
    probe<<<148, 512>>>(d, mode, iters, dc);
    unsigned long long c = 0;
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    // columns read per iteration per CTA: 16 warps x 32 lanes x 64 columns x 4 bytes (mode 1);
    // mode 2 reads x32 packed (the semantics line says how many columns that is)
    printf("mode %d: %.1f cycles per iteration (16 warps), %s\n", mode, double(c) / iters,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
