// Exhaustive batched k-NN on the 5th-generation tensor cores (K7): scan_knn (scan.hpp:43-68) as
// an integer GEMM. sm_100a has no binary MMA, but the int8 tcgen05 MMA is
// exact for 0/1 data: with the database bit x_i in {0, 1} (u8) and the query bit as
// a_i = 1 - 2 q_i in {+1, -1} (s8),
//     sum_i x_i a_i = popc(x) - 2 popc(x & q) = d(q, x) - popc(q),
// so the s32 accumulator is the Hamming distance up to the per-query constant popc(q). One
// M=128 x N=256 x K=32 instruction evaluates 32768 (query, code) pairs on 32 bits; the POPC pipe
// needs 2048 instructions for the same work.
//
// Persistent CTAs (one per SM), each over a contiguous range of (128-query tile, id chunk) work
// items; consecutive items of one query tile form a segment (one id range, one set of lists).
// 22 warps, warp-specialised:
//   warps 0-15  epilogue: thread (warp % 4, lane) owns query row 32 (warp % 4) + lane; group
//               g = warp / 4 drains columns [64 g, 64 g + 64) of every 256-code tile and keeps its
//               own candidate list per query (id order, compacted to the exact top-k when it reaches
//               2k entries; scanlist.cuh, as in K6), under a bound shared by all lists of the query.
//   warps 16-19 producers: each thread takes two codes per tile from the raw ring and expands them
//               to K bytes of 0/1 in the 128-byte-swizzled K-major layout of the B operand.
//   warp 20     TMEM allocation and the single-thread tcgen05.mma issue.
//   warp 21     loader: one thread keeps kRaw raw code tiles in flight from HBM/L2 into shared
//               memory with 1-D TMA bulk copies (cp.async.bulk, mbarrier complete_tx).
// Pipelines: B stages full/empty (producers <-> MMA, mbarriers; tcgen05.commit frees a stage) and
// two TMEM accumulators of 256 columns (MMA <-> epilogue), so the MMA runs one tile ahead of the
// accumulator drain. The query tile (A operand) sits in shared memory in B's layout.
// The per-query selection over the lists is K6's (gather + select_topk), so ties resolve to the
// smaller id exactly as scan.hpp:24-26.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "knn.cuh"
#include "scanlist.cuh"
#include "select.cuh"

namespace mihg {

namespace {

constexpr int kTcM = 128;        // queries per CTA (TMEM lanes)
constexpr int kTcN = 256;        // codes per tile (MMA N)
constexpr int kAcc = 2;          // TMEM accumulators of kTcN columns (all 512 columns)
constexpr int kEpiGroups = 4;    // epilogue groups of 4 warps; group g drains columns [32 g, 32 g + 32)
constexpr int kEpiCols = kTcN / kEpiGroups;
// a list is compacted to its exact top-k when it holds kListSlack * k entries (MIHG_TC_SLACK
// builds: A/B of compaction frequency vs size)
#ifndef MIHG_TC_SLACK
#define MIHG_TC_SLACK 2
#endif
constexpr uint32_t kListSlack = MIHG_TC_SLACK;
constexpr int kEpiWarps = 4 * kEpiGroups;
constexpr int kProdWarps = 4;    // 128 producer threads: one code each per tile
constexpr int kRaw = 4;          // raw code tiles in flight (TMA bulk ring)
constexpr int kTcThreads = (kEpiWarps + kProdWarps + 2) * 32;
constexpr int kMmaWarp = kEpiWarps + kProdWarps;
constexpr int kLoadWarp = kMmaWarp + 1;

struct TcArgs {
  const uint64_t* codes;
  uint64_t n;
  uint32_t bits, k;
  const uint64_t* queries;
  uint64_t nq;
  uint32_t qtiles;
  uint32_t nch;      // id chunks per query tile; work item = (query tile, chunk), tile-major
  uint64_t chunk;    // codes per chunk (multiple of kTcN)
  uint32_t ipc;      // work items per CTA (a contiguous range)
  uint32_t spq;      // CTAs touching one query tile, at most (list slots = spq * kEpiGroups)
  uint32_t L;
  uint64_t* lists;   // [q][slot][L], slot = (CTA - first CTA of the tile) * kEpiGroups + group
  uint32_t* counts;  // [q][slot], zero for unused slots
  uint32_t slots;
  int32_t* dump;     // debug: nq x n distances (tests only), or nullptr
  uint32_t* gbound;  // [q]: smallest k-th distance proven by any list of the query (0xFFFFFFFF = none)
#ifdef MIHG_TC_DEBUG
  unsigned long long* prof;  // debug build only: [32 warps][8] cycle counters summed over CTAs
  uint32_t tl0;              // debug build only: first tile of CTA 0's recorded timeline (MIHG_TC_TL0)
  uint32_t mma_only;         // debug build only: only the MMA stream runs (2: rotating B stages);
                             // results are NOT produced — measures the tensor ceiling
#endif
};

// ---- PTX wrappers (tcgen05 / mbarrier) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
// ---- CTA-pair (cta_group::2) helpers ----
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same shared-memory offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// (the CUTLASS 2x1SM pattern: default .release.cta semantics; the operand bytes reach the tensor
// core through the async proxy, ordered by the writer's fence.proxy.async)
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// wait with cluster-scope acquire (arrivals come from the peer CTA)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!ok);
}
// arrive on the barrier at this offset in both CTAs of the pair once the issued MMAs complete
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(uint16_t(3))
      : "memory");
}
// D[tmem, both SMs] (+)= A[smem, 128 rows per CTA] . B[smem, N/2 rows per CTA]^T, kind::i8, M = 256
__device__ __forceinline__ void tc_mma_i8_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// D[tmem] (+)= A[smem] . B[smem]^T, kind::i8 (A signed, B unsigned, s32 accumulate)
__device__ __forceinline__ void tc_mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Shared-memory matrix descriptor, K-major, 128-byte swizzle: rows of 128 bytes in 1024-byte
// atoms of 8 rows (SBO = 1024), the 16-byte chunk c of row r stored at c ^ (r mod 8); a K extent
// above 128 bytes continues in the next 128-byte K block (a separate rows x 128 B region).
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t addr) {
  return uint64_t((addr & 0x3FFFFu) >> 4) | (uint64_t(16 >> 4) << 16) | (uint64_t(1024 >> 4) << 32) |
         (uint64_t(1) << 46) | (uint64_t(2) << 61);  // version 1, base offset 0, SWIZZLE_128B
}

// Instruction descriptor: kind::i8, D = s32, A = s8 (signed), B = u8, both K-major, M x N.
constexpr uint32_t tc_idesc(uint32_t M, uint32_t N) {
  return (2u << 4) | (1u << 7) | (0u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}


#define TC_R8U(i) "=r"(v[i + 0]), "=r"(v[i + 1]), "=r"(v[i + 2]), "=r"(v[i + 3]), "=r"(v[i + 4]), \
                  "=r"(v[i + 5]), "=r"(v[i + 6]), "=r"(v[i + 7])
// 32 TMEM lanes x 64 consecutive 32-bit columns -> 32 registers per thread, each holding the low
// 16 bits of two adjacent columns (column 2i in bits 0-15, 2i+1 in bits 16-31; measured layout,
// tools/probe/tmem_ld.cu). The accumulators are d(q, x) - popc(q) in [-256, 256], exact in 16
// bits; the packed load moves half the register bytes: 64 columns x 16 warps in 162 clk vs 408
// clk for two plain .x32 loads (B200, same probe), and the minimum tree runs on halfword pairs.
__device__ __forceinline__ void tmem_ld64_pack16(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.pack::16b.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : TC_R8U(0), TC_R8U(8), TC_R8U(16), TC_R8U(24)
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
#undef TC_R8U

// 4 bits -> 4 bytes of 0/1 (bit i -> byte i)
__device__ __forceinline__ uint32_t spread4(uint32_t x) { return (x * 0x00204081u) & 0x01010101u; }

// byte offset of (row r, 16-byte K chunk c) in a 128B-swizzled K-major operand of `rows` rows
template <int KB>
__device__ __forceinline__ uint32_t core_off(uint32_t r, uint32_t c, uint32_t rows) {
  return (c >> 3) * (rows * 128) + (r >> 3) * 1024 + (r & 7) * 128 + (((c & 7) ^ (r & 7)) << 4);
}

// start address of MMA k-step kk (32 bytes of K) in such an operand
__device__ __forceinline__ uint32_t kstep_addr(uint32_t base, int kk, uint32_t rows) {
  return base + (kk >> 2) * (rows * 128) + (kk & 3) * 32;
}

// The 16-byte-aligned part of a raw tile's code bytes (TMA bulk copies need 16-byte alignment and
// size): it starts `skip` bytes into the tile and is `bytes` long; codes outside it (a misaligned
// head, an odd tail) are read with plain loads.
template <int W, int kCodes>
__device__ __forceinline__ void raw_span(const uint64_t* codes, uint64_t id0, uint64_t hi, uint32_t& skip,
                                         uint32_t& bytes) {
  const uintptr_t s = reinterpret_cast<uintptr_t>(codes + min(hi, id0) * W);
  const uintptr_t e = reinterpret_cast<uintptr_t>(codes + min(hi, id0 + kCodes) * W);
  const uintptr_t s16 = (s + 15) & ~uintptr_t(15), e16 = e & ~uintptr_t(15);
  skip = uint32_t(s16 - s);
  bytes = e16 > s16 ? uint32_t(e16 - s16) : 0u;
}

// kPair: a CTA pair (cluster of 2, cta_group::2) shares each 256-code tile: M = 256 queries (128
// rows of A per CTA), each CTA expands and holds N/2 = 128 codes of B, and each SM's TMEM receives
// its 128 query rows x all 256 codes. Per SM, the expansion and the B operand bytes halve.
template <int KB, bool kPair = false>
struct TcCfg {
  static constexpr int W = KB / 64;
  static constexpr uint32_t kOpBytes = KB;
  static constexpr int kSteps = kOpBytes / 32;
  static constexpr uint32_t kKBp = (kOpBytes + 127) / 128 * 128;  // whole 128-byte swizzle rows
  static constexpr int kCodes = kPair ? kTcN / 2 : kTcN;           // codes per CTA per tile
  static constexpr uint32_t kA = kTcM * kKBp;  // A (queries) in shared memory
  static constexpr uint32_t kB = kCodes * kKBp;
  static constexpr int kStages = (kKBp <= 128 ? 4 : 2) * (kPair ? 2 : 1);
  static constexpr uint32_t kRawBytes = kCodes * W * 8;  // one raw tile of packed codes
  static constexpr uint32_t kSmem = 1024 + kA + kStages * kB + kRaw * kRawBytes;  // + barriers/hist
};

template <int KB, bool kDump, bool kPair>
__global__ void __launch_bounds__(kTcThreads, 1) tc_scan_kernel(TcArgs a) {
  using Cfg = TcCfg<KB, kPair>;
  constexpr int kCodes = Cfg::kCodes;
  constexpr int W = Cfg::W;
  constexpr int S = Cfg::kStages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = base;
  uint8_t* sB = base + Cfg::kA;
  uint8_t* sRaw = sB + S * Cfg::kB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sRaw + kRaw * Cfg::kRawBytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + S;
  uint64_t* tfull = bars + 2 * S;
  uint64_t* tempty = bars + 2 * S + kAcc;
  uint64_t* rfull = bars + 2 * S + 2 * kAcc;
  uint64_t* rempty = rfull + kRaw;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rempty + kRaw);
  uint32_t* hist_all = tmem_slot + 4;  // kEpiWarps * (bits + 1)

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef MIHG_TC_DEBUG
  // per-tile event timeline of CTA 0 (tiles kTl0 .. kTl0+63 of the launch): [tile][event] clock64
  const uint32_t kTl0 = a.tl0;
  unsigned long long* tl = a.prof ? a.prof + 32 * 8 : nullptr;
#define TC_TL(t, ev)                                                                        \
  do {                                                                                      \
    if (tl && blockIdx.x < 2 && (t) >= kTl0 && (t) < kTl0 + 64)                               \
      tl[blockIdx.x * 512 + ((t) - kTl0) * 8 + (ev)] = clock64();                             \
  } while (0)
  unsigned long long wcyc[4] = {0, 0, 0, 0};
  auto wait_k = [&](uint64_t* bar, uint32_t parity, int kind) {
    const unsigned long long c0 = a.prof ? clock64() : 0;
    mbar_wait(bar, parity);
    if (a.prof) wcyc[kind] += clock64() - c0;
  };
  const unsigned long long t_start = clock64();
#else
  auto wait_k = [&](uint64_t* bar, uint32_t parity, int) { mbar_wait(bar, parity); };
#define TC_TL(t, ev) ((void)0)
#endif

  const uint32_t rank = kPair ? cluster_rank() : 0u;  // 0: the pair's MMA issuer
  constexpr uint32_t kSides = kPair ? 2 : 1;
  if (warp == kMmaWarp) {
    if (lane == 0) {
      for (int s = 0; s < S; ++s) {
        mbar_init(full + s, kProdWarps * kSides);  // (pair: used in rank 0 only)
        mbar_init(empty + s, 1);
      }
      for (int b = 0; b < kAcc; ++b) {
        mbar_init(tfull + b, 1);
        mbar_init(tempty + b, kEpiWarps * kSides);  // (pair: used in rank 0 only)
      }
      for (int r = 0; r < kRaw; ++r) {
        mbar_init(rfull + r, 1);
        mbar_init(rempty + r, kProdWarps);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    if constexpr (kPair) {  // both CTAs' MMA warps (same warp id) allocate the pair's TMEM
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  if constexpr (kPair) cluster_sync();  // barriers of both CTAs initialised before any remote arrive
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // pair: producers and epilogues report to rank 0's full / tempty barriers
  const uint32_t full_c = kPair ? mapa(smem_u32(full), 0) : 0u;
  const uint32_t tempty_c = kPair ? mapa(smem_u32(tempty), 0) : 0u;

  // This CTA's work items [i0, i1) (tile-major): consecutive items of one query tile form a
  // segment over one contiguous id range, with one candidate list per (query, group).
  // work unit: one CTA, or one CTA pair (both CTAs walk the same items)
  const uint32_t unit = kPair ? blockIdx.x / 2 : blockIdx.x;
  const uint64_t items = uint64_t(a.qtiles) * a.nch;
  const uint64_t i0 = uint64_t(unit) * a.ipc, i1 = min(items, i0 + a.ipc);
  uint32_t tg = 0;  // tiles processed by this CTA so far: drives every pipeline phase
#ifdef MIHG_TC_DEBUG
  uint32_t mo_phase = 0;  // mma_only probe
  uint32_t tiles_total = 0;
#endif
  for (uint64_t it = i0; it < i1;) {
    const uint32_t Q = uint32_t(it / a.nch);
    const uint64_t it_end = min(i1, uint64_t(Q + 1) * a.nch);
    const uint64_t lo = (it - uint64_t(Q) * a.nch) * a.chunk;
    const uint64_t hi = min(a.n, (it_end - uint64_t(Q) * a.nch) * a.chunk);
    const uint32_t T = uint32_t((hi - lo + kTcN - 1) / kTcN);
    const uint32_t slot0 = (unit - uint32_t((uint64_t(Q) * a.nch) / a.ipc)) * kEpiGroups;
    const uint64_t q0 = uint64_t(Q) * kTcM * kSides + rank * kTcM;  // this CTA's 128 query rows
    it = it_end;

    // A operand in shared memory (128B-swizzled K-major, like B): row r = query q0 + r as K bytes
    // of +1 (bit 0) / -1 (bit 1); padding rows zero. Written by warps 0-3 (rows 32 w..).
    if (warp < 4) {
      const uint32_t r = warp * 32 + lane;
      const uint64_t q = q0 + r;
#pragma unroll
      for (int c = 0; c < KB / 16; ++c) {  // 16-byte chunk c = query bits [16 c, 16 c + 16)
        uint4 o = make_uint4(0, 0, 0, 0);
        if (q < a.nq) {
          const uint32_t h = uint32_t(__ldg(a.queries + q * W + (c >> 2)) >> ((c & 3) * 16)) & 0xFFFFu;
          o.x = (spread4(h & 0xF) * 0xFEu) ^ 0x01010101u;
          o.y = (spread4((h >> 4) & 0xF) * 0xFEu) ^ 0x01010101u;
          o.z = (spread4((h >> 8) & 0xF) * 0xFEu) ^ 0x01010101u;
          o.w = (spread4(h >> 12) * 0xFEu) ^ 0x01010101u;
        }
        *reinterpret_cast<uint4*>(sA + core_off<KB>(r, c, kTcM)) = o;
      }
    }
    fence_proxy_async();
    tc_fence_before();
    if constexpr (kPair) cluster_sync();  // both halves of A written before the pair's MMAs
    else __syncthreads();
    tc_fence_after();

#ifdef MIHG_TC_DEBUG
    if (a.mma_only) {
      if (warp == kMmaWarp && lane == 0 && rank == 0) {
        constexpr uint32_t idesc = tc_idesc(kTcM * kSides, kTcN);
        const uint32_t b_addr = smem_u32(sB);
        for (uint32_t t = tg; t < tg + T; ++t) {
#pragma unroll
          for (int kk = 0; kk < Cfg::kSteps; ++kk) {
            const uint64_t ad = smem_desc_sw128(kstep_addr(smem_u32(sA), kk, kTcM));
            const uint64_t bd =
                smem_desc_sw128(kstep_addr(b_addr + (a.mma_only == 2 ? (t % S) * Cfg::kB : 0), kk, kCodes));
            if constexpr (kPair) tc_mma_i8_pair(tmem + (t % kAcc) * kTcN, ad, bd, idesc, kk > 0);
            else tc_mma_i8(tmem + (t % kAcc) * kTcN, ad, bd, idesc, kk > 0);
          }
        }
        if constexpr (kPair) tc_commit_pair(tfull);
        else tc_commit(tfull);
        mbar_wait(tfull, mo_phase);  // drains this segment's MMAs
        mo_phase ^= 1;
      } else if (kPair && warp == kMmaWarp && lane == 0) {
        mbar_wait(tfull, mo_phase);  // the peer's copy of the commit
        mo_phase ^= 1;
      }
      __syncwarp();
    } else
#endif
    if (warp == kMmaWarp) {
      // ===== MMA issuer (pair: rank 0 only, for both SMs) =====
      if (lane == 0 && rank == 0) {
        constexpr uint32_t idesc = tc_idesc(kTcM * kSides, kTcN);
        const uint32_t b_addr = smem_u32(sB);
        for (uint32_t t = tg; t < tg + T; ++t) {
          const uint32_t s = t % S, ph = (t / S) & 1, b = t % kAcc, bph = (t / kAcc) & 1;
          TC_TL(t, 0);
          if constexpr (kPair) {
#ifdef MIHG_TC_DEBUG
            const unsigned long long c0 = a.prof ? clock64() : 0;
            mbar_wait_cluster(tempty + b, bph ^ 1);
            const unsigned long long c1 = a.prof ? clock64() : 0;
            TC_TL(t, 1);
            mbar_wait_cluster(full + s, ph);
            if (a.prof) {
              wcyc[0] += c1 - c0;
              wcyc[1] += clock64() - c1;
            }
#else
            mbar_wait_cluster(tempty + b, bph ^ 1);
            mbar_wait_cluster(full + s, ph);
#endif
          } else {
            wait_k(tempty + b, bph ^ 1, 0);
            TC_TL(t, 1);
            wait_k(full + s, ph, 1);
          }
          TC_TL(t, 2);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < Cfg::kSteps; ++kk) {  // 32 bytes of K per step
            const uint64_t bd = smem_desc_sw128(kstep_addr(b_addr + s * Cfg::kB, kk, kCodes));
            const uint64_t ad = smem_desc_sw128(kstep_addr(smem_u32(sA), kk, kTcM));
            if constexpr (kPair) tc_mma_i8_pair(tmem + b * kTcN, ad, bd, idesc, kk > 0);
            else tc_mma_i8(tmem + b * kTcN, ad, bd, idesc, kk > 0);
          }
          if constexpr (kPair) {
            tc_commit_pair(empty + s);  // frees the B stage in both CTAs
            tc_commit_pair(tfull + b);  // publishes the accumulator in both SMs
          } else {
            tc_commit(empty + s);
            tc_commit(tfull + b);
          }
          TC_TL(t, 3);
        }
      }
      __syncwarp();
    } else if (warp == kLoadWarp) {
      // ===== loader: raw code tiles -> shared memory (TMA bulk copies) =====
      if (lane == 0) {
        for (uint32_t t = tg; t < tg + T; ++t) {
          const uint32_t r = t % kRaw;
          wait_k(rempty + r, ((t / kRaw) & 1) ^ 1, 0);
          const uint64_t id0 = lo + uint64_t(t - tg) * kTcN + rank * kCodes;  // this CTA's codes
          uint32_t skip, bytes;
          raw_span<W, kCodes>(a.codes, id0, hi, skip, bytes);
          const uint32_t bar = smem_u32(rfull + r);
          if (bytes) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(sRaw + r * Cfg::kRawBytes)),
                "l"(reinterpret_cast<const uint8_t*>(a.codes + id0 * W) + skip), "r"(bytes), "r"(bar)
                : "memory");
          } else {
            mbar_arrive(rfull + r);
          }
        }
      }
      __syncwarp();
    } else if (warp >= kEpiWarps) {
      // ===== producers: raw code -> 0/1 bytes (kCodes / 128 codes per thread per tile) =====
      const uint32_t p0 = threadIdx.x - kEpiWarps * 32;
      for (uint32_t t = tg; t < tg + T; ++t) {
        const uint32_t s = t % S, ph = (t / S) & 1, r = t % kRaw;
        const uint64_t id0 = lo + uint64_t(t - tg) * kTcN + rank * kCodes;
        uint32_t skip, tbytes;
        raw_span<W, kCodes>(a.codes, id0, hi, skip, tbytes);
        wait_k(rfull + r, (t / kRaw) & 1, 0);
        uint64_t cur[kCodes / 128][W];
#pragma unroll
        for (int h = 0; h < kCodes / 128; ++h) {
          const uint32_t p = p0 + 128 * h;
          const uint64_t id = id0 + p;
          if (p * W * 8 >= skip && (p + 1) * W * 8 <= skip + tbytes) {
            const uint64_t* src = reinterpret_cast<const uint64_t*>(sRaw + r * Cfg::kRawBytes + p * W * 8 - skip);
#pragma unroll
            for (int w = 0; w < W; ++w) cur[h][w] = src[w];
          } else if (id < hi) {  // misaligned head / odd tail of the tile
#pragma unroll
            for (int w = 0; w < W; ++w) cur[h][w] = __ldg(a.codes + id * W + w);
          } else {
#pragma unroll
            for (int w = 0; w < W; ++w) cur[h][w] = 0;
          }
        }
        wait_k(empty + s, ph ^ 1, 1);
        uint8_t* dst = sB + s * Cfg::kB;
#pragma unroll
        for (int h = 0; h < kCodes / 128; ++h) {
          const uint32_t p = p0 + 128 * h;
#pragma unroll
          for (int c = 0; c < KB / 16; ++c) {
            const uint32_t hh = uint32_t(cur[h][c >> 2] >> ((c & 3) * 16)) & 0xFFFFu;
            const uint4 o = make_uint4(spread4(hh & 0xF), spread4((hh >> 4) & 0xF), spread4((hh >> 8) & 0xF),
                                       spread4(hh >> 12));
            *reinterpret_cast<uint4*>(dst + core_off<KB>(p, c, kCodes)) = o;
          }
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          if constexpr (kPair) mbar_arrive_cluster(full_c + s * 8);  // rank 0's barrier
          else mbar_arrive(full + s);
          mbar_arrive(rempty + r);  // the raw words were consumed by the expansion above

        }
      }
    } else {
      // ===== epilogue: TMEM -> registers -> bound test -> candidate list =====
      // Accept bound per query: min(own, shared). own = bits until the list is first compacted,
      // then (its k-th distance) - 1: a later id at that distance ranks below all k kept entries.
      // shared = gbound[q], the smallest k-th distance any list of this query has proven
      // (atomicMin after each compaction); ties at it are still accepted (another slot may hold
      // smaller ids).
      const uint32_t g = warp >> 2, quad = warp & 3;
      const uint32_t row = quad * 32 + lane;
      const uint64_t q = q0 + row;
      const bool qvalid = q < a.nq;
      const uint64_t* qp = a.queries + (qvalid ? q : 0) * W;
      int32_t pq = 0;
      if (qvalid)
        for (int w = 0; w < W; ++w) pq += __popcll(__ldg(qp + w));
      int32_t own = qvalid ? int32_t(a.bits) : -1;
      uint32_t cnt = 0;
      const uint32_t slot = slot0 + g;
      uint64_t* list = a.lists + ((qvalid ? q : 0) * a.slots + slot) * uint64_t(a.L);
      uint32_t* hist = hist_all + warp * (a.bits + 1);
      const uint32_t taddr0 = tmem + ((quad * 32) << 16) + g * kEpiCols;
      // the shared bound is refreshed every 4 tiles from a load issued 4 tiles earlier (L2 latency)
      uint32_t gb_next = qvalid ? __ldcg(a.gbound + q) : 0u;
      int32_t shared_b = qvalid ? int32_t(a.bits) : -1;
      for (uint32_t t = tg; t < tg + T; ++t) {
        const uint32_t b = t % kAcc;
        if (((t - tg) & 3) == 0 && qvalid) {
          shared_b = int32_t(min(gb_next, a.bits));
          gb_next = __ldcg(a.gbound + q);
        }
        wait_k(tfull + b, (t / kAcc) & 1, 0);  // the tile's MMAs are complete
        if (warp == 0 && lane == 0) TC_TL(t, 4);
#ifdef MIHG_TC_DEBUG
        if (tl && blockIdx.x == 0 && lane == 0 && t >= kTl0 && t < kTl0 + 64)  // per-warp: tile seen
          tl[2 * 512 + (warp * 64 + (t - kTl0)) * 2] = clock64();
#endif
        tc_fence_after();
        static_assert(kEpiCols == 64, "packed epilogue drains 64 columns per group");
        {
        uint32_t v[32];
        tmem_ld64_pack16(taddr0 + b * kTcN, v);
        tc_fence_before();  // accumulator drained into registers: hand it back
        __syncwarp();
        if (lane == 0) {
          if constexpr (kPair) mbar_arrive_cluster(tempty_c + b * 8);  // rank 0's barrier
          else mbar_arrive(tempty + b);
          if (warp == 0) TC_TL(t, 5);
#ifdef MIHG_TC_DEBUG
          if (tl && blockIdx.x == 0 && t >= kTl0 && t < kTl0 + 64)  // per-warp: tile released
            tl[2 * 512 + (warp * 64 + (t - kTl0)) * 2 + 1] = clock64();
          if (tl && blockIdx.x < 2 && t >= kTl0 && t < kTl0 + 64)  // the last epilogue warp's release
            atomicMax(tl + blockIdx.x * 512 + (t - kTl0) * 8 + 6, clock64());
#endif
        }
        const uint64_t id0 = lo + uint64_t(t - tg) * kTcN + g * kEpiCols;
        if constexpr (kDump) {
          if (qvalid)
            for (int j = 0; j < 64; ++j) {
              const int32_t x = int32_t(int16_t(uint16_t(v[j >> 1] >> ((j & 1) * 16))));
              if (id0 + j < hi) a.dump[q * a.n + id0 + j] = x + pq;
            }
        }
        const int32_t thr = min(own, shared_b) - pq;
        // halfword-SIMD tree minimum over the 64 packed values
        uint32_t m16[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) m16[i] = __vmins2(v[2 * i], v[2 * i + 1]);
#pragma unroll
        for (int w = 8; w >= 1; w >>= 1)
#pragma unroll
          for (int i = 0; i < w; ++i) m16[i] = __vmins2(m16[i], m16[i + w]);
        const int32_t mn = min(int32_t(int16_t(uint16_t(m16[0]))), int32_t(int16_t(uint16_t(m16[0] >> 16))));
        if (mn <= thr) {
          // hits straight from the accumulator: d = value + popc(q) exactly, no code word re-read.
          // The values go to a thread-local copy first (L1), read back by dynamic column index,
          // so the register-resident drain loop keeps its budget.
          uint32_t tmp[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) tmp[i] = v[i];
          const uint32_t t2 = uint32_t(uint16_t(int16_t(thr))) * 0x00010001u;
          uint64_t m = 0;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const uint32_t le = __vcmples2(v[i], t2);  // 0xFFFF per halfword <= thr
            m |= uint64_t((le & 1u) | ((le >> 15) & 2u)) << (2 * i);
          }
          while (m) {
            const uint32_t j = __ffsll(static_cast<long long>(m)) - 1;
            m &= m - 1;
            const uint64_t id = id0 + j;
            if (id >= hi) break;
            const int32_t val = int32_t(int16_t(uint16_t(tmp[j >> 1] >> ((j & 1) * 16))));
            list[cnt++] = (uint64_t(val + pq) << 32) | uint32_t(id);
          }
        }
        // warp-cooperative compaction of every list that reached 2k entries (scanlist.cuh)
        uint32_t need = __ballot_sync(~0u, cnt >= kListSlack * a.k);
        while (need) {
          const int src = __ffs(need) - 1;
          need &= need - 1;
          uint64_t* l2 = reinterpret_cast<uint64_t*>(__shfl_sync(~0u, reinterpret_cast<uintptr_t>(list), src));
          uint32_t c2 = __shfl_sync(~0u, cnt, src);
          __syncwarp();
          // every entry of the list is <= the owner's bound + 1 (own = last k-th distance - 1)
          const uint32_t tau = min(a.bits, uint32_t(__shfl_sync(~0u, own, src) + 1));
#ifdef MIHG_TC_DEBUG
          const unsigned long long cc0 = clock64();
#endif
          const uint32_t nt = compact_list(l2, c2, tau, a.k, hist);
#ifdef MIHG_TC_DEBUG
          if (a.prof) {
            wcyc[2] += clock64() - cc0;
            wcyc[3] += 1;
          }
#endif
          if (lane == uint32_t(src)) {
            cnt = c2;
            own = int32_t(nt) - 1;
            atomicMin(a.gbound + q, nt);
#ifdef MIHG_TC_DEBUG
            if (tl && blockIdx.x < 2 && t >= kTl0 && t < kTl0 + 64)  // compactions during this tile
              atomicAdd(tl + blockIdx.x * 512 + (t - kTl0) * 8 + 7, 1ull);
#endif
          }
          __syncwarp();
        }
        }
      }
      if (qvalid) a.counts[q * a.slots + slot] = cnt;
    }
    tg += T;
#ifdef MIHG_TC_DEBUG
    tiles_total += T;
#endif
    // segment end: every MMA of the segment was drained by the epilogue, so A may be reloaded
    tc_fence_before();
    if constexpr (kPair) cluster_sync();
    else __syncthreads();
    tc_fence_after();
  }
#ifdef MIHG_TC_DEBUG
  if (a.prof && lane == 0) {
    unsigned long long* pr = a.prof + warp * 8;
    atomicAdd(pr + 0, clock64() - t_start);
    for (int i = 0; i < 4; ++i) atomicAdd(pr + 1 + i, wcyc[i]);
    atomicAdd(pr + 5, (unsigned long long)tiles_total);
  }
#endif
  if constexpr (kPair) {
    tc_fence_before();
    cluster_sync();  // both SMs done with the pair's TMEM and barriers
    tc_fence_after();
    if (warp == kMmaWarp) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  } else if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int KB, bool kPair>
size_t tc_smem_bytes(uint32_t bits) {
  using Cfg = TcCfg<KB, kPair>;
  return Cfg::kSmem + (2 * Cfg::kStages + 2 * kAcc + 2 * kRaw) * 8 + 16 + size_t(kEpiWarps) * (bits + 1) * 4;
}

template <int KB, bool kDump, bool kPair>
void launch_tc_k(const TcArgs& a, uint32_t grid, cudaStream_t st) {
  const size_t smem = tc_smem_bytes<KB, kPair>(a.bits);
  auto* fn = tc_scan_kernel<KB, kDump, kPair>;
  MIHG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  if constexpr (kPair) {  // clusters of two CTAs on one TPC
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kTcThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    MIHG_CUDA(cudaLaunchKernelEx(&cfg, fn, a));
  } else {
    fn<<<grid, kTcThreads, smem, st>>>(a);
  }
  MIHG_LAUNCH();
}

template <int KB, bool kPair>
void launch_tc(const TcArgs& a, uint32_t grid, cudaStream_t st) {
  if (a.dump) launch_tc_k<KB, true, kPair>(a, grid, st);
  else launch_tc_k<KB, false, kPair>(a, grid, st);
}

}  // namespace

bool tc_scan_supported(uint32_t bits) { return bits >= 1 && bits <= 256; }

namespace {
__global__ void kth_column_kernel(const uint32_t* __restrict__ dists, uint64_t nq, uint32_t k,
                                  uint32_t* __restrict__ out) {
  const uint64_t q = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (q < nq) out[q] = dists[q * k + (k - 1)];
}
}  // namespace

// Codes in the bound-seeding sample (0: none): MIHG_TC_SEED=<codes> enables it when the database
// is at least 64x larger and the sample holds at least 16 k codes. Off by default: measured
// neutral to -2% at n = 1e8 (the lists' own bounds tighten within the first tiles of a segment).
uint64_t tc_seed_codes(uint64_t n, uint32_t k) {
  const char* e = std::getenv("MIHG_TC_SEED");
  const uint64_t s = e ? std::strtoull(e, nullptr, 10) : 0;
  return (s >= 16ull * k && n >= 64 * s) ? s : 0;
}

// CTA-pair (cta_group::2) geometry by default (n = 1e8 x 256-bit, 1e4 queries: 39.4K -> 48.9K
// q/s; 64-bit: same within noise); MIHG_TC_PAIR=0 selects one CTA per tile.
bool tc_pair_enabled() {
  const char* e = std::getenv("MIHG_TC_PAIR");  // read per call: tests run both geometries
  return !(e && e[0] == '0');
}

// K7: the exhaustive k-NN of scan_knn_device on the tensor cores (same results bit for bit).
void tc_scan_knn_device(const uint64_t* d_codes, uint64_t n, uint32_t bits, uint32_t id_base,
                        const uint64_t* d_queries, uint64_t nq, uint32_t k, uint32_t* d_ids,
                        uint32_t* d_dists, cudaStream_t st, int32_t* d_dump) {
  if (k > n) throw InvalidArgument("scan_knn: k exceeds database size");
  if (!tc_scan_supported(bits)) throw InvalidArgument("tc_scan: code width must be 1..256 bits");
  if (nq == 0 || k == 0) return;
  const uint32_t W = words_per_code(bits);
  const uint32_t L = kListSlack * k + kEpiCols;
  const bool pair = tc_pair_enabled();
  const uint64_t tileq = pair ? 2 * kTcM : kTcM;  // queries per work unit (CTA or CTA pair)
  const uint64_t sms = uint64_t(device_sm_count()) / (pair ? 2 : 1);  // work units in flight
  for (uint64_t q0 = 0; q0 < nq;) {
    uint64_t qn = nq - q0;
    uint64_t qtiles = (qn + tileq - 1) / tileq;
    // Persistent CTAs, one per SM, each over a contiguous range of (query tile, chunk) items.
    // nch is a multiple of sms / gcd(qtiles, sms) so the items divide evenly over the SMs, with
    // at least 8 items per CTA; chunks of at least 16 tiles.
    uint64_t g = sms, r = qtiles;
    while (r) { const uint64_t t = g % r; g = r; r = t; }
    const uint64_t step = sms / g;
    uint64_t nch = step;
    while (nch * qtiles < 8 * sms) nch += step;
    nch = std::min<uint64_t>(nch, std::max<uint64_t>(1, n / (16 * kTcN)));
    uint64_t chunk = ((n + nch - 1) / nch + kTcN - 1) / kTcN * kTcN;
    nch = (n + chunk - 1) / chunk;
    uint64_t items = qtiles * nch, ipc = (items + sms - 1) / sms;
    auto spq_of = [&](uint64_t qt, uint64_t nchv, uint64_t ipcv) {
      uint64_t m = 1;
      for (uint64_t Q = 0; Q < qt; ++Q) m = std::max(m, ((Q + 1) * nchv - 1) / ipcv - (Q * nchv) / ipcv + 1);
      return m;
    };
    uint64_t spq = spq_of(qtiles, nch, ipc);
    // list memory bound (~2 GiB): fewer queries per pass when k is large
    const uint64_t per_q = kEpiGroups * spq * uint64_t(L) * 8 * 2;
    const uint64_t qmax = std::max<uint64_t>(tileq, (uint64_t(2) << 30) / per_q / tileq * tileq);
    if (qn > qmax) {
      qn = qmax;
      qtiles = qn / tileq;
      items = qtiles * nch;
      ipc = (items + sms - 1) / sms;
      spq = spq_of(qtiles, nch, ipc);
    }
    const uint32_t grid = uint32_t((items + ipc - 1) / ipc) * (pair ? 2 : 1);
    TcArgs a{};
    a.codes = d_codes;
    a.n = n;
    a.bits = bits;
    a.k = k;
    a.queries = d_queries + q0 * W;
    a.nq = qn;
    a.qtiles = uint32_t(qtiles);
    a.nch = uint32_t(nch);
    a.chunk = chunk;
    a.ipc = uint32_t(ipc);
    a.spq = uint32_t(spq);
    a.L = L;
    a.slots = uint32_t(kEpiGroups * spq);
    a.dump = d_dump;
#ifdef MIHG_TC_DEBUG  // timing probes of a debug build (make TCDEBUG=1); never in the product .so
    if (const char* mo = std::getenv("MIHG_TC_MMA_ONLY")) a.mma_only = uint32_t(std::atoi(mo));
    a.tl0 = 200;
    if (const char* t0 = std::getenv("MIHG_TC_TL0")) a.tl0 = uint32_t(std::atoi(t0));
    const char* pe = std::getenv("MIHG_TC_PROF");
    const bool dbg_prof = pe && pe[0] == '1';
    constexpr size_t kProfWords = 32 * 8 + 2 * 64 * 8 + 16 * 64 * 2;
    DeviceBuffer<unsigned long long> profbuf(dbg_prof ? kProfWords : 1, st);
    if (dbg_prof) {
      MIHG_CUDA(cudaMemsetAsync(profbuf.get(), 0, kProfWords * 8, st));
      a.prof = profbuf.get();
    }
#endif
    DeviceBuffer<uint64_t> lists(qn * a.slots * L, st), gathered(qn * a.slots * L, st);
    DeviceBuffer<uint32_t> counts(qn * a.slots, st), gcount(qn, st), gbound(qn, st);
    MIHG_CUDA(cudaMemsetAsync(counts.get(), 0, qn * a.slots * 4, st));
    MIHG_CUDA(cudaMemsetAsync(gbound.get(), 0xFF, qn * 4, st));
    // Seed every query's shared bound with the k-th smallest distance over a sample of the database
    // (the first `seed` codes, K6 on the POPC pipe): an upper bound on the global k-th distance, so
    // the lists start filtered instead of accepting everything until their first compactions
    // (the hit storm at the start of every segment). Exact: only codes with d > bound are dropped,
    // and the bound is inclusive (ties kept).
    const uint64_t seed = tc_seed_codes(n, k);
    if (seed) {
      DeviceBuffer<uint32_t> si(qn * k, st), sd(qn * k, st);
      popc_scan_knn_device(d_codes, seed, bits, 0, d_queries + q0 * W, qn, k, si.get(), sd.get(), st);
      kth_column_kernel<<<unsigned((qn + 255) / 256), 256, 0, st>>>(sd.get(), qn, k, gbound.get());
      MIHG_LAUNCH();
    }
    a.gbound = gbound.get();
    a.lists = lists.get();
    a.counts = counts.get();
    // live kernel timing for the bench's roofline (mihg_profile), on the launching stream
    static thread_local cudaEvent_t ev[2] = {nullptr, nullptr};
    const bool prof = profile().enabled;
    if (prof) {
      if (!ev[0]) {
        MIHG_CUDA(cudaEventCreate(&ev[0]));
        MIHG_CUDA(cudaEventCreate(&ev[1]));
      }
      MIHG_CUDA(cudaEventRecord(ev[0], st));
    }
    if (pair) {
      switch (W) {
        case 1: launch_tc<64, true>(a, grid, st); break;
        case 2: launch_tc<128, true>(a, grid, st); break;
        case 3: launch_tc<192, true>(a, grid, st); break;
        default: launch_tc<256, true>(a, grid, st); break;
      }
    } else {
      switch (W) {
        case 1: launch_tc<64, false>(a, grid, st); break;
        case 2: launch_tc<128, false>(a, grid, st); break;
        case 3: launch_tc<192, false>(a, grid, st); break;
        default: launch_tc<256, false>(a, grid, st); break;
      }
    }
    if (prof) MIHG_CUDA(cudaEventRecord(ev[1], st));
#ifdef MIHG_TC_DEBUG
    if (dbg_prof) {
      static unsigned long long h[32 * 8 + 2 * 64 * 8 + 16 * 64 * 2];
      MIHG_CUDA(cudaMemcpyAsync(h, a.prof, sizeof(h), cudaMemcpyDeviceToHost, st));
      MIHG_CUDA(cudaStreamSynchronize(st));
      for (int w = 0; w <= kLoadWarp; ++w) {
        const double tl = double(h[w * 8 + 5] ? h[w * 8 + 5] : 1);
        fprintf(stderr, "tcprof warp %2d: tiles %llu cyc/tile %.0f wait0 %.0f wait1 %.0f compaction cyc/call %.0f calls/tile %.4f\n", w,
                h[w * 8 + 5], h[w * 8] / tl, h[w * 8 + 1] / tl, h[w * 8 + 2] / tl,
                h[w * 8 + 3] / double(h[w * 8 + 4] ? h[w * 8 + 4] : 1), h[w * 8 + 4] / tl);
      }
      fprintf(stderr, "tcprof grid %u ipc %u nch %u spq %u\n", grid, a.ipc, a.nch, a.spq);
      // timeline of CTA 0 (relative to the MMA's wait start of the first recorded tile)
      const unsigned long long* T = h + 32 * 8;
      const unsigned long long z = T[0];
      fprintf(stderr, "tctl tile: mma_wait_start tempty_ok full_ok issued | epi_seen epi_released epi_max_released | compactions\n");
      // per epilogue warp of CTA 0: tile seen / released, relative to warp 0's seen time of the tile
      const unsigned long long* PW = T + 2 * 512;
      for (int i = 0; i < 16; ++i) {
        fprintf(stderr, "tcwarp tile %2d:", i);
        for (int w = 0; w < 16; ++w)
          fprintf(stderr, " %5lld/%5lld", (long long)(PW[(w * 64 + i) * 2] - PW[i * 2]),
                  (long long)(PW[(w * 64 + i) * 2 + 1] - PW[i * 2]));
        fprintf(stderr, "\n");
      }
      // CTA 1 (the pair's second SM) on its own clock: deltas to its first epi_seen
      const unsigned long long* U = T + 512;
      const unsigned long long z1 = U[4];
      for (int i = 0; i < 64; i += 1)
        fprintf(stderr, "tctl %2d: %8lld %8lld %8lld %8lld | %8lld %8lld %8lld | %8lld || cta1 epi %8lld %8lld %8lld prod %8lld\n", i,
                (long long)(T[i * 8] - z), (long long)(T[i * 8 + 1] - z), (long long)(T[i * 8 + 2] - z),
                (long long)(T[i * 8 + 3] - z), (long long)(T[i * 8 + 4] - z), (long long)(T[i * 8 + 5] - z),
                (long long)(T[i * 8 + 6] - z), (long long)T[i * 8 + 7], (long long)(U[i * 8 + 4] - z1),
                (long long)(U[i * 8 + 5] - z1), (long long)(U[i * 8 + 6] - z1), (long long)U[i * 8 + 7]);
    }
#endif
    gather_lists_kernel<<<unsigned(qn), 256, 0, st>>>(lists.get(), counts.get(), a.slots, L, gathered.get(),
                                                      gcount.get());
    MIHG_LAUNCH();
    SelectArgs sa;
    sa.keys = gathered.get();
    sa.seg_stride = uint64_t(a.slots) * L;
    sa.seg_count = gcount.get();
    sa.k = k;
    sa.max_dist = bits;
    sa.id_base = id_base;
    sa.out_ids = d_ids + q0 * k;
    sa.out_dists = d_dists + q0 * k;
    select_topk(sa, uint32_t(qn), st);
    if (prof) {
      float ms = 0;
      MIHG_CUDA(cudaEventSynchronize(ev[1]));
      MIHG_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[1]));
      profile().scan_ms += ms;
      profile().scan_launches += 1;
    }
    q0 += qn;
  }
}

}  // namespace mihg
