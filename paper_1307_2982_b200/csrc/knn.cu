// Batched exact MIH k-nearest-neighbour search on the GPU (K4/K5 in SURVEY.md §2.2).
//
// Reference semantics: MihIndex::knn_search (index.hpp:185-253, paper Alg. 3). Step r probes
// ring floor(r/m) of table r mod m; every newly seen id is verified by its full Hamming distance
// and binned; the search stops after step r once the bins at distance <= r hold >= k ids; the
// result is the k smallest (dist, id) pairs.
//
// GPU restatement (bulk-synchronous over a batch of queries; all active queries run the same
// step r in one launch):
//  * mih_probe_kernel: flat work list over (active query, ring index) chunks. A thread unranks
//    its first flip combination (colex combinatorial number system) and walks the rest with
//    Gosper's hack; the enumeration order differs from RingEnumerator's lexicographic order
//    (enumerate.hpp:59-82), which only affects the order trace counters accumulate in.
//  * Dedup without the n-bit mark vector (index.hpp:55-76): a candidate x found at step r is
//    "new" iff r is its first discovery step, r == min_j (m * d_j(q, x) + j), a pure function of
//    x's code. Exactly-once, stateless, and it reproduces unique_candidates.
//  * Verified candidates with dist <= U_q (a per-query upper bound on the k-th distance, tightened
//    every round from the exact histogram) are histogrammed and appended to a bounded per-query
//    buffer; a per-query drop-minimum records whether anything relevant overflowed.
//  * mih_round_end_kernel: termination test sum_{d<=r} hist >= k (index.hpp:209, :232), U update,
//    next active list, and the list of buffers mih_compact_kernel trims to the new bound.
//  * selection: exact top-k of the buffered keys (dist << 32 | id) — select.cu. Queries whose
//    buffer overflowed with a relevant key re-run their steps with the final radius as the bound
//    into exactly-sized buffers.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "knn.cuh"
#include "select.cuh"

namespace mihg {

// A slice of one big bucket, processed by a warp (load balancing for skewed buckets).
struct Piece {
  uint32_t q, lo, cnt, pad;
};

struct Workspace {
  uint64_t nq_cap = 0;
  uint32_t b1 = 0, m = 0, cap = 0;
  DeviceBuffer<uint64_t> qcodes_pad;
  DeviceBuffer<uint32_t> hist_g;  // all-reduced histograms (partitioned calls)
  DeviceBuffer<uint32_t> qsub, hist, ubound, bufcnt, dropmin, act0, act1, counters, final_r;
  DeviceBuffer<uint64_t> buf;
  DeviceBuffer<unsigned long long> trc;
  DeviceBuffer<uint64_t> lookups_prefix;
  DeviceBuffer<Piece> pieces;
  DeviceBuffer<uint32_t> piece_count;
  DeviceBuffer<uint32_t> gstart, grouped;
  DeviceBuffer<uint32_t> compact_list, compact_n;  // (query, new bound) pairs of a round's buffer compactions
  DeviceBuffer<uint64_t> pair_prefix;
  DeviceBuffer<unsigned long long> work_counter;
  uint32_t* h_counter = nullptr;
  cudaStream_t st = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // device-planned radius rounds: nact_dev[r] = queries active entering round r (written by the
  // previous round's end kernel), mirrored into pinned h_nact[r] behind event ev_round[r - 1];
  // ev_probe[2r], [2r+1] bracket round r's probe kernels (profiling)
  DeviceBuffer<uint32_t> nact_dev;
  uint32_t* h_nact = nullptr;
  std::vector<cudaEvent_t> ev_round, ev_probe;
  ~Workspace() {
    if (h_counter) cudaFreeHost(h_counter);
    if (h_nact) cudaFreeHost(h_nact);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    for (cudaEvent_t e : ev_round) cudaEventDestroy(e);
    for (cudaEvent_t e : ev_probe) cudaEventDestroy(e);
  }
};

Index::~Index() {
  if (stream) cudaStreamSynchronize(stream);
  delete ws;
  ws = nullptr;
  stage_q.reset();
  stage_ids.reset();
  stage_dists.reset();
  stage_tr.reset();
  codes.reset();
  d_positions.reset();
  d_subs.reset();
  d_submask.reset();
  for (auto& t : tables)
    if (t) t->release();
  d_tables.reset();
  if (stream) {
    cudaStreamSynchronize(stream);
    cudaStreamDestroy(stream);
  }
}

namespace {

// colex unranking: the idx-th z-subset of {0..s-1} (Gosper order) as a bit mask. Substrings are
// at most 32 bits (table.hpp:31), so masks, ring sizes (<= C(32,16)) and indices fit 32 bits.
__device__ __forceinline__ uint32_t unrank_comb(const uint64_t* __restrict__ binom, uint32_t idx,
                                                uint32_t s, uint32_t z) {
  uint32_t mask = 0;
  uint32_t c = s;
  for (uint32_t t = z; t >= 2; --t) {
    // largest cc < c with C(cc, t) <= idx (C(t - 1, t) = 0 always qualifies): binary search
    uint32_t lo = t - 1, hi = c;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (uint32_t(__ldg(binom + mid * kBinomStride + t)) <= idx) lo = mid;
      else hi = mid;
    }
    mask |= 1u << lo;
    idx -= uint32_t(__ldg(binom + lo * kBinomStride + t));
    c = lo;
  }
  if (z >= 1) mask |= 1u << idx;  // C(cc, 1) = cc
  return mask;
}

// next subset of the same size in increasing numeric order (Gosper's hack); past the last
// subset of a 32-bit ring the value is garbage, never used (the walk stops at the ring end)
__device__ __forceinline__ uint32_t next_comb(uint32_t x) {
  if (x == 0) return 0;
  const uint32_t u = x & (~x + 1);
  const uint32_t v = x + u;
  return v | (((v ^ x) >> 2) >> (__ffs(int(u)) - 1));
}

template <int W>
__device__ __forceinline__ uint64_t pick(const uint64_t* d, uint32_t i) {
  uint64_t r = d[0];
#pragma unroll
  for (int w = 1; w < W; ++w)
    if (i == uint32_t(w)) r = d[w];
  return r;
}

// XOR of the query and one candidate code, held in registers (W > 0) or read from memory.
template <int W>
struct Diff {
  uint64_t d[W];
  __device__ __forceinline__ void load(const uint64_t* __restrict__ codes, uint32_t id,
                                       const uint64_t* qc, uint32_t) {
    uint64_t x[W];
    load_code<W>(codes, id, x);
#pragma unroll
    for (int w = 0; w < W; ++w) d[w] = qc[w] ^ x[w];
  }
  __device__ __forceinline__ uint32_t dist(uint32_t) const {
    uint32_t s = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) s += __popcll(d[w]);
    return s;
  }
  __device__ __forceinline__ uint32_t subdist(const DevSubstring& sb, const uint64_t* submask_j,
                                              uint32_t) const {
    if (sb.contiguous) {
      const uint32_t w = sb.offset >> 6, sh = sb.offset & 63;
      uint64_t v = pick<W>(d, w) >> sh;
      if (sh + sb.len > 64) v |= pick<W>(d, w + 1) << (64 - sh);
      if (sb.len < 64) v &= (uint64_t(1) << sb.len) - 1;
      return __popcll(v);
    }
    uint32_t s = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) s += __popcll(d[w] & __ldg(submask_j + w));
    return s;
  }
};

template <>
struct Diff<0> {
  const uint64_t* x;
  const uint64_t* q;
  __device__ __forceinline__ void load(const uint64_t* __restrict__ codes, uint32_t id,
                                       const uint64_t* qc, uint32_t nw) {
    x = codes + uint64_t(id) * nw;
    q = qc;
  }
  __device__ __forceinline__ uint32_t dist(uint32_t nw) const {
    uint32_t s = 0;
    for (uint32_t w = 0; w < nw; ++w) s += __popcll(__ldg(q + w) ^ __ldg(x + w));
    return s;
  }
  __device__ __forceinline__ uint32_t subdist(const DevSubstring&, const uint64_t* submask_j,
                                              uint32_t nw) const {
    uint32_t s = 0;
    for (uint32_t w = 0; w < nw; ++w)
      s += __popcll((__ldg(q + w) ^ __ldg(x + w)) & __ldg(submask_j + w));
    return s;
  }
};

// Buckets up to inline_max entries are verified by the probing warp; bigger ones are cut into
// pieces of piece_size entries for the warp-per-piece kernel (MIHG_INLINE_MAX / MIHG_PIECE_SIZE).
uint32_t env_u32(const char* name, uint32_t dflt) {
  const char* e = std::getenv(name);
  return e ? uint32_t(std::atoi(e)) : dflt;
}

struct ProbeArgs {
  const uint64_t* codes;
  uint64_t n_codes;        // codes in the index (assert build)
  const uint64_t* qcodes;  // nq * nw
  const uint32_t* qsub;    // nq * m
  const DevTable* tables;  // the index's m tables on the device (mih_solo_kernel switches per step)
  DevTable tab;
  const DevSubstring* subs;
  const uint64_t* submask;
  uint32_t m, a, rr, nw;
  const uint32_t* active;
  uint64_t ring, cpq, total;
  uint32_t chunk;
  uint32_t* hist;  // nullable (re-run pass)
  uint32_t b1;
  const uint32_t* ubound;
  const uint32_t* rlimit;  // re-run: skip queries whose final radius < r
  uint32_t r;
  uint64_t* buf;
  const uint64_t* bufbase;  // nullable: base = q * cap_fixed
  const uint32_t* bufcap;   // nullable: cap = cap_fixed
  uint32_t cap_fixed;
  uint32_t* bufcnt;
  uint32_t* dropmin;
  unsigned long long* trc;  // nullable: 2 per query (candidates, unique)
  Piece* pieces;            // nullable: no piece queue
  uint32_t* piece_count;
  uint32_t piece_cap;
  uint32_t inline_max, inline_max_sparse, piece_size;
  const uint64_t* binom;    // device_binomials()
  // L2-sliced rounds (slice_bits > 0): active queries grouped by the top t bits G of their
  // substring; units enumerated per (slice P, group G) pair, P-major, claimed in order.
  uint32_t slice_bits;
  // device-planned rounds (the host runs ahead of the GPU): the round's active count is read from
  // *d_nact and the work split derived on the device (chunk from *d_chunk when sliced)
  const uint32_t* d_nact;
  uint32_t* d_chunk;
  uint64_t lane_target;  // lanes to keep busy (plan_round)
  double chunk_scale;    // sliced rounds: chunk = nact * ring * chunk_scale (plan_slicing)
  uint32_t prefetch;            // sparse tables: 0 off, 1 next iteration's directory sectors -> L1, 2 -> L2
#ifdef MIHG_TC_DEBUG
  uint32_t debug_probe_only;    // debug build: skip verification (MIHG_DEBUG_PROBE_ONLY=1)
#endif
  uint32_t part_bits, part_id;  // probe-space partition (multi-GPU): top key bits owned
  const uint64_t* pair_prefix;  // 4^t + 1 exclusive unit prefix over (P, G) pairs
  const uint32_t* gstart;       // 2^t + 1 group starts into grouped[]
  const uint32_t* grouped;      // active slots sorted by group
  unsigned long long* work_counter;
};

// Chunking of a round's (queries x ring) work list into warp units of 32 lanes x chunk probes.
__host__ __device__ __forceinline__ uint32_t plan_chunk(uint64_t nact, uint64_t ring, uint64_t target) {
  uint64_t chunk = (nact * ring + target - 1) / target;
  chunk = chunk < 1 ? 1 : (chunk > 256 ? 256 : chunk);
  const uint64_t cap = (ring + 31) / 32 < 1 ? 1 : (ring + 31) / 32;
  return uint32_t(chunk < cap ? chunk : cap);
}

// Per sliced round (one block): group the active queries by G = top t bits of their substring,
// then the unit prefix over (P, G) pairs: within slice P a query of group G has the sub-ring
// with top flip pattern T = P ^ G fixed and rr - popc(T) flips in the low s' = s - t bits.
__global__ void __launch_bounds__(1024) slice_plan_kernel(ProbeArgs p, uint32_t nact, uint64_t span,
                                                          uint32_t* __restrict__ gstart,
                                                          uint32_t* __restrict__ grouped,
                                                          uint64_t* __restrict__ pair_prefix) {
  __shared__ uint32_t hist[256], cur[256];
  __shared__ unsigned long long part[1024];
  if (p.d_nact) {  // device-planned round: this round's count and chunk
    nact = *p.d_nact;
    const double c = floor(double(nact) * double(p.ring) * p.chunk_scale);
    const uint32_t chunk = uint32_t(c < 1.0 ? 1.0 : (c > 256.0 ? 256.0 : c));
    span = uint64_t(chunk) * 32;
    if (threadIdx.x == 0) *p.d_chunk = chunk;
  }
  const uint32_t t = p.slice_bits, G = 1u << t, sb = p.tab.s - t;
  for (uint32_t i = threadIdx.x; i < G; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < nact; i += blockDim.x) {
    const uint32_t q = p.active[i];
    if (p.rlimit && p.r > p.rlimit[q]) continue;
    atomicAdd(&hist[p.qsub[uint64_t(q) * p.m + p.a] >> sb], 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t acc = 0;
    for (uint32_t g = 0; g < G; ++g) {
      gstart[g] = acc;
      cur[g] = acc;
      acc += hist[g];
    }
    gstart[G] = acc;
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < nact; i += blockDim.x) {
    const uint32_t q = p.active[i];
    if (p.rlimit && p.r > p.rlimit[q]) continue;
    grouped[atomicAdd(&cur[p.qsub[uint64_t(q) * p.m + p.a] >> sb], 1u)] = i;
  }
  // units per pair, then a block-wide exclusive scan in P-major order
  const uint32_t npairs = G * G, per = (npairs + blockDim.x - 1) / blockDim.x;
  unsigned long long run = 0;
  for (uint32_t j = 0; j < per; ++j) {
    const uint32_t idx = threadIdx.x * per + j;
    if (idx >= npairs) break;
    const uint32_t P = idx >> t, g = idx & (G - 1), h = __popc(P ^ g);
    uint64_t c = 0;
    const bool owned = p.part_bits == 0 || (P >> (t - p.part_bits)) == p.part_id;
    if (owned && h <= p.rr && p.rr - h <= sb)
      c = uint64_t(hist[g]) * ((p.binom[sb * kBinomStride + (p.rr - h)] + span - 1) / span);
    pair_prefix[idx] = c;  // temporarily the count
    run += c;
  }
  // block-wide exclusive scan of the per-thread sums (warp shuffles, then the 32 warp totals)
  __shared__ unsigned long long wsum[32];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned long long incl = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(~0u, incl, o);
    if (lane >= uint32_t(o)) incl += y;
  }
  if (lane == 31) wsum[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    unsigned long long w = lane < (blockDim.x >> 5) ? wsum[lane] : 0ull;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(~0u, w, o);
      if (lane >= uint32_t(o)) w += y;
    }
    wsum[lane] = w;  // inclusive over warps
    if (lane == 31) {
      pair_prefix[npairs] = w;
      *p.work_counter = 0;
    }
  }
  __syncthreads();
  part[threadIdx.x] = (wid ? wsum[wid - 1] : 0ull) + incl - run;
  __syncthreads();
  unsigned long long acc = part[threadIdx.x];
  for (uint32_t j = 0; j < per; ++j) {
    const uint32_t idx = threadIdx.x * per + j;
    if (idx >= npairs) break;
    const uint64_t c = pair_prefix[idx];
    pair_prefix[idx] = acc;
    acc += c;
  }
}


// Is step (a, rr) the first step that reaches a candidate whose substring distances are d_j?
// New iff for j < a: d_j > rr, and for j > a: d_j >= rr (r == min_j m*d_j + j).
template <int W>
__device__ __forceinline__ bool first_discovery(const Diff<W>& df, const ProbeArgs& p) {
  for (uint32_t j = 0; j < p.m; ++j) {
    if (j == p.a) continue;
    if (j > p.a && p.rr == 0) continue;
    const uint32_t lim = j < p.a ? p.rr : p.rr - 1;
    const uint32_t dj = df.subdist(p.subs[j], p.submask + uint64_t(j) * p.nw, p.nw);
    if (dj <= lim) return false;
  }
  return true;
}

// Per-unit query state kept in registers (the buffer base and capacity are derived on the rare
// append path, which keeps the probe kernel inside its 32-register budget).
struct QueryCtx {
  uint32_t q, U;
};

__device__ __forceinline__ QueryCtx query_ctx(const ProbeArgs& p, uint32_t q) {
  QueryCtx c;
  c.q = q;
  c.U = p.ubound[q];
  return c;
}

// Keepers of a verified pair of entries: histogram + append (one atomic per warp), shared by the
// residual and the full-code verification paths.
__device__ __forceinline__ void keep_entries(const ProbeArgs& p, const QueryCtx& c, bool k0, uint32_t dist0,
                                             uint32_t id0, bool k1, uint32_t dist1, uint32_t id1,
                                             uint32_t b0, uint32_t b1);

// Residual verification (64-bit codes, m = 2 tables of 32 bits): the entry's bits in this table's
// substring are the bucket key v with popc(v ^ q_a) = rr (the ring), so d(q, x) = rr +
// popc(q_other ^ residual), and the other table's substring distance is that popcount itself.
// First discovery (index.hpp:219-230 dedup, see first_discovery): new iff d_other > rr when the
// other table precedes this one (j < a), d_other >= rr when it follows (j > a, rr >= 1).
template <bool kTrace>
__device__ __forceinline__ void verify_residual(const ProbeArgs& p, const QueryCtx& c, bool v0, uint32_t e0,
                                                bool v1, uint32_t e1, uint64_t q, uint64_t& n_new) {
  const uint32_t qo = uint32_t(q >> p.tab.rshift);
  MIHG_DASSERT((!v0 || e0 < p.tab.n_entries) && (!v1 || e1 < p.tab.n_entries));
  uint32_t r0 = 0, r1 = 0;  // candidate codes stream through L2: evict first
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  if (v0) asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r0) : "l"(p.tab.rcodes + e0), "l"(pol));
  if (v1) asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r1) : "l"(p.tab.rcodes + e1), "l"(pol));
  const uint32_t do0 = __popc(qo ^ r0), do1 = __popc(qo ^ r1);
  const uint32_t dist0 = p.rr + do0, dist1 = p.rr + do1;
  const bool other_first = p.a == 1;  // the other table (j = 1 - a) precedes this one
  const bool f0 = other_first ? do0 > p.rr : (p.rr == 0 || do0 >= p.rr);
  const bool f1 = other_first ? do1 > p.rr : (p.rr == 0 || do1 >= p.rr);
  bool k0, k1;
  if constexpr (kTrace) {
    n_new += uint64_t(v0 && f0) + uint64_t(v1 && f1);
    k0 = v0 && f0 && dist0 <= c.U;
    k1 = v1 && f1 && dist1 <= c.U;
  } else {
    k0 = v0 && dist0 <= c.U && f0;
    k1 = v1 && dist1 <= c.U && f1;
  }
  const uint32_t b0 = __ballot_sync(~0u, k0), b1 = __ballot_sync(~0u, k1);
  if ((b0 | b1) == 0) return;
  const uint32_t id0 = k0 ? __ldg(p.tab.ids + e0) : 0u, id1 = k1 ? __ldg(p.tab.ids + e1) : 0u;
  keep_entries(p, c, k0, dist0, id0, k1, dist1, id1, b0, b1);
}

// Verify up to two table entries per lane (index.hpp:219-230): dedup by first discovery, full
// distance, keep if d <= U. All 32 lanes call it together (warp-uniform query, `valid` masks
// lanes without an entry); keepers are appended with ONE atomic per warp and histogrammed with
// one atomic per distinct distance. With inline codes the id is fetched for keepers only.
template <int W, bool kTrace>
__device__ __forceinline__ void verify_entries(const ProbeArgs& p, const QueryCtx& c, bool v0,
                                               uint32_t e0, bool v1, uint32_t e1, const uint64_t* qc,
                                               uint32_t nw, uint64_t& n_new) {
  if constexpr (W == 1) {
    if (p.tab.rcodes) {  // 4-byte residual codes (two 32-bit substrings, see DevTable)
      verify_residual<kTrace>(p, c, v0, e0, v1, e1, qc[0], n_new);
      return;
    }
  }
  Diff<W> d0, d1;
  uint32_t id0 = 0, id1 = 0;
  MIHG_DASSERT((!v0 || e0 < p.tab.n_entries) && (!v1 || e1 < p.tab.n_entries));
  if (p.tab.codes) {
    if (v0) d0.load(p.tab.codes, e0, qc, nw);
    if (v1) d1.load(p.tab.codes, e1, qc, nw);
  } else {
    if (v0) id0 = __ldg(p.tab.ids + e0);
    if (v1) id1 = __ldg(p.tab.ids + e1);
    MIHG_DASSERT((!v0 || id0 < p.n_codes) && (!v1 || id1 < p.n_codes));
    if (v0) d0.load(p.codes, id0, qc, nw);
    if (v1) d1.load(p.codes, id1, qc, nw);
  }
  const uint32_t dist0 = v0 ? d0.dist(nw) : 0u, dist1 = v1 ? d1.dist(nw) : 0u;
  bool k0, k1;
  if constexpr (kTrace) {  // unique_candidates counts every first discovery
    const bool f0 = v0 && first_discovery<W>(d0, p), f1 = v1 && first_discovery<W>(d1, p);
    n_new += uint64_t(f0) + uint64_t(f1);
    k0 = f0 && dist0 <= c.U;
    k1 = f1 && dist1 <= c.U;
  } else {  // only keepers matter: bound first, dedup second
    k0 = v0 && dist0 <= c.U && first_discovery<W>(d0, p);
    k1 = v1 && dist1 <= c.U && first_discovery<W>(d1, p);
  }
  const uint32_t b0 = __ballot_sync(~0u, k0), b1 = __ballot_sync(~0u, k1);
  if ((b0 | b1) == 0) return;
  if (p.tab.codes) {
    if (k0) id0 = __ldg(p.tab.ids + e0);
    if (k1) id1 = __ldg(p.tab.ids + e1);
  }
  keep_entries(p, c, k0, dist0, id0, k1, dist1, id1, b0, b1);
}

__device__ __forceinline__ void keep_entries(const ProbeArgs& p, const QueryCtx& c, bool k0, uint32_t dist0,
                                             uint32_t id0, bool k1, uint32_t dist1, uint32_t id1,
                                             uint32_t b0, uint32_t b1) {
  const uint32_t lane = threadIdx.x & 31, lt = lanemask_lt();
  const uint32_t n0 = __popc(b0), total = n0 + __popc(b1);
  MIHG_DASSERT((!k0 || (dist0 < p.b1 && id0 < p.n_codes)) && (!k1 || (dist1 < p.b1 && id1 < p.n_codes)));
  uint32_t base = 0;
  if (lane == 0) base = atomicAdd(p.bufcnt + c.q, total);
  base = __shfl_sync(~0u, base, 0);
  if (p.hist) {
    const uint32_t key0 = k0 ? dist0 : 0xFFFFFFFFu, key1 = k1 ? dist1 : 0xFFFFFFFEu;
    const uint32_t m0 = __match_any_sync(~0u, key0);
    if (k0 && (m0 & lt) == 0) atomicAdd(p.hist + uint64_t(c.q) * p.b1 + dist0, __popc(m0));
    const uint32_t m1 = __match_any_sync(~0u, key1);
    if (k1 && (m1 & lt) == 0) atomicAdd(p.hist + uint64_t(c.q) * p.b1 + dist1, __popc(m1));
  }
  const uint64_t qbase = p.bufbase ? p.bufbase[c.q] : uint64_t(c.q) * p.cap_fixed;
  const uint32_t qcap = p.bufcap ? p.bufcap[c.q] : p.cap_fixed;
  if (k0) {
    const uint32_t pos = base + __popc(b0 & lt);
    if (pos < qcap) p.buf[qbase + pos] = (uint64_t(dist0) << 32) | id0;
    else atomicMin(p.dropmin + c.q, dist0);
  }
  if (k1) {
    const uint32_t pos = base + n0 + __popc(b1 & lt);
    if (pos < qcap) p.buf[qbase + pos] = (uint64_t(dist1) << 32) | id1;
    else atomicMin(p.dropmin + c.q, dist1);
  }
}

constexpr int kProbeThreads = 256;
constexpr int kProbeWarps = kProbeThreads / 32;

// One warp unit of an MIH step: query q, ring indices [part * 32 * pchunk, ... + 32 * pchunk) of a
// (sub-)ring of `ring` indices with zbits flips among the low sbits key bits (`high` = the fixed
// top flip pattern of a sliced round). s_lo / s_off: the warp's bucket list in shared memory.
template <int W, bool kTrace, int kLaneProbes>
__device__ __forceinline__ void probe_unit(const ProbeArgs& p, uint32_t q, uint32_t part, uint32_t pchunk,
                                           uint32_t ring, uint32_t high, uint32_t zbits, uint32_t sbits,
                                           uint32_t (*s_lo)[32 * kLaneProbes], uint32_t (*s_off)[32 * kLaneProbes]) {
  constexpr int kNzBits = kLaneProbes == 1 ? 1 : kLaneProbes == 2 ? 2 : kLaneProbes == 4 ? 3 : 4;
  const uint32_t nw = W ? W : p.nw;
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5, lt = lanemask_lt();
  const uint32_t span = pchunk * 32;
  const uint32_t ubeg = part * span;
  const uint32_t uend = uint32_t(min(uint64_t(ring), uint64_t(ubeg) + span));
  uint32_t i = ubeg + lane * pchunk;
  const uint32_t iend = min(uend, i + pchunk);
  uint32_t mask = i < iend ? unrank_comb(p.binom, i, sbits, zbits) : 0u;
  const uint32_t qa = p.qsub[uint64_t(q) * p.m + p.a];
  // the query's words stay in memory (L1 hits at verification time): holding them in registers
  // across the probe loop cost more in spills than the reloads (config 2 +2.2%, config 4 +1.5%)
  const uint64_t* qc = p.qcodes + uint64_t(q) * nw;
  const QueryCtx ctx = query_ctx(p, q);
  uint64_t n_cand = 0, n_new = 0;
  for (uint32_t it = 0; it < pchunk; it += kLaneProbes) {
    uint32_t lo[kLaneProbes], cnt[kLaneProbes];
#pragma unroll
    for (int b = 0; b < kLaneProbes; ++b) {
      uint32_t l = 0, h = 0;
      if (i < iend && it + b < pchunk) {
        const uint32_t v = qa ^ (high | mask);
        if (p.part_bits == 0 || (v >> (p.tab.s - p.part_bits)) == p.part_id) probe_bucket(p.tab, v, l, h);
        mask = next_comb(mask);
        ++i;
      }
      lo[b] = l;
      cnt[b] = h - l;
    }
    if (p.prefetch && !p.tab.dense) {
      // the next iteration's directory sectors start their DRAM trip now, overlapping this
      // iteration's verification (no registers held: a cache prefetch)
      uint32_t mk = mask, ii = i;
#pragma unroll
      for (int b = 0; b < kLaneProbes; ++b) {
        if (ii < iend && it + kLaneProbes + b < pchunk) {
          const DirGroup* blk = p.tab.dir + ((qa ^ (high | mk)) >> kDirBucketsLog2);
          if (p.prefetch == 1) asm volatile("prefetch.global.L1 [%0];" ::"l"(blk));
          else asm volatile("prefetch.global.L2 [%0];" ::"l"(blk));
          mk = next_comb(mk);
          ++ii;
        }
      }
    }
    uint32_t mine = 0;
#pragma unroll
    for (int b = 0; b < kLaneProbes; ++b) {
      n_cand += cnt[b];
      if (cnt[b] > (p.tab.dense ? p.inline_max : p.inline_max_sparse) && p.pieces) {
        const uint32_t np = (cnt[b] + p.piece_size - 1) / p.piece_size;
        const uint32_t at = atomicAdd(p.piece_count, np);
        if (at + np <= p.piece_cap) {
          for (uint32_t t = 0; t < np; ++t)
            p.pieces[at + t] = Piece{q, lo[b] + t * p.piece_size, min(p.piece_size, cnt[b] - t * p.piece_size), 0};
          cnt[b] = 0;
        } else {
          for (uint32_t t = at; t < p.piece_cap && t < at + np; ++t) p.pieces[t] = Piece{q, 0, 0, 0};
        }
      }
      mine += cnt[b];
    }
    // warp exclusive prefix of the per-lane totals; buckets laid out lane-major
    uint32_t incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(~0u, incl, o);
      if (lane >= uint32_t(o)) incl += y;
    }
    const uint32_t total = __shfl_sync(~0u, incl, 31);
    if (total == 0) continue;
#ifdef MIHG_TC_DEBUG
    if (p.debug_probe_only) continue;  // traffic attribution: directory probes alone
#endif
    // the non-empty buckets, compacted in lane-major order: (first entry, offset in the union)
    uint32_t nz = 0;
#pragma unroll
    for (int b = 0; b < kLaneProbes; ++b) nz += cnt[b] != 0;
    uint32_t sp = 0, n_ne = 0;
#pragma unroll
    for (int bit = 0; bit < kNzBits; ++bit) {
      const uint32_t bal = __ballot_sync(~0u, (nz >> bit) & 1u);
      sp += __popc(bal & lt) << bit;
      n_ne += __popc(bal) << bit;
    }
    uint32_t off = incl - mine;
#pragma unroll
    for (int b = 0; b < kLaneProbes; ++b) {
      if (cnt[b]) {
        MIHG_DASSERT(sp < uint32_t(32 * kLaneProbes));
        s_lo[wib][sp] = lo[b];
        s_off[wib][sp] = off;
        ++sp;
        off += cnt[b];
      }
    }
    __syncwarp();
    // Entry t of the union belongs to the last bucket whose offset is <= t. Offsets are distinct
    // and ascending, so the buckets starting inside a 64-entry window are the next <= 64 list
    // slots after `cur` (the count of buckets that started before the window): their start
    // positions, OR-reduced into a 64-bit mask, rank every entry with one popcount.
    uint32_t cur = 0;
    const uint32_t le = 0xFFFFFFFFu >> (31 - lane);
    for (uint32_t t0 = 0; t0 < total; t0 += 64) {
      const uint32_t i0 = cur + lane, i1 = i0 + 32;
      const uint32_t o0 = i0 < n_ne ? s_off[wib][i0] - t0 : 64u, o1 = i1 < n_ne ? s_off[wib][i1] - t0 : 64u;
      uint32_t mlo = (o0 < 32 ? 1u << o0 : 0u) | (o1 < 32 ? 1u << o1 : 0u);
      uint32_t mhi = (o0 - 32 < 32 ? 1u << (o0 - 32) : 0u) | (o1 - 32 < 32 ? 1u << (o1 - 32) : 0u);
      mlo = __reduce_or_sync(~0u, mlo);
      mhi = __reduce_or_sync(~0u, mhi);
      const uint32_t nlo = __popc(mlo);
      const uint32_t a0 = cur + __popc(mlo & le) - 1, a1 = cur + nlo + __popc(mhi & le) - 1;
      MIHG_DASSERT(a0 < n_ne && a1 < n_ne && s_off[wib][a0] <= t0 + lane && s_off[wib][a1] <= t0 + 32 + lane);
      uint32_t e[2];
      bool v[2];
      v[0] = t0 + lane < total;
      v[1] = t0 + 32 + lane < total;
      e[0] = s_lo[wib][a0] + (t0 + lane - s_off[wib][a0]);
      e[1] = s_lo[wib][a1] + (t0 + 32 + lane - s_off[wib][a1]);
      cur += nlo + __popc(mhi);
      verify_entries<W, kTrace>(p, ctx, v[0], e[0], v[1], e[1], qc, nw, n_new);
    }
    __syncwarp();
  }
  if (kTrace) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      n_cand += __shfl_xor_sync(~0u, n_cand, o);
      n_new += __shfl_xor_sync(~0u, n_new, o);
    }
    if (lane == 0 && n_cand) {
      atomicAdd(p.trc + 2 * uint64_t(q), (unsigned long long)n_cand);
      if (n_new) atomicAdd(p.trc + 2 * uint64_t(q) + 1, (unsigned long long)n_new);
    }
  }
}

// Warp-cooperative MIH step. A work unit is (active query, warp chunk of 32*chunk ring indices);
// lane l walks its own `chunk` consecutive ring indices, kLaneProbes per iteration (independent
// directory loads in flight). The warp prefix-sums the bucket sizes and verifies the union of the
// entries lane-parallel, two per lane per pass (entry t belongs to the bucket whose
// [off, off + cnt) holds t: a popcount rank over the window's bucket starts), so bucket-size skew
// never idles the warp. Buckets above the inline limit go to the piece queue.
// Resident blocks per SM (MIHG_PROBE_MINB overrides the W <= 2 value): 8 (32 registers) for
// 1-2 probes per lane, 6 (40 registers, spills 172 -> 40 B) for the 4-probe sparse variant.
// Measured B200 sweep: config 4 (4 probes) 8/6/5/4 blocks = 951K/970K/872K/852K q/s; config 3
// (2 probes) 271K/242K/227K/194K — occupancy wins over spills except for the 4-probe kernel.
// (W = 2 at 6 blocks: config 2 895K -> 879K.)
#ifdef MIHG_PROBE_MINB
constexpr int probe_min_blocks(int W, int) { return W <= 2 ? MIHG_PROBE_MINB : 5; }
#else
constexpr int probe_min_blocks(int W, int lane_probes) { return W <= 2 ? (lane_probes >= 4 ? 6 : 8) : 5; }
#endif
template <int W, bool kTrace, int kLaneProbes>
__global__ void __launch_bounds__(kProbeThreads, probe_min_blocks(W, kLaneProbes)) mih_probe_kernel(ProbeArgs p) {
  constexpr int kWarpBuckets = 32 * kLaneProbes;
  __shared__ uint32_t s_lo[kProbeWarps][kWarpBuckets];
  __shared__ uint32_t s_off[kProbeWarps][kWarpBuckets];
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint32_t pchunk = p.chunk;
  uint64_t pcpq = p.cpq, ptotal = p.total;
  if (p.d_nact) {  // device-planned round
    const uint32_t nact = *p.d_nact;
    if (p.slice_bits) {
      pchunk = *p.d_chunk;
    } else {
      pchunk = plan_chunk(nact, p.ring, p.lane_target);
      pcpq = (p.ring + 32ull * pchunk - 1) / (32ull * pchunk);
      ptotal = uint64_t(nact) * pcpq;
    }
  }
  const uint32_t span = pchunk * 32;  // ring indices per warp unit
  const uint64_t nwarps = uint64_t(gridDim.x) * kProbeWarps;
  uint64_t u = blockIdx.x * uint64_t(kProbeWarps) + wib;
  for (;; u += nwarps) {
    uint32_t slot, part;
    uint32_t ring = uint32_t(p.ring), high = 0;
    uint32_t zbits = p.rr, sbits = p.tab.s;
    if (p.slice_bits) {
      // sliced round: units are claimed in order (slice-major), so the warps in flight probe
      // one L2-sized slice of the table at a time
      if (lane == 0) u = atomicAdd(p.work_counter, 1ull);
      u = __shfl_sync(~0u, u, 0);
      const uint32_t npairs = 1u << (2 * p.slice_bits);
      if (u >= __ldg(p.pair_prefix + npairs)) break;
      uint32_t lo_i = 0, hi_i = npairs;  // last pair with prefix <= u (L1-resident table)
      while (hi_i - lo_i > 1) {
        const uint32_t mid = (lo_i + hi_i) >> 1;
        if (__ldg(p.pair_prefix + mid) <= u) lo_i = mid;
        else hi_i = mid;
      }
      const uint32_t P = lo_i >> p.slice_bits, G = lo_i & ((1u << p.slice_bits) - 1);
      sbits = p.tab.s - p.slice_bits;
      const uint32_t T = P ^ G;  // flip pattern of the top slice bits
      zbits = p.rr - __popc(T);
      ring = uint32_t(__ldg(p.binom + sbits * kBinomStride + zbits));
      const uint32_t upq = (ring + span - 1) / span;
      const uint64_t rel = u - __ldg(p.pair_prefix + lo_i);
      const uint32_t kq = uint32_t(rel / upq);
      part = uint32_t(rel - uint64_t(kq) * upq);
      slot = p.grouped[p.gstart[G] + kq];
      high = sbits < 32 ? T << sbits : 0u;
    } else {
      if (u >= ptotal) break;
      slot = uint32_t(u / pcpq);
      part = uint32_t(u - uint64_t(slot) * pcpq);
    }
    const uint32_t q = p.active[slot];
    if (p.rlimit && p.r > p.rlimit[q]) continue;
    probe_unit<W, kTrace, kLaneProbes>(p, q, part, pchunk, ring, high, zbits, sbits, s_lo, s_off);
  }
}

// Small batches: ONE block per query runs the query's whole radius loop (index.hpp:208-234) —
// step r probes ring r / m of table r mod m with the block's warps (probe_unit), a block barrier
// replaces the per-round kernel launches, warp 0 applies the stopping rule and tightens the
// bound. With a few hundred lookups per round the round-synchronous path is bound by launch and
// dependent-load latency per round (config 1: 13 rounds x ~70 us); here a query's rounds cost a
// block barrier each and different queries do not wait for one another. The step's ProbeArgs
// live in shared memory (table, a, rr, r change per step).
template <int W, bool kTrace, int kLaneProbes>
__global__ void __launch_bounds__(kProbeThreads, probe_min_blocks(W, kLaneProbes))
    mih_solo_kernel(ProbeArgs p0, uint32_t nq, uint32_t k, uint32_t bits, uint32_t* __restrict__ ubound,
                    uint32_t* __restrict__ final_r) {
  constexpr int kWarpBuckets = 32 * kLaneProbes;
  __shared__ uint32_t s_lo[kProbeWarps][kWarpBuckets];
  __shared__ uint32_t s_off[kProbeWarps][kWarpBuckets];
  constexpr uint32_t kSoloTables = 16;  // tables kept in shared memory (more: read per step)
  __shared__ ProbeArgs sp;
  __shared__ DevTable s_tab[kSoloTables];
  __shared__ uint32_t s_done;
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  if (threadIdx.x < min(p0.m, kSoloTables)) s_tab[threadIdx.x] = p0.tables[threadIdx.x];
  for (uint32_t q = blockIdx.x; q < nq; q += gridDim.x) {
    __syncthreads();
    if (threadIdx.x == 0) sp = p0;
    for (uint32_t r = 0; r <= bits; ++r) {
      const uint32_t a = r % p0.m, rr = r / p0.m;
      __syncthreads();
      if (threadIdx.x == 0) {
        sp.tab = a < kSoloTables ? s_tab[a] : p0.tables[a];
        sp.a = a;
        sp.rr = rr;
        sp.r = r;
      }
      __syncthreads();
      const uint32_t s = sp.tab.s;
      const uint32_t ring = rr <= s ? uint32_t(__ldg(p0.binom + s * kBinomStride + rr)) : 0u;
      if (ring) {
        const uint32_t want = (ring + 32 * kProbeWarps - 1) / (32 * kProbeWarps);  // one unit per warp
        const uint32_t pchunk = min(max(want, 1u), 256u);
        const uint32_t cpq = (ring + 32 * pchunk - 1) / (32 * pchunk);
        for (uint32_t part = wib; part < cpq; part += kProbeWarps)
          probe_unit<W, kTrace, kLaneProbes>(sp, q, part, pchunk, ring, 0u, rr, s, s_lo, s_off);
      }
      __threadfence();
      __syncthreads();
      if (wib == 0) {  // the stopping rule and the bound, as mih_round_end_kernel (L2 reads: the
                       // histogram is updated by atomics, which bypass L1)
        const uint32_t U = __ldcg(ubound + q);
        const uint32_t* h = p0.hist + uint64_t(q) * p0.b1;
        uint32_t run = 0, settled = 0, newU = U;
        bool found = false;
        for (uint32_t d0 = 0; d0 <= U; d0 += 32) {
          const uint32_t d = d0 + lane;
          uint32_t v = d <= U ? __ldcg(h + d) : 0u;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(~0u, v, o);
            if (lane >= uint32_t(o)) v += y;
          }
          const uint32_t cum = run + v;
          if (r >= d0 && r < d0 + 32) settled = __shfl_sync(~0u, cum, r - d0);
          const uint32_t ok = __ballot_sync(~0u, d <= U && cum >= k);
          if (!found && ok) {
            newU = d0 + __ffs(ok) - 1;
            found = true;
          }
          run = __shfl_sync(~0u, cum, 31);
        }
        if (r > U) settled = run;
        if (lane == 0) {
          if (settled >= k) {
            final_r[q] = r;
            s_done = 1;
          } else {
            ubound[q] = newU;
            s_done = 0;
          }
        }
      }
      __threadfence();
      __syncthreads();
      if (s_done) break;
    }
  }
}

// One warp per queued piece of a big bucket (64 entries per pass).
template <int W, bool kTrace>
__global__ void __launch_bounds__(kProbeThreads, 8) mih_piece_kernel(ProbeArgs p) {
  const uint32_t nw = W ? W : p.nw;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t npieces = min(*p.piece_count, p.piece_cap);
  const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
  for (uint64_t w = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; w < npieces; w += warps) {
    const Piece pc = p.pieces[w];
    if (pc.cnt == 0) continue;
    uint64_t qreg[W ? W : 1];
    const uint64_t* qptr = p.qcodes + uint64_t(pc.q) * nw;
    if constexpr (W > 0) {
#pragma unroll
      for (int x = 0; x < W; ++x) qreg[x] = __ldg(qptr + x);
    }
    const uint64_t* qc = W ? qreg : qptr;
    const QueryCtx ctx = query_ctx(p, pc.q);
    uint64_t n_new = 0;
    for (uint32_t t0 = 0; t0 < pc.cnt; t0 += 64)
      verify_entries<W, kTrace>(p, ctx, t0 + lane < pc.cnt, pc.lo + t0 + lane, t0 + 32 + lane < pc.cnt,
                                pc.lo + t0 + 32 + lane, qc, nw, n_new);
    if (kTrace) {
#pragma unroll
      for (int o = 16; o; o >>= 1) n_new += __shfl_xor_sync(~0u, n_new, o);
      if (lane == 0 && n_new) atomicAdd(p.trc + 2 * uint64_t(pc.q) + 1, (unsigned long long)n_new);
    }
  }
}

__global__ void mih_init_kernel(uint64_t nq, uint32_t bits, uint32_t* ubound, uint32_t* bufcnt,
                                uint32_t* dropmin, uint32_t* act, uint32_t* final_r,
                                uint32_t* nact_dev = nullptr) {
  if (nact_dev && blockIdx.x == 0 && threadIdx.x == 0) nact_dev[0] = uint32_t(nq);
  for (uint64_t q = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; q < nq;
       q += uint64_t(gridDim.x) * blockDim.x) {
    ubound[q] = bits;
    bufcnt[q] = 0;
    dropmin[q] = 0xFFFFFFFFu;
    act[q] = uint32_t(q);
    final_r[q] = 0xFFFFFFFFu;
  }
}

// One warp per active query: termination test, bound update, compaction list.
__global__ void mih_round_end_kernel(const uint32_t* __restrict__ act_in, uint32_t nact,
                                     const uint32_t* __restrict__ d_nact_in,
                                     uint32_t* __restrict__ act_out, uint32_t* __restrict__ nact_out,
                                     const uint32_t* __restrict__ hist, uint32_t b1,
                                     uint32_t* __restrict__ ubound, uint32_t k, uint32_t r,
                                     uint32_t* __restrict__ final_r, const uint32_t* __restrict__ bufcnt,
                                     uint32_t cap, uint32_t* __restrict__ compact_list,
                                     uint32_t* __restrict__ compact_n) {
  __shared__ uint32_t s_n, s_base;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  if (d_nact_in) nact = *d_nact_in;  // device-planned round (grid sized by an upper bound)
  if (blockIdx.x * uint64_t(blockDim.x) >= uint64_t(nact) * 32) return;  // whole block idle
  if (threadIdx.x == 0) s_n = 0;
  __syncthreads();
  const bool active = warp < nact;
  const uint32_t q = active ? act_in[warp] : 0u;
  const uint32_t U = active ? ubound[q] : 0u;
  bool survive = false;
  uint32_t newU = U;
  if (active) {
    const uint32_t* h = hist + uint64_t(q) * b1;
    uint32_t run = 0, settled = 0;
    bool found = false;
    for (uint32_t d0 = 0; d0 <= U; d0 += 32) {
      const uint32_t d = d0 + lane;
      uint32_t v = d <= U ? h[d] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(~0u, v, o);
        if (lane >= o) v += y;
      }
      const uint32_t cum = run + v;
      if (r >= d0 && r < d0 + 32) settled = __shfl_sync(~0u, cum, r - d0);
      const uint32_t ok = __ballot_sync(~0u, d <= U && cum >= k);
      if (!found && ok) {
        newU = d0 + __ffs(ok) - 1;
        found = true;
      }
      run = __shfl_sync(~0u, cum, 31);
    }
    if (r > U) settled = run;  // cannot happen while active (r <= U); kept for safety
    if (settled >= k) {
      if (lane == 0) final_r[q] = r;
    } else {
      survive = true;
    }
  }
  // survivors: one shared-memory slot each, one global atomic per block (the next round's count)
  uint32_t slot = 0;
  if (survive && lane == 0) {
    ubound[q] = newU;
    slot = atomicAdd(&s_n, 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0 && s_n) s_base = atomicAdd(nact_out, s_n);
  __syncthreads();
  if (survive && lane == 0) act_out[s_base + slot] = q;
  // drop buffered keys above the tightened bound once the buffer is half full: such queries are
  // listed for mih_compact_kernel (one block each; in here, the 32 queries of a block would be
  // compacted one after another and a single block would set the kernel's length)
  if (survive && lane == 0 && newU < U && min(bufcnt[q], cap) > cap / 2) {
    const uint32_t at = atomicAdd(compact_n, 1u);
    compact_list[2 * at] = q;
    compact_list[2 * at + 1] = newU;
  }
}

// In-place compaction of the listed queries' candidate buffers to the keys with dist <= the new
// bound (one block per query, block-stride over the list). The buffer's order is irrelevant.
__global__ void __launch_bounds__(1024) mih_compact_kernel(const uint32_t* __restrict__ compact_list,
                                                          const uint32_t* __restrict__ compact_n,
                                                          uint32_t* __restrict__ bufcnt,
                                                          uint64_t* __restrict__ buf, uint32_t cap) {
  __shared__ uint32_t s_w;
  const uint32_t lane = threadIdx.x & 31, njobs = *compact_n;
  for (uint32_t c = blockIdx.x; c < njobs; c += gridDim.x) {
    const uint32_t cq = compact_list[2 * c], cu = compact_list[2 * c + 1];
    const uint32_t cnt = min(bufcnt[cq], cap);
    uint64_t* bq = buf + uint64_t(cq) * cap;
    if (threadIdx.x == 0) s_w = 0;
    __syncthreads();
    for (uint32_t i0 = 0; i0 < cnt; i0 += blockDim.x) {
      const uint32_t i = i0 + threadIdx.x;
      const uint64_t key = i < cnt ? bq[i] : ~0ull;
      const bool keep = i < cnt && uint32_t(key >> 32) <= cu;
      __syncthreads();  // every key of this pass is read before any is overwritten
      const uint32_t bal = __ballot_sync(~0u, keep);
      uint32_t wbase = 0;
      if (lane == 0 && bal) wbase = atomicAdd(&s_w, __popc(bal));
      wbase = __shfl_sync(~0u, wbase, 0);
      if (keep) bq[wbase + __popc(bal & lanemask_lt())] = key;
      __syncthreads();
    }
    if (threadIdx.x == 0) bufcnt[cq] = s_w;
    __syncthreads();
  }
}

// Per query: final trace, candidate count for selection, and the re-run flag.
__global__ void mih_finish_kernel(uint64_t nq, const uint32_t* __restrict__ final_r,
                                  const uint32_t* __restrict__ hist, uint32_t b1,
                                  const uint32_t* __restrict__ bufcnt, uint32_t cap,
                                  const uint32_t* __restrict__ dropmin,
                                  const unsigned long long* __restrict__ trc,
                                  const uint64_t* __restrict__ lookups_prefix, Trace* traces,
                                  uint32_t* __restrict__ seg_count, uint32_t* __restrict__ need,
                                  uint32_t* __restrict__ rerun_list, uint32_t* __restrict__ rerun_n) {
  for (uint64_t q = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; q < nq;
       q += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t R = final_r[q];
    uint64_t tot = 0;
    for (uint32_t d = 0; d <= R; ++d) tot += hist[q * b1 + d];
    need[q] = uint32_t(tot);
    seg_count[q] = min(bufcnt[q], cap);
    if (dropmin[q] <= R) rerun_list[atomicAdd(rerun_n, 1u)] = uint32_t(q);
    if (traces) {
      Trace t;
      t.lookups = lookups_prefix[R];
      t.candidates = trc[2 * q];
      t.unique_candidates = trc[2 * q + 1];
      t.distance_evaluations = t.unique_candidates;
      t.final_radius = R;
      t.reserved = 0;
      traces[q] = t;
    }
  }
}

__global__ void zero_trace_kernel(uint64_t nq, Trace* traces) {
  for (uint64_t q = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; q < nq;
       q += uint64_t(gridDim.x) * blockDim.x)
    traces[q] = Trace{0, 0, 0, 0, 0, 0};
}

// Buckets probed per lane per iteration (MIHG_LANE_PROBES=1|2|4 overrides): 4 for the sparse
// directory of 32-bit tables (more independent DRAM sectors in flight: config 4 +2.5%; 8 at 6 or 5 blocks/SM: -13%), 2 for dense
// offsets (fewer registers: config 3 -7% at 4; measured B200 sweep).
int lane_probes(const DevTable& t) {
  static const int v = [] {
    const char* e = std::getenv("MIHG_LANE_PROBES");
    return e ? std::atoi(e) : 0;
  }();
  return v ? v : (t.dense ? 2 : 4);
}

template <int W, bool kTrace>
void launch_probe(const ProbeArgs& p, cudaStream_t st) {
  const uint64_t blocks_needed = (p.total + kProbeWarps - 1) / kProbeWarps;
  const int lp = lane_probes(p.tab);
  const int minb = lp == 1 ? probe_min_blocks(W, 1) : lp == 4 ? probe_min_blocks(W, 4) : probe_min_blocks(W, 2);
  const uint64_t max_blocks = uint64_t(device_sm_count()) * minb;  // one resident wave
  // unsliced rounds: the host's plan (made with an upper bound of the active count) sizes the
  // grid — small rounds launch few blocks; the unit loop strides, so any grid is correct
  const unsigned grid = p.slice_bits ? unsigned(max_blocks)
                                     : unsigned(std::max<uint64_t>(1, std::min(blocks_needed, max_blocks)));
  if (p.pieces) MIHG_CUDA(cudaMemsetAsync(p.piece_count, 0, 4, st));
  switch (lp) {
    case 1: mih_probe_kernel<W, kTrace, 1><<<grid, kProbeThreads, 0, st>>>(p); break;
    case 4: mih_probe_kernel<W, kTrace, 4><<<grid, kProbeThreads, 0, st>>>(p); break;
    default: mih_probe_kernel<W, kTrace, 2><<<grid, kProbeThreads, 0, st>>>(p);
  }
  MIHG_LAUNCH();
  if (p.pieces) {
    mih_piece_kernel<W, kTrace><<<unsigned(device_sm_count() * 8), kProbeThreads, 0, st>>>(p);
    MIHG_LAUNCH();
  }
}

void dispatch_probe(const ProbeArgs& p, bool trace, cudaStream_t st) {
  switch (p.nw) {
#define MIHG_W(w)                                                   \
  case w:                                                           \
    trace ? launch_probe<w, true>(p, st) : launch_probe<w, false>(p, st); \
    break;
    MIHG_W(1)
    MIHG_W(2)
    MIHG_W(3)
    MIHG_W(4)
#undef MIHG_W
    default:
      trace ? launch_probe<0, true>(p, st) : launch_probe<0, false>(p, st);
  }
}

// Per-query blocks for small batches (mih_solo_kernel; MIHG_SOLO=0 disables, MIHG_SOLO_BUDGET =
// expected lookups of the whole batch below which it is used).
template <int W>
void launch_solo(const ProbeArgs& p, bool trace, uint32_t nq, uint32_t k, uint32_t bits, uint32_t* ubound,
                 uint32_t* final_r, cudaStream_t st) {
  const unsigned grid = unsigned(std::min<uint64_t>(nq, uint64_t(device_sm_count()) * probe_min_blocks(W, 2)));
  if (trace) mih_solo_kernel<W, true, 2><<<grid, kProbeThreads, 0, st>>>(p, nq, k, bits, ubound, final_r);
  else mih_solo_kernel<W, false, 2><<<grid, kProbeThreads, 0, st>>>(p, nq, k, bits, ubound, final_r);
  MIHG_LAUNCH();
}

void dispatch_solo(const ProbeArgs& p, bool trace, uint32_t nq, uint32_t k, uint32_t bits, uint32_t* ubound,
                   uint32_t* final_r, cudaStream_t st) {
  switch (p.nw) {
    case 1: launch_solo<1>(p, trace, nq, k, bits, ubound, final_r, st); break;
    case 2: launch_solo<2>(p, trace, nq, k, bits, ubound, final_r, st); break;
    case 3: launch_solo<3>(p, trace, nq, k, bits, ubound, final_r, st); break;
    case 4: launch_solo<4>(p, trace, nq, k, bits, ubound, final_r, st); break;
    default: launch_solo<0>(p, trace, nq, k, bits, ubound, final_r, st);
  }
}

// Chunking of a round's (queries x ring) work list into warp units of 32 lanes x chunk probes.
void plan_round(ProbeArgs& p, uint64_t nact) {
  p.lane_target = uint64_t(device_sm_count()) * 2048 * 4;  // lanes to keep busy
  const uint64_t chunk = plan_chunk(nact, p.ring, p.lane_target);
  p.chunk = uint32_t(chunk);
  p.cpq = (p.ring + 32 * chunk - 1) / (32 * chunk);
  p.total = nact * p.cpq;
}

// Key-sliced probing for tables whose probe structure is much larger than L2/TLB reach (the
// 32-bit sparse tables of configs 4/5): the ring of every query splits exactly by the top t key
// bits, so a round's work is ordered slice-major and the warps in flight probe one ~128 MB
// region of the directory (and of the table-order codes) at a time. Measured on config 4:
// 546K -> 706K q/s (slice 128 MB, ~128 MB in flight; sweep in DESIGN.md §3). MIHG_SLICE=0
// disables; MIHG_SLICE_MB / MIHG_INFLIGHT_MB tune.
bool slicing_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("MIHG_SLICE");
    return !(e && e[0] == '0');
  }();
  return on;
}

double slice_mb() {
  static const double v = [] {
    const char* e = std::getenv("MIHG_SLICE_MB");
    return e ? std::atof(e) : 128.0;
  }();
  return v;
}

double inflight_mb() {
  static const double v = [] {
    const char* e = std::getenv("MIHG_INFLIGHT_MB");
    return e ? std::atof(e) : 128.0;
  }();
  return v;
}

void plan_slicing(ProbeArgs& p, Workspace& ws, uint64_t nact, cudaStream_t st) {
  p.slice_bits = 0;
  const uint32_t s = p.tab.s;
  const double bytes = p.tab.dense ? double((uint64_t(1) << s) + 1) * 4
                                   : double(uint64_t(1) << (s - kDirBucketsLog2)) * sizeof(DirGroup);
  if (!slicing_enabled() || bytes <= 64.0 * (1 << 20) || double(nact) * double(p.ring) < 4.0e6) return;
  uint32_t t = 0;
  while (bytes / double(1u << t) > slice_mb() * (1 << 20) && t < 8) ++t;
  t = std::max<uint32_t>(t, p.part_bits);  // slices nest inside the rank's key range
  t = std::min<uint32_t>(t, s - 1);
  if (t == 0) return;
  // the in-flight wavefront may span `inflight` slices (~half of L2): units per slice >=
  // resident warps / inflight
  const double resident_warps = double(device_sm_count()) * 64;
  const double inflight = std::max(1.0, std::floor(inflight_mb() * (1 << 20) / (bytes / double(1u << t))));
  p.chunk_scale = inflight / (double(1u << t) * resident_warps * 32.0);
  const double chunk = std::floor(double(nact) * double(p.ring) * p.chunk_scale);
  p.chunk = uint32_t(std::max(1.0, std::min(chunk, 256.0)));
  p.slice_bits = t;
  if (ws.grouped.size() < nact) ws.grouped = DeviceBuffer<uint32_t>(nact, st);
  p.gstart = ws.gstart.get();
  p.grouped = ws.grouped.get();
  p.pair_prefix = ws.pair_prefix.get();
  p.work_counter = ws.work_counter.get();
  slice_plan_kernel<<<1, 1024, 0, st>>>(p, uint32_t(nact), uint64_t(p.chunk) * 32, ws.gstart.get(),
                                        ws.grouped.get(), ws.pair_prefix.get());
  MIHG_LAUNCH();
}

constexpr uint32_t kPieceQueue = 1u << 24;  // 16M pieces (256 MB); overflow falls back inline

void ensure_workspace(Index& idx, uint64_t nq, uint32_t cap, cudaStream_t st) {
  Workspace*& ws = idx.ws;
  const uint32_t b1 = idx.bits + 1;
  if (ws && ws->nq_cap >= nq && ws->b1 == b1 && ws->cap == cap && ws->st == st) return;
  delete ws;
  ws = new Workspace();
  ws->st = st;
  ws->nq_cap = nq;
  ws->b1 = b1;
  ws->m = idx.m;
  ws->cap = cap;
  ws->qsub = DeviceBuffer<uint32_t>(nq * idx.m, st);
  ws->hist = DeviceBuffer<uint32_t>(nq * b1, st);
  ws->ubound = DeviceBuffer<uint32_t>(nq, st);
  ws->bufcnt = DeviceBuffer<uint32_t>(nq, st);
  ws->dropmin = DeviceBuffer<uint32_t>(nq, st);
  ws->act0 = DeviceBuffer<uint32_t>(nq, st);
  ws->act1 = DeviceBuffer<uint32_t>(nq, st);
  ws->counters = DeviceBuffer<uint32_t>(4, st);
  ws->final_r = DeviceBuffer<uint32_t>(nq, st);
  ws->buf = DeviceBuffer<uint64_t>(nq * cap, st);
  ws->trc = DeviceBuffer<unsigned long long>(2 * nq, st);
  ws->lookups_prefix = DeviceBuffer<uint64_t>(b1 + 1, st);
  ws->pieces = DeviceBuffer<Piece>(kPieceQueue, st);
  ws->piece_count = DeviceBuffer<uint32_t>(1, st);
  ws->gstart = DeviceBuffer<uint32_t>(257, st);
  ws->compact_list = DeviceBuffer<uint32_t>(2 * nq, st);
  ws->compact_n = DeviceBuffer<uint32_t>(b1 + 2, st);  // one counter per round, zeroed per search
  ws->pair_prefix = DeviceBuffer<uint64_t>((1u << 16) + 1, st);
  ws->work_counter = DeviceBuffer<unsigned long long>(1, st);
  MIHG_CUDA(cudaMallocHost(reinterpret_cast<void**>(&ws->h_counter), 16));
  MIHG_CUDA(cudaEventCreate(&ws->ev0));
  MIHG_CUDA(cudaEventCreate(&ws->ev1));
  ws->nact_dev = DeviceBuffer<uint32_t>(b1 + 2, st);
  MIHG_CUDA(cudaMallocHost(reinterpret_cast<void**>(&ws->h_nact), (b1 + 2) * 4));
  ws->ev_round.resize(b1 + 2);
  for (cudaEvent_t& e : ws->ev_round) MIHG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  ws->ev_probe.resize(2 * (b1 + 2));
  for (cudaEvent_t& e : ws->ev_probe) MIHG_CUDA(cudaEventCreate(&e));
}

uint32_t read_counter(const uint32_t* d, uint32_t* h, cudaStream_t st) {
  MIHG_CUDA(cudaMemcpyAsync(h, d, 4, cudaMemcpyDeviceToHost, st));
  MIHG_CUDA(cudaStreamSynchronize(st));
  return *h;
}

// Hybrid switch: queries still active when the probe budget is exhausted are finished by the
// exact exhaustive scan. Their MIH state is neutralised so finish/select skip them.
__global__ void neutralise_kernel(const uint32_t* __restrict__ act, uint32_t nact, uint32_t* final_r,
                                  uint32_t* bufcnt, uint32_t* dropmin) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nact; i += gridDim.x * blockDim.x) {
    const uint32_t q = act[i];
    final_r[q] = 0;
    bufcnt[q] = 0;
    dropmin[q] = 0xFFFFFFFFu;
  }
}

__global__ void gather_rows_kernel(const uint64_t* __restrict__ src, const uint32_t* __restrict__ rows,
                                   uint32_t nrows, uint32_t width, uint64_t* __restrict__ dst) {
  const uint64_t total = uint64_t(nrows) * width;
  for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < total;
       t += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t i = t / width;
    dst[t] = src[uint64_t(rows[i]) * width + (t - i * width)];
  }
}

__global__ void scatter_rows_kernel(const uint32_t* __restrict__ ids, const uint32_t* __restrict__ dists,
                                    const uint32_t* __restrict__ rows, uint32_t nrows, uint32_t k,
                                    uint32_t* __restrict__ out_ids, uint32_t* __restrict__ out_dists) {
  const uint64_t total = uint64_t(nrows) * k;
  for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < total;
       t += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t i = t / k;
    out_ids[uint64_t(rows[i]) * k + (t - i * k)] = ids[t];
    out_dists[uint64_t(rows[i]) * k + (t - i * k)] = dists[t];
  }
}

// Cost of one more MIH round for each active query vs an exhaustive scan of that query, in
// 64-bit popcount units (the scan costs n*W per query): one probe ~ 36 + 15*(W-1) units,
// measured on B200 from the MIH probe rate vs the K6 scan rate (config 4, W=1: 36; config 5,
// W=4: ~80). MIHG_HYBRID_ALPHA (default 0.5) scales the scan budget; MIHG_HYBRID=0 disables
// the switch. Traced calls never switch (the trace is defined by the MIH probe sequence).
double hybrid_alpha() {
  static const double v = [] {
    const char* h = std::getenv("MIHG_HYBRID");
    if (h && h[0] == '0') return 0.0;
    const char* e = std::getenv("MIHG_HYBRID_ALPHA");
    return e ? std::atof(e) : 0.5;
  }();
  return v;
}

// Exhaustive-scan cost per (query, code) pair in the same 64-bit-popcount units: W on the POPC
// pipe (K6); the tensor-core scan (K7) is cheaper by the measured B200 ratio of the two kernels'
// pair rates (tools/bench_tcscan.py; MIHG_TC_SPEEDUP overrides).
double scan_cost_per_code(uint32_t bits) {
  const uint32_t W = words_per_code(bits);
  if (scan_kernel_for(bits) != ScanKernel::Tensor) return W;
  const char* e = std::getenv("MIHG_TC_SPEEDUP");
  // measured pair rates on B200 (bench.py --method scan, 1e4 queries): K7 (CTA pairs) 6.4e12
  // pairs/s (64-bit, n = 1e8) ... 5.8e12 (256-bit, n = 1e9); K6 1.95e12 (W=1) ... 5.3e11 (W=4)
  // (W <= 2: no credit — MIH's candidate verification, not charged by the probe count, dominates
  // there; measured config 2 at k = 100 lost 17% when stragglers were switched on the rate ratio)
  const double f = e ? std::atof(e) : (W <= 2 ? 1.0 : W == 3 ? 8.0 : 10.9);
  return W / f;
}

// MIH lookups a query needs under the uniform-code model: R = the first radius
// with n * sum_{d <= R} C(b, d) / 2^b >= k, lookups = sum_{r <= R} C(s_{r mod m}, r / m). Used only
// to skip an MIH prefix that cannot win: clustered data needs fewer lookups than this, so the model
// errs towards MIH, and the caller demands a wide margin before it switches up front.
double uniform_model_lookups(const Index& idx, uint32_t k) {
  const uint32_t b = idx.bits, m = idx.m;
  const double ln2 = std::log(2.0);
  double ln_cum = -INFINITY;  // ln sum_{d <= R} C(b, d)
  uint32_t R = 0;
  for (; R <= b; ++R) {
    const double ln_c = std::lgamma(double(b) + 1) - std::lgamma(double(R) + 1) - std::lgamma(double(b - R) + 1);
    ln_cum = ln_cum == -INFINITY ? ln_c : std::max(ln_cum, ln_c) + std::log1p(std::exp(-std::fabs(ln_cum - ln_c)));
    if (std::log(double(idx.n)) + ln_cum - b * ln2 >= std::log(double(k))) break;
  }
  double lookups = 0;
  for (uint32_t r = 0; r <= std::min(R, b); ++r) {
    const uint32_t s = idx.lengths[r % m], rr = r / m;
    if (rr <= s) lookups += double(host_binom(s, rr));
  }
  return lookups;
}

ProbeArgs make_probe_args(Index& idx, Workspace& ws, const uint64_t* d_q) {
  ProbeArgs p{};
  p.codes = idx.codes.get();
  p.tables = idx.d_tables.get();
  p.n_codes = idx.n;
  p.qcodes = d_q;
  p.qsub = ws.qsub.get();
  p.subs = idx.d_subs.get();
  p.submask = idx.d_submask.get();
  p.m = idx.m;
  p.nw = idx.W;
  p.hist = ws.hist.get();
  p.b1 = idx.bits + 1;
  p.ubound = ws.ubound.get();
  p.buf = ws.buf.get();
  p.cap_fixed = ws.cap;
  p.bufcnt = ws.bufcnt.get();
  p.dropmin = ws.dropmin.get();
  p.trc = ws.trc.get();
  p.pieces = ws.pieces.get();
  p.piece_count = ws.piece_count.get();
  p.piece_cap = kPieceQueue;
  p.binom = device_binomials();
  // dense tables 64, sparse 128 (config 4 +2.1% at 128; config 2 -9% at 128, configs 1/3 neutral)
  static const uint32_t inline_max = env_u32("MIHG_INLINE_MAX", 64);
  static const uint32_t inline_max_sparse = env_u32("MIHG_INLINE_MAX", 128);
  static const uint32_t piece_size = env_u32("MIHG_PIECE_SIZE", 256);
  static const uint32_t prefetch = env_u32("MIHG_PREFETCH", 0);
  p.prefetch = prefetch;
#ifdef MIHG_TC_DEBUG
  p.debug_probe_only = env_u32("MIHG_DEBUG_PROBE_ONLY", 0);
#endif
  p.inline_max = inline_max;
  p.inline_max_sparse = inline_max_sparse;
  p.piece_size = std::max<uint32_t>(32, piece_size);
  return p;
}

// Re-run of the queries whose bounded buffer dropped a key with dist <= final radius: their
// steps 0..R are probed again with U = R into exactly-sized buffers (need = sum_{d<=R} hist),
// without histogram or trace updates. Exact because first discovery is stateless.
struct RerunResult {
  std::vector<uint32_t> list, need, R;
  std::vector<uint64_t> base;
  DeviceBuffer<uint64_t> big;
};

RerunResult rerun_pass(Index& idx, const ProbeArgs& p, const uint32_t* d_rerun, uint32_t nre,
                       const uint32_t* d_need, uint64_t nq, cudaStream_t st) {
  Workspace& ws = *idx.ws;
  const uint32_t m = idx.m;
  RerunResult res;
  res.list.resize(nre);
  res.need.resize(nq);
  res.R.resize(nq);
  MIHG_CUDA(cudaMemcpyAsync(res.list.data(), d_rerun, nre * 4, cudaMemcpyDeviceToHost, st));
  MIHG_CUDA(cudaMemcpyAsync(res.need.data(), d_need, nq * 4, cudaMemcpyDeviceToHost, st));
  MIHG_CUDA(cudaMemcpyAsync(res.R.data(), ws.final_r.get(), nq * 4, cudaMemcpyDeviceToHost, st));
  MIHG_CUDA(cudaStreamSynchronize(st));
  std::sort(res.list.begin(), res.list.end());
  res.base.assign(nq, 0);
  std::vector<uint32_t> hcap(nq, 0);
  uint64_t total = 0;
  uint32_t maxR = 0;
  for (uint32_t q : res.list) {
    res.base[q] = total;
    hcap[q] = res.need[q];
    total += res.need[q];
    maxR = std::max(maxR, res.R[q]);
  }
  res.big = DeviceBuffer<uint64_t>(std::max<uint64_t>(total, 1), st);
  DeviceBuffer<uint64_t> dbase(nq, st);
  DeviceBuffer<uint32_t> dcap(nq, st), dlist(nre, st);
  MIHG_CUDA(cudaMemcpyAsync(dbase.get(), res.base.data(), nq * 8, cudaMemcpyHostToDevice, st));
  MIHG_CUDA(cudaMemcpyAsync(dcap.get(), hcap.data(), nq * 4, cudaMemcpyHostToDevice, st));
  MIHG_CUDA(cudaMemcpyAsync(dlist.get(), res.list.data(), nre * 4, cudaMemcpyHostToDevice, st));
  MIHG_CUDA(cudaMemsetAsync(ws.bufcnt.get(), 0, nq * 4, st));
  ProbeArgs rp = p;
  rp.d_nact = nullptr;  // host-planned: the re-run list size is known
  rp.pieces = ws.pieces.get();
  rp.hist = nullptr;
  rp.trc = nullptr;
  rp.ubound = ws.final_r.get();
  rp.rlimit = ws.final_r.get();
  rp.buf = res.big.get();
  rp.bufbase = dbase.get();
  rp.bufcap = dcap.get();
  rp.active = dlist.get();
  for (uint32_t r = 0; r <= maxR; ++r) {
    const uint32_t a = r % m, rr = r / m, s = idx.lengths[a];
    const uint64_t ring = rr <= s ? host_binom(s, rr) : 0;
    if (!ring) continue;
    rp.tab = idx.tables[a]->view();
    rp.a = a;
    rp.rr = rr;
    rp.r = r;
    rp.ring = ring;
    plan_round(rp, nre);
    plan_slicing(rp, ws, nre, st);
    dispatch_probe(rp, false, st);
  }
  MIHG_CUDA(cudaStreamSynchronize(st));
  return res;
}

void call_allreduce(const Partition* part, void* ptr, uint64_t count, int dtype, cudaStream_t st) {
  if (part->comm) {  // the library's own NCCL communicator: enqueued on the index stream
    comm_allreduce_sum(part->comm, ptr, count, dtype, st);
    return;
  }
  if (!part->allreduce) throw InvalidArgument("partitioned knn: no all-reduce callback");
  const int rc = part->allreduce(part->user, ptr, count, dtype, st);
  if (rc) throw CudaError("partitioned knn: all-reduce callback failed (" + std::to_string(rc) + ")");
}

void knn_chunk(Index& idx, const uint64_t* d_q, uint64_t nq, uint32_t k, uint32_t* d_ids,
               uint32_t* d_dists, Trace* d_tr, cudaStream_t st, const KnnOptions& opt) {
  // a library communicator keeps the collective path even at count 1 (one-rank NCCL group)
  const Partition* part = opt.part && (opt.part->count > 1 || opt.part->comm) ? opt.part : nullptr;
  Workspace& ws = *idx.ws;
  const uint32_t m = idx.m, b1 = idx.bits + 1, cap = ws.cap;
  const unsigned g1 = unsigned(std::min<uint64_t>((nq + 255) / 256, 4096));
  extract_all_keys(idx, d_q, nq, ws.qsub.get(), st);
  MIHG_CUDA(cudaMemsetAsync(ws.hist.get(), 0, nq * b1 * 4, st));
  MIHG_CUDA(cudaMemsetAsync(ws.trc.get(), 0, 2 * nq * 8, st));
  MIHG_CUDA(cudaMemsetAsync(ws.nact_dev.get(), 0, ws.nact_dev.size() * 4, st));
  MIHG_CUDA(cudaMemsetAsync(ws.compact_n.get(), 0, ws.compact_n.size() * 4, st));
  mih_init_kernel<<<g1, 256, 0, st>>>(nq, idx.bits, ws.ubound.get(), ws.bufcnt.get(),
                                       ws.dropmin.get(), ws.act0.get(), ws.final_r.get(), ws.nact_dev.get());
  MIHG_LAUNCH();

  ProbeArgs p = make_probe_args(idx, ws, d_q);
  uint64_t part_lo = 0, part_hi = idx.n;  // id range this rank scans if queries switch to K6
  // the stopping rule's k: the caller's global k when shards hold fewer than k codes (id_shards)
  const uint32_t kstop = part && part->k_stop ? part->k_stop : k;
  if (part && part->k_stop && part->k_stop < k) throw InvalidArgument("partitioned knn: k_stop below k");
  bool hybrid_ok = true;  // the scan switch must be the same decision on every rank
  if (part && part->id_shards) {  // every shard probes every ring; only the counts are global
    if (part->rank >= part->count) throw InvalidArgument("partitioned knn: rank must be < count");
    if (ws.hist_g.size() < nq * b1) ws.hist_g = DeviceBuffer<uint32_t>(ws.nq_cap * b1, st);
  } else if (part) {
    uint32_t bits = 0;
    while ((1u << bits) < part->count) ++bits;
    if ((1u << bits) != part->count || part->rank >= part->count)
      throw InvalidArgument("partitioned knn: count must be a power of two and rank < count");
    for (uint32_t j = 0; j < m; ++j)
      if (idx.lengths[j] < bits) throw InvalidArgument("partitioned knn: substring narrower than log2(count)");
    p.part_bits = bits;
    p.part_id = part->rank;
    if (ws.hist_g.size() < nq * b1) ws.hist_g = DeviceBuffer<uint32_t>(ws.nq_cap * b1, st);
    const uint64_t per = (idx.n + part->count - 1) / part->count;
    part_lo = std::min<uint64_t>(idx.n, uint64_t(part->rank) * per);
    part_hi = std::min<uint64_t>(idx.n, part_lo + per);
    // the last rank's range is the smallest; every rank evaluates the same condition
    const uint64_t last_lo = std::min<uint64_t>(idx.n, uint64_t(part->count - 1) * per);
    hybrid_ok = idx.n - last_lo >= k;
  }

  std::vector<uint64_t> lookups_prefix;
  // Radius rounds, planned on the device: round r reads its active count from nact_dev[r] and
  // its end kernel writes nact_dev[r + 1]; the host enqueues rounds ahead of the GPU and learns
  // the counts from a pinned mirror up to kRunAhead rounds late, so the stream never drains
  // between rounds. Rounds enqueued after the last query stopped see a count of 0 and exit at
  // once. nact_known (the newest count read back) bounds the current count from above (counts
  // never grow): it sizes grids and the slicing decision.
  constexpr uint32_t kRunAhead = 2;
  uint32_t* act_buf[2] = {ws.act0.get(), ws.act1.get()};
  uint64_t nact_known = nq;
  uint32_t r_known = 0;  // nact_known == nact entering round r_known
  uint64_t acc = 0, cand_bound = 0;
  const double alpha = (d_tr || (part && part->id_shards) || !hybrid_ok) ? 0.0 : hybrid_alpha();
  const double scan_pairs = double(idx.n) * scan_cost_per_code(idx.bits),
               probe_pairs = 36.0 + 15.0 * (idx.W - 1);
  uint32_t* switched = nullptr;
  uint64_t nswitched = 0;
  ProfileState& profst = profile();
  std::vector<uint32_t> probed_rounds;
  // read back round `upto`'s end (the count entering round upto + 1), blocking on its event
  auto learn = [&](uint32_t upto) {
    while (r_known <= upto) {
      MIHG_CUDA(cudaEventSynchronize(ws.ev_round[r_known]));
      nact_known = ws.h_nact[r_known + 1];
      ++r_known;
      if (nact_known == 0) return;
    }
  };
  // hopeless MIH: when the uniform model puts the lookups above 16x the scan budget, every query
  // goes to the exhaustive scan at round 0 (config 5, 256-bit uniform: ~220x; configs 1-4: < 1x)
  const bool pre_switch = alpha > 0 && uniform_model_lookups(idx, kstop) * probe_pairs >= 16.0 * alpha * scan_pairs;
  // small batches of light queries: one block per query runs all its rounds (mih_solo_kernel)
  const char* solo_env = std::getenv("MIHG_SOLO");  // read per call: tests run both paths
  const bool solo_on = !(solo_env && solo_env[0] == '0');
  const double solo_budget = std::getenv("MIHG_SOLO_BUDGET") ? std::atof(std::getenv("MIHG_SOLO_BUDGET")) : 4.0e6;
  // (measured: a block per query loses to the round kernels once a query needs thousands of
  // lookups — config 2 / 3 / 4 at 100 queries: 0.6x / 0.45x / 0.1x — and ties at config 1 x 10000)
  const double model_lookups = uniform_model_lookups(idx, kstop);
  bool solo = solo_on && !part && !pre_switch && nq <= 65536 && model_lookups <= 4096.0 &&
              double(nq) * model_lookups <= solo_budget;
  for (uint32_t j = 0; solo && j < m; ++j) {  // no piece queue in there: buckets must fit the inline limit
    const TableStorage& t = *idx.tables[j];
    solo = t.max_bucket <= (t.dense ? p.inline_max : p.inline_max_sparse);
  }
  if (solo) {
    for (uint32_t rr2 = 0; rr2 <= idx.bits; ++rr2) {
      const uint32_t s2 = idx.lengths[rr2 % m];
      acc += rr2 / m <= s2 ? host_binom(s2, rr2 / m) : 0;
      lookups_prefix.push_back(acc);
    }
    ProbeArgs sp = p;
    sp.d_nact = nullptr;
    sp.pieces = nullptr;
    sp.slice_bits = 0;
    sp.part_bits = 0;
    sp.rlimit = nullptr;
    if (profst.enabled) MIHG_CUDA(cudaEventRecord(ws.ev_probe[0], st));
    dispatch_solo(sp, d_tr != nullptr, uint32_t(nq), kstop, idx.bits, ws.ubound.get(), ws.final_r.get(), st);
    if (profst.enabled) {
      MIHG_CUDA(cudaEventRecord(ws.ev_probe[1], st));
      probed_rounds.push_back(0);
    }
    nact_known = 0;
  }
  uint32_t r = 0;
  for (; nact_known > 0; ++r) {
    if (r > idx.bits) throw CudaError("knn: radius loop exceeded the code width (internal error)");
    if (pre_switch && r == 0) {
      switched = act_buf[0];
      nswitched = nq;
      neutralise_kernel<<<unsigned(std::min<uint64_t>((nq + 255) / 256, 1024)), 256, 0, st>>>(
          act_buf[0], uint32_t(nq), ws.final_r.get(), ws.bufcnt.get(), ws.dropmin.get());
      MIHG_LAUNCH();
      break;
    }
    const uint32_t a = r % m, rr = r / m;
    const uint32_t s = idx.lengths[a];
    const uint64_t ring = rr <= s ? host_binom(s, rr) : 0;
    uint32_t* act_in = act_buf[r & 1];
    uint32_t* act_out = act_buf[(r + 1) & 1];
    if (alpha > 0) {
      // the scan of a switched batch costs whole 128-query tiles on the tensor cores (K7), so a few
      // stragglers are charged a full tile's pass over the database
      auto wants_switch = [&](uint64_t nact) {
        const double scan_q = scan_kernel_for(idx.bits) == ScanKernel::Tensor ? double((nact + 127) / 128 * 128)
                                                                               : double(nact);
        return double(acc + ring) * probe_pairs * double(nact) >= alpha * scan_pairs * scan_q;
      };
      if (wants_switch(nact_known)) {  // decide on the exact count entering round r
        if (r > 0) learn(r - 1);
        if (nact_known == 0) break;
        if (wants_switch(nact_known)) {
          switched = act_in;  // every active query has probed the same `acc` buckets so far
          nswitched = nact_known;
          neutralise_kernel<<<unsigned(std::min<uint64_t>((nswitched + 255) / 256, 1024)), 256, 0, st>>>(
              act_in, uint32_t(nswitched), ws.final_r.get(), ws.bufcnt.get(), ws.dropmin.get());
          MIHG_LAUNCH();
          break;
        }
      }
    }
    acc += ring;
    lookups_prefix.push_back(acc);
    // no query can hold more keys than ring x (largest bucket) per round: below the inline limit
    // the round has no piece queue, and below half a buffer no compaction (launch-bound batches)
    const uint64_t maxb = idx.tables[a]->max_bucket;
    cand_bound = std::min<uint64_t>(cand_bound + ring * maxb, uint64_t(1) << 62);
    if (ring) {
      p.tab = idx.tables[a]->view();
      p.pieces = maxb > (p.tab.dense ? p.inline_max : p.inline_max_sparse) ? ws.pieces.get() : nullptr;
      p.a = a;
      p.rr = rr;
      p.r = r;
      p.active = act_in;
      p.ring = ring;
      p.d_nact = ws.nact_dev.get() + r;
      p.d_chunk = ws.counters.get() + 1;
      plan_round(p, nact_known);
      plan_slicing(p, ws, nact_known, st);
      if (profst.enabled) MIHG_CUDA(cudaEventRecord(ws.ev_probe[2 * r], st));
      dispatch_probe(p, d_tr != nullptr, st);
      if (profst.enabled) {
        MIHG_CUDA(cudaEventRecord(ws.ev_probe[2 * r + 1], st));
        probed_rounds.push_back(r);
      }
    }
    const uint32_t* hist_end = ws.hist.get();
    if (part) {  // global histograms: every rank takes the same stopping / bound decision
      MIHG_CUDA(cudaMemcpyAsync(ws.hist_g.get(), ws.hist.get(), nq * b1 * 4, cudaMemcpyDeviceToDevice, st));
      call_allreduce(part, ws.hist_g.get(), nq * b1, 0, st);
      hist_end = ws.hist_g.get();
    }
    // 32 queries (warps) per block: one global atomic per 32 survivors (same-address atomics
    // serialise at the L2)
    const unsigned g = unsigned((nact_known * 32 + 1023) / 1024);
    mih_round_end_kernel<<<g, 1024, 0, st>>>(act_in, uint32_t(nact_known), ws.nact_dev.get() + r, act_out,
                                             ws.nact_dev.get() + r + 1, hist_end, b1, ws.ubound.get(), kstop, r,
                                             ws.final_r.get(), ws.bufcnt.get(), cap, ws.compact_list.get(),
                                             ws.compact_n.get() + r);
    MIHG_LAUNCH();
    if (cand_bound > cap / 2) {
      mih_compact_kernel<<<unsigned(std::min<uint64_t>(nact_known, uint64_t(device_sm_count()) * 2)), 1024, 0, st>>>(
          ws.compact_list.get(), ws.compact_n.get() + r, ws.bufcnt.get(), ws.buf.get(), cap);
      MIHG_LAUNCH();
    }
    MIHG_CUDA(cudaMemcpyAsync(ws.h_nact + r + 1, ws.nact_dev.get() + r + 1, 4, cudaMemcpyDeviceToHost, st));
    MIHG_CUDA(cudaEventRecord(ws.ev_round[r], st));
    // keep at most kRunAhead rounds unread; read any that already finished. Partitioned calls read
    // on the fixed lag only, so every rank enqueues the same rounds (each round carries a
    // collective: an opportunistic early read on one rank would leave the ranks' all-reduces
    // unpaired)
    while (r_known <= r && (r + 1 - r_known > kRunAhead ||
                            (!part && cudaEventQuery(ws.ev_round[r_known]) == cudaSuccess))) {
      learn(r_known);
      if (nact_known == 0) break;
    }
    if (r == idx.bits && nact_known > 0) learn(r);  // the last possible round: drain
  }
  if (profst.enabled) {
    for (uint32_t pr : probed_rounds) {
      float ms = 0;
      MIHG_CUDA(cudaEventSynchronize(ws.ev_probe[2 * pr + 1]));
      MIHG_CUDA(cudaEventElapsedTime(&ms, ws.ev_probe[2 * pr], ws.ev_probe[2 * pr + 1]));
      profst.probe_ms += ms;
      profst.probe_launches += 1;
    }
  }
  MIHG_CUDA(cudaMemcpyAsync(ws.lookups_prefix.get(), lookups_prefix.data(),
                            lookups_prefix.size() * 8, cudaMemcpyHostToDevice, st));
  if (part && d_tr) call_allreduce(part, ws.trc.get(), 2 * nq, 1, st);  // global candidates/unique
  DeviceBuffer<uint32_t> seg_count(nq, st), need(nq, st), rerun(nq, st);
  MIHG_CUDA(cudaMemsetAsync(ws.counters.get(), 0, 4, st));
  mih_finish_kernel<<<g1, 256, 0, st>>>(nq, ws.final_r.get(), ws.hist.get(), b1, ws.bufcnt.get(),
                                        cap, ws.dropmin.get(), ws.trc.get(), ws.lookups_prefix.get(),
                                        d_tr, seg_count.get(), need.get(), rerun.get(),
                                        ws.counters.get());
  MIHG_LAUNCH();
  const uint32_t nre = read_counter(ws.counters.get(), ws.h_counter, st);

  // main selection over the fixed-stride buffers (re-run queries are overwritten below)
  SelectArgs sa;
  sa.keys = ws.buf.get();
  sa.seg_stride = cap;
  sa.seg_count = seg_count.get();
  sa.seg_maxd = ws.final_r.get();
  sa.k = k;
  sa.max_dist = idx.bits;
  sa.id_base = idx.id_base;
  sa.out_ids = d_ids;
  sa.out_dists = d_dists;
  select_topk(sa, uint32_t(nq), st);

  if (nswitched) {  // exhaustive K6 scan for the queries MIH would have spent longer on
    DeviceBuffer<uint64_t> tq(nswitched * idx.W, st);
    DeviceBuffer<uint32_t> ti(nswitched * k, st), td(nswitched * k, st);
    const unsigned gg = unsigned(std::min<uint64_t>((nswitched * idx.W + 255) / 256, 4096));
    gather_rows_kernel<<<gg, 256, 0, st>>>(d_q, switched, uint32_t(nswitched), idx.W, tq.get());
    MIHG_LAUNCH();
    scan_knn_device(idx.codes.get() + part_lo * idx.W, part_hi - part_lo, idx.bits,
                    idx.id_base + uint32_t(part_lo), tq.get(), nswitched, k, ti.get(), td.get(), st);
    scatter_rows_kernel<<<unsigned(std::min<uint64_t>((nswitched * k + 255) / 256, 4096)), 256, 0, st>>>(
        ti.get(), td.get(), switched, uint32_t(nswitched), k, d_ids, d_dists);
    MIHG_LAUNCH();
    profile().switched_queries += nswitched;
  }

  if (nre == 0) return;
  const bool prof = profile().enabled;
  const auto t_re = std::chrono::steady_clock::now();
  if (prof) profile().rerun_queries += nre;
  RerunResult rr_res = rerun_pass(idx, p, rerun.get(), nre, need.get(), nq, st);
  std::vector<uint32_t>& hre = rr_res.list;
  std::vector<uint64_t>& hbase = rr_res.base;
  std::vector<uint32_t>& hneed = rr_res.need;
  std::vector<uint32_t>& hR = rr_res.R;
  DeviceBuffer<uint64_t>& big = rr_res.big;
  // select the re-run queries from their exact buffers
  DeviceBuffer<uint64_t> rows(nre, st), sbase(nre, st);
  DeviceBuffer<uint32_t> scount(nre, st), smaxd(nre, st);
  std::vector<uint64_t> hrows(nre), hsb(nre);
  std::vector<uint32_t> hsc(nre), hmd(nre);
  for (uint32_t i = 0; i < nre; ++i) {
    hrows[i] = hre[i];
    hsb[i] = hbase[hre[i]];
    hsc[i] = hneed[hre[i]];
    hmd[i] = hR[hre[i]];
  }
  MIHG_CUDA(cudaMemcpyAsync(rows.get(), hrows.data(), nre * 8, cudaMemcpyHostToDevice, st));
  MIHG_CUDA(cudaMemcpyAsync(sbase.get(), hsb.data(), nre * 8, cudaMemcpyHostToDevice, st));
  MIHG_CUDA(cudaMemcpyAsync(scount.get(), hsc.data(), nre * 4, cudaMemcpyHostToDevice, st));
  MIHG_CUDA(cudaMemcpyAsync(smaxd.get(), hmd.data(), nre * 4, cudaMemcpyHostToDevice, st));
  SelectArgs sr = sa;
  sr.keys = big.get();
  sr.seg_base_arr = sbase.get();
  sr.seg_stride = 0;
  sr.seg_count = scount.get();
  sr.seg_maxd = smaxd.get();
  sr.out_row = rows.get();
  select_topk(sr, nre, st);
  if (prof) {
    MIHG_CUDA(cudaStreamSynchronize(st));
    profile().rerun_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_re).count();
  }
}

}  // namespace

void knn_device(Index& idx, const uint64_t* d_queries, uint64_t nq, uint32_t k, uint32_t* d_ids,
                uint32_t* d_dists, Trace* d_traces, cudaStream_t st, const KnnOptions& opt) {
  if (k > idx.n) throw InvalidArgument("knn_search: k exceeds database size");
  if (nq == 0) return;
  if (k == 0) {  // index.hpp:189-194: empty result, zero trace
    if (d_traces) {
      zero_trace_kernel<<<unsigned(std::min<uint64_t>((nq + 255) / 256, 4096)), 256, 0, st>>>(nq, d_traces);
      MIHG_LAUNCH();
    }
    return;
  }
  const uint64_t chunk = std::min<uint64_t>(nq, opt.query_chunk);
  // per-query candidate buffer: large k keeps many ties at the k-th distance, so scale the
  // buffer with k (64 k, up to 64K keys) rather than overflowing into the exact re-run pass
  // (config 4, k = 1000: 8192 -> 65536 keys removes ~1.3k re-runs per 10k queries, 189K -> 240K q/s)
  const uint32_t scaled = uint32_t(std::min<uint64_t>(64ull * k, 65536));
  const uint32_t cap = std::max<uint32_t>({env_u32("MIHG_BUFFER_CAP", std::max(opt.buffer_cap, scaled)), 2 * k + 64});
  ensure_workspace(idx, chunk, cap, st);
  for (uint64_t q0 = 0; q0 < nq; q0 += chunk) {  // (partitioned: every rank runs the same chunks)
    const uint64_t cn = std::min(chunk, nq - q0);
    knn_chunk(idx, d_queries + q0 * idx.W, cn, k, d_ids + q0 * k, d_dists + q0 * k,
              d_traces ? d_traces + q0 : nullptr, st, opt);
  }
}


// ---- range_search (index.hpp:149-176, paper Alg. 2) --------------------------------------------
// Steps 0..r of the kNN loop probe exactly the reference's split balls (table j gets rings
// 0..floor((r-j)/m), i.e. ball(r') for j <= a and ball(r'-1) for j > a with r = m r' + a), so
// range search is those rounds with the bound fixed at U = r and no stopping test; every key with
// d <= r is kept and the result is sorted by (dist, id) with one radix sort of
// (query << 45 | dist << 32 | id) keys.
namespace {

__global__ void range_init_kernel(uint64_t nq, uint32_t r, uint32_t* ubound, uint32_t* bufcnt,
                                  uint32_t* dropmin, uint32_t* act, uint32_t* final_r) {
  for (uint64_t q = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; q < nq;
       q += uint64_t(gridDim.x) * blockDim.x) {
    ubound[q] = r;
    bufcnt[q] = 0;
    dropmin[q] = 0xFFFFFFFFu;
    act[q] = uint32_t(q);
    final_r[q] = r;
  }
}

__global__ void range_compose_kernel(const uint64_t* __restrict__ buf, uint32_t cap,
                                     const uint32_t* __restrict__ seg_count,
                                     const uint64_t* __restrict__ rbase, const uint64_t* __restrict__ big,
                                     const uint32_t* __restrict__ need,
                                     const uint64_t* __restrict__ out_off, uint32_t r,
                                     uint64_t* __restrict__ out_keys) {
  __shared__ uint32_t s_at;
  const uint64_t q = blockIdx.x;
  const bool rerun = rbase && rbase[q] != ~0ull;
  const uint64_t* src = rerun ? big + rbase[q] : buf + q * cap;
  const uint32_t cnt = rerun ? need[q] : seg_count[q];
  if (threadIdx.x == 0) s_at = 0;
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) {
    const uint64_t key = src[i];
    if (uint32_t(key >> 32) <= r) out_keys[out_off[q] + atomicAdd(&s_at, 1u)] = (q << 45) | key;
  }
}

__global__ void range_split_kernel(const uint64_t* __restrict__ keys, uint64_t total, uint32_t id_base,
                                   uint32_t* __restrict__ ids, uint32_t* __restrict__ dists) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total;
       i += uint64_t(gridDim.x) * blockDim.x) {
    ids[i] = uint32_t(keys[i]) + id_base;
    dists[i] = uint32_t(keys[i] >> 32) & 0x1FFFu;
  }
}

__global__ void range_trace_fix_kernel(uint64_t nq, Trace* traces) {
  for (uint64_t q = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; q < nq;
       q += uint64_t(gridDim.x) * blockDim.x)
    traces[q].final_radius = 0;  // SearchTrace::final_radius is kNN-only (index.hpp:50)
}

}  // namespace

// One chunk of queries; returns per-query result counts (host) and the sorted device results.
void range_chunk(Index& idx, const uint64_t* d_q, uint64_t nq, uint32_t r, std::vector<uint64_t>& counts,
                 DeviceBuffer<uint32_t>& out_ids, DeviceBuffer<uint32_t>& out_dists, Trace* d_tr,
                 cudaStream_t st) {
  Workspace& ws = *idx.ws;
  const uint32_t m = idx.m, b1 = idx.bits + 1, cap = ws.cap;
  const unsigned g1 = unsigned(std::min<uint64_t>((nq + 255) / 256, 4096));
  extract_all_keys(idx, d_q, nq, ws.qsub.get(), st);
  MIHG_CUDA(cudaMemsetAsync(ws.hist.get(), 0, nq * b1 * 4, st));
  MIHG_CUDA(cudaMemsetAsync(ws.trc.get(), 0, 2 * nq * 8, st));
  range_init_kernel<<<g1, 256, 0, st>>>(nq, r, ws.ubound.get(), ws.bufcnt.get(), ws.dropmin.get(),
                                         ws.act0.get(), ws.final_r.get());
  MIHG_LAUNCH();
  ProbeArgs p = make_probe_args(idx, ws, d_q);
  std::vector<uint64_t> lookups_prefix;
  uint64_t acc = 0;
  for (uint32_t t = 0; t <= r; ++t) {
    const uint32_t a = t % m, rr = t / m, s = idx.lengths[a];
    const uint64_t ring = rr <= s ? host_binom(s, rr) : 0;
    acc += ring;
    lookups_prefix.push_back(acc);
    if (!ring) continue;
    p.tab = idx.tables[a]->view();
    p.a = a;
    p.rr = rr;
    p.r = t;
    p.active = ws.act0.get();
    p.ring = ring;
    plan_round(p, nq);
    plan_slicing(p, ws, nq, st);
    dispatch_probe(p, d_tr != nullptr, st);
  }
  MIHG_CUDA(cudaMemcpyAsync(ws.lookups_prefix.get(), lookups_prefix.data(), lookups_prefix.size() * 8,
                            cudaMemcpyHostToDevice, st));
  DeviceBuffer<uint32_t> seg_count(nq, st), need(nq, st), rerun(nq, st);
  MIHG_CUDA(cudaMemsetAsync(ws.counters.get(), 0, 4, st));
  mih_finish_kernel<<<g1, 256, 0, st>>>(nq, ws.final_r.get(), ws.hist.get(), b1, ws.bufcnt.get(), cap,
                                        ws.dropmin.get(), ws.trc.get(), ws.lookups_prefix.get(), d_tr,
                                        seg_count.get(), need.get(), rerun.get(), ws.counters.get());
  MIHG_LAUNCH();
  if (d_tr) {
    range_trace_fix_kernel<<<g1, 256, 0, st>>>(nq, d_tr);
    MIHG_LAUNCH();
  }
  const uint32_t nre = read_counter(ws.counters.get(), ws.h_counter, st);
  std::vector<uint32_t> hneed(nq);
  MIHG_CUDA(cudaMemcpyAsync(hneed.data(), need.get(), nq * 4, cudaMemcpyDeviceToHost, st));
  MIHG_CUDA(cudaStreamSynchronize(st));
  RerunResult rr_res;
  DeviceBuffer<uint64_t> rbase;
  if (nre) {
    rr_res = rerun_pass(idx, p, rerun.get(), nre, need.get(), nq, st);
    std::vector<uint64_t> hb(nq, ~0ull);
    for (uint32_t q : rr_res.list) hb[q] = rr_res.base[q];
    rbase = DeviceBuffer<uint64_t>(nq, st);
    MIHG_CUDA(cudaMemcpyAsync(rbase.get(), hb.data(), nq * 8, cudaMemcpyHostToDevice, st));
  }
  counts.assign(nq, 0);
  std::vector<uint64_t> off(nq);
  uint64_t total = 0;
  for (uint64_t q = 0; q < nq; ++q) {
    off[q] = total;
    counts[q] = hneed[q];
    total += hneed[q];
  }
  DeviceBuffer<uint64_t> d_off(nq, st), keys(std::max<uint64_t>(total, 1), st);
  MIHG_CUDA(cudaMemcpyAsync(d_off.get(), off.data(), nq * 8, cudaMemcpyHostToDevice, st));
  range_compose_kernel<<<unsigned(nq), 256, 0, st>>>(ws.buf.get(), cap, seg_count.get(), rbase.get(),
                                                      rr_res.big.get(), need.get(), d_off.get(), r,
                                                      keys.get());
  MIHG_LAUNCH();
  uint32_t qbits = 0;
  while ((uint64_t(1) << qbits) < nq) ++qbits;
  radix_sort_keys_u64(keys.get(), total, 45 + qbits, st);
  out_ids = DeviceBuffer<uint32_t>(std::max<uint64_t>(total, 1), st);
  out_dists = DeviceBuffer<uint32_t>(std::max<uint64_t>(total, 1), st);
  if (total) {
    range_split_kernel<<<unsigned(std::min<uint64_t>((total + 255) / 256, 65535)), 256, 0, st>>>(
        keys.get(), total, idx.id_base, out_ids.get(), out_dists.get());
    MIHG_LAUNCH();
  }
  MIHG_CUDA(cudaStreamSynchronize(st));
}

void range_host(Index& idx, const uint64_t* h_q, uint64_t nq, uint32_t r, uint64_t* h_offsets,
                uint32_t* h_ids, uint32_t* h_dists, uint64_t capacity, Trace* h_tr, cudaStream_t st,
                const KnnOptions& opt) {
  if (r > idx.bits) throw InvalidArgument("range_search: radius exceeds code width");
  h_offsets[0] = 0;
  if (nq == 0) return;
  const uint64_t chunk = std::min<uint64_t>(nq, std::min<uint64_t>(opt.query_chunk, uint64_t(1) << 18));
  ensure_workspace(idx, chunk, opt.buffer_cap, st);
  DeviceBuffer<uint64_t> dq(chunk * idx.W, st);
  DeviceBuffer<Trace> dt(h_tr ? chunk : 0, st);
  uint64_t written = 0;
  for (uint64_t q0 = 0; q0 < nq; q0 += chunk) {
    const uint64_t cn = std::min(chunk, nq - q0);
    MIHG_CUDA(cudaMemcpyAsync(dq.get(), h_q + q0 * idx.W, cn * idx.W * 8, cudaMemcpyHostToDevice, st));
    std::vector<uint64_t> counts;
    DeviceBuffer<uint32_t> ids, dists;
    range_chunk(idx, dq.get(), cn, r, counts, ids, dists, h_tr ? dt.get() : nullptr, st);
    uint64_t tot = 0;
    for (uint64_t q = 0; q < cn; ++q) {
      tot += counts[q];
      h_offsets[q0 + q + 1] = written + tot;
    }
    if (h_ids && written + tot <= capacity && tot) {
      MIHG_CUDA(cudaMemcpyAsync(h_ids + written, ids.get(), tot * 4, cudaMemcpyDeviceToHost, st));
      MIHG_CUDA(cudaMemcpyAsync(h_dists + written, dists.get(), tot * 4, cudaMemcpyDeviceToHost, st));
    }
    if (h_tr) MIHG_CUDA(cudaMemcpyAsync(h_tr + q0, dt.get(), cn * sizeof(Trace), cudaMemcpyDeviceToHost, st));
    MIHG_CUDA(cudaStreamSynchronize(st));
    written += tot;
  }
}

}  // namespace mihg
