// Per-(slot, query) candidate lists shared by the exhaustive scans (K6 scan.cu, K7 tcscan.cu):
// an append-only list of packed keys (dist << 32 | id) in id order per slot, compacted in place
// to its exact top-k when it fills, then gathered per query for the final selection.
#pragma once
#include "common.cuh"

namespace mihg {
namespace {

// Register-resident variant for lists of at most 32 * R entries: every load of the list is issued
// at once (one memory round trip instead of one per 32 entries in each of the two passes), then
// the k-th distance (radix select on ballots) and the in-order compaction work on registers.
template <int R>
__device__ __forceinline__ uint32_t compact_list_regs(uint64_t* list, uint32_t& cnt, uint32_t tau, uint32_t k,
                                                      uint32_t* hist) {
  const uint32_t lane = threadIdx.x & 31;
  uint64_t v[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const uint32_t i = uint32_t(r) * 32 + lane;
    v[r] = i < cnt ? list[i] : ~0ull;
  }
  // k-th smallest distance by a radix select over the registers (ballots, no shared-memory
  // histogram: the distances of a list cluster under its bound, so histogram atomics would
  // serialise up to 32 ways)
  if (cnt < k) return tau;  // fewer than k entries: nothing to drop
  uint32_t prefix = 0, rank = k;  // 1-based rank of the target among the candidates left
  for (int bit = 31 - __clz(max(tau, 1u)); bit >= 0; --bit) {  // every entry's distance is <= tau
    uint32_t zeros = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const uint32_t d = uint32_t(v[r] >> 32);
      const bool e = uint32_t(r) * 32 + lane < cnt && (d >> (bit + 1)) == (prefix >> (bit + 1)) && !((d >> bit) & 1u);
      zeros += __popc(__ballot_sync(~0u, e));
    }
    if (rank > zeros) {
      rank -= zeros;
      prefix |= 1u << bit;
    }
  }
  const uint32_t newtau = prefix, before = k - rank;
  (void)hist;
  const uint32_t need_eq = k - before;
  uint32_t wpos = 0, eq_seen = 0;
#pragma unroll
  for (int r = 0; r < R; ++r) {  // entries in list order: i = 32 r + lane
    const bool valid = uint32_t(r) * 32 + lane < cnt;
    const uint32_t d = uint32_t(v[r] >> 32);
    const bool eq = valid && d == newtau;
    const uint32_t eqbal = __ballot_sync(~0u, eq);
    const bool keep = (valid && d < newtau) || (eq && eq_seen + __popc(eqbal & lanemask_lt()) < need_eq);
    const uint32_t bal = __ballot_sync(~0u, keep);
    if (keep) list[wpos + __popc(bal & lanemask_lt())] = v[r];
    wpos += __popc(bal);
    eq_seen += __popc(eqbal);
  }
  __syncwarp();
  cnt = wpos;
  return newtau;
}

// In-place exact top-k of a warp's list (ids ascending in list order); returns the new bound.
__device__ __noinline__ uint32_t compact_list(uint64_t* list, uint32_t& cnt, uint32_t tau, uint32_t k,
                                 uint32_t* hist) {
  const uint32_t lane = threadIdx.x & 31;
  if (cnt <= 32 * 12) return compact_list_regs<12>(list, cnt, tau, k, hist);
  if (cnt <= 32 * 24) return compact_list_regs<24>(list, cnt, tau, k, hist);
  MIHG_DASSERT(tau < 4097);
  for (uint32_t d = lane; d <= tau; d += 32) hist[d] = 0;
  __syncwarp();
  for (uint32_t i = lane; i < cnt; i += 32) atomicAdd(&hist[uint32_t(list[i] >> 32)], 1u);
  __syncwarp();
  uint32_t run = 0, newtau = tau, before = 0;
  bool found = false;
  for (uint32_t d0 = 0; d0 <= tau && !found; d0 += 32) {
    const uint32_t d = d0 + lane;
    uint32_t v = d <= tau ? hist[d] : 0;
    const uint32_t own = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(~0u, v, o);
      if (lane >= o) v += y;
    }
    const uint32_t ok = __ballot_sync(~0u, d <= tau && run + v >= k);
    if (ok) {
      const int src = __ffs(ok) - 1;
      newtau = d0 + src;
      before = run + __shfl_sync(~0u, v - own, src);
      found = true;
    }
    run += __shfl_sync(~0u, v, 31);
  }
  if (!found) return tau;  // fewer than k entries: nothing to drop
  const uint32_t need_eq = k - before;
  uint32_t wpos = 0, eq_seen = 0;
  for (uint32_t i0 = 0; i0 < cnt; i0 += 32) {
    const uint32_t i = i0 + lane;
    const uint64_t key = i < cnt ? list[i] : ~0ull;
    const uint32_t d = uint32_t(key >> 32);
    const bool eq = i < cnt && d == newtau;
    const uint32_t eqbal = __ballot_sync(~0u, eq);
    const bool keep = (i < cnt && d < newtau) ||
                      (eq && eq_seen + __popc(eqbal & lanemask_lt()) < need_eq);
    const uint32_t bal = __ballot_sync(~0u, keep);
    __syncwarp();
    if (keep) list[wpos + __popc(bal & lanemask_lt())] = key;
    __syncwarp();
    wpos += __popc(bal);
    eq_seen += __popc(eqbal);
  }
  cnt = wpos;
  return newtau;
}

// Gather the per-warp lists of one query into a contiguous segment (one CTA per query).
__global__ void gather_lists_kernel(const uint64_t* __restrict__ lists,
                                    const uint32_t* __restrict__ counts, uint32_t slots, uint32_t L,
                                    uint64_t* __restrict__ out, uint32_t* __restrict__ out_count) {
  __shared__ uint32_t s_off[1025];
  const uint64_t q = blockIdx.x;
  if (threadIdx.x == 0) {
    uint32_t acc = 0;
    for (uint32_t s = 0; s < slots; ++s) {
      s_off[s] = acc;
      acc += counts[q * slots + s];
    }
    s_off[slots] = acc;
    out_count[q] = acc;
  }
  __syncthreads();
  const uint64_t obase = q * uint64_t(slots) * L;
  for (uint32_t s = threadIdx.x >> 5; s < slots; s += blockDim.x >> 5) {
    const uint32_t c = s_off[s + 1] - s_off[s];
    const uint64_t* src = lists + (q * slots + s) * uint64_t(L);
    for (uint32_t i = threadIdx.x & 31; i < c; i += 32) out[obase + s_off[s] + i] = src[i];
  }
}

}  // namespace
}  // namespace mihg
