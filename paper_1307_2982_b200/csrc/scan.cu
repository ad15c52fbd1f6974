// Exhaustive batched k-NN (K6): the in-repo comparator and small-n path.
// Reference: scan_knn (scan.hpp:43-68) — XOR+popcount distance to every code, the k smallest
// (dist, id) pairs, ties at the cut to smaller ids.
//
// sm_100a has no native binary MMA (mma .b1 lowers to an emulation call), so
// this runs on the INT/POPC pipe: POPC at 16/clk/SM (measured 4.56e12 popc32/s on B200).
//
// Work split: a warp owns a contiguous id range and a tile of QT queries held in registers; it
// streams 32 codes per step (one per lane, coalesced) and tests each against every query of the
// tile. Per (warp, query) it keeps a bound tau and an append-only list of keys with d <= tau in
// id order; when the list reaches 2k entries it is compacted in place to its exact top-k (ties
// at tau keep the earliest = smallest ids) and tau tightens. A final per-query selection over
// all warp lists gives the exact global top-k.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "knn.cuh"
#include "scanlist.cuh"
#include "select.cuh"

namespace mihg {

namespace {

constexpr int kScanWarps = 8;

struct ScanArgs {
  const uint64_t* codes;
  uint64_t n;
  uint32_t nw, bits, k;
  const uint64_t* queries;
  uint64_t nq;
  uint32_t nsplit;       // id splits per query tile (blocks per tile)
  uint64_t range;        // ids per warp
  uint32_t L;            // list capacity per (warp, query)
  uint64_t* lists;       // [q][split*8 + warp][L]
  uint32_t* counts;      // [q][split*8 + warp]
  uint32_t slots;        // nsplit * kScanWarps
};

template <int W, int QT>
__global__ void __launch_bounds__(kScanWarps * 32, 2) scan_kernel(ScanArgs a) {
  extern __shared__ uint32_t s_hist[];  // kScanWarps * (bits + 1)
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t nw = W ? W : a.nw;
  const uint32_t tile = blockIdx.x / a.nsplit, split = blockIdx.x % a.nsplit;
  const uint32_t slot = split * kScanWarps + warp;
  const uint64_t lo = uint64_t(slot) * a.range;
  const uint64_t hi = min(a.n, lo + a.range);
  uint32_t* hist = s_hist + warp * (a.bits + 1);
  const uint64_t q0 = uint64_t(tile) * QT;
  uint64_t qr[QT][W ? W : 1];
  uint32_t tau[QT], cnt[QT];
#pragma unroll
  for (int t = 0; t < QT; ++t) {
    const uint64_t q = min(q0 + t, a.nq - 1);
    if constexpr (W > 0) {
#pragma unroll
      for (int w = 0; w < W; ++w) qr[t][w] = __ldg(a.queries + q * W + w);
    }
    tau[t] = q0 + t < a.nq ? a.bits : 0xFFFFFFFFu;  // padding queries: never accept (tau sentinel)
    cnt[t] = 0;
  }
  auto list_of = [&](int t) -> uint64_t* {
    return a.lists + ((q0 + t) * a.slots + slot) * uint64_t(a.L);
  };
  const uint32_t lt = lanemask_lt();
  // register double buffer: the next 32 codes are in flight while this chunk is tested
  uint64_t xn[W ? W : 1];
  if constexpr (W > 0) {
    if (lo < hi) load_code<W>(a.codes, min(lo + lane, hi - 1), xn);
  }
  for (uint64_t base = lo; base < hi; base += 32) {
    const uint64_t id = base + lane;
    const bool valid = id < hi;
    uint64_t x[W ? W : 1];
    const uint64_t* xp = a.codes + (valid ? id : lo) * nw;
    if constexpr (W > 0) {
#pragma unroll
      for (int w = 0; w < W; ++w) x[w] = xn[w];
      if (base + 32 < hi) load_code<W>(a.codes, min(base + 32 + lane, hi - 1), xn);
    }
    uint32_t d[QT];
    bool anyp = false;
#pragma unroll
    for (int t = 0; t < QT; ++t) {
      if constexpr (W > 0) {
        d[t] = hamming<W>(qr[t], x, W);
      } else {
        const uint64_t* qp = a.queries + min(q0 + t, a.nq - 1) * nw;
        uint32_t dd = 0;
        for (uint32_t w = 0; w < nw; ++w) dd += __popcll(__ldg(qp + w) ^ __ldg(xp + w));
        d[t] = dd;
      }
      anyp |= valid && d[t] <= tau[t];  // padding queries have tau = 0xFFFFFFFF: checked below
    }
    if (!__any_sync(~0u, anyp)) continue;  // fast path: nothing in this chunk beats any bound
#pragma unroll
    for (int t = 0; t < QT; ++t) {
      const bool pass = valid && d[t] <= tau[t] && tau[t] != 0xFFFFFFFFu;
      const uint32_t bal = __ballot_sync(~0u, pass);
      if (bal) {
        uint64_t* list = list_of(t);
        MIHG_DASSERT(q0 + t < a.nq);
        MIHG_DASSERT(cnt[t] + 32 <= a.L);
        if (pass) list[cnt[t] + __popc(bal & lt)] = (uint64_t(d[t]) << 32) | uint32_t(id);
        cnt[t] += __popc(bal);
        if (cnt[t] >= 2 * a.k) {
          __syncwarp();
          tau[t] = compact_list(list, cnt[t], tau[t], a.k, hist);
        }
      }
    }
  }
#pragma unroll
  for (int t = 0; t < QT; ++t)
    if (q0 + t < a.nq && lane == 0) a.counts[(q0 + t) * a.slots + slot] = cnt[t];
}

template <int W, int QT>
void launch_scan(ScanArgs a, cudaStream_t st) {
  const uint32_t tiles = uint32_t((a.nq + QT - 1) / QT);
  const size_t smem = size_t(kScanWarps) * (a.bits + 1) * 4;
  MIHG_CUDA(cudaFuncSetAttribute(scan_kernel<W, QT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(std::max<size_t>(smem, 1024))));
  scan_kernel<W, QT><<<tiles * a.nsplit, kScanWarps * 32, smem, st>>>(a);
  MIHG_LAUNCH();
}

}  // namespace

// Which exhaustive kernel serves scan_knn: K7 (tensor cores, tcscan.cu) for codes up to 256 bits,
// K6 (POPC pipe) otherwise. MIHG_SCAN_KERNEL=popc|tc forces one (A/B measurement, tests).
ScanKernel scan_kernel_for(uint32_t bits) {
  const char* e = std::getenv("MIHG_SCAN_KERNEL");
  if (e && e[0] == 'p') return ScanKernel::Popc;
  if (e && e[0] == 't' && tc_scan_supported(bits)) return ScanKernel::Tensor;
  return tc_scan_supported(bits) ? ScanKernel::Tensor : ScanKernel::Popc;
}

void scan_knn_device(const uint64_t* d_codes, uint64_t n, uint32_t bits, uint32_t id_base,
                     const uint64_t* d_queries, uint64_t nq, uint32_t k, uint32_t* d_ids,
                     uint32_t* d_dists, cudaStream_t st) {
  if (k > n) throw InvalidArgument("scan_knn: k exceeds database size");
  if (scan_kernel_for(bits) == ScanKernel::Tensor) {
    tc_scan_knn_device(d_codes, n, bits, id_base, d_queries, nq, k, d_ids, d_dists, st, nullptr);
    return;
  }
  popc_scan_knn_device(d_codes, n, bits, id_base, d_queries, nq, k, d_ids, d_dists, st);
}

// K6 on the POPC pipe.
void popc_scan_knn_device(const uint64_t* d_codes, uint64_t n, uint32_t bits, uint32_t id_base,
                          const uint64_t* d_queries, uint64_t nq, uint32_t k, uint32_t* d_ids,
                          uint32_t* d_dists, cudaStream_t st) {
  if (k > n) throw InvalidArgument("scan_knn: k exceeds database size");
  if (nq == 0 || k == 0) return;
  const uint32_t nw = words_per_code(bits);
  const int QT = nw <= 2 ? 16 : (nw <= 4 ? 8 : 4);
  const uint32_t L = 2 * k + 32;
  const uint64_t sms = uint64_t(device_sm_count());
  // query chunk bounded by list memory (~2 GiB)
  const uint64_t per_q_slot = uint64_t(L) * 8;
  for (uint64_t q0 = 0; q0 < nq;) {
    uint64_t qn = nq - q0;
    const uint64_t tiles_all = (qn + QT - 1) / QT;
    // enough warps to fill the GPU ~4 waves, but each warp scans >= 32 codes per list
    uint64_t nsplit = std::max<uint64_t>(1, (sms * 8 + tiles_all - 1) / tiles_all);
    nsplit = std::min<uint64_t>(nsplit, std::max<uint64_t>(1, n / (kScanWarps * 256)));
    nsplit = std::min<uint64_t>(nsplit, 1024 / kScanWarps);
    const uint64_t slots = nsplit * kScanWarps;
    const uint64_t budget = uint64_t(2) << 30;
    const uint64_t qmax = std::max<uint64_t>(QT, budget / (2 * slots * per_q_slot) / QT * QT);
    qn = std::min(qn, qmax);
    ScanArgs a{};
    a.codes = d_codes;
    a.n = n;
    a.nw = nw;
    a.bits = bits;
    a.k = k;
    a.queries = d_queries + q0 * nw;
    a.nq = qn;
    a.nsplit = uint32_t(nsplit);
    a.slots = uint32_t(slots);
    a.range = (n + slots - 1) / slots;
    a.L = L;
    DeviceBuffer<uint64_t> lists(qn * slots * L, st), gathered(qn * slots * L, st);
    DeviceBuffer<uint32_t> counts(qn * slots, st), gcount(qn, st);
    a.lists = lists.get();
    a.counts = counts.get();
    switch (nw) {
      case 1: launch_scan<1, 16>(a, st); break;
      case 2: launch_scan<2, 16>(a, st); break;
      case 3: launch_scan<3, 8>(a, st); break;
      case 4: launch_scan<4, 8>(a, st); break;
      default: launch_scan<0, 4>(a, st);
    }
    gather_lists_kernel<<<unsigned(qn), 256, 0, st>>>(lists.get(), counts.get(), uint32_t(slots), L,
                                                      gathered.get(), gcount.get());
    MIHG_LAUNCH();
    SelectArgs sa;
    sa.keys = gathered.get();
    sa.seg_stride = slots * L;
    sa.seg_count = gcount.get();
    sa.k = k;
    sa.max_dist = bits;
    sa.id_base = id_base;
    sa.out_ids = d_ids + q0 * k;
    sa.out_dists = d_dists + q0 * k;
    select_topk(sa, uint32_t(qn), st);
    q0 += qn;
  }
}

// ---- K9: exact k-way merge of per-shard results -----------------------------------------
namespace {
__global__ void pack_shard_keys_kernel(const uint32_t* __restrict__ ids,
                                       const uint32_t* __restrict__ dists, uint32_t G, uint64_t nq,
                                       uint32_t k_in, uint64_t* __restrict__ keys,
                                       uint32_t* __restrict__ cnt) {
  // input layout: [g][q][k_in]; output segment per query: G * k_in keys
  const uint64_t total = uint64_t(G) * nq * k_in;
  for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < total;
       t += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t g = t / (nq * k_in);
    const uint64_t rem = t - g * nq * k_in;
    const uint64_t q = rem / k_in, i = rem - q * k_in;
    const uint32_t d = dists[t], id = ids[t];
    keys[q * G * k_in + g * k_in + i] = d == 0xFFFFFFFFu ? ~0ull : (uint64_t(d) << 32) | id;
    if (t < nq) cnt[t] = G * k_in;
  }
}
}  // namespace

void merge_topk_device(const uint32_t* d_ids, const uint32_t* d_dists, uint32_t G, uint64_t nq,
                       uint32_t k_in, uint32_t k_out, uint32_t* d_out_ids, uint32_t* d_out_dists,
                       cudaStream_t st) {
  if (nq == 0 || k_out == 0) return;
  DeviceBuffer<uint64_t> keys(uint64_t(G) * nq * k_in, st);
  DeviceBuffer<uint32_t> cnt(nq, st);
  const uint64_t total = uint64_t(G) * nq * k_in;
  pack_shard_keys_kernel<<<unsigned(std::min<uint64_t>((total + 255) / 256, 65535)), 256, 0, st>>>(
      d_ids, d_dists, G, nq, k_in, keys.get(), cnt.get());
  MIHG_LAUNCH();
  SelectArgs sa;
  sa.keys = keys.get();
  sa.seg_stride = uint64_t(G) * k_in;
  sa.seg_count = cnt.get();
  sa.seg_maxd = nullptr;
  sa.k = k_out;
  sa.id_base = 0;
  sa.out_ids = d_out_ids;
  sa.out_dists = d_out_dists;
  select_topk(sa, uint32_t(nq), st);
}

}  // namespace mihg
