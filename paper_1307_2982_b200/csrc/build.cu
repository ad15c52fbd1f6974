// GPU index build: MihIndex::build (index.hpp:101-121) + SubstringTable::build (table.hpp:91-159).
//
//   K1 extract_keys_kernel   substring key of every code (codes.hpp:214-231)
//   K2 radix_sort_pairs_u32  stable sort of (key, id) -> ids in (key, id) order (table.hpp:98-99)
//   K3 dense:  bucket histogram + exclusive scan -> offsets[2^s + 1]
//      sparse: one warp per 32-bucket directory group -> 3-bit-plane counts + entry base in 16
//              bytes, escape records (33 exact starts) for groups holding a bucket of >= 7 entries.
#include <algorithm>
#include <cstdio>
#include <atomic>
#include <cstdlib>
#include <mutex>
#include <string>

#include "index.cuh"

namespace mihg {


uint64_t host_binom(uint32_t n, uint32_t k) {
  if (k > n) return 0;
  uint64_t c = 1;
  for (uint32_t i = 0; i < k; ++i) c = c * (n - i) / (i + 1);
  return c;
}

const uint64_t* device_binomials() {
  static std::mutex mu;
  static uint64_t* per_device[64] = {};
  int dev = 0;
  MIHG_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if (!per_device[dev]) {
    static uint64_t tab[65][65];
    for (uint32_t n = 0; n <= 64; ++n)
      for (uint32_t k = 0; k <= 64; ++k)  // C(64,32) ~ 1.8e18 fits; recurrence avoids overflow
        tab[n][k] = k > n ? 0 : (k == 0 || k == n) ? 1 : tab[n - 1][k - 1] + tab[n - 1][k];
    MIHG_CUDA(cudaMalloc(reinterpret_cast<void**>(&per_device[dev]), sizeof(tab)));
    MIHG_CUDA(cudaMemcpy(per_device[dev], tab, sizeof(tab), cudaMemcpyHostToDevice));
  }
  return per_device[dev];
}

static std::atomic<uint64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
uint64_t launch_count() { return g_launches.load(); }
ProfileState& profile() {
  static ProfileState p;
  return p;
}

bool sync_debug() {
  static const bool on = [] {
    const char* e = std::getenv("MIHG_SYNC_DEBUG");
    return e && e[0] == '1';
  }();
  return on;
}

int device_sm_count() {
  int dev = 0, sms = 0;
  MIHG_CUDA(cudaGetDevice(&dev));
  MIHG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  return sms;
}

// The stream-ordered pool returns freed memory to the driver at every synchronisation by
// default, so a step's temporaries (selection buffers, re-run buffers) would be re-mapped on each
// call. Keep up to MIHG_POOL_KEEP_MB (default 16 GB) cached in the device's default pool.
// Release threshold of the device's default stream-ordered pool. While an index is being built
// it is 16 GB — below what a large build holds, so freed temporaries go back to the driver at the
// next synchronisation and the index's long-lived arrays are carved out of freshly mapped memory
// (measured on config 4: with 32 GB or more the arrays reuse cached build temporaries and the
// probe kernel runs 3% slower, 8.82 -> 9.10 ms; so do arrays from plain cudaMalloc; a threshold
// of 0 gives the same placement but a 0.6 s longer build). Once the index stands, freed memory stays cached (MIHG_POOL_KEEP_MB, default 64 GB),
// so a search's workspace and temporaries are not trimmed at every synchronisation and re-grown
// through the driver by the next call (config 4, k = 1000: 30 ms steps became 40-120 ms).
void set_pool_threshold(int device, uint64_t bytes) {
  cudaMemPool_t pool;
  MIHG_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t v = bytes;
  MIHG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &v));
}

void configure_mempool(int device) { set_pool_threshold(device, uint64_t(16384) << 20); }

void settle_mempool(int device) {
  const char* e = std::getenv("MIHG_POOL_KEEP_MB");
  cudaMemPool_t pool;
  MIHG_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
  MIHG_CUDA(cudaMemPoolTrimTo(pool, 0));  // the build's temporaries
  set_pool_threshold(device, uint64_t(e ? std::strtoull(e, nullptr, 10) : 65536) << 20);
}

void validate_partition(uint32_t bits, uint32_t m, const uint32_t* lengths,
                        const uint32_t* positions) {
  if (bits == 0 || bits > kMaxCodeBits) throw InvalidArgument("Partition: bad width");
  if (m == 0 || m > bits) throw InvalidArgument("Partition: substring count must be in [1, bits]");
  std::vector<char> seen(bits, 0);
  uint64_t total = 0, at = 0;
  uint32_t lo = bits, hi = 0;
  for (uint32_t j = 0; j < m; ++j) {
    lo = std::min(lo, lengths[j]);
    hi = std::max(hi, lengths[j]);
    total += lengths[j];
    if (total > bits) throw InvalidArgument("Partition: positions do not cover the code");
    for (uint32_t i = 0; i < lengths[j]; ++i) {
      const uint32_t p = positions[at++];
      if (p >= bits)
        throw InvalidArgument("Partition: bit position " + std::to_string(p) + " out of range");
      if (seen[p])
        throw InvalidArgument("Partition: bit position " + std::to_string(p) + " assigned twice");
      seen[p] = 1;
    }
  }
  if (total != bits) throw InvalidArgument("Partition: positions do not cover the code");
  if (hi - lo > 1) throw InvalidArgument("Partition: substring sizes differ by more than 1");
}

namespace {

__global__ void extract_keys_kernel(const uint64_t* __restrict__ codes, uint32_t W, uint64_t n,
                                    DevSubstring sub, const uint32_t* __restrict__ positions,
                                    uint32_t* __restrict__ keys, uint32_t* __restrict__ ids) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    keys[i] = extract_key(codes + i * W, sub, positions);
    ids[i] = uint32_t(i);
  }
}

// Loaded tables: entry i of table j must hold an id seen exactly once whose substring key is
// keys[i] (bit 0 of *bad: key mismatch, bit 1: repeated id).
__global__ void verify_pre_kernel(const uint64_t* __restrict__ codes, uint32_t W, uint64_t n,
                                  DevSubstring sub, const uint32_t* __restrict__ positions,
                                  const uint32_t* __restrict__ keys, const uint32_t* __restrict__ ids,
                                  uint32_t* __restrict__ seen, uint32_t* __restrict__ bad) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t id = ids[i];
    uint32_t f = 0;
    if (extract_key(codes + uint64_t(id) * W, sub, positions) != keys[i]) f |= 1;
    if (atomicOr(seen + (id >> 5), 1u << (id & 31)) & (1u << (id & 31))) f |= 2;
    if (f) atomicOr(bad, f);
  }
}

__global__ void extract_all_keys_kernel(const uint64_t* __restrict__ codes, uint32_t W,
                                        uint64_t count, uint32_t m, const DevSubstring* __restrict__ subs,
                                        const uint32_t* __restrict__ positions, uint32_t* __restrict__ keys) {
  const uint64_t total = count * m;
  for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < total;
       t += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t i = t / m;
    const uint32_t j = uint32_t(t - i * m);
    keys[t] = extract_key(codes + i * W, subs[j], positions);
  }
}

__global__ void gather_codes_kernel(const uint64_t* __restrict__ codes, uint32_t W,
                                    const uint32_t* __restrict__ ids, uint64_t n,
                                    uint64_t* __restrict__ out) {
  const uint64_t total = n * W;
  for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < total;
       t += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t e = t / W;
    out[t] = __ldg(codes + uint64_t(__ldg(ids + e)) * W + (t - e * W));
  }
}

// 32-bit residuals in table order: the bits of the other 32-bit substring of each entry's code.
__global__ void gather_residuals_kernel(const uint64_t* __restrict__ codes, const uint32_t* __restrict__ ids,
                                        uint64_t n, uint32_t shift, uint32_t* __restrict__ out) {
  for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < n; e += uint64_t(gridDim.x) * blockDim.x)
    out[e] = uint32_t(__ldg(codes + __ldg(ids + e)) >> shift);
}

__global__ void occupancy_kernel(const uint32_t* __restrict__ keys, uint64_t n, uint32_t* __restrict__ occ) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t k = keys[i];
    if (i == 0 || keys[i - 1] != k) atomicOr(occ + (k >> 5), 1u << (k & 31));  // first of its bucket
  }
}

__global__ void bucket_hist_kernel(const uint32_t* __restrict__ keys, uint64_t n,
                                   uint32_t* __restrict__ cnt) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    atomicAdd(cnt + keys[i], 1u);
}

// stats[0] non-empty buckets, [1] max bucket size, [2] non-empty 32-bucket groups
__global__ void dense_stats_kernel(const uint32_t* __restrict__ off, uint64_t groups,
                                   unsigned long long* __restrict__ stats) {
  for (uint64_t g = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; g < groups;
       g += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t ne = 0, mx = 0;
    for (uint32_t t = 0; t < 32; ++t) {
      const uint32_t c = off[g * 32 + t + 1] - off[g * 32 + t];
      ne += c != 0;
      mx = max(mx, c);
    }
    if (ne) {
      atomicAdd(stats, (unsigned long long)ne);
      atomicMax(stats + 1, (unsigned long long)mx);
      atomicAdd(stats + 2, 1ull);
    }
  }
}

__device__ __forceinline__ uint64_t lower_bound_u32(const uint32_t* __restrict__ keys, uint64_t n,
                                                    uint64_t target) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (uint64_t(__ldg(keys + mid)) < target) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// One warp per 32-bucket directory group (lane = bucket). Phase 0 writes the group and an escape
// flag; phase 1 (escaped groups only) writes the 33 exact starts at esc_idx[g] and points the
// group's base at that record.
template <int kPhase>
__global__ void dir_build_kernel(const uint32_t* __restrict__ keys, uint64_t n, uint64_t ngroups,
                                 DirGroup* __restrict__ dir, uint32_t* __restrict__ flags,
                                 const uint32_t* __restrict__ esc_idx, uint32_t* __restrict__ esc,
                                 unsigned long long* __restrict__ stats) {
  __shared__ uint32_t cnt[8][32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
  // A warp takes 32 consecutive groups at a time: the 33 group boundaries are 32 + 1 binary
  // searches run by the lanes in parallel (one dependent-load chain per 32 groups instead of one
  // per group: the searches were the kernel's whole length), then the groups are built one by one.
  for (uint64_t g0 = (blockIdx.x * uint64_t(blockDim.x >> 5) + wib) * 32; g0 < ngroups; g0 += warps * 32) {
    if (kPhase == 1 && !__any_sync(~0u, g0 + lane < ngroups && flags[g0 + lane])) continue;
    uint64_t lbv = lower_bound_u32(keys, n, (g0 + lane) << kDirBucketsLog2);
    uint64_t ubv = __shfl_down_sync(~0u, lbv, 1);
    {
      uint64_t endv = 0;
      if (lane == 0) endv = lower_bound_u32(keys, n, (g0 + 32) << kDirBucketsLog2);
      endv = __shfl_sync(~0u, endv, 0);
      if (lane == 31) ubv = endv;
    }
  for (uint32_t j = 0; j < 32; ++j) {
    const uint64_t g = g0 + j;
    if (g >= ngroups) break;
    const uint64_t lb = __shfl_sync(~0u, lbv, j), ub = __shfl_sync(~0u, ubv, j);
    if (kPhase == 1 && !flags[g]) continue;
    __syncwarp();
    cnt[wib][lane] = 0;
    __syncwarp();
    for (uint64_t p = lb + lane; p < ub; p += 32) atomicAdd(&cnt[wib][keys[p] & 31u], 1u);
    __syncwarp();
    const uint32_t c = cnt[wib][lane];
    if (kPhase == 0) {
      const uint32_t sc = min(c, 7u);
      DirGroup grp;
      grp.p0 = __ballot_sync(~0u, sc & 1);
      grp.p1 = __ballot_sync(~0u, sc & 2);
      grp.p2 = __ballot_sync(~0u, sc & 4);
      grp.base = uint32_t(lb);
      const bool escaped = __any_sync(~0u, c > kMaxInlineCount);
      const uint32_t ne = __popc(__ballot_sync(~0u, c != 0));
      uint32_t mx = c;
#pragma unroll
      for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(~0u, mx, o));
      if (lane == 0) {
        dir[g] = grp;
        flags[g] = escaped ? 1u : 0u;
        if (ne) {
          atomicAdd(stats, (unsigned long long)ne);
          atomicMax(stats + 1, (unsigned long long)mx);
          atomicAdd(stats + 2, 1ull);  // non-empty 32-bucket groups (the reference's unit)
        }
      }
    } else {
      uint32_t x = c;  // exclusive prefix of the 32 counts
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(~0u, x, o);
        if (lane >= o) x += y;
      }
      const uint32_t e = esc_idx[g];
      uint32_t* rec = esc + uint64_t(e) * kEscStarts;
      rec[lane] = uint32_t(lb) + x - c;
      if (lane == 0) {
        rec[32] = uint32_t(ub);
        dir[g].base = e;
      }
    }
  }
  }
}

inline unsigned grid_for(uint64_t work, unsigned threads) {
  const uint64_t want = (work + threads - 1) / threads;
  const uint64_t cap = uint64_t(device_sm_count()) * 16;
  return unsigned(std::max<uint64_t>(1, std::min(want, cap)));
}

void build_table(Index& idx, uint32_t j, const BuildOptions& opt) {
  cudaStream_t st = idx.stream;
  const uint64_t n = idx.n;
  auto t = std::make_unique<TableStorage>();
  const uint32_t s = idx.lengths[j];
  t->s = s;
  const uint64_t nb = uint64_t(1) << s;
  bool dense = nb <= std::max<uint64_t>(uint64_t(1) << opt.dense_max_bits, opt.dense_ratio * n);
  if (opt.force == 1) dense = true;
  if (opt.force == 2) dense = false;
  if (s < kDirBucketsLog2) dense = true;
  t->dense = dense;

  DeviceBuffer<uint32_t> keys(std::max<uint64_t>(n, 1), st);
  t->ids = DeviceBuffer<uint32_t>(std::max<uint64_t>(n, 1), st);
  if (n && opt.pre) {  // tables from an index file: already in (key, id) order
    MIHG_CUDA(cudaMemcpyAsync(keys.get(), (*opt.pre)[j].keys.data(), n * 4, cudaMemcpyHostToDevice, st));
    MIHG_CUDA(cudaMemcpyAsync(t->ids.get(), (*opt.pre)[j].ids.data(), n * 4, cudaMemcpyHostToDevice, st));
    // ids < n was checked by the loader
    DeviceBuffer<uint32_t> seen((n + 31) / 32 + 1, st);
    MIHG_CUDA(cudaMemsetAsync(seen.get(), 0, ((n + 31) / 32 + 1) * 4, st));
    uint32_t* bad = seen.get() + (n + 31) / 32;
    verify_pre_kernel<<<grid_for(n, 256), 256, 0, st>>>(idx.codes.get(), idx.W, n, idx.subs[j],
                                                        idx.d_positions.get(), keys.get(), t->ids.get(),
                                                        seen.get(), bad);
    MIHG_LAUNCH();
    uint32_t hbad = 0;
    MIHG_CUDA(cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, st));
    MIHG_CUDA(cudaStreamSynchronize(st));
    if (hbad & 2) throw InconsistentTable(j, "table " + std::to_string(j) + " lists an id more than once");
    if (hbad & 1)
      throw InconsistentTable(j, "table " + std::to_string(j) + " files an id under a key other than its substring");
  } else if (n) {
    extract_keys_kernel<<<grid_for(n, 256), 256, 0, st>>>(idx.codes.get(), idx.W, n, idx.subs[j],
                                                          idx.d_positions.get(), keys.get(),
                                                          t->ids.get());
    MIHG_LAUNCH();
    radix_sort_pairs_u32(keys.get(), t->ids.get(), n, s, st);
  }
  DeviceBuffer<unsigned long long> stats(3, st);
  MIHG_CUDA(cudaMemsetAsync(stats.get(), 0, 3 * sizeof(unsigned long long), st));
  if (dense) {
    DeviceBuffer<uint32_t> cnt(nb + 1, st);
    MIHG_CUDA(cudaMemsetAsync(cnt.get(), 0, (nb + 1) * 4, st));
    if (n) {
      bucket_hist_kernel<<<grid_for(n, 256), 256, 0, st>>>(keys.get(), n, cnt.get());
      MIHG_LAUNCH();
    }
    t->offsets = DeviceBuffer<uint32_t>(nb + 1, st);
    exclusive_scan<uint32_t>(cnt.get(), t->offsets.get(), nb + 1, st);
    const uint64_t groups = (nb + 31) / 32;
    if (nb >= 32) {
      dense_stats_kernel<<<grid_for(groups, 256), 256, 0, st>>>(t->offsets.get(), groups, stats.get());
      MIHG_LAUNCH();
    }
  } else {
    const uint64_t nblocks = nb >> kDirBucketsLog2;  // 32-bucket groups
    t->dir = DeviceBuffer<DirGroup>(nblocks, st);
    DeviceBuffer<uint32_t> flags(nblocks, st), esc_idx(nblocks, st);
    const unsigned grid = grid_for(nblocks * 32, 256);
    dir_build_kernel<0><<<grid, 256, 0, st>>>(keys.get(), n, nblocks, t->dir.get(), flags.get(),
                                             nullptr, nullptr, stats.get());
    MIHG_LAUNCH();
    exclusive_scan<uint32_t>(flags.get(), esc_idx.get(), nblocks, st);
    uint32_t last_idx = 0, last_flag = 0;
    MIHG_CUDA(cudaMemcpyAsync(&last_idx, esc_idx.get() + nblocks - 1, 4, cudaMemcpyDeviceToHost, st));
    MIHG_CUDA(cudaMemcpyAsync(&last_flag, flags.get() + nblocks - 1, 4, cudaMemcpyDeviceToHost, st));
    MIHG_CUDA(cudaStreamSynchronize(st));
    t->escaped_blocks = uint64_t(last_idx) + last_flag;
    if (opt.occupancy && s >= 20) {  // 2^s bits; 512 MB for a 32-bit table
      const uint64_t words = nb / 32;
      t->occ = DeviceBuffer<uint32_t>(words, st);
      MIHG_CUDA(cudaMemsetAsync(t->occ.get(), 0, words * 4, st));
      if (n) {
        occupancy_kernel<<<grid_for(n, 256), 256, 0, st>>>(keys.get(), n, t->occ.get());
        MIHG_LAUNCH();
      }
    }
    if (t->escaped_blocks) {
      t->esc = DeviceBuffer<uint32_t>(t->escaped_blocks * kEscStarts, st);
      dir_build_kernel<1><<<grid, 256, 0, st>>>(keys.get(), n, nblocks, t->dir.get(), flags.get(),
                                               esc_idx.get(), t->esc.get(), nullptr);
      MIHG_LAUNCH();
    }
  }
  // 64-bit codes, two contiguous 32-bit substrings (config 4's shape): the other substring alone
  // identifies the code within a bucket, so table-order codes shrink to 4 bytes per entry
  const bool residual = idx.inline_codes && n && idx.W == 1 && idx.m == 2 && idx.lengths[0] == 32 &&
                        idx.lengths[1] == 32 && idx.subs[0].contiguous && idx.subs[1].contiguous &&
                        opt.residual_codes && !(std::getenv("MIHG_RESIDUAL") && std::getenv("MIHG_RESIDUAL")[0] == '0');
  keys.reset();  // the sorted keys are not needed any more: 4 bytes per code less at the build's peak
  if (residual) {
    t->rshift = idx.subs[1 - j].offset;  // 0 or 32
    t->rcodes = DeviceBuffer<uint32_t>(n, st);
    gather_residuals_kernel<<<grid_for(n, 256), 256, 0, st>>>(idx.codes.get(), t->ids.get(), n, t->rshift,
                                                              t->rcodes.get());
    MIHG_LAUNCH();
  } else if (idx.inline_codes && n) {
    t->tcodes = DeviceBuffer<uint64_t>(n * idx.W, st);
    gather_codes_kernel<<<grid_for(n * idx.W, 256), 256, 0, st>>>(idx.codes.get(), idx.W, t->ids.get(), n,
                                                                  t->tcodes.get());
    MIHG_LAUNCH();
  }
  unsigned long long hs[3];
  MIHG_CUDA(cudaMemcpyAsync(hs, stats.get(), sizeof(hs), cudaMemcpyDeviceToHost, st));
  MIHG_CUDA(cudaStreamSynchronize(st));
  t->non_empty_buckets = hs[0];
  t->max_bucket = hs[1];
  t->non_empty_groups = hs[2];
  if (dense && nb < 32) {  // tiny table: stats on the host
    std::vector<uint32_t> off(nb + 1);
    MIHG_CUDA(cudaMemcpy(off.data(), t->offsets.get(), (nb + 1) * 4, cudaMemcpyDeviceToHost));
    for (uint64_t v = 0; v < nb; ++v) {
      const uint64_t c = off[v + 1] - off[v];
      t->non_empty_buckets += c != 0;
      t->max_bucket = std::max<uint64_t>(t->max_bucket, c);
    }
    t->non_empty_groups = t->non_empty_buckets ? 1 : 0;
  }
  idx.tables[j] = std::move(t);
}

}  // namespace

void extract_all_keys(const Index& idx, const uint64_t* d_codes, uint64_t count, uint32_t* d_keys,
                      cudaStream_t st) {
  if (!count) return;
  extract_all_keys_kernel<<<grid_for(count * idx.m, 256), 256, 0, st>>>(
      d_codes, idx.W, count, idx.m, idx.d_subs.get(), idx.d_positions.get(), d_keys);
  MIHG_LAUNCH();
}

Index* build_index(const uint64_t* codes, bool codes_on_device, uint64_t n, uint32_t bits,
                   uint32_t m, const uint32_t* lengths, const uint32_t* positions, int device,
                   uint32_t id_base, const BuildOptions& opt) {
  std::vector<uint32_t> len, pos;
  if (lengths) {
    len.assign(lengths, lengths + m);
    uint64_t tot = 0;
    for (uint32_t j = 0; j < m; ++j) tot += lengths[j];
    if (!positions) throw InvalidArgument("Partition: positions missing");
    pos.assign(positions, positions + std::min<uint64_t>(tot, uint64_t(bits) + 1));
    if (tot != bits) throw InvalidArgument("Partition: positions do not cover the code");
  } else {
    // consecutive_partition, codes.hpp:198-211
    if (m == 0 || m > bits)
      throw InvalidArgument("consecutive_partition: need 1 <= m <= bits, got m=" +
                            std::to_string(m) + ", bits=" + std::to_string(bits));
    const uint32_t base = bits / m, extra = bits % m;
    for (uint32_t j = 0, p = 0; j < m; ++j) {
      len.push_back(base + (j < extra ? 1 : 0));
      for (uint32_t i = 0; i < len.back(); ++i) pos.push_back(p++);
    }
  }
  validate_partition(bits, m, len.data(), pos.data());
  for (uint32_t j = 0; j < m; ++j)
    if (len[j] > kMaxTableBits)
      throw InvalidArgument("MihIndex::build: substring " + std::to_string(j) + " is " +
                            std::to_string(len[j]) +
                            " bits; direct addressing supports at most 32 (use more substrings)");
  if (n > 0xFFFFFFFFull)
    throw InvalidArgument("CodeDatabase: the GPU index supports at most 2^32-1 codes");
  if (uint64_t(id_base) + n > (uint64_t(1) << 32))
    throw InvalidArgument("shard id range exceeds 2^32");

  MIHG_CUDA(cudaSetDevice(device));
  configure_mempool(device);
  auto idx = std::make_unique<Index>();
  idx->device = device;
  MIHG_CUDA(cudaStreamCreateWithFlags(&idx->stream, cudaStreamNonBlocking));
  cudaStream_t st = idx->stream;
  device_binomials();
  idx->bits = bits;
  idx->W = words_per_code(bits);
  idx->m = m;
  idx->n = n;
  idx->id_base = id_base;
  idx->lengths = len;
  idx->positions = pos;
  const uint32_t W = idx->W;
  // padding bits must be zero (codes.hpp:87-95) — checked by the host facade on append.
  idx->codes = DeviceBuffer<uint64_t>(std::max<uint64_t>(n * W, 1), st);
  if (n)
    MIHG_CUDA(cudaMemcpyAsync(idx->codes.get(), codes, n * W * 8,
                              codes_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
  std::vector<uint64_t> submask(uint64_t(m) * W, 0);
  for (uint32_t j = 0, at = 0; j < m; ++j) {
    DevSubstring s{len[j], 1u, len[j] ? pos[at] : 0u, at};
    for (uint32_t i = 0; i < len[j]; ++i) {
      const uint32_t p = pos[at + i];
      submask[uint64_t(j) * W + (p >> 6)] |= uint64_t(1) << (p & 63);
      if (i && p != pos[at + i - 1] + 1) s.contiguous = 0;
    }
    idx->subs.push_back(s);
    at += len[j];
  }
  idx->d_positions = DeviceBuffer<uint32_t>(std::max<size_t>(pos.size(), 1), st);
  MIHG_CUDA(cudaMemcpyAsync(idx->d_positions.get(), pos.data(), pos.size() * 4, cudaMemcpyHostToDevice, st));
  idx->d_subs = DeviceBuffer<DevSubstring>(m, st);
  MIHG_CUDA(cudaMemcpyAsync(idx->d_subs.get(), idx->subs.data(), m * sizeof(DevSubstring),
                            cudaMemcpyHostToDevice, st));
  idx->d_submask = DeviceBuffer<uint64_t>(submask.size(), st);
  MIHG_CUDA(cudaMemcpyAsync(idx->d_submask.get(), submask.data(), submask.size() * 8,
                            cudaMemcpyHostToDevice, st));
  MIHG_CUDA(cudaStreamSynchronize(st));
  {
    size_t free_b = 0, total_b = 0;
    MIHG_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const double inline_bytes = double(n) * m * W * 8;
    idx->inline_codes = opt.inline_codes == 1 || (opt.inline_codes == -1 && inline_bytes <= 0.4 * double(free_b));
  }
  idx->tables.resize(m);
  for (uint32_t j = 0; j < m; ++j) build_table(*idx, j, opt);
  std::vector<DevTable> views;
  for (auto& t : idx->tables) views.push_back(t->view());
  idx->d_tables = DeviceBuffer<DevTable>(m, st);
  MIHG_CUDA(cudaMemcpyAsync(idx->d_tables.get(), views.data(), m * sizeof(DevTable),
                            cudaMemcpyHostToDevice, st));
  MIHG_CUDA(cudaStreamSynchronize(st));
  settle_mempool(device);
  return idx.release();
}

}  // namespace mihg
