// Shared device helpers for the B200 multi-index-hashing kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>

#include <cassert>
#include <cstdint>
#include <stdexcept>
#include <string>

namespace mihg {

// ---- error plumbing: CUDA failures become mihg::CudaError, mapped to MIHG_ECUDA at the C ABI.
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess)
    throw CudaError(std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
                    std::to_string(line) + ")");
}
#define MIHG_CUDA(x) ::mihg::cuda_check((x), #x, __FILE__, __LINE__)
// MIHG_SYNC_DEBUG=1 in the environment: synchronize after every launch to localize faults.
bool sync_debug();
void count_launch();  // process-wide counter of this library's kernel launches (mihg_profile)
#define MIHG_LAUNCH()                                                                     \
  do {                                                                                    \
    ::mihg::count_launch();                                                               \
    ::mihg::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__);          \
    if (::mihg::sync_debug())                                                             \
      ::mihg::cuda_check(cudaDeviceSynchronize(), "kernel execution", __FILE__, __LINE__); \
  } while (0)

#ifdef MIHG_DEBUG
#define MIHG_DASSERT(c) assert(c)
#else
#define MIHG_DASSERT(c) ((void)0)
#endif

constexpr uint32_t kMaxTableBits = 32;   // table.hpp:31
constexpr uint32_t kMaxCodeBits = 4096;  // codes.hpp:16
constexpr uint32_t kWarp = 32;

__host__ __device__ constexpr uint32_t words_per_code(uint32_t bits) { return (bits + 63) / 64; }

// Directory group of a sparse (blocked-count) table: 32 consecutive buckets — one of the
// reference's 32-bucket groups (table.hpp:40-47) — in 16 bytes. Bucket t's entry count c_t (0..6
// exact, 7 = saturated) is spread over three 32-bit planes (bit i of c_t is bit t of plane i);
//   start(t) = base + popc(p0 & below) + 2 popc(p1 & below) + 4 popc(p2 & below).
// A group holding a saturated bucket (p0 & p1 & p2 != 0) keeps its exact starts in a 33-entry
// escape record, and `base` is that record's index (probes of its non-empty buckets read the
// record). A probe reads 16 bytes (4 registers).
struct __align__(16) DirGroup {
  uint32_t p0, p1, p2;
  uint32_t base;  // index into ids[] of the group's first entry, or (escaped) the record index
};
static_assert(sizeof(DirGroup) == 16, "half a sector per directory group");
constexpr uint32_t kDirBucketsLog2 = 5;
constexpr uint32_t kEscStarts = 33;  // exact starts per escape record (32 buckets + end)
constexpr uint32_t kMaxInlineCount = 6;

// One substring table on the device.
struct DevTable {
  const uint32_t* ids;      // n ids sorted by (substring key, id)
  const uint32_t* offsets;  // dense: 2^s + 1 bucket starts (nullptr when sparse)
  const DirGroup* dir;      // sparse: 2^(s-5) groups (nullptr when dense)
  const uint32_t* esc;      // sparse: 33 absolute starts per escaped group
  const uint64_t* codes;    // inline codes in table order (W words per entry), or nullptr
  const uint32_t* occ;      // sparse: 1 bit per bucket (non-empty), or nullptr
  uint32_t s;
  uint32_t dense;
  // 64-bit codes split into two 32-bit substrings: the table-order codes keep only the OTHER
  // substring (4 bytes per entry; this table's 32 bits equal the bucket key). rshift: position of
  // the other substring in the code word (0 or 32). rcodes != nullptr replaces `codes`.
  const uint32_t* rcodes;
  uint32_t rshift;
  // bounds for the assert build (make EXTRA=-DMIHG_DEBUG): entries in the table, escape records
  uint32_t n_entries, n_esc;
};

// Substring j of the partition: contiguous run (offset, len) or explicit positions.
struct DevSubstring {
  uint32_t len;
  uint32_t contiguous;
  uint32_t offset;    // first bit when contiguous
  uint32_t pos_base;  // index into positions[] otherwise
};

// Binomial coefficients C(n, k) for n, k <= 64 (ring sizes, colex unranking), in global memory:
// lanes index it divergently, which constant memory would serialise.
constexpr int kBinomStride = 65;
const uint64_t* device_binomials();  // [65][65] on the current device
uint64_t host_binom(uint32_t n, uint32_t k);

// One 256-bit global load (sm_100a LDG.E.ENL2.256): a whole directory block or 256-bit code.
__device__ __forceinline__ void ldg256(const void* p, uint32_t (&r)[8]) {
  asm("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                 "=r"(r[7])
               : "l"(p));
}

// One directory group of a sparse table (16 bytes). The directory is re-read by other queries of
// the same key slice: keep it in L2 (evict last); the candidate codes behind it stream through
// (evict first, verify_residual).
__device__ __forceinline__ uint4 load_dir_group(const DevTable& t, uint32_t gi) {
  MIHG_DASSERT(t.dir && t.s >= kDirBucketsLog2 && uint64_t(gi) < (uint64_t(1) << (t.s - kDirBucketsLog2)));
  uint4 g;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(g.x), "=r"(g.y), "=r"(g.z), "=r"(g.w)
               : "l"(t.dir + gi), "l"(pol));
  return g;
}

// [lo, hi) of bucket tt (0..31) of a loaded directory group.
__device__ __forceinline__ void decode_dir_group(const DevTable& t, const uint4& g, uint32_t tt, uint32_t& lo,
                                                 uint32_t& hi) {
  const uint32_t c = ((g.x >> tt) & 1u) | (((g.y >> tt) & 1u) << 1) | (((g.z >> tt) & 1u) << 2);
  if (c == 0) {
    lo = hi = 0;
    return;
  }
  const uint32_t below = (1u << tt) - 1u;
  // Escaped group (some bucket saturated at count 7): `base` holds the escape record's index, so
  // every non-empty bucket of the group reads its exact start from the record.
  if (g.x & g.y & g.z) {
    MIHG_DASSERT(g.w < t.n_esc);
    const uint32_t* e = t.esc + uint64_t(g.w) * kEscStarts + tt;
    lo = __ldg(e);
    hi = __ldg(e + 1);
    MIHG_DASSERT(lo < hi && hi <= t.n_entries);
    return;
  }
  lo = g.w + __popc(g.x & below) + 2u * __popc(g.y & below) + 4u * __popc(g.z & below);
  hi = lo + c;
  MIHG_DASSERT(hi <= t.n_entries);
}

// ---- bucket probe: [lo, hi) slice of ids[] for bucket `v` (table.hpp:178-188 semantics).
__device__ __forceinline__ void probe_bucket(const DevTable& t, uint32_t v, uint32_t& lo,
                                             uint32_t& hi) {
  if (t.dense) {
    MIHG_DASSERT(uint64_t(v) < (uint64_t(1) << t.s));
    lo = __ldg(t.offsets + v);
    hi = __ldg(t.offsets + v + 1);
    MIHG_DASSERT(lo <= hi && hi <= t.n_entries);
    return;
  }
  if (t.occ && !((__ldg(t.occ + (v >> 5)) >> (v & 31)) & 1u)) {  // empty: an L2 hit, no sector
    lo = hi = 0;
    return;
  }
  const uint4 g = load_dir_group(t, v >> kDirBucketsLog2);
  decode_dir_group(t, g, v & 31u, lo, hi);
}

// Full-code Hamming distance (codes.hpp:38-42). W > 0: compile-time word count.
template <int W>
__device__ __forceinline__ uint32_t hamming(const uint64_t* q, const uint64_t* x, uint32_t) {
  uint32_t d = 0;
#pragma unroll
  for (int w = 0; w < W; ++w) d += __popcll(q[w] ^ x[w]);
  return d;
}
template <>
__device__ __forceinline__ uint32_t hamming<0>(const uint64_t* q, const uint64_t* x, uint32_t nw) {
  uint32_t d = 0;
  for (uint32_t w = 0; w < nw; ++w) d += __popcll(q[w] ^ x[w]);
  return d;
}

// Load code `id` into registers (vectorised for W = 2, 4).
template <int W>
__device__ __forceinline__ void load_code(const uint64_t* __restrict__ codes, uint64_t id,
                                          uint64_t* x) {
  const uint64_t* p = codes + id * W;
  if constexpr (W == 2) {
    const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(p));
    x[0] = v.x;
    x[1] = v.y;
  } else if constexpr (W == 4) {
    uint32_t r[8];
    ldg256(p, r);
#pragma unroll
    for (int w = 0; w < 4; ++w) x[w] = (uint64_t(r[2 * w + 1]) << 32) | r[2 * w];
  } else {
#pragma unroll
    for (int w = 0; w < W; ++w) x[w] = __ldg(p + w);
  }
}

// Substring extraction (codes.hpp:214-231) of code words `c`.
__device__ __forceinline__ uint32_t extract_key(const uint64_t* c, const DevSubstring& sub,
                                                const uint32_t* __restrict__ positions) {
  if (sub.len == 0) return 0;
  if (sub.contiguous) {
    const uint32_t w = sub.offset >> 6, sh = sub.offset & 63;
    uint64_t v = c[w] >> sh;
    if (sh + sub.len > 64) v |= c[w + 1] << (64 - sh);
    return uint32_t(sub.len >= 64 ? v : (v & ((uint64_t(1) << sub.len) - 1)));
  }
  uint32_t v = 0;
  for (uint32_t i = 0; i < sub.len; ++i) {
    const uint32_t p = positions[sub.pos_base + i];
    v |= uint32_t((c[p >> 6] >> (p & 63)) & 1u) << i;
  }
  return v;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

inline uint32_t ceil_div_u32(uint64_t a, uint64_t b) { return uint32_t((a + b - 1) / b); }

int device_sm_count();
void configure_mempool(int device);  // pool release threshold while an index is built (build.cu)
void set_last_error(const std::string& msg);

// Live per-kernel timing (CUDA events on the launching stream), enabled by mihg_profile_enable.
struct ProfileState {
  bool enabled = false;
  double probe_ms = 0;
  uint64_t probe_launches = 0;
  double scan_ms = 0;
  uint64_t scan_launches = 0;
  uint64_t switched_queries = 0;  // queries finished by the exhaustive scan (hybrid switch)
  uint64_t rerun_queries = 0;     // queries whose candidate buffer overflowed (exact re-run pass)
  double rerun_ms = 0;            // host wall time of the re-run passes
};
ProfileState& profile();  // thread-local message behind mihg_last_error()

}  // namespace mihg
