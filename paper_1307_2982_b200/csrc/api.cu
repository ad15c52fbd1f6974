// C ABI (include/mihg.h) over the device index and kernels. No C++ exception crosses it.
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/mihg.h"
#include "knn.cuh"
#include "optimize.cuh"
#include "persist.cuh"

struct mihg_index {
  mihg::Index* impl;
};

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return MIHG_OK;
  } catch (const mihg::FormatError& e) {
    g_err = e.what();
    return MIHG_EFORMAT;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return MIHG_EINVAL;
  } catch (const std::bad_alloc&) {
    g_err = "bad_alloc";
    return MIHG_ENOMEM;
  } catch (const mihg::NcclError& e) {
    mihg::set_last_error(e.what());
    return MIHG_ENCCL;
  } catch (const mihg::CudaError& e) {
    g_err = e.what();
    // surface allocation failures as ENOMEM
    if (std::strstr(e.what(), "out of memory")) return MIHG_ENOMEM;
    return MIHG_ECUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    const std::string m = e.what();
    if (m.rfind("cannot open", 0) == 0 || m.rfind("read failed", 0) == 0 || m.rfind("write failed", 0) == 0)
      return MIHG_EIO;
    return MIHG_EINTERNAL;
  } catch (...) {
    g_err = "unknown error";
    return MIHG_EINTERNAL;
  }
}

mihg::Index& impl(const mihg_index* idx) {
  if (!idx || !idx->impl) throw mihg::InvalidArgument("null index");
  return *idx->impl;
}

// Runs the index's work on its own stream, ordered after / before the caller's stream with events:
// the library's stream-ordered workspace allocations then always live on one stream (cross-stream
// frees defeat the pool's reuse; measured: config 4 k=1000 through a caller stream 112-211K q/s vs
// 233K through the index stream).
struct StreamJoin {
  cudaStream_t user, own;
  explicit StreamJoin(cudaStream_t user_stream, cudaStream_t index_stream) : user(user_stream), own(index_stream) {
    if (user == own) return;
    cudaEvent_t e;
    MIHG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    MIHG_CUDA(cudaEventRecord(e, user));
    MIHG_CUDA(cudaStreamWaitEvent(own, e, 0));
    cudaEventDestroy(e);
  }
  ~StreamJoin() {
    if (user == own) return;
    cudaEvent_t e;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return;
    cudaEventRecord(e, own);
    cudaStreamWaitEvent(user, e, 0);
    cudaEventDestroy(e);
  }
};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    MIHG_CUDA(cudaGetDevice(&prev));
    if (prev != dev) MIHG_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// std::mt19937_64 (io.hpp:268); the parameters are fixed by the C++ standard.
struct Mt64 {
  uint64_t s[312];
  int i = 312;
  explicit Mt64(uint64_t seed) {
    s[0] = seed;
    for (int k = 1; k < 312; ++k) s[k] = 6364136223846793005ULL * (s[k - 1] ^ (s[k - 1] >> 62)) + k;
  }
  uint64_t operator()() {
    if (i >= 312) {
      for (int k = 0; k < 312; ++k) {
        const uint64_t y = (s[k] & 0xFFFFFFFF80000000ULL) | (s[(k + 1) % 312] & 0x7FFFFFFFULL);
        s[k] = s[(k + 156) % 312] ^ (y >> 1) ^ ((y & 1) ? 0xB5026F5AA96619E9ULL : 0);
      }
      i = 0;
    }
    uint64_t z = s[i++];
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= z >> 43;
    return z;
  }
};

}  // namespace

namespace mihg {
void set_last_error(const std::string& msg) { g_err = msg; }
uint64_t launch_count();
}  // namespace mihg

extern "C" {

const char* mihg_last_error(void) { return g_err.c_str(); }
int mihg_abi_version(void) { return MIHG_ABI_VERSION; }

int mihg_device_count(int* count) {
  return guarded([&] { MIHG_CUDA(cudaGetDeviceCount(count)); });
}

int mihg_index_build_ex(const mihg_build_params* p, mihg_index** out) {
  return guarded([&] {
    if (!p || !out) throw mihg::InvalidArgument("null argument");
    if (p->n && !p->codes) throw mihg::InvalidArgument("null codes");
    if (p->bits == 0 || p->bits > mihg::kMaxCodeBits)
      throw mihg::InvalidArgument("CodeDatabase: code width must be in [1, 4096], got " +
                                  std::to_string(p->bits));
    mihg::BuildOptions opt;
    if (p->dense_max_bits) opt.dense_max_bits = p->dense_max_bits;
    opt.force = p->layout;
    if (const char* e = std::getenv("MIHG_OCC")) opt.occupancy = e[0] == '1';  // A/B switch
    DeviceGuard g(p->device);
    mihg::Index* ix = mihg::build_index(p->codes, p->codes_on_device != 0, p->n, p->bits, p->m,
                                        p->lengths, p->positions, p->device, p->id_base, opt);
    *out = new mihg_index{ix};
  });
}

int mihg_index_build(const uint64_t* codes, uint64_t n, uint32_t bits, uint32_t m,
                     const uint32_t* lengths, const uint32_t* positions, int device,
                     mihg_index** out) {
  mihg_build_params p{};
  p.codes = codes;
  p.n = n;
  p.bits = bits;
  p.m = m;
  p.lengths = lengths;
  p.positions = positions;
  p.device = device;
  return mihg_index_build_ex(&p, out);
}

void mihg_index_free(mihg_index* idx) {
  if (!idx) return;
  guarded([&] {
    if (idx->impl) {
      DeviceGuard g(idx->impl->device);
      delete idx->impl;
    }
  });
  delete idx;
}

int mihg_index_get_info(const mihg_index* idx, mihg_index_info* out) {
  return guarded([&] {
    const mihg::Index& ix = impl(idx);
    out->n = ix.n;
    out->bits = ix.bits;
    out->m = ix.m;
    out->id_base = ix.id_base;
    out->device = ix.device;
    uint64_t bytes = ix.codes.size() * 8;
    for (auto& t : ix.tables) bytes += t->bytes();
    out->device_bytes = bytes;
  });
}

int mihg_table_get_info(const mihg_index* idx, uint32_t j, mihg_table_info* out) {
  return guarded([&] {
    const mihg::Index& ix = impl(idx);
    if (j >= ix.m) throw mihg::InvalidArgument("table index out of range");
    const mihg::TableStorage& t = *ix.tables[j];
    out->s = t.s;
    out->dense = t.dense ? 1 : 0;
    out->non_empty_buckets = t.non_empty_buckets;
    out->max_bucket_size = t.max_bucket;
    out->total_entries = ix.n;
    out->device_bytes = t.bytes();
    out->escaped_blocks = t.escaped_blocks;
    // TableStats::estimate_bytes (table.hpp:42-46): the reference's accounting model.
    const uint64_t groups = uint64_t(1) << (t.s >= 5 ? t.s - 5 : 0);
    out->estimated_bytes = groups * 12 + t.non_empty_groups * 12 + t.non_empty_buckets * 4 + ix.n * 4;
  });
}

int mihg_bucket_lookup(const mihg_index* idx, uint32_t j, uint64_t value, uint32_t* out_ids,
                       uint64_t cap, uint64_t* count) {
  return guarded([&] {
    mihg::Index& ix = impl(idx);
    if (j >= ix.m) throw mihg::InvalidArgument("table index out of range");
    const mihg::TableStorage& t = *ix.tables[j];
    if (value >> t.s)
      throw mihg::InvalidArgument("bucket_lookup: value " + std::to_string(value) +
                                  " does not fit in " + std::to_string(t.s) + " bits");
    DeviceGuard g(ix.device);
    std::lock_guard<std::mutex> lk(ix.mu);
    uint32_t lo = 0, hi = 0;
    if (t.dense) {
      uint32_t two[2];
      MIHG_CUDA(cudaMemcpy(two, t.offsets.get() + value, 8, cudaMemcpyDeviceToHost));
      lo = two[0];
      hi = two[1];
    } else {
      mihg::DirGroup gp;
      MIHG_CUDA(cudaMemcpy(&gp, t.dir.get() + (value >> mihg::kDirBucketsLog2), sizeof(gp),
                           cudaMemcpyDeviceToHost));
      const uint32_t tt = uint32_t(value & 31);
      const uint32_t c = ((gp.p0 >> tt) & 1u) | (((gp.p1 >> tt) & 1u) << 1) | (((gp.p2 >> tt) & 1u) << 2);
      if (c) {
        const uint32_t below = (1u << tt) - 1u;
        if (gp.p0 & gp.p1 & gp.p2) {  // escaped group: base is the record index
          uint32_t two[2];
          MIHG_CUDA(cudaMemcpy(two, t.esc.get() + uint64_t(gp.base) * mihg::kEscStarts + tt, 8,
                               cudaMemcpyDeviceToHost));
          lo = two[0];
          hi = two[1];
        } else {
          lo = gp.base + __builtin_popcount(gp.p0 & below) + 2 * __builtin_popcount(gp.p1 & below) +
               4 * __builtin_popcount(gp.p2 & below);
          hi = lo + c;
        }
      }
    }
    *count = hi - lo;
    const uint64_t w = std::min<uint64_t>(cap, hi - lo);
    if (w) {
      MIHG_CUDA(cudaMemcpy(out_ids, t.ids.get() + lo, w * 4, cudaMemcpyDeviceToHost));
      for (uint64_t i = 0; i < w; ++i) out_ids[i] += ix.id_base;
    }
  });
}

int mihg_index_write(mihg_index* idx, const char* path) {
  return guarded([&] {
    mihg::Index& ix = impl(idx);
    if (!path) throw mihg::InvalidArgument("null path");
    if (ix.id_base) throw mihg::InvalidArgument("write_index: shard indexes (id_base != 0) are not files");
    DeviceGuard g(ix.device);
    std::lock_guard<std::mutex> lk(ix.mu);
    mihg::write_index(ix, path);
  });
}

int mihg_index_read(const char* path, int device, mihg_index** out) {
  return guarded([&] {
    if (!path || !out) throw mihg::InvalidArgument("null argument");
    DeviceGuard g(device);
    mihg::BuildOptions opt;
    *out = new mihg_index{mihg::read_index(path, device, opt)};
  });
}

int mihg_index_codes(const mihg_index* idx, const uint64_t** d_codes) {
  return guarded([&] { *d_codes = impl(idx).codes.get(); });
}

int mihg_knn_batch_device(mihg_index* idx, const uint64_t* d_queries, uint64_t nq, uint32_t k,
                          uint32_t* d_ids, uint32_t* d_dists, mihg_trace* d_traces, void* stream) {
  return guarded([&] {
    mihg::Index& ix = impl(idx);
    DeviceGuard g(ix.device);
    std::lock_guard<std::mutex> lk(ix.mu);
    StreamJoin j(static_cast<cudaStream_t>(stream), ix.stream);
    mihg::knn_device(ix, d_queries, nq, k, d_ids, d_dists, reinterpret_cast<mihg::Trace*>(d_traces), ix.stream);
  });
}

int mihg_knn_batch_device_part(mihg_index* idx, const uint64_t* d_queries, uint64_t nq, uint32_t k,
                               uint32_t* d_ids, uint32_t* d_dists, mihg_trace* d_traces,
                               const mihg_partition* part, void* stream) {
  return guarded([&] {
    mihg::Index& ix = impl(idx);
    DeviceGuard g(ix.device);
    std::lock_guard<std::mutex> lk(ix.mu);
    mihg::Partition pt;
    if (part) {
      pt.count = part->count;
      pt.rank = part->rank;
      pt.allreduce = part->allreduce;
      pt.user = part->user;
      pt.id_shards = part->id_shards != 0;
      pt.k_stop = part->k_stop;
      pt.comm = reinterpret_cast<mihg::Comm*>(part->comm);
      if (pt.comm && (uint32_t(mihg::comm_size(pt.comm)) != pt.count || uint32_t(mihg::comm_rank(pt.comm)) != pt.rank))
        throw mihg::InvalidArgument("partitioned knn: count/rank do not match the communicator");
    }
    mihg::KnnOptions opt;
    opt.part = part ? &pt : nullptr;
    StreamJoin j(static_cast<cudaStream_t>(stream), ix.stream);
    mihg::knn_device(ix, d_queries, nq, k, d_ids, d_dists, reinterpret_cast<mihg::Trace*>(d_traces), ix.stream,
                     opt);
  });
}

int mihg_comm_unique_id(uint8_t out_id[128]) {
  return guarded([&] {
    if (!out_id) throw mihg::InvalidArgument("null argument");
    mihg::comm_unique_id(out_id);
  });
}

int mihg_comm_init(const uint8_t id[128], int nranks, int rank, int device, mihg_comm** out) {
  return guarded([&] {
    if (!id || !out) throw mihg::InvalidArgument("null argument");
    DeviceGuard g(device);
    *out = reinterpret_cast<mihg_comm*>(mihg::comm_init(id, nranks, rank, device));
  });
}

void mihg_comm_free(mihg_comm* comm) {
  guarded([&] { mihg::comm_free(reinterpret_cast<mihg::Comm*>(comm)); });
}

int mihg_nccl_version(int* version) {
  return guarded([&] { *version = mihg::nccl_version(); });
}

int mihg_knn_sharded_device(mihg_index* idx, mihg_comm* comm, int layout, uint64_t n_total,
                            const uint64_t* d_queries, uint64_t nq, uint32_t k, uint32_t* d_ids,
                            uint32_t* d_dists, mihg_trace* d_traces, void* stream) {
  return guarded([&] {
    mihg::Index& ix = impl(idx);
    if (!comm) throw mihg::InvalidArgument("sharded knn: null communicator");
    if (layout != 0 && layout != 1) throw mihg::InvalidArgument("sharded knn: layout must be 0 or 1");
    auto* c = reinterpret_cast<mihg::Comm*>(comm);
    const uint32_t G = uint32_t(mihg::comm_size(c)), rank = uint32_t(mihg::comm_rank(c));
    if (k > n_total) throw mihg::InvalidArgument("knn_search: k exceeds database size");
    DeviceGuard g(ix.device);
    std::lock_guard<std::mutex> lk(ix.mu);
    StreamJoin j(static_cast<cudaStream_t>(stream), ix.stream);
    cudaStream_t st = ix.stream;
    mihg::Partition pt;
    pt.count = G;
    pt.rank = rank;
    pt.comm = c;
    uint32_t kk = k;
    bool collective = true;
    if (layout == 1) {
      const uint64_t per = (n_total + G - 1) / G;
      const uint64_t lo = std::min<uint64_t>(n_total, uint64_t(rank) * per), hi = std::min<uint64_t>(n_total, lo + per);
      if (ix.n != hi - lo || (ix.n && ix.id_base != lo))
        throw mihg::InvalidArgument("sharded knn: the index is not id shard " + std::to_string(rank) + " of n_total");
      kk = uint32_t(std::min<uint64_t>(k, ix.n));
      pt.id_shards = true;
      pt.k_stop = k;
      collective = n_total > uint64_t(G - 1) * per;  // every shard non-empty: global stopping
    } else if (ix.n != n_total) {
      throw mihg::InvalidArgument("sharded knn: layout 0 needs the full index on every rank");
    }
    if (nq == 0 || k == 0) return;
    mihg::DeviceBuffer<uint32_t> li(nq * k, st), ld(nq * k, st);
    if (kk < k) {  // a shard smaller than k: its list is padded (0xFFFFFFFF sorts last)
      MIHG_CUDA(cudaMemsetAsync(li.get(), 0xFF, nq * k * 4, st));
      MIHG_CUDA(cudaMemsetAsync(ld.get(), 0xFF, nq * k * 4, st));
    }
    if (kk > 0) {
      mihg::KnnOptions opt;
      opt.part = collective ? &pt : nullptr;
      if (kk == k) {
        mihg::knn_device(ix, d_queries, nq, kk, li.get(), ld.get(), reinterpret_cast<mihg::Trace*>(d_traces), st, opt);
      } else {
        mihg::DeviceBuffer<uint32_t> ti(nq * kk, st), td(nq * kk, st);
        mihg::knn_device(ix, d_queries, nq, kk, ti.get(), td.get(), reinterpret_cast<mihg::Trace*>(d_traces), st, opt);
        MIHG_CUDA(cudaMemcpy2DAsync(li.get(), k * 4, ti.get(), kk * 4, kk * 4, nq, cudaMemcpyDeviceToDevice, st));
        MIHG_CUDA(cudaMemcpy2DAsync(ld.get(), k * 4, td.get(), kk * 4, kk * 4, nq, cudaMemcpyDeviceToDevice, st));
      }
    }
    mihg::DeviceBuffer<uint32_t> gi(uint64_t(G) * nq * k, st), gd(uint64_t(G) * nq * k, st);
    mihg::comm_allgather(c, li.get(), gi.get(), nq * k * 4, st);
    mihg::comm_allgather(c, ld.get(), gd.get(), nq * k * 4, st);
    mihg::merge_topk_device(gi.get(), gd.get(), G, nq, k, k, d_ids, d_dists, st);
  });
}

int mihg_knn_batch(mihg_index* idx, const uint64_t* queries, uint64_t nq, uint32_t k,
                   uint32_t* out_ids, uint32_t* out_dists, mihg_trace* traces) {
  return guarded([&] {
    mihg::Index& ix = impl(idx);
    if (k > ix.n) throw mihg::InvalidArgument("knn_search: k exceeds database size");
    if (nq == 0) return;
    DeviceGuard g(ix.device);
    std::lock_guard<std::mutex> lk(ix.mu);
    cudaStream_t st = ix.stream;
    uint64_t* dq = mihg::Index::grow(ix.stage_q, nq * ix.W, st);
    uint32_t* di = mihg::Index::grow(ix.stage_ids, std::max<uint64_t>(nq * k, 1), st);
    uint32_t* dd = mihg::Index::grow(ix.stage_dists, std::max<uint64_t>(nq * k, 1), st);
    mihg::Trace* dt = traces ? reinterpret_cast<mihg::Trace*>(mihg::Index::grow(ix.stage_tr, nq * sizeof(mihg::Trace), st))
                             : nullptr;
    MIHG_CUDA(cudaMemcpyAsync(dq, queries, nq * ix.W * 8, cudaMemcpyHostToDevice, st));
    mihg::knn_device(ix, dq, nq, k, di, dd, dt, st);
    if (k) {
      MIHG_CUDA(cudaMemcpyAsync(out_ids, di, nq * k * 4, cudaMemcpyDeviceToHost, st));
      MIHG_CUDA(cudaMemcpyAsync(out_dists, dd, nq * k * 4, cudaMemcpyDeviceToHost, st));
    }
    if (traces) MIHG_CUDA(cudaMemcpyAsync(traces, dt, nq * sizeof(mihg::Trace), cudaMemcpyDeviceToHost, st));
    MIHG_CUDA(cudaStreamSynchronize(st));
  });
}

int mihg_range_batch(mihg_index* idx, const uint64_t* queries, uint64_t nq, uint32_t r,
                     uint64_t* out_offsets, uint32_t* out_ids, uint32_t* out_dists, uint64_t capacity,
                     mihg_trace* traces) {
  return guarded([&] {
    mihg::Index& ix = impl(idx);
    if (!out_offsets) throw mihg::InvalidArgument("range_search: null offsets");
    DeviceGuard g(ix.device);
    std::lock_guard<std::mutex> lk(ix.mu);
    mihg::range_host(ix, queries, nq, r, out_offsets, out_ids, out_dists, capacity,
                     reinterpret_cast<mihg::Trace*>(traces), ix.stream);
  });
}

int mihg_scan_knn_batch_device(mihg_index* idx, const uint64_t* d_queries, uint64_t nq, uint32_t k,
                               uint32_t* d_ids, uint32_t* d_dists, void* stream) {
  return guarded([&] {
    mihg::Index& ix = impl(idx);
    DeviceGuard g(ix.device);
    std::lock_guard<std::mutex> lk(ix.mu);
    mihg::scan_knn_device(ix.codes.get(), ix.n, ix.bits, ix.id_base, d_queries, nq, k, d_ids,
                          d_dists, static_cast<cudaStream_t>(stream));
  });
}

int mihg_scan_knn_batch(mihg_index* idx, const uint64_t* queries, uint64_t nq, uint32_t k,
                        uint32_t* out_ids, uint32_t* out_dists) {
  return guarded([&] {
    mihg::Index& ix = impl(idx);
    if (k > ix.n) throw mihg::InvalidArgument("scan_knn: k exceeds database size");
    if (nq == 0 || k == 0) return;
    DeviceGuard g(ix.device);
    std::lock_guard<std::mutex> lk(ix.mu);
    cudaStream_t st = ix.stream;
    uint64_t* dq = mihg::Index::grow(ix.stage_q, nq * ix.W, st);
    uint32_t* di = mihg::Index::grow(ix.stage_ids, nq * k, st);
    uint32_t* dd = mihg::Index::grow(ix.stage_dists, nq * k, st);
    MIHG_CUDA(cudaMemcpyAsync(dq, queries, nq * ix.W * 8, cudaMemcpyHostToDevice, st));
    mihg::scan_knn_device(ix.codes.get(), ix.n, ix.bits, ix.id_base, dq, nq, k, di, dd, st);
    MIHG_CUDA(cudaMemcpyAsync(out_ids, di, nq * k * 4, cudaMemcpyDeviceToHost, st));
    MIHG_CUDA(cudaMemcpyAsync(out_dists, dd, nq * k * 4, cudaMemcpyDeviceToHost, st));
    MIHG_CUDA(cudaStreamSynchronize(st));
  });
}

int mihg_scan_knn_raw_device(const uint64_t* d_codes, uint64_t n, uint32_t bits, uint32_t id_base,
                             const uint64_t* d_queries, uint64_t nq, uint32_t k, uint32_t* d_ids,
                             uint32_t* d_dists, void* stream) {
  return guarded([&] {
    if (bits == 0 || bits > mihg::kMaxCodeBits) throw mihg::InvalidArgument("bad code width");
    mihg::scan_knn_device(d_codes, n, bits, id_base, d_queries, nq, k, d_ids, d_dists,
                          static_cast<cudaStream_t>(stream));
  });
}

int mihg_scan_kernel_for(uint32_t bits) {
  return mihg::scan_kernel_for(bits) == mihg::ScanKernel::Tensor ? 1 : 0;
}

int mihg_tc_distances_device(const uint64_t* d_codes, uint64_t n, uint32_t bits,
                             const uint64_t* d_queries, uint64_t nq, int32_t* d_out, void* stream) {
  return guarded([&] {
    if (n == 0 || nq == 0) return;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    mihg::DeviceBuffer<uint32_t> di(nq, st), dd(nq, st);
    mihg::tc_scan_knn_device(d_codes, n, bits, 0, d_queries, nq, 1, di.get(), dd.get(), st, d_out);
    MIHG_CUDA(cudaStreamSynchronize(st));
  });
}

int mihg_merge_topk_device(const uint32_t* d_ids, const uint32_t* d_dists, uint32_t G, uint64_t nq,
                           uint32_t k_in, uint32_t k_out, uint32_t* d_out_ids,
                           uint32_t* d_out_dists, void* stream) {
  return guarded([&] {
    if (G == 0 || k_out > uint64_t(G) * k_in) throw mihg::InvalidArgument("merge: bad shard shape");
    mihg::merge_topk_device(d_ids, d_dists, G, nq, k_in, k_out, d_out_ids, d_out_dists,
                            static_cast<cudaStream_t>(stream));
  });
}

// ---- calibration: random-access lookup rate of the device (see include/mihg.h)
namespace {
__device__ __forceinline__ uint64_t calib_mix(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}
// Four independent lookups in flight per lane, like the sparse probe kernel.
__global__ void __launch_bounds__(256) calib_lookup_kernel(const uint8_t* __restrict__ dir, uint64_t dir_bytes,
                                                           const uint8_t* __restrict__ codes, uint64_t codes_bytes,
                                                           uint32_t nonempty_pct, uint64_t per_thread, uint64_t seed,
                                                           uint32_t* sink) {
  const uint64_t tid = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  uint32_t acc = 0;
  for (uint64_t i = 0; i < per_thread; i += 4) {
    uint4 g[4];
    uint64_t h[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      h[u] = calib_mix(seed + tid * per_thread + i + u);
      g[u] = __ldg(reinterpret_cast<const uint4*>(dir + ((h[u] % dir_bytes) & ~15ull)));
    }
    uint32_t r[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool ne = ((h[u] >> 40) % 100) < nonempty_pct;
      const uint64_t pos = (((h[u] >> 8) + g[u].x) % codes_bytes) & ~3ull;
      r[u] = ne ? __ldg(reinterpret_cast<const uint32_t*>(codes + pos)) : g[u].y;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc ^= r[u];
  }
  if (acc == 0x12345u) *sink = acc;  // keeps the loads alive
}
}  // namespace

int mihg_calibrate_random_lookups(int device, uint64_t dir_bytes, uint64_t codes_bytes, uint32_t nonempty_pct,
                                  double* lookups_per_s) {
  return guarded([&] {
    if (!lookups_per_s || dir_bytes < 16 || codes_bytes < 4 || nonempty_pct > 100)
      throw mihg::InvalidArgument("calibrate: bad arguments");
    MIHG_CUDA(cudaSetDevice(device));
    uint8_t* buf = nullptr;
    uint32_t* sink = nullptr;
    MIHG_CUDA(cudaMalloc(&buf, dir_bytes + codes_bytes));
    MIHG_CUDA(cudaMalloc(&sink, 4));
    MIHG_CUDA(cudaMemset(buf, 0, dir_bytes + codes_bytes));
    cudaEvent_t a, b;
    MIHG_CUDA(cudaEventCreate(&a));
    MIHG_CUDA(cudaEventCreate(&b));
    const int blocks = mihg::device_sm_count() * 6, threads = 256;
    const uint64_t per_thread = 1024;
    float ms = 0;
    for (int rep = 0; rep < 2; ++rep) {  // the second run is the measurement
      MIHG_CUDA(cudaEventRecord(a, nullptr));
      calib_lookup_kernel<<<blocks, threads>>>(buf, dir_bytes, buf + dir_bytes, codes_bytes, nonempty_pct,
                                               per_thread, 7 + rep, sink);
      MIHG_LAUNCH();
      MIHG_CUDA(cudaEventRecord(b, nullptr));
      MIHG_CUDA(cudaEventSynchronize(b));
      MIHG_CUDA(cudaEventElapsedTime(&ms, a, b));
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(buf);
    cudaFree(sink);
    *lookups_per_s = double(blocks) * threads * double(per_thread) / (double(ms) * 1e-3);
  });
}

int mihg_profile_enable(int on) {
  mihg::profile().enabled = on != 0;
  return MIHG_OK;
}

void mihg_profile_reset(void) {
  mihg::ProfileState& p = mihg::profile();
  p.probe_ms = p.scan_ms = 0;
  p.probe_launches = p.scan_launches = 0;
  p.switched_queries = 0;
  p.rerun_queries = 0;
  p.rerun_ms = 0;
}

int mihg_profile_read(mihg_profile* out) {
  const mihg::ProfileState& p = mihg::profile();
  out->kernel_launches = mihg::launch_count();
  out->probe_ms = p.probe_ms;
  out->probe_launches = p.probe_launches;
  out->scan_ms = p.scan_ms;
  out->scan_launches = p.scan_launches;
  out->switched_queries = p.switched_queries;
  out->rerun_queries = p.rerun_queries;
  out->rerun_ms = p.rerun_ms;
  return MIHG_OK;
}

struct mihg_mt64 {
  Mt64 g;
  explicit mihg_mt64(uint64_t seed) : g(seed) {}
};

int mihg_mt64_create(uint64_t seed, mihg_mt64** out) {
  return guarded([&] { *out = new mihg_mt64(seed); });
}

void mihg_mt64_free(mihg_mt64* s) { delete s; }

int mihg_mt64_next_codes(mihg_mt64* s, uint64_t n, uint32_t bits, uint64_t* out) {
  return guarded([&] {
    if (bits == 0 || bits > mihg::kMaxCodeBits) throw mihg::InvalidArgument("gen_uniform: bad width");
    const uint32_t wpc = mihg::words_per_code(bits);
    const uint64_t mask = (bits & 63) == 0 ? ~uint64_t(0) : ((uint64_t(1) << (bits & 63)) - 1);
    for (uint64_t i = 0; i < n; ++i) {
      uint64_t* w = out ? out + i * wpc : nullptr;
      for (uint32_t k = 0; k < wpc; ++k) {
        const uint64_t v = s->g();
        if (w) w[k] = v;
      }
      if (w) w[wpc - 1] &= mask;
    }
  });
}

int mihg_gen_uniform(uint64_t n, uint32_t bits, uint64_t seed, uint64_t* out) {
  return mihg_gen_uniform_range(0, n, bits, seed, out);
}

int mihg_gen_uniform_range(uint64_t first, uint64_t n, uint32_t bits, uint64_t seed, uint64_t* out) {
  return guarded([&] {
    if (bits == 0 || bits > mihg::kMaxCodeBits) throw mihg::InvalidArgument("gen_uniform: bad width");
    Mt64 rng(seed);
    const uint32_t wpc = mihg::words_per_code(bits);
    const uint64_t mask = (bits & 63) == 0 ? ~uint64_t(0) : ((uint64_t(1) << (bits & 63)) - 1);
    for (uint64_t i = 0; i < first * wpc; ++i) rng();  // the stream is sequential: skip draws
    for (uint64_t i = 0; i < n; ++i) {
      uint64_t* w = out + i * wpc;
      for (uint32_t k = 0; k < wpc; ++k) w[k] = rng();
      w[wpc - 1] &= mask;
    }
  });
}

int mihg_estimate_correlations(const uint64_t* codes, uint64_t n, uint32_t bits, int device,
                               int codes_on_device, double* out_corr, uint8_t* out_constant,
                               uint64_t* out_counts) {
  return guarded([&] {
    if (n < 2) throw mihg::InvalidArgument("estimate_correlations: need at least 2 codes");
    if (bits == 0 || bits > mihg::kMaxCodeBits) throw mihg::InvalidArgument("estimate_correlations: bad width");
    if (!codes || !out_corr || !out_constant) throw mihg::InvalidArgument("estimate_correlations: null pointer");
    DeviceGuard g(device);
    cudaStream_t st;
    MIHG_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    std::vector<uint64_t> counts(uint64_t(bits) * bits);
    try {
      mihg::DeviceBuffer<uint64_t> d_counts(counts.size(), st);
      MIHG_CUDA(cudaMemsetAsync(d_counts.get(), 0, counts.size() * 8, st));
      mihg::and_count_gram(codes, n, bits, codes_on_device != 0, d_counts.get(), st);
      MIHG_CUDA(cudaMemcpyAsync(counts.data(), d_counts.get(), counts.size() * 8, cudaMemcpyDeviceToHost, st));
      MIHG_CUDA(cudaStreamSynchronize(st));
    } catch (...) {
      cudaStreamDestroy(st);
      throw;
    }
    cudaStreamDestroy(st);
    for (uint32_t i = 0; i < bits; ++i)  // the kernel fills the upper-triangle tiles only
      for (uint32_t j = i + 1; j < bits; ++j) counts[uint64_t(j) * bits + i] = counts[uint64_t(i) * bits + j];
    if (out_counts) std::memcpy(out_counts, counts.data(), counts.size() * 8);
    mihg::finish_correlations(counts.data(), n, bits, out_corr, out_constant);
  });
}

int mihg_greedy_assign(const double* corr, const uint8_t* constant, uint32_t bits, uint32_t m,
                       uint64_t seed, uint32_t* out_lengths, uint32_t* out_positions) {
  return guarded([&] {
    if (!corr || !constant || !out_lengths || !out_positions) throw mihg::InvalidArgument("greedy_assign: null pointer");
    mihg::greedy_assign(corr, constant, bits, m, seed, out_lengths, out_positions);
  });
}

}  // extern "C"
