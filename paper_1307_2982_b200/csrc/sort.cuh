#pragma once
#include <utility>

#include "common.cuh"

namespace mihg {

// Stream-ordered device allocation (cudaMallocAsync); freed on the same stream.
template <typename T>
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  DeviceBuffer(uint64_t n, cudaStream_t st) : st_(st), n_(n) {
    if (n) MIHG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p_), n * sizeof(T), st));
  }
  DeviceBuffer(DeviceBuffer&& o) noexcept : p_(o.p_), st_(o.st_), n_(o.n_) {
    o.p_ = nullptr;
    o.n_ = 0;
  }
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    if (this != &o) {
      reset();
      p_ = o.p_;
      st_ = o.st_;
      n_ = o.n_;
      o.p_ = nullptr;
      o.n_ = 0;
    }
    return *this;
  }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  ~DeviceBuffer() { reset(); }
  void reset() {
    if (p_) cudaFreeAsync(p_, st_);
    p_ = nullptr;
    n_ = 0;
  }
  T* get() const { return p_; }
  uint64_t size() const { return n_; }
  T* release() {
    T* p = p_;
    p_ = nullptr;
    n_ = 0;
    return p;
  }

 private:
  T* p_ = nullptr;
  cudaStream_t st_ = nullptr;
  uint64_t n_ = 0;
};

template <typename T>
void exclusive_scan(const T* in, T* out, uint64_t n, cudaStream_t st);

// Stable LSD radix sort of (key, value) pairs by the low `key_bits` key bits.
void radix_sort_pairs_u32(uint32_t* keys, uint32_t* vals, uint64_t n, uint32_t key_bits,
                          cudaStream_t st);
void radix_sort_keys_u64(uint64_t* keys, uint64_t n, uint32_t key_bits, cudaStream_t st);

}  // namespace mihg
