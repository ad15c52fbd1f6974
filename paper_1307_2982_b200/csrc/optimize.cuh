// Substring optimisation on the GPU: the integer core of
// estimate_correlations (/root/reference/proj/include/mih/optimize.hpp:47-92) and the host-side
// greedy_assign (optimize.hpp:101-172).
#pragma once
#include <cstdint>

#include <cuda_runtime.h>

namespace mihg {

// AND-popcount Gram matrix of the bit columns: counts[i*bits+j] = #{x : bit_i(x) & bit_j(x)}
// (diagonal = ones(i)) over n codes of ceil(bits/64) words, accumulated into the DEVICE buffer
// `d_counts` (bits*bits u64, caller-zeroed). Codes are read from `codes` (device pointer when
// on_device, else host memory streamed through in chunks).
void and_count_gram(const uint64_t* codes, uint64_t n, uint32_t bits, bool on_device,
                    uint64_t* d_counts, cudaStream_t st);

// The reference's floating-point finish over exact integer counts (bitwise equal to the
// reference compiled by its CMake on an FMA host; see optimize.cu).
void finish_correlations(const uint64_t* counts, uint64_t n, uint32_t bits, double* corr,
                         uint8_t* constant);

// greedy_assign over a row-major bits*bits matrix; lengths[m] + concatenated sorted positions.
void greedy_assign(const double* corr, const uint8_t* constant, uint32_t bits, uint32_t m,
                   uint64_t seed, uint32_t* lengths, uint32_t* positions);

}  // namespace mihg
