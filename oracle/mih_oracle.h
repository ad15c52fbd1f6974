/* TEST INFRASTRUCTURE ONLY — CPU restatement of the reference hot path (see mih_oracle.c).
 * Never linked into the product library; only tests/, smoke() and bench.py's CPU legs use it.
 * Return codes: 0 ok, 1 invalid argument (reference: std::invalid_argument), 3 out of memory. */
#ifndef MIH_ORACLE_H
#define MIH_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct or_index or_index;

const char* or_last_error(void);
int or_gen_uniform(uint64_t n, uint32_t bits, uint64_t seed, uint64_t* out);
int or_consecutive_partition(uint32_t bits, uint32_t m, uint32_t* lengths, uint32_t* positions);
uint32_t or_hamming(const uint64_t* a, const uint64_t* b, uint32_t nwords);
int or_index_build(const uint64_t* codes, uint64_t n, uint32_t bits, uint32_t m,
                   const uint32_t* lengths, const uint32_t* positions, or_index** out);
void or_index_free(or_index* idx);
int or_bucket(const or_index* idx, uint32_t j, uint64_t value, uint32_t* out, uint64_t cap,
              uint64_t* count);
int or_knn(const or_index* idx, const uint64_t* queries, uint64_t nq, uint32_t k, uint32_t* ids,
           uint32_t* dists, uint64_t* traces);
int or_range(const or_index* idx, const uint64_t* q, uint32_t r, uint32_t* ids, uint32_t* dists,
             uint64_t cap, uint64_t* count, uint64_t* trace);
int or_scan_knn(const uint64_t* codes, uint64_t n, uint32_t bits, const uint64_t* queries,
                uint64_t nq, uint32_t k, uint32_t* ids, uint32_t* dists);

int or_gen_mixture(uint64_t first, uint64_t n, uint32_t bits, uint32_t dim, uint32_t comps,
                   uint64_t model_seed, uint64_t data_seed, uint64_t* out, int nthreads);

int or_estimate_correlations(const uint64_t* codes, uint64_t n, uint32_t bits, double* corr,
                             uint8_t* constant, uint64_t* counts);
int or_greedy_assign(const double* corr, const uint8_t* constant, uint32_t bits, uint32_t m,
                     uint64_t seed, uint32_t* lengths, uint32_t* positions);

#ifdef __cplusplus
}
#endif
#endif
