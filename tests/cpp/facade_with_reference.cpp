// Drop-in check: the reference's own types and its CPU MihIndex next to mihg::MihIndex in one
// program (test infrastructure; compiled in the dev container against
// /root/reference/proj/include, the binary travels to the GPU box like oracle/_ref).
//
// A caller switches by replacing `mih::MihIndex::build(db, p)` with
// `mihg::MihIndex<mih::Neighbor>::build(db, p)`; everything else (CodeDatabase, Partition,
// BinaryCode, SearchTrace, Neighbors, exceptions) stays the reference's.
#include <cstdio>
#include <cstdlib>
#include <stdexcept>

#include "mih/index.hpp"
#include "mih/io.hpp"
#include "mih/optimize.hpp"
#include "mih/scan.hpp"
#include "mihg/mih_gpu.hpp"

int main() {
  int bad = 0;
  // shapes whose reference CPU search is cheap (substrings <= 24 bits: 32-bit substrings at
  // n = 2e4 put the reference in its exhaustive-probing regime, minutes per query)
  for (uint32_t bits : {64u, 70u, 128u}) {
    mih::CodeDatabase db = mih::gen_uniform(20000, bits, 900 + bits);
    mih::CodeDatabase qs = mih::gen_uniform(30, bits, 901 + bits);
    for (uint32_t m : {3u, 4u, 6u}) {
      if ((bits + m - 1) / m > 24) continue;
      mih::Partition p = mih::consecutive_partition(bits, m);
      mih::MihIndex cpu = mih::MihIndex::build(db, p);
      auto gpu = mihg::MihIndex<mih::Neighbor>::build(db, p);
      for (uint64_t qi = 0; qi < qs.size(); ++qi)
        for (uint32_t k : {1u, 10u, 100u}) {
          mih::SearchTrace tc, tg;
          mih::Neighbors a = cpu.knn_search(qs.code(qi), k, &tc);
          mih::Neighbors b = gpu.knn_search(qs.code(qi), k, &tg);
          if (!(a == b) || tc.lookups != tg.lookups || tc.candidates != tg.candidates ||
              tc.unique_candidates != tg.unique_candidates || tc.final_radius != tg.final_radius) {
            std::printf("mismatch bits=%u m=%u q=%llu k=%u\n", bits, m, (unsigned long long)qi, k);
            ++bad;
          }
        }
    }
  }
  // error contract (index_test.cpp:250-268)
  mih::CodeDatabase db = mih::gen_uniform(10, 64, 1);
  auto gpu = mihg::MihIndex<mih::Neighbor>::build(db, mih::consecutive_partition(64, 2));
  uint64_t qw[1] = {5};
  try {
    gpu.knn_search(mih::BinaryCode{qw, 64}, 11);
    ++bad;
  } catch (const std::invalid_argument&) {
  }
  if (!gpu.knn_search(mih::BinaryCode{qw, 64}, 0).empty()) ++bad;
  try {
    mihg::MihIndex<mih::Neighbor>::build(db, mih::consecutive_partition(32, 2));
    ++bad;
  } catch (const std::invalid_argument&) {
  }
  // substring optimisation: the GPU Gram path vs the reference's estimate_correlations (bitwise)
  // and greedy_assign over the reference's own matrix type (optimize.hpp)
  for (uint32_t bits : {16u, 100u, 256u}) {
    mih::CodeDatabase d = mih::gen_duplicated_bits(3000, bits, 4, 40 + bits);
    const mih::CorrelationMatrix want = mih::estimate_correlations(d);
    const auto got = mihg::estimate_correlations<mih::CorrelationMatrix>(d);
    for (uint32_t i = 0; i < bits; ++i) {
      if (want.is_constant(i) != got.is_constant(i)) ++bad;
      for (uint32_t j = 0; j < bits; ++j)
        if (want.at(i, j) != got.at(i, j)) ++bad;
    }
    for (uint32_t m : {2u, 4u}) {
      if (!(mih::greedy_assign(want, m, 7 + m) == mihg::greedy_assign<mih::Partition>(got, m, 7 + m))) {
        std::printf("greedy_assign mismatch bits=%u m=%u\n", bits, m);
        ++bad;
      }
    }
  }
  try {
    mihg::estimate_correlations<mih::CorrelationMatrix>(mih::CodeDatabase::zeros(3, 1));
    ++bad;
  } catch (const std::invalid_argument&) {
  }
  std::printf(bad ? "FAIL %d\n" : "OK drop-in parity (reference MihIndex vs mihg::MihIndex)\n", bad);
  return bad ? 1 : 0;
}
