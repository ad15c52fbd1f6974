// Drop-in check: the reference's own types and its CPU MihIndex next to mihg::MihIndex in one
// program (test infrastructure; compiled in the dev container against
// /root/reference/proj/include, the binary travels to the GPU box like oracle/_ref).
//
// A caller switches by `using mihg::dropin::MihIndex;` (include/mihg/mih_dropin.hpp) in place of
// `mih::MihIndex`; everything else (CodeDatabase, Partition, BinaryCode, SearchTrace, Neighbors,
// TableStats, exceptions) stays the reference's.
#include <cstdio>
#include <cstdlib>
#include <stdexcept>

#include "mih/index.hpp"
#include "mih/io.hpp"
#include "mih/optimize.hpp"
#include "mih/scan.hpp"
#include "mihg/mih_dropin.hpp"
#include "mihg/mih_gpu.hpp"

int main() {
  std::setvbuf(stdout, nullptr, _IONBF, 0);
  int bad = 0;
  // shapes whose reference CPU search is cheap (substrings <= 24 bits: 32-bit substrings at
  // n = 2e4 put the reference in its exhaustive-probing regime, minutes per query)
  for (uint32_t bits : {64u, 70u, 128u}) {
    mih::CodeDatabase db = mih::gen_uniform(20000, bits, 900 + bits);
    mih::CodeDatabase qs = mih::gen_uniform(30, bits, 901 + bits);
    for (uint32_t m : {3u, 4u, 6u}) {
      if ((bits + m - 1) / m > 24) continue;
      mih::Partition p = mih::consecutive_partition(bits, m);
      std::fprintf(stderr, "stage build bits=%u m=%u\n", bits, m);
      mih::MihIndex cpu = mih::MihIndex::build(db, p);
      mihg::dropin::MihIndex gpu = mihg::dropin::MihIndex::build(db, p);
      std::fprintf(stderr, "stage accessors\n");
      // accessors (index.hpp:143-146): the index owns copies of the caller's db and partition
      if (!(gpu.db() == cpu.db()) || !(gpu.partition() == cpu.partition()) || gpu.num_tables() != cpu.num_tables()) {
        std::printf("accessor mismatch bits=%u m=%u\n", bits, m);
        ++bad;
      }
      for (uint32_t j = 0; j < m; ++j) {  // table(j): stats and bucket contents (table.hpp:169-197)
        const mih::TableStats a = cpu.table(j).stats(), b = gpu.table(j).stats();
        if (a.non_empty_buckets != b.non_empty_buckets || a.max_bucket_size != b.max_bucket_size ||
            a.total_entries != b.total_entries || a.estimated_bytes != b.estimated_bytes ||
            cpu.table(j).s() != gpu.table(j).s()) {
          std::printf("table stats mismatch bits=%u m=%u j=%u\n", bits, m, j);
          ++bad;
        }
        for (uint64_t v : {uint64_t{0}, uint64_t{1}, uint64_t{12345} % (uint64_t{1} << cpu.table(j).s()),
                           mih::extract_substring(db.code(7), p, j), mih::extract_substring(db.code(99), p, j)}) {
          const auto sa = cpu.table(j).bucket_lookup(v);
          const std::vector<uint32_t> va(sa.begin(), sa.end());
          if (va != gpu.table(j).bucket_lookup(v)) {
            std::printf("bucket mismatch bits=%u m=%u j=%u v=%llu\n", bits, m, j, (unsigned long long)v);
            ++bad;
          }
        }
      }
      std::fprintf(stderr, "stage range\n");
      for (uint64_t qi = 0; qi < 5; ++qi)  // range_search (index.hpp:149-176)
        for (uint32_t r : {0u, bits / 8, bits / 4}) {
          mih::SearchTrace tc, tg;
          if (!(cpu.range_search(qs.code(qi), r, &tc) == gpu.range_search(qs.code(qi), r, &tg)) ||
              tc.lookups != tg.lookups || tc.candidates != tg.candidates) {
            std::printf("range mismatch bits=%u m=%u q=%llu r=%u\n", bits, m, (unsigned long long)qi, r);
            ++bad;
          }
        }
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
  std::fprintf(stderr, "stage build_index\n");
  // build_index (index.hpp:287-289) and the error contract (index_test.cpp:250-268)
  mih::CodeDatabase db = mih::gen_uniform(10, 64, 1);
  mihg::dropin::MihIndex gpu = mihg::dropin::build_index(db, mih::consecutive_partition(64, 2));
  if (gpu.db().size() != 10 || gpu.partition().m() != 2) ++bad;
  try {
    gpu.range_search(mih::BinaryCode{nullptr, 32}, 1);
    ++bad;
  } catch (const std::invalid_argument&) {
  }
  uint64_t qw[1] = {5};
  try {
    gpu.knn_search(mih::BinaryCode{qw, 64}, 11);
    ++bad;
  } catch (const std::invalid_argument&) {
  }
  if (!gpu.knn_search(mih::BinaryCode{qw, 64}, 0).empty()) ++bad;
  try {
    mihg::dropin::MihIndex::build(db, mih::consecutive_partition(32, 2));
    ++bad;
  } catch (const std::invalid_argument&) {
  }
  std::fprintf(stderr, "stage optimize\n");
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
    std::fprintf(stderr, "stage optimize bits=%u gram done\n", bits);
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
  std::fprintf(stderr, "stage done\n");
  std::printf(bad ? "FAIL %d\n" : "OK drop-in parity (reference MihIndex vs mihg::MihIndex)\n", bad);
  return bad ? 1 : 0;
}
