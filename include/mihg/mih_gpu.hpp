// mihg::MihIndex — header-only C++ facade over the C ABI (include/mihg.h) that keeps the
// reference's index-build / kNN-query interface (/root/reference/proj/include/mih/index.hpp):
//
//   auto idx = mihg::MihIndex<>::build(db, partition);            // index.hpp:101-121
//   auto res = idx.knn_search(q, k, &trace, &scratch);             // index.hpp:185-253
//   idx.db(); idx.partition(); idx.num_tables();                    // index.hpp:143-146
//   auto c = mihg::estimate_correlations<mih::CorrelationMatrix>(db); // optimize.hpp:47-92
//   auto p = mihg::greedy_assign<mih::Partition>(c, m, seed);         // optimize.hpp:101-172
//
// It is duck-typed over the reference's own types, so a caller holding mih::CodeDatabase,
// mih::Partition, mih::BinaryCode, mih::SearchTrace and mih::Neighbors switches by replacing
// `mih::MihIndex` with `mihg::MihIndex<mih::Neighbor>`. The C ABI's status
// codes are rethrown as the reference's exception types: MIHG_EINVAL -> std::invalid_argument,
// MIHG_ENOMEM -> std::bad_alloc, others -> mihg::Error.
#pragma once

#include <cstdint>
#include <memory>
#include <new>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../mihg.h"

namespace mihg {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline void check(int rc) {
  if (rc == MIHG_OK) return;
  const std::string msg = mihg_last_error();
  if (rc == MIHG_EINVAL) throw std::invalid_argument(msg);
  if (rc == MIHG_ENOMEM) throw std::bad_alloc();
  throw Error(rc, msg);
}

// Layout-compatible with mih::Neighbor (scan.hpp:14-19).
struct Neighbor {
  uint32_t id = 0;
  uint32_t dist = 0;
  friend bool operator==(const Neighbor&, const Neighbor&) = default;
};

// Layout-compatible with mih::SearchTrace's fields (index.hpp:45-51).
struct SearchTrace {
  uint64_t lookups = 0, candidates = 0, unique_candidates = 0, distance_evaluations = 0;
  uint32_t final_radius = 0;
};

// Minimal standalone code/partition types (used when the reference headers are not included).
struct CodeArray {
  uint32_t bits_ = 0;
  uint64_t n_ = 0;
  std::vector<uint64_t> words_;
  uint32_t bits() const { return bits_; }
  uint64_t size() const { return n_; }
  const std::vector<uint64_t>& raw_words() const { return words_; }
};

template <class NeighborT = Neighbor>
class MihIndex {
 public:
  using Neighbors = std::vector<NeighborT>;

  // MihIndex::build(CodeDatabase db, Partition partition) — any DB type with bits(), size(),
  // raw_words(); any partition type with bits(), m(), positions(j).
  template <class DB, class Part>
  static MihIndex build(const DB& db, const Part& partition, int device = 0) {
    if (partition.bits() != db.bits())
      throw std::invalid_argument("MihIndex::build: partition width does not match codes");
    std::vector<uint32_t> lengths, positions;
    for (uint32_t j = 0; j < partition.m(); ++j) {
      const auto& pos = partition.positions(j);
      lengths.push_back(static_cast<uint32_t>(pos.size()));
      positions.insert(positions.end(), pos.begin(), pos.end());
    }
    MihIndex idx;
    mihg_index* h = nullptr;
    check(mihg_index_build(db.raw_words().data(), db.size(), db.bits(), partition.m(), lengths.data(),
                           positions.data(), device, &h));
    idx.h_.reset(h);
    idx.bits_ = db.bits();
    idx.n_ = db.size();
    idx.m_ = partition.m();
    return idx;
  }

  uint32_t num_tables() const { return m_; }
  uint64_t size() const { return n_; }
  uint32_t bits() const { return bits_; }
  mihg_index* handle() const { return h_.get(); }

  // knn_search(BinaryCode q, uint32_t k, SearchTrace*, SearchScratch*) — index.hpp:185-253.
  // Code: any type with `.words` (const uint64_t*) and `.bits`; TraceT: fields as SearchTrace.
  template <class Code, class TraceT = SearchTrace>
  Neighbors knn_search(const Code& q, uint32_t k, TraceT* trace = nullptr, void* /*scratch*/ = nullptr) const {
    if (q.bits != bits_) throw std::invalid_argument("knn_search: query width mismatch");
    if (k > n_) throw std::invalid_argument("knn_search: k exceeds database size");
    std::vector<uint32_t> ids(k), dists(k);
    mihg_trace t{};
    check(mihg_knn_batch(h_.get(), q.words, 1, k, ids.data(), dists.data(), trace ? &t : nullptr));
    if (trace) {
      trace->lookups = t.lookups;
      trace->candidates = t.candidates;
      trace->unique_candidates = t.unique_candidates;
      trace->distance_evaluations = t.distance_evaluations;
      trace->final_radius = t.final_radius;
    }
    Neighbors out(k);
    for (uint32_t i = 0; i < k; ++i) {
      out[i].id = ids[i];
      out[i].dist = dists[i];
    }
    return out;
  }

  // Batched form (the GPU-native call): queries nq*ceil(bits/64) words, outputs nq*k.
  void knn_search_batch(const uint64_t* queries, uint64_t nq, uint32_t k, uint32_t* ids,
                        uint32_t* dists, mihg_trace* traces = nullptr) const {
    check(mihg_knn_batch(h_.get(), queries, nq, k, ids, dists, traces));
  }

  void scan_knn_batch(const uint64_t* queries, uint64_t nq, uint32_t k, uint32_t* ids,
                      uint32_t* dists) const {
    check(mihg_scan_knn_batch(h_.get(), queries, nq, k, ids, dists));
  }

  // SubstringTable::bucket_lookup (table.hpp:169-175) of table j.
  std::vector<uint32_t> bucket_lookup(uint32_t j, uint64_t value) const {
    uint64_t count = 0;
    check(mihg_bucket_lookup(h_.get(), j, value, nullptr, 0, &count));
    std::vector<uint32_t> out(count);
    check(mihg_bucket_lookup(h_.get(), j, value, out.data(), count, &count));
    return out;
  }

 private:
  struct Free {
    void operator()(mihg_index* h) const { mihg_index_free(h); }
  };
  std::unique_ptr<mihg_index, Free> h_;
  uint32_t bits_ = 0, m_ = 0;
  uint64_t n_ = 0;
};

// estimate_correlations(sample) — optimize.hpp:47-92, Gram kernel on the GPU. CorrT: any type
// constructible from the width with set(i, j, v) / set_constant(i) (mih::CorrelationMatrix).
template <class CorrT, class DB>
CorrT estimate_correlations(const DB& sample, int device = 0) {
  const uint32_t b = sample.bits();
  std::vector<double> corr(uint64_t{b} * b);
  std::vector<uint8_t> constant(b);
  check(mihg_estimate_correlations(sample.raw_words().data(), sample.size(), b, device, 0, corr.data(),
                                   constant.data(), nullptr));
  CorrT out(b);
  for (uint32_t i = 0; i < b; ++i) {
    if (constant[i]) out.set_constant(i);
    for (uint32_t j = i + 1; j < b; ++j) out.set(i, j, corr[uint64_t{i} * b + j]);
  }
  return out;
}

// greedy_assign(corr, m, seed) — optimize.hpp:101-172 (host). PartT: constructible from
// (bits, std::vector<std::vector<uint32_t>>) (mih::Partition); CorrT: bits(), at(), is_constant().
template <class PartT, class CorrT>
PartT greedy_assign(const CorrT& corr, uint32_t m, uint64_t seed) {
  const uint32_t b = corr.bits();
  std::vector<double> v(uint64_t{b} * b);
  std::vector<uint8_t> constant(b);
  for (uint32_t i = 0; i < b; ++i) {
    constant[i] = corr.is_constant(i) ? 1 : 0;
    for (uint32_t j = 0; j < b; ++j) v[uint64_t{i} * b + j] = corr.at(i, j);
  }
  std::vector<uint32_t> lengths(m), positions(b);
  check(mihg_greedy_assign(v.data(), constant.data(), b, m, seed, lengths.data(), positions.data()));
  std::vector<std::vector<uint32_t>> subs(m);
  uint32_t at = 0;
  for (uint32_t j = 0; j < m; ++j)
    for (uint32_t t = 0; t < lengths[j]; ++t) subs[j].push_back(positions[at++]);
  return PartT(b, std::move(subs));
}

}  // namespace mihg
