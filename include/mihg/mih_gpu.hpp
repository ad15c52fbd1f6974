// mihg::MihIndex — header-only C++ facade over the C ABI (include/mihg.h) that keeps the
// reference's index-build / kNN-query interface (/root/reference/proj/include/mih/index.hpp):
//
//   auto idx = mihg::MihIndex<>::build(db, partition);            // index.hpp:101-121
//   auto idx = mihg::build_index(db, partition);                   // index.hpp:287-289
//   auto res = idx.knn_search(q, k, &trace, &scratch);             // index.hpp:185-253
//   auto res = idx.range_search(q, r, &trace);                     // index.hpp:149-176
//   idx.db(); idx.partition(); idx.num_tables();                    // index.hpp:143-145
//   idx.table(j).bucket_lookup(v); idx.table(j).stats();            // index.hpp:146, table.hpp:169-197
//   auto c = mihg::estimate_correlations<mih::CorrelationMatrix>(db); // optimize.hpp:47-92
//   auto p = mihg::greedy_assign<mih::Partition>(c, m, seed);         // optimize.hpp:101-172
//
// The index is generic over the caller's code-database, partition and neighbour types
// (BasicMihIndex<DB, Part, NeighborT>), and holds the database and partition by value as the
// reference does (MihIndex owns its CodeDatabase, index.hpp:101 / :256-257), so db() and
// partition() return the caller's own types. With the reference's headers included first,
// include/mihg/mih_dropin.hpp defines mihg::dropin::MihIndex / build_index over mih::CodeDatabase,
// mih::Partition, mih::Neighbor — a same-named drop-in. The C ABI's status
// codes are rethrown as the reference's exception types: MIHG_EINVAL -> std::invalid_argument,
// MIHG_ENOMEM -> std::bad_alloc, others -> mihg::Error. SearchScratch is accepted and unused
// (the GPU workspace is per index; calls on one index are serialised).
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

// Layout-compatible with mih::TableStats (table.hpp:33-47).
struct TableStats {
  uint64_t non_empty_buckets = 0;
  uint64_t max_bucket_size = 0;
  uint64_t total_entries = 0;
  uint64_t estimated_bytes = 0;
};

// Minimal consecutive partition (codes.hpp:124-211 subset) for callers without the reference.
struct ConsecutivePartition {
  uint32_t bits_ = 0;
  std::vector<std::vector<uint32_t>> subs_;
  ConsecutivePartition() = default;
  ConsecutivePartition(uint32_t bits, uint32_t m) : bits_(bits) {
    if (m == 0 || m > bits)
      throw std::invalid_argument("consecutive_partition: need 1 <= m <= bits, got m=" + std::to_string(m) +
                                  ", bits=" + std::to_string(bits));
    for (uint32_t j = 0, p = 0; j < m; ++j) {
      subs_.emplace_back();
      for (uint32_t i = 0; i < bits / m + (j < bits % m ? 1u : 0u); ++i) subs_.back().push_back(p++);
    }
  }
  uint32_t bits() const { return bits_; }
  uint32_t m() const { return static_cast<uint32_t>(subs_.size()); }
  const std::vector<uint32_t>& positions(uint32_t j) const { return subs_.at(j); }
  uint32_t length(uint32_t j) const { return static_cast<uint32_t>(subs_.at(j).size()); }
};

// SubstringTable view of one GPU table (table.hpp:160-197 read-only surface).
template <class StatsT = TableStats>
class TableView {
 public:
  TableView(mihg_index* h, uint32_t j) : h_(h), j_(j) {
    check(mihg_table_get_info(h_, j_, &info_));
  }
  uint32_t s() const { return info_.s; }
  uint64_t size() const { return info_.total_entries; }
  uint64_t bucket_count() const { return uint64_t{1} << info_.s; }
  // bucket_lookup(value) — table.hpp:169-175: ids in ascending order; value >= 2^s throws.
  std::vector<uint32_t> bucket_lookup(uint64_t value) const {
    uint64_t count = 0;
    check(mihg_bucket_lookup(h_, j_, value, nullptr, 0, &count));
    std::vector<uint32_t> out(count);
    if (count) check(mihg_bucket_lookup(h_, j_, value, out.data(), count, &count));
    return out;
  }
  // stats() — table.hpp:190-197 (the reference's own accounting model for estimated_bytes).
  StatsT stats() const {
    StatsT st{};
    st.non_empty_buckets = info_.non_empty_buckets;
    st.max_bucket_size = info_.max_bucket_size;
    st.total_entries = info_.total_entries;
    st.estimated_bytes = info_.estimated_bytes;
    return st;
  }
  const mihg_table_info& gpu_info() const { return info_; }

 private:
  mihg_index* h_;
  uint32_t j_;
  mihg_table_info info_{};
};

template <class DB = CodeArray, class Part = ConsecutivePartition, class NeighborT = Neighbor,
          class StatsT = TableStats>
class BasicMihIndex {
 public:
  using Neighbors = std::vector<NeighborT>;

  // MihIndex::build(CodeDatabase db, Partition partition) — index.hpp:101-121, by value like the
  // reference (the index owns the database). DB: bits(), size(), raw_words(); Part: bits(), m(),
  // positions(j). Validation and messages are the library's (= the reference's).
  static BasicMihIndex build(DB db, Part partition, int device = 0) {
    if (partition.bits() != db.bits())
      throw std::invalid_argument("MihIndex::build: partition width does not match codes");
    std::vector<uint32_t> lengths, positions;
    for (uint32_t j = 0; j < partition.m(); ++j) {
      const auto& pos = partition.positions(j);
      lengths.push_back(static_cast<uint32_t>(pos.size()));
      positions.insert(positions.end(), pos.begin(), pos.end());
    }
    mihg_index* h = nullptr;
    check(mihg_index_build(db.raw_words().data(), db.size(), db.bits(), partition.m(), lengths.data(),
                           positions.data(), device, &h));
    return BasicMihIndex(h, std::move(db), std::move(partition));
  }

  // MihIndex accessors (index.hpp:143-146).
  const DB& db() const { return db_; }
  const Part& partition() const { return part_; }
  uint32_t num_tables() const { return static_cast<uint32_t>(part_.m()); }
  TableView<StatsT> table(uint32_t j) const {
    if (j >= num_tables()) throw std::out_of_range("MihIndex::table: index out of range");
    return TableView<StatsT>(h_.get(), j);
  }
  uint64_t size() const { return db_.size(); }
  uint32_t bits() const { return db_.bits(); }
  mihg_index* handle() const { return h_.get(); }

  // knn_search(BinaryCode q, uint32_t k, SearchTrace*, SearchScratch*) — index.hpp:185-253.
  // Code: any type with `.words` (const uint64_t*) and `.bits`; TraceT: fields as SearchTrace.
  template <class Code, class TraceT = SearchTrace>
  Neighbors knn_search(const Code& q, uint32_t k, TraceT* trace = nullptr, void* /*scratch*/ = nullptr) const {
    if (q.bits != bits()) throw std::invalid_argument("knn_search: query width mismatch");
    if (k > size()) throw std::invalid_argument("knn_search: k exceeds database size");
    std::vector<uint32_t> ids(k), dists(k);
    mihg_trace t{};
    check(mihg_knn_batch(h_.get(), q.words, 1, k, ids.data(), dists.data(), trace ? &t : nullptr));
    if (trace) put_trace(t, trace);
    Neighbors out(k);
    for (uint32_t i = 0; i < k; ++i) {
      out[i].id = ids[i];
      out[i].dist = dists[i];
    }
    return out;
  }

  // range_search(BinaryCode q, uint32_t r, SearchTrace*, SearchScratch*) — index.hpp:149-176:
  // every code within distance r, in (dist, id) order.
  template <class Code, class TraceT = SearchTrace>
  Neighbors range_search(const Code& q, uint32_t r, TraceT* trace = nullptr, void* /*scratch*/ = nullptr) const {
    if (q.bits != bits()) throw std::invalid_argument("range_search: query width mismatch");
    uint64_t offs[2] = {0, 0};
    mihg_trace t{};
    check(mihg_range_batch(h_.get(), q.words, 1, r, offs, nullptr, nullptr, 0, nullptr));
    std::vector<uint32_t> ids(offs[1]), dists(offs[1]);
    check(mihg_range_batch(h_.get(), q.words, 1, r, offs, ids.data(), dists.data(), offs[1], trace ? &t : nullptr));
    if (trace) put_trace(t, trace);
    Neighbors out(offs[1]);
    for (uint64_t i = 0; i < offs[1]; ++i) {
      out[i].id = ids[i];
      out[i].dist = dists[i];
    }
    return out;
  }

  // Batched forms (the GPU-native calls): queries nq*ceil(bits/64) words, outputs nq*k.
  void knn_search_batch(const uint64_t* queries, uint64_t nq, uint32_t k, uint32_t* ids,
                        uint32_t* dists, mihg_trace* traces = nullptr) const {
    check(mihg_knn_batch(h_.get(), queries, nq, k, ids, dists, traces));
  }

  void scan_knn_batch(const uint64_t* queries, uint64_t nq, uint32_t k, uint32_t* ids,
                      uint32_t* dists) const {
    check(mihg_scan_knn_batch(h_.get(), queries, nq, k, ids, dists));
  }

  // SubstringTable::bucket_lookup (table.hpp:169-175) of table j.
  std::vector<uint32_t> bucket_lookup(uint32_t j, uint64_t value) const { return table(j).bucket_lookup(value); }

 private:
  BasicMihIndex(mihg_index* h, DB db, Part part) : h_(h), db_(std::move(db)), part_(std::move(part)) {}
  template <class TraceT>
  static void put_trace(const mihg_trace& t, TraceT* trace) {
    trace->lookups = t.lookups;
    trace->candidates = t.candidates;
    trace->unique_candidates = t.unique_candidates;
    trace->distance_evaluations = t.distance_evaluations;
    trace->final_radius = t.final_radius;
  }
  struct Free {
    void operator()(mihg_index* h) const { mihg_index_free(h); }
  };
  std::unique_ptr<mihg_index, Free> h_;
  DB db_;
  Part part_;
};

// The round-1 spelling: MihIndex<NeighborT> builds from any DB / partition types (copied in).
template <class NeighborT = Neighbor>
class MihIndex {
 public:
  template <class DB, class Part>
  static BasicMihIndex<DB, Part, NeighborT> build(const DB& db, const Part& partition, int device = 0) {
    return BasicMihIndex<DB, Part, NeighborT>::build(db, partition, device);
  }
};

// build_index(db, partition) — index.hpp:287-289.
template <class DB, class Part>
BasicMihIndex<DB, Part> build_index(DB db, Part partition, int device = 0) {
  return BasicMihIndex<DB, Part>::build(std::move(db), std::move(partition), device);
}

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
