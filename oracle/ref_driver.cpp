// TEST INFRASTRUCTURE ONLY — never linked into, or called by, the product path.
//
// C-ABI driver around the UNMODIFIED reference headers at
// /root/reference/proj/include/mih/{codes,table,scan,index,io}.hpp. `oracle/Makefile`
// compiles this file against those headers where they lie and writes the result to
// oracle/_ref/libmihref.so (git-ignored; it travels to the GPU box as a prebuilt file).
// Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / --impl reference legs
// load it, as the checker or the timed CPU baseline.
//
// optimize.hpp (estimate_correlations / greedy_assign) needs only codes.hpp and is included.
// mih.hpp / costmodel.hpp are deliberately NOT included: they pull in <gmpxx.h>, which is
// absent. Every entry point catches C++ exceptions and maps them to
// integer codes (1 = std::invalid_argument, 2 = FormatError/other, 3 = bad_alloc).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <new>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "mih/codes.hpp"
#include "mih/index.hpp"
#include "mih/io.hpp"
#include "mih/optimize.hpp"
#include "mih/scan.hpp"
#include "mih/table.hpp"

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::bad_alloc& e) {
    g_err = "bad_alloc";
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

mih::CodeDatabase make_db(const uint64_t* words, uint64_t n, uint32_t bits) {
  mih::CodeDatabase db = mih::CodeDatabase::zeros(bits, n);
  if (n) std::memcpy(db.mutable_words(0), words, n * db.words_per_entry() * sizeof(uint64_t));
  return db;
}

mih::Partition make_partition(uint32_t bits, uint32_t m, const uint32_t* lengths,
                              const uint32_t* positions) {
  if (!lengths) return mih::consecutive_partition(bits, m);
  std::vector<std::vector<uint32_t>> subs(m);
  uint64_t at = 0;
  for (uint32_t j = 0; j < m; ++j) {
    subs[j].assign(positions + at, positions + at + lengths[j]);
    at += lengths[j];
  }
  return mih::Partition(bits, std::move(subs));
}

void put_trace(const mih::SearchTrace& t, uint64_t* out) {
  out[0] = t.lookups;
  out[1] = t.candidates;
  out[2] = t.unique_candidates;
  out[3] = t.distance_evaluations;
  out[4] = t.final_radius;
}

template <typename F>
void parallel_for(uint64_t count, int nthreads, F&& f) {
  if (nthreads <= 1 || count <= 1) {
    for (uint64_t i = 0; i < count; ++i) f(i, 0);
    return;
  }
  std::vector<std::thread> pool;
  std::vector<std::exception_ptr> errs(nthreads);
  for (int t = 0; t < nthreads; ++t)
    pool.emplace_back([&, t] {
      try {
        // strided assignment, as tools/mih.cpp:363
        for (uint64_t i = t; i < count; i += nthreads) f(i, t);
      } catch (...) {
        errs[t] = std::current_exception();
      }
    });
  for (auto& th : pool) th.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_gen_uniform(uint64_t n, uint32_t bits, uint64_t seed, uint64_t* out) {
  return guarded([&] {
    mih::CodeDatabase db = mih::gen_uniform(n, bits, seed);
    if (n) std::memcpy(out, db.raw_words().data(), db.raw_words().size() * sizeof(uint64_t));
  });
}

// Codes from the reference's non-uniform lane: gen_correlated_vectors + LshSpec::from_data
// + lsh_encode (io.hpp:312-331, :232-262), as used by acceptance.cpp:151-156 and
// io_test.cpp:288-292. `fit_*` vectors define the LSH spec (mean), `enc_*` are encoded.
int ref_gen_lsh(uint64_t fit_n, uint64_t enc_n, uint32_t dim, uint32_t group, double noise,
                uint64_t fit_seed, uint64_t enc_seed, uint32_t bits, uint64_t spec_seed,
                uint64_t* out) {
  return guarded([&] {
    mih::VectorData fit = mih::gen_correlated_vectors(fit_n, dim, group, noise, fit_seed);
    mih::LshSpec spec = mih::LshSpec::from_data(fit, bits, spec_seed);
    mih::VectorData enc =
        enc_seed == fit_seed && enc_n == fit_n ? fit
                                               : mih::gen_correlated_vectors(enc_n, dim, group, noise, enc_seed);
    mih::CodeDatabase db = mih::lsh_encode(enc, spec);
    if (enc_n) std::memcpy(out, db.raw_words().data(), db.raw_words().size() * sizeof(uint64_t));
  });
}

// gen_duplicated_bits (io.hpp:281-297), pins the CLI's `gen --mode correlated`.
int ref_gen_duplicated(uint64_t n, uint32_t bits, uint32_t block, uint64_t seed, uint64_t* out) {
  return guarded([&] {
    mih::CodeDatabase db = mih::gen_duplicated_bits(n, bits, block, seed);
    if (n) std::memcpy(out, db.raw_words().data(), db.raw_words().size() * sizeof(uint64_t));
  });
}

int ref_index_build(const uint64_t* codes, uint64_t n, uint32_t bits, uint32_t m,
                    const uint32_t* lengths, const uint32_t* positions, void** out) {
  return guarded([&] {
    mih::MihIndex idx =
        mih::MihIndex::build(make_db(codes, n, bits), make_partition(bits, m, lengths, positions));
    *out = new mih::MihIndex(std::move(idx));
  });
}

// Same index as ref_index_build, with the m tables built concurrently (one thread per table)
// through the reference's public SubstringTable::build (table.hpp:91-159) and
// MihIndex::assemble (index.hpp:124-141); pairs are formed exactly as MihIndex::build does
// (index.hpp:113-117), so every table is identical. Only the wall time of the setup differs.
int ref_index_build_parallel(const uint64_t* codes, uint64_t n, uint32_t bits, uint32_t m,
                             void** out) {
  return guarded([&] {
    mih::CodeDatabase db = make_db(codes, n, bits);
    mih::Partition part = mih::consecutive_partition(bits, m);
    std::vector<mih::SubstringTable> tables(m);
    std::vector<std::exception_ptr> errs(m);
    std::vector<std::thread> pool;
    for (uint32_t j = 0; j < m; ++j)
      pool.emplace_back([&, j] {
        try {
          std::vector<std::pair<uint64_t, uint32_t>> pairs;
          pairs.reserve(n);
          for (uint64_t i = 0; i < n; ++i)
            pairs.emplace_back(mih::extract_substring(db.code(i), part, j), static_cast<uint32_t>(i));
          tables[j] = mih::SubstringTable::build(part.length(j), std::move(pairs));
        } catch (...) {
          errs[j] = std::current_exception();
        }
      });
    for (auto& t : pool) t.join();
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
    *out = new mih::MihIndex(mih::MihIndex::assemble(std::move(db), std::move(part), std::move(tables)));
  });
}

void ref_index_free(void* h) { delete static_cast<mih::MihIndex*>(h); }

int ref_index_table_s(void* h, uint32_t j, uint32_t* s) {
  return guarded([&] { *s = static_cast<mih::MihIndex*>(h)->table(j).s(); });
}

// Bucket contents of table j (table.hpp:169-175). Writes min(count, cap) ids.
int ref_bucket(void* h, uint32_t j, uint64_t value, uint32_t* out, uint64_t cap, uint64_t* count) {
  return guarded([&] {
    auto seg = static_cast<mih::MihIndex*>(h)->table(j).bucket_lookup(value);
    *count = seg.size();
    for (uint64_t i = 0; i < seg.size() && i < cap; ++i) out[i] = seg[i];
  });
}

// Table statistics (table.hpp:190-197): non_empty_buckets, max_bucket_size, total_entries,
// estimated_bytes.
int ref_table_stats(void* h, uint32_t j, uint64_t* out4) {
  return guarded([&] {
    mih::TableStats st = static_cast<mih::MihIndex*>(h)->table(j).stats();
    out4[0] = st.non_empty_buckets;
    out4[1] = st.max_bucket_size;
    out4[2] = st.total_entries;
    out4[3] = st.estimated_bytes;
  });
}

// Batched MihIndex::knn_search (index.hpp:185-253), one SearchScratch per thread
// (tools/mih.cpp:357-391). ids/dists: nq*k; traces (nullable): nq*5 u64.
int ref_knn(void* h, const uint64_t* queries, uint64_t nq, uint32_t k, uint32_t* ids,
            uint32_t* dists, uint64_t* traces, int nthreads) {
  return guarded([&] {
    const mih::MihIndex& idx = *static_cast<mih::MihIndex*>(h);
    const uint32_t bits = idx.db().bits(), wpc = mih::words_per_code(bits);
    std::vector<mih::SearchScratch> scratch(nthreads > 0 ? nthreads : 1);
    parallel_for(nq, nthreads, [&](uint64_t qi, int t) {
      mih::SearchTrace tr;
      mih::Neighbors res = idx.knn_search({queries + qi * wpc, bits}, k, &tr, &scratch[t]);
      for (uint32_t i = 0; i < res.size(); ++i) {
        ids[qi * k + i] = res[i].id;
        dists[qi * k + i] = res[i].dist;
      }
      if (traces) put_trace(tr, traces + qi * 5);
    });
  });
}

// ref_knn with the wall time of every query (seconds, measured inside its thread): the
// per-query statistics of tools/mih.cpp:198-213 / :316-339. secs: nq doubles or NULL.
int ref_knn_timed(void* h, const uint64_t* queries, uint64_t nq, uint32_t k, uint32_t* ids,
                  uint32_t* dists, uint64_t* traces, int nthreads, double* secs) {
  return guarded([&] {
    const mih::MihIndex& idx = *static_cast<mih::MihIndex*>(h);
    const uint32_t bits = idx.db().bits(), wpc = mih::words_per_code(bits);
    std::vector<mih::SearchScratch> scratch(nthreads > 0 ? nthreads : 1);
    parallel_for(nq, nthreads, [&](uint64_t qi, int t) {
      mih::SearchTrace tr;
      const auto t0 = std::chrono::steady_clock::now();
      mih::Neighbors res = idx.knn_search({queries + qi * wpc, bits}, k, &tr, &scratch[t]);
      if (secs) secs[qi] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      for (uint32_t i = 0; i < res.size(); ++i) {
        ids[qi * k + i] = res[i].id;
        dists[qi * k + i] = res[i].dist;
      }
      if (traces) put_trace(tr, traces + qi * 5);
    });
  });
}

namespace {
void scan_timed(const mih::CodeDatabase& db, const uint64_t* queries, uint64_t nq, uint32_t k,
                uint32_t* ids, uint32_t* dists, int nthreads, double* secs) {
  const uint32_t bits = db.bits(), wpc = mih::words_per_code(bits);
  parallel_for(nq, nthreads, [&](uint64_t qi, int) {
    const auto t0 = std::chrono::steady_clock::now();
    mih::Neighbors res = mih::scan_knn(db, {queries + qi * wpc, bits}, k);
    if (secs) secs[qi] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (uint32_t i = 0; i < res.size(); ++i) {
      ids[qi * k + i] = res[i].id;
      dists[qi * k + i] = res[i].dist;
    }
  });
}
}  // namespace

// scan_knn (scan.hpp:43-68) over an index's own database (MihIndex::db(), index.hpp:143): the
// reference's linear-scan baseline beside its MIH on the same codes, no second copy.
int ref_index_scan_knn_timed(void* h, const uint64_t* queries, uint64_t nq, uint32_t k, uint32_t* ids,
                             uint32_t* dists, int nthreads, double* secs) {
  return guarded([&] {
    scan_timed(static_cast<mih::MihIndex*>(h)->db(), queries, nq, k, ids, dists, nthreads, secs);
  });
}

// A CodeDatabase held by the driver (configs whose reference index does not fit host memory:
// only scan_knn runs over it).
int ref_db_new(const uint64_t* codes, uint64_t n, uint32_t bits, void** out) {
  return guarded([&] { *out = new mih::CodeDatabase(make_db(codes, n, bits)); });
}

// gen_uniform (io.hpp:266-277) straight into a held CodeDatabase.
int ref_db_gen_uniform(uint64_t n, uint32_t bits, uint64_t seed, void** out) {
  return guarded([&] { *out = new mih::CodeDatabase(mih::gen_uniform(n, bits, seed)); });
}

const uint64_t* ref_db_words(void* h) { return static_cast<mih::CodeDatabase*>(h)->raw_words().data(); }

void ref_db_free(void* h) { delete static_cast<mih::CodeDatabase*>(h); }

int ref_db_scan_knn_timed(void* h, const uint64_t* queries, uint64_t nq, uint32_t k, uint32_t* ids,
                          uint32_t* dists, int nthreads, double* secs) {
  return guarded([&] {
    scan_timed(*static_cast<mih::CodeDatabase*>(h), queries, nq, k, ids, dists, nthreads, secs);
  });
}

// MihIndex::range_search (index.hpp:149-176) for one query. Writes min(count, cap).
int ref_range(void* h, const uint64_t* q, uint32_t r, uint32_t* ids, uint32_t* dists,
              uint64_t cap, uint64_t* count, uint64_t* trace) {
  return guarded([&] {
    const mih::MihIndex& idx = *static_cast<mih::MihIndex*>(h);
    mih::SearchTrace tr;
    mih::Neighbors res = idx.range_search({q, idx.db().bits()}, r, &tr);
    *count = res.size();
    for (uint64_t i = 0; i < res.size() && i < cap; ++i) {
      ids[i] = res[i].id;
      dists[i] = res[i].dist;
    }
    if (trace) put_trace(tr, trace);
  });
}

// Batched scan_knn (scan.hpp:43-68) over a raw code array.
int ref_scan_knn(const uint64_t* codes, uint64_t n, uint32_t bits, const uint64_t* queries,
                 uint64_t nq, uint32_t k, uint32_t* ids, uint32_t* dists, int nthreads) {
  return guarded([&] {
    // scan_knn only reads db.raw_words(); build the database view once.
    mih::CodeDatabase db = make_db(codes, n, bits);
    const uint32_t wpc = mih::words_per_code(bits);
    parallel_for(nq, nthreads, [&](uint64_t qi, int) {
      mih::Neighbors res = mih::scan_knn(db, {queries + qi * wpc, bits}, k);
      for (uint32_t i = 0; i < res.size(); ++i) {
        ids[qi * k + i] = res[i].id;
        dists[qi * k + i] = res[i].dist;
      }
    });
  });
}

// scan_range (scan.hpp:29-40) for one query. Writes min(count, cap).
int ref_scan_range(const uint64_t* codes, uint64_t n, uint32_t bits, const uint64_t* q,
                   uint32_t r, uint32_t* ids, uint32_t* dists, uint64_t cap, uint64_t* count) {
  return guarded([&] {
    mih::CodeDatabase db = make_db(codes, n, bits);
    mih::Neighbors res = mih::scan_range(db, {q, bits}, r);
    *count = res.size();
    for (uint64_t i = 0; i < res.size() && i < cap; ++i) {
      ids[i] = res[i].id;
      dists[i] = res[i].dist;
    }
  });
}

// write_codes / read_codes (io.hpp:151-171): the BMIH interchange format.
int ref_write_codes(const uint64_t* codes, uint64_t n, uint32_t bits, const char* path) {
  return guarded([&] { mih::write_codes(make_db(codes, n, bits), path); });
}

int ref_read_codes_header(const char* path, uint32_t* bits, uint64_t* n) {
  return guarded([&] {
    mih::CodeDatabase db = mih::read_codes(path);
    *bits = db.bits();
    *n = db.size();
  });
}

// write_index (io.hpp:335-358): the BMIX index file.
int ref_write_index(void* h, const char* path) {
  return guarded([&] { mih::write_index(*static_cast<mih::MihIndex*>(h), path); });
}

int ref_read_index(const char* path, void** out) {
  return guarded([&] { *out = new mih::MihIndex(mih::read_index(path)); });
}

// estimate_correlations (optimize.hpp:47-92): b*b |Pearson| matrix (row-major) + constant flags.
int ref_estimate_correlations(const uint64_t* codes, uint64_t n, uint32_t bits, double* corr,
                              uint8_t* constant) {
  return guarded([&] {
    const mih::CorrelationMatrix c = mih::estimate_correlations(make_db(codes, n, bits));
    for (uint32_t i = 0; i < bits; ++i) {
      constant[i] = c.is_constant(i) ? 1 : 0;
      for (uint32_t j = 0; j < bits; ++j) corr[uint64_t{i} * bits + j] = c.at(i, j);
    }
  });
}

// greedy_assign (optimize.hpp:101-172) over a given matrix; lengths[m] + concatenated positions.
int ref_greedy_assign(const double* corr, const uint8_t* constant, uint32_t bits, uint32_t m,
                      uint64_t seed, uint32_t* lengths, uint32_t* positions) {
  return guarded([&] {
    mih::CorrelationMatrix c(bits);
    for (uint32_t i = 0; i < bits; ++i) {
      if (constant[i]) c.set_constant(i);
      for (uint32_t j = i + 1; j < bits; ++j) c.set(i, j, corr[uint64_t{i} * bits + j]);
    }
    const mih::Partition p = mih::greedy_assign(c, m, seed);
    uint32_t at = 0;
    for (uint32_t j = 0; j < p.m(); ++j) {
      lengths[j] = p.length(j);
      for (uint32_t pos : p.positions(j)) positions[at++] = pos;
    }
  });
}

}  // extern "C"
