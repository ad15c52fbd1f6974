// Same-named drop-in for the reference's MihIndex, over the reference's own types. Include AFTER
// the reference headers (mih/codes.hpp, mih/scan.hpp, mih/table.hpp):
//
//   #include "mih/index.hpp"          // or just codes/scan/table
//   #include "mihg/mih_dropin.hpp"
//   using mihg::dropin::MihIndex;     // was: using mih::MihIndex;
//   using mihg::dropin::build_index;  // was: using mih::build_index;
//
//   MihIndex idx = MihIndex::build(std::move(db), partition);   // index.hpp:101-121
//   mih::Neighbors res = idx.knn_search(q, k, &trace, &scratch); // index.hpp:185-253
//   idx.range_search(q, r); idx.db(); idx.partition(); idx.num_tables();
//   idx.table(j).bucket_lookup(v); idx.table(j).stats();        // -> mih::TableStats
#pragma once

#include "mih_gpu.hpp"

namespace mihg::dropin {

using MihIndex = mihg::BasicMihIndex<mih::CodeDatabase, mih::Partition, mih::Neighbor, mih::TableStats>;

// build_index(CodeDatabase db, Partition partition) — index.hpp:287-289.
inline MihIndex build_index(mih::CodeDatabase db, mih::Partition partition, int device = 0) {
  return MihIndex::build(std::move(db), std::move(partition), device);
}

}  // namespace mihg::dropin
