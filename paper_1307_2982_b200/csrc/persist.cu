// BMIX index files: write_index / read_index (io.hpp:335-425, table.hpp:224-270).
//
//   "BMIX" | u32 version=1 | codes block (u32 bits, u64 n, n*W u64 words) |
//   u32 m | per substring: u32 len, len u32 positions |
//   per table: u32 s | u64 entries | u64 groups | per non-empty 32-bucket group, ascending:
//              u64 group id | u32 mask | (c+1) u32 group-local starts | entry u32 ids
//
// The writer produces the reference's bytes exactly (same group order, same local starts, ids in
// insertion order). The reader applies the reference's structural checks (read_codes_block,
// Partition, SubstringTable::from_groups, MihIndex::assemble) with its messages, reports errors as
// FormatError(byte offset), and loads the FILE's tables onto the GPU as given (no re-sort).
#include <bit>
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include "index.cuh"
#include "persist.cuh"

namespace mihg {

namespace {

constexpr char kIndexMagic[4] = {'B', 'M', 'I', 'X'};
constexpr uint32_t kVersion = 1;

struct Reader {
  std::ifstream in;
  std::string path;
  uint64_t size = 0, off = 0;
  explicit Reader(const std::string& p) : in(p, std::ios::binary), path(p) {
    if (!in) throw std::runtime_error("cannot open for reading: " + p);
    in.seekg(0, std::ios::end);
    size = uint64_t(in.tellg());
    in.seekg(0, std::ios::beg);
  }
  void raw(void* dst, uint64_t n, const char* what) {
    if (off + n > size)
      throw FormatError("truncated file " + path + ": reading " + what + " needs " + std::to_string(n) +
                            " bytes, " + std::to_string(size - off) + " remain",
                        off);
    in.read(static_cast<char*>(dst), std::streamsize(n));
    if (!in) throw std::runtime_error("read failed: " + path);
    off += n;
  }
  template <typename T>
  T get(const char* what) {
    T v;
    raw(&v, sizeof(T), what);
    return v;
  }
};

uint64_t host_extract(const uint64_t* c, const std::vector<uint32_t>& pos, uint32_t at, uint32_t len) {
  uint64_t v = 0;
  for (uint32_t i = 0; i < len; ++i) {
    const uint32_t p = pos[at + i];
    v |= ((c[p >> 6] >> (p & 63)) & 1ull) << i;
  }
  return v;
}

}  // namespace

void write_index(Index& idx, const std::string& path) {
  const uint64_t n = idx.n;
  const uint32_t W = idx.W, m = idx.m;
  std::vector<uint64_t> codes(n * W);
  if (n) MIHG_CUDA(cudaMemcpy(codes.data(), idx.codes.get(), n * W * 8, cudaMemcpyDeviceToHost));
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("cannot open for writing: " + path);
  auto put = [&](const void* p, size_t b) { out.write(static_cast<const char*>(p), std::streamsize(b)); };
  put(kIndexMagic, 4);
  put(&kVersion, 4);
  put(&idx.bits, 4);
  put(&n, 8);
  put(codes.data(), codes.size() * 8);
  put(&m, 4);
  for (uint32_t j = 0, at = 0; j < m; ++j) {
    put(&idx.lengths[j], 4);
    put(idx.positions.data() + at, idx.lengths[j] * 4ull);
    at += idx.lengths[j];
  }
  std::vector<uint32_t> ids(n);
  std::vector<uint32_t> keys(n);
  for (uint32_t j = 0, at = 0; j < m; ++j) {
    const TableStorage& t = *idx.tables[j];
    if (n) MIHG_CUDA(cudaMemcpy(ids.data(), t.ids.get(), n * 4, cudaMemcpyDeviceToHost));
    for (uint64_t e = 0; e < n; ++e)
      keys[e] = uint32_t(host_extract(codes.data() + uint64_t(ids[e]) * W, idx.positions, at, idx.lengths[j]));
    at += idx.lengths[j];
    uint64_t groups = 0;
    for (uint64_t e = 0; e < n;) {  // count non-empty 32-bucket groups
      const uint64_t g = keys[e] >> 5;
      while (e < n && (keys[e] >> 5) == g) ++e;
      ++groups;
    }
    put(&t.s, 4);
    put(&n, 8);
    put(&groups, 8);
    std::vector<uint32_t> block;
    for (uint64_t e = 0; e < n;) {  // table.hpp:137-157 group emit
      const uint64_t g = keys[e] >> 5;
      uint64_t ge = e;
      uint32_t mask = 0;
      block.clear();
      block.push_back(0);
      while (ge < n && (keys[ge] >> 5) == g) {
        const uint32_t v = keys[ge];
        mask |= 1u << (v & 31);
        while (ge < n && keys[ge] == v) ++ge;
        block.push_back(uint32_t(ge - e));
      }
      put(&g, 8);
      put(&mask, 4);
      put(block.data(), block.size() * 4);
      put(ids.data() + e, (ge - e) * 4);
      e = ge;
    }
  }
  out.close();
  if (!out) throw std::runtime_error("write failed: " + path);
}

Index* read_index(const std::string& path, int device, const BuildOptions& base_opt) {
  Reader r(path);
  char magic[4];
  r.raw(magic, 4, "magic");
  if (std::string(magic, 4) != std::string(kIndexMagic, 4)) throw FormatError("not an index file (bad magic)", 0);
  const uint32_t version = r.get<uint32_t>("version");
  if (version != kVersion) throw FormatError("unsupported index file version " + std::to_string(version), 4);
  // codes block (io.hpp:124-145)
  const uint64_t header_at = r.off;
  const uint32_t bits = r.get<uint32_t>("code width");
  if (bits == 0 || bits > kMaxCodeBits) throw FormatError("bad code width " + std::to_string(bits), header_at);
  const uint64_t n = r.get<uint64_t>("code count");
  if (n > (uint64_t(1) << 32)) throw FormatError("code count exceeds 2^32", header_at + 4);
  const uint32_t W = words_per_code(bits);
  std::vector<uint64_t> codes(n * W);
  const uint64_t payload_at = r.off;
  if (n) r.raw(codes.data(), n * W * 8, "code words");
  const uint64_t pad = (bits & 63) == 0 ? 0 : ~((uint64_t(1) << (bits & 63)) - 1);
  for (uint64_t i = 0; i < n; ++i)
    if (codes[i * W + W - 1] & pad)
      throw FormatError("nonzero padding bits in record " + std::to_string(i), payload_at + (i * W + W - 1) * 8);
  // partition (io.hpp:372-388)
  const uint64_t part_at = r.off;
  const uint32_t m = r.get<uint32_t>("substring count");
  if (m == 0 || m > bits) throw FormatError("bad substring count", part_at);
  std::vector<uint32_t> lengths(m), positions;
  for (uint32_t j = 0; j < m; ++j) {
    const uint32_t len = r.get<uint32_t>("substring length");
    if (len > bits) throw FormatError("bad substring length", r.off - 4);
    lengths[j] = len;
    const size_t at = positions.size();
    positions.resize(at + len);
    if (len) r.raw(positions.data() + at, uint64_t(len) * 4, "substring positions");
  }
  try {
    validate_partition(bits, m, lengths.data(), positions.data());
  } catch (const std::invalid_argument& e) {
    throw FormatError(std::string("invalid partition: ") + e.what(), part_at);
  }
  // tables (io.hpp:390-418 + SubstringTable::from_groups, table.hpp:224-270)
  std::vector<PreTable> pre(m);
  std::vector<uint64_t> table_at(m);
  for (uint32_t j = 0; j < m; ++j) {
    table_at[j] = r.off;
    const uint32_t s = r.get<uint32_t>("table width");
    const uint64_t entries = r.get<uint64_t>("table entry count");
    const uint64_t groups = r.get<uint64_t>("table group count");
    auto invalid = [&](const std::string& what) {
      return FormatError("invalid table " + std::to_string(j) + ": " + what, table_at[j]);
    };
    if (s == 0 || s > kMaxTableBits)
      throw invalid("SubstringTable: key width must be in [1, 32], got " + std::to_string(s));
    const uint64_t num_groups = ((uint64_t(1) << s) + 31) / 32;
    PreTable& t = pre[j];
    uint64_t prev_g = 0, arena = 0, total = 0;
    bool first = true;
    std::vector<uint32_t> starts;
    for (uint64_t gi = 0; gi < groups; ++gi) {
      const uint64_t gid = r.get<uint64_t>("group id");
      const uint32_t mask = r.get<uint32_t>("group mask");
      if (mask == 0) throw FormatError("empty group mask", r.off - 4);
      const uint32_t c = uint32_t(__builtin_popcount(mask));
      starts.resize(c + 1);
      r.raw(starts.data(), uint64_t(c + 1) * 4, "group starts");
      const uint32_t e = starts[c];
      const size_t at = t.ids.size();
      t.ids.resize(at + e);
      if (e) r.raw(t.ids.data() + at, uint64_t(e) * 4, "group entries");
      if (gid >= num_groups) throw invalid("table group id out of range");
      if (!first && gid <= prev_g) throw invalid("table group ids not ascending");
      if (starts[0] != 0) throw invalid("table group starts must begin at 0");
      for (uint32_t i = 0; i < c; ++i)
        if (starts[i] > starts[i + 1]) throw invalid("table group starts not monotone");
      arena += uint64_t(c) + 1 + e;
      if (arena > (uint64_t(1) << 32)) throw invalid("table arena exceeds 2^32 slots");
      uint32_t mm = mask;
      t.keys.resize(at + e);
      // buckets past 2^s (possible when s < 5) are unreachable by any probe: a table holding
      // entries there is rejected (the reference keeps them, dead; the GPU directory has no slot)
      if (s < 5 && (uint64_t(mask) >> (uint64_t(1) << s)) != 0) throw invalid("table group mask has buckets >= 2^s");
      for (uint32_t i = 0; i < c; ++i) {  // bucket i of the group = i-th set bit of the mask
        const uint32_t bit = uint32_t(__builtin_ctz(mm));
        mm &= mm - 1;
        for (uint32_t x = starts[i]; x < starts[i + 1]; ++x) t.keys[at + x] = uint32_t(gid * 32 + bit);
      }
      total += e;
      prev_g = gid;
      first = false;
    }
    if (total != entries)
      throw invalid("table entry count mismatch: header says " + std::to_string(entries) + ", groups hold " +
                    std::to_string(total));
    // MihIndex::assemble (index.hpp:124-141)
    if (s != lengths[j])
      throw FormatError("inconsistent index: MihIndex: table " + std::to_string(j) +
                            " width does not match its substring", 8);
    if (entries != n)
      throw FormatError("inconsistent index: MihIndex: table " + std::to_string(j) +
                            " entry count does not match the database", 8);
    for (uint32_t id : t.ids)
      if (id >= n) throw invalid("entry id out of range");
  }
  if (r.off != r.size)
    throw FormatError("trailing bytes after index payload in " + path + ": expected size " +
                          std::to_string(r.off) + ", file has " + std::to_string(r.size),
                      r.off);
  BuildOptions opt = base_opt;
  opt.pre = &pre;
  try {
    return build_index(codes.data(), false, n, bits, m, lengths.data(), positions.data(), device, 0, opt);
  } catch (const InconsistentTable& e) {
    throw FormatError(std::string("inconsistent index: ") + e.what(), table_at[e.table]);
  }
}

}  // namespace mihg
