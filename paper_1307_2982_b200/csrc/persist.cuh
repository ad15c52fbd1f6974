#pragma once
#include <string>

#include "index.cuh"

namespace mihg {

// io.hpp:35-44: format errors carry the byte offset at which they were detected.
struct FormatError : std::runtime_error {
  uint64_t offset;
  FormatError(const std::string& what, uint64_t off)
      : std::runtime_error(what + " (byte offset " + std::to_string(off) + ")"), offset(off) {}
};

void write_index(Index& idx, const std::string& path);
Index* read_index(const std::string& path, int device, const BuildOptions& opt);

}  // namespace mihg
