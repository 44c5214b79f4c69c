// Per-edge derived outputs (gd_derive.cu).
#pragma once

#include "gd_common.cuh"

namespace gd {

struct CsvText {
  DBuf<char> text;  // device, header + one line per edge
  int64_t bytes = 0;
};

// Return -1, or (edge << 4 | k) for the first negative derived count (k in
// the order tt0 susv0 ts0 ss0 ti0 ti1 si0 si1 ii0 ii1).
int64_t micro_roles(const DevGraph& g, const long long* table, bool table_dev,
                    const int64_t* orig_host, long long* roles_host, cudaStream_t s);
int64_t micro_csv(const DevGraph& g, const long long* table, bool table_dev,
                  const int64_t* orig_host, CsvText& out, cudaStream_t s);

}  // namespace gd
