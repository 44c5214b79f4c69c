// Device edge-list parser (gd_parse.cu).
#pragma once

#include "gd_common.cuh"

namespace gd {

struct ParseOut {
  // [0] pairs  [1] MatrixMarket rows (-1: no size header)
  // [2] error kind (0 none, 1 fewer than 2 tokens, 2 non-integer id,
  //     3 malformed MatrixMarket size header, 4 no data lines)
  // [3] error line (1-based)  [4] its byte offset  [5] its byte length
  // [6] fallback (input the ASCII rules cannot decide)
  // [7] min id  [8] max id (before the shift)  [9] shift applied  [10] lines
  int64_t info[12];
  DBuf<int64_t> pairs;  // device, (pairs x 2)
};

void parse_edge_list(const char* text, int64_t len, const char* const* prefixes, int nprefixes,
                     int cr_newline, int mm_shift, ParseOut& out, cudaStream_t s);

}  // namespace gd
