// Incremental selections over a device graph (gd_select.cu).
#pragma once

#include "gd_common.cuh"

namespace gd {

class Selection {
 public:
  Selection(const DevGraph& g, cudaStream_t graph_stream);
  ~Selection();
  Selection(const Selection&) = delete;
  Selection& operator=(const Selection&) = delete;
  // action: 0 add_vertex, 1 remove_vertex (a = dense vertex id),
  //         2 readmit edge, 3 exclude edge (a = canonical edge id);
  // moments: 11 x (lo, hi) two's complement 128-bit running sums
  void apply(int action, int64_t a, uint64_t* moments);

 private:
  const DevGraph& g_;
  cudaStream_t s_;
  struct Impl;
  Impl* p_ = nullptr;
};

}  // namespace gd
