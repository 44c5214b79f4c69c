#pragma once
#include "gd_common.cuh"

namespace gd {
void build_graph(DevGraph& g, const int64_t* pairs, int64_t k, int64_t n_decl, int mode,
                 int flags, cudaStream_t s);
void build_graph_batch(DevGraph& g, const int64_t* pairs, const int64_t* poff_h,
                       const int64_t* gn_h, int64_t G, int flags, cudaStream_t s);
void export_graph(const DevGraph& g, int64_t* edges, int64_t* orig_ids, int64_t* indptr,
                  int64_t* indices, int64_t* slot_ids, int64_t* degrees, cudaStream_t s);
}  // namespace gd
