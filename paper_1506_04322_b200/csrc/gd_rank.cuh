// Edge analytics over the per-edge table (gd_rank.cu).
#pragma once

#include "gd_common.cuh"

namespace gd {

void edge_weights(const DevGraph& g, const long long* table, bool dev, int pattern,
                  int64_t* weights_host, cudaStream_t s);
void rank_edges(const DevGraph& g, const long long* table, bool dev, int pattern, int64_t k,
                int64_t* index, int64_t* u, int64_t* v, int64_t* weight, cudaStream_t s);
void vertex_triangles(const DevGraph& g, const long long* table, bool dev, int64_t* out_host,
                      cudaStream_t s);

}  // namespace gd
