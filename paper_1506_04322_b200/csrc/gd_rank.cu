// Analytics consumers of the per-edge table on the B200:
// rank_edges / edge_weights / vertex_triangle_counts (analytics.py:142-194).
// Weights come straight from the (device) micro table; the ranking is a
// stable descending radix sort of (weight, canonical index) pairs, so ties
// keep canonical order exactly like the reference's argsort(-w, stable); only
// the top-k rows cross PCIe.
#include <cub/cub.cuh>

#include "gd_common.cuh"
#include "gd_rank.cuh"

namespace gd {

namespace {

__global__ void k_edge_weights(const long long* __restrict__ table, int64_t m, int pattern,
                               int64_t* __restrict__ w, int64_t* __restrict__ idx) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const long long* r = table + 10 * e;
    int64_t x;
    if (pattern == 0) x = r[0];        // triangle: common neighbours
    else if (pattern == 1) x = r[3];   // clique4
    else if (pattern == 2) x = r[4];   // cycle4
    else {                             // star4: C(su,2)+C(sv,2)-uu-vv
      const int64_t su = r[1], sv = r[2];
      x = su * (su - 1) / 2 + sv * (sv - 1) / 2 - r[5] - r[6];
    }
    w[e] = x;
    if (idx) idx[e] = e;
  }
}

__global__ void k_vertex_tri(const long long* __restrict__ table, const int32_t* __restrict__ eu,
                             const int32_t* __restrict__ ev, int64_t m,
                             unsigned long long* __restrict__ acc) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long t = (unsigned long long)table[10 * e];
    if (t) {
      atomicAdd(&acc[eu[e]], t);
      atomicAdd(&acc[ev[e]], t);
    }
  }
}

__global__ void k_halve(const unsigned long long* __restrict__ acc, int64_t n,
                        int64_t* __restrict__ out) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    out[v] = (int64_t)(acc[v] >> 1);
}

__global__ void k_gather_ends(const int64_t* __restrict__ idx, int64_t k,
                              const int32_t* __restrict__ eu, const int32_t* __restrict__ ev,
                              int64_t* __restrict__ u, int64_t* __restrict__ v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k;
       i += (int64_t)gridDim.x * blockDim.x) {
    u[i] = eu[idx[i]];
    v[i] = ev[idx[i]];
  }
}

int grid_for(int64_t work) {
  const int64_t b = (work + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)num_sms() * 16));
}

struct Table {
  DBuf<long long> copy;
  const long long* p = nullptr;
};

void stage_table(const DevGraph& g, const long long* table, bool dev, Table& T, cudaStream_t s) {
  if (g.G != 1) throw Error(GD_EINVAL, "edge analytics need a single graph (not a batch)");
  if (dev) {
    T.p = table;
    return;
  }
  T.copy.alloc((size_t)g.m * 10, s);
  if (g.m)
    GD_CUDA(cudaMemcpyAsync(T.copy.p, table, (size_t)g.m * 80, cudaMemcpyHostToDevice, s));
  T.p = T.copy.p;
}

}  // namespace

void edge_weights(const DevGraph& g, const long long* table, bool dev, int pattern,
                  int64_t* weights_host, cudaStream_t s) {
  Table T;
  stage_table(g, table, dev, T, s);
  DBuf<int64_t> w;
  w.alloc(g.m, s);
  if (g.m) {
    k_edge_weights<<<grid_for(g.m), 256, 0, s>>>(T.p, g.m, pattern, w.p, nullptr);
    GD_LAUNCH_CHECK("edge_weights");
    GD_CUDA(cudaMemcpyAsync(weights_host, w.p, g.m * 8, cudaMemcpyDeviceToHost, s));
  }
  GD_CUDA(cudaStreamSynchronize(s));
}

void rank_edges(const DevGraph& g, const long long* table, bool dev, int pattern, int64_t k,
                int64_t* index, int64_t* u, int64_t* v, int64_t* weight, cudaStream_t s) {
  const int64_t m = g.m;
  if (k < 0 || k > m) k = m;
  Table T;
  stage_table(g, table, dev, T, s);
  DBuf<int64_t> w, idx, w2, idx2, du, dv;
  w.alloc(m, s);
  idx.alloc(m, s);
  w2.alloc(m, s);
  idx2.alloc(m, s);
  if (m) {
    k_edge_weights<<<grid_for(m), 256, 0, s>>>(T.p, m, pattern, w.p, idx.p);
    GD_LAUNCH_CHECK("rank_weights");
    size_t tb = 0;
    GD_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, w.p, w2.p, idx.p, idx2.p, m,
                                                      0, 64, s));
    DBuf<char> tmp;
    tmp.alloc(tb, s);
    GD_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp.p, tb, w.p, w2.p, idx.p, idx2.p, m, 0,
                                                      64, s));
  }
  du.alloc(k, s);
  dv.alloc(k, s);
  if (k) {
    k_gather_ends<<<grid_for(k), 256, 0, s>>>(idx2.p, k, g.eu.p, g.ev.p, du.p, dv.p);
    GD_LAUNCH_CHECK("rank_gather");
    GD_CUDA(cudaMemcpyAsync(index, idx2.p, k * 8, cudaMemcpyDeviceToHost, s));
    GD_CUDA(cudaMemcpyAsync(weight, w2.p, k * 8, cudaMemcpyDeviceToHost, s));
    GD_CUDA(cudaMemcpyAsync(u, du.p, k * 8, cudaMemcpyDeviceToHost, s));
    GD_CUDA(cudaMemcpyAsync(v, dv.p, k * 8, cudaMemcpyDeviceToHost, s));
  }
  GD_CUDA(cudaStreamSynchronize(s));
}

void vertex_triangles(const DevGraph& g, const long long* table, bool dev, int64_t* out_host,
                      cudaStream_t s) {
  Table T;
  stage_table(g, table, dev, T, s);
  DBuf<unsigned long long> acc;
  DBuf<int64_t> out;
  acc.alloc(g.n, s);
  acc.zero();
  out.alloc(g.n, s);
  if (g.m) {
    k_vertex_tri<<<grid_for(g.m), 256, 0, s>>>(T.p, g.eu.p, g.ev.p, g.m, acc.p);
    GD_LAUNCH_CHECK("vertex_triangles");
  }
  if (g.n) {
    k_halve<<<grid_for(g.n), 256, 0, s>>>(acc.p, g.n, out.p);
    GD_LAUNCH_CHECK("vertex_triangles_halve");
    GD_CUDA(cudaMemcpyAsync(out_host, out.p, g.n * 8, cudaMemcpyDeviceToHost, s));
  }
  GD_CUDA(cudaStreamSynchronize(s));
}

}  // namespace gd
