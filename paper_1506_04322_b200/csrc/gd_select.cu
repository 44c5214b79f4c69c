// Incremental induced-subgraph selections on the B200:
// the reference's SelectionState._refresh_region / _local_tuple / _close
// (selection.py:120-205).
//
// State on the device, over the base graph's rank-space CSR: active flags
// (per rank id), excluded flags and selected flags (per canonical edge), the
// per-edge tuple (t, su, sv, cl, cy) inside the selection, and eleven running
// 128-bit moments of the selected edges' tuples from which the closure
// (_close) is evaluated in O(1) on the host:
//   [0] m_sel  [1] S t  [2] S s  [3] S cl  [4] S cy  [5] S C(t,2)
//   [6] S su*sv  [7] S t*s  [8] S C(su,2)+C(sv,2)  [9] S t^2  [10] S s^2
// (s = su + sv).  One mutation touches only the edges incident to its region
// (the vertex and its base neighbours, or both endpoints and theirs): each
// candidate edge subtracts its old contribution if it was selected and, if
// it is selected now, recomputes its tuple with the reference's marks
// protocol over the selection-filtered adjacency (one CTA per edge, a
// private n-byte marks array per CTA) and adds the new one.
#include <cub/cub.cuh>

#include "gd_common.cuh"
#include "gd_select.cuh"

namespace gd {

namespace {

typedef __int128 i128;
constexpr int kMoments = 11;

struct SelView {
  int64_t n, m;
  const int64_t* rp;
  const int32_t* col;
  const int32_t* seid;
  const int32_t* eu;  // dense ids
  const int32_t* ev;
  const int32_t* d2r;
  unsigned char* active;    // [n] by rank id
  unsigned char* excluded;  // [m]
  unsigned char* selected;  // [m]
  unsigned char* cand;      // [m] candidate dedupe flags (kept zero between ops)
  long long* tup;           // [m][5]
  unsigned long long* mom;  // [kMoments][2] two's complement 128-bit
};

__device__ __forceinline__ void add_i128(unsigned long long* lohi, i128 v) {
  const unsigned long long lo = (unsigned long long)v;
  const unsigned long long hi = (unsigned long long)((unsigned __int128)v >> 64);
  const unsigned long long old = atomicAdd(lohi, lo);
  const unsigned long long carry = (old + lo < old) ? 1ull : 0ull;
  if (hi + carry) atomicAdd(lohi + 1, hi + carry);
}

// region rows: the op's vertices (rank ids) and, per vertex, its neighbours
__global__ void k_collect(SelView S, const int32_t* __restrict__ seeds, int nseeds,
                          int64_t* __restrict__ list, unsigned long long* __restrict__ count) {
  // one warp per region vertex: seeds[i] itself, then each of its neighbours
  const int warps = gridDim.x * (blockDim.x >> 5);
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  for (int si = 0; si < nseeds; si++) {
    const int x = seeds[si];
    const int64_t b = S.rp[x], e = S.rp[x + 1];
    // region vertex y: x (index -1) or col[b + k]
    for (int64_t k = (int64_t)wid - 1; k < e - b; k += warps) {
      const int y = k < 0 ? x : S.col[b + k];
      for (int64_t q = S.rp[y] + lane; q < S.rp[y + 1]; q += 32) {
        const int ed = S.seid[q];
        if (S.cand[ed]) continue;
        // byte flag set with a 32-bit atomicOr on its word (buffer padded)
        unsigned* w = (unsigned*)((uintptr_t)(S.cand + ed) & ~(uintptr_t)3);
        const unsigned sh = (unsigned)((uintptr_t)(S.cand + ed) & 3u) * 8u;
        const unsigned old = atomicOr(w, 1u << sh);
        if (!((old >> sh) & 0xffu)) list[atomicAdd(count, 1ull)] = ed;
      }
    }
  }
}

template <int NT>
__global__ void __launch_bounds__(NT)
k_refresh(SelView S, const int64_t* __restrict__ list, int64_t nlist, unsigned char* marks_all) {
  typedef cub::BlockReduce<long long, NT> BR;
  __shared__ typename BR::TempStorage tmp;
  __shared__ int s_now;
  unsigned char* marks = marks_all + (size_t)blockIdx.x * S.n;
  for (int64_t li = blockIdx.x; li < nlist; li += gridDim.x) {
    const int e = (int)list[li];
    const int u = S.d2r[S.eu[e]], v = S.d2r[S.ev[e]];
    if (threadIdx.x == 0) {
      const int was = S.selected[e];
      const int now = S.active[u] && S.active[v] && !S.excluded[e];
      s_now = now;
      if (was) {
        const long long* o = S.tup + 5 * e;
        const i128 t = o[0], su = o[1], sv = o[2], s = su + sv;
        add_i128(S.mom + 0, -1);
        add_i128(S.mom + 2, -t);
        add_i128(S.mom + 4, -s);
        add_i128(S.mom + 6, -(i128)o[3]);
        add_i128(S.mom + 8, -(i128)o[4]);
        add_i128(S.mom + 10, -(t * (t - 1) / 2));
        add_i128(S.mom + 12, -(su * sv));
        add_i128(S.mom + 14, -(t * s));
        add_i128(S.mom + 16, -(su * (su - 1) / 2 + sv * (sv - 1) / 2));
        add_i128(S.mom + 18, -(t * t));
        add_i128(S.mom + 20, -(s * s));
      }
      S.selected[e] = (unsigned char)now;
      S.cand[e] = 0;
    }
    __syncthreads();
    if (!s_now) {
      __syncthreads();
      continue;
    }
    // marks protocol (selection.py:155-190) over filtered adjacency
    const int64_t bu = S.rp[u], eu_ = S.rp[u + 1], bv = S.rp[v], ev_ = S.rp[v + 1];
    long long du = 0;
    for (int64_t q = bu + threadIdx.x; q < eu_; q += NT) {
      const int w = S.col[q];
      if (w != v && S.active[w] && !S.excluded[S.seid[q]]) {
        marks[w] = 1;
        du++;
      }
    }
    __syncthreads();
    long long t = 0, sv = 0;
    for (int64_t q = bv + threadIdx.x; q < ev_; q += NT) {
      const int w = S.col[q];
      if (w != u && S.active[w] && !S.excluded[S.seid[q]]) {
        if (marks[w] == 1) {
          marks[w] = 2;
          t++;
        } else {
          marks[w] = 3;
          sv++;
        }
      }
    }
    __syncthreads();
    // 4-cliques: selected edges inside Tri (each pair once: r > w);
    // 4-cycles: selected edges from Star_u to Star_v
    long long cl = 0, cy = 0;
    for (int64_t q = bu + threadIdx.x; q < eu_; q += NT) {
      const int w = S.col[q];
      const unsigned char mw = marks[w];
      if (w == v || (mw != 1 && mw != 2) || S.excluded[S.seid[q]] || !S.active[w]) continue;
      const unsigned char want = mw == 2 ? 2 : 3;
      for (int64_t p = S.rp[w]; p < S.rp[w + 1]; p++) {
        const int r = S.col[p];
        if (marks[r] != want || S.excluded[S.seid[p]]) continue;
        if (want == 2) cl += r > w;
        else cy++;
      }
    }
    const long long T = BR(tmp).Sum(t);
    __syncthreads();
    const long long SV = BR(tmp).Sum(sv);
    __syncthreads();
    const long long DU = BR(tmp).Sum(du);
    __syncthreads();
    const long long CL = BR(tmp).Sum(cl);
    __syncthreads();
    const long long CY = BR(tmp).Sum(cy);
    __syncthreads();
    // clear the marks of N(u), N(v)
    for (int64_t q = bu + threadIdx.x; q < eu_; q += NT) marks[S.col[q]] = 0;
    for (int64_t q = bv + threadIdx.x; q < ev_; q += NT) marks[S.col[q]] = 0;
    if (threadIdx.x == 0) {
      const long long SU = DU - T;
      long long* o = S.tup + 5 * e;
      o[0] = T;
      o[1] = SU;
      o[2] = SV;
      o[3] = CL;
      o[4] = CY;
      const i128 ti = T, su = SU, svv = SV, s = su + svv;
      add_i128(S.mom + 0, 1);
      add_i128(S.mom + 2, ti);
      add_i128(S.mom + 4, s);
      add_i128(S.mom + 6, (i128)CL);
      add_i128(S.mom + 8, (i128)CY);
      add_i128(S.mom + 10, ti * (ti - 1) / 2);
      add_i128(S.mom + 12, su * svv);
      add_i128(S.mom + 14, ti * s);
      add_i128(S.mom + 16, su * (su - 1) / 2 + svv * (svv - 1) / 2);
      add_i128(S.mom + 18, ti * ti);
      add_i128(S.mom + 20, s * s);
    }
    __syncthreads();
  }
}

}  // namespace

struct Selection::Impl {
  DBuf<unsigned char> active, excluded, selected, cand, marks;
  DBuf<long long> tup;
  DBuf<unsigned long long> mom, count;
  DBuf<int64_t> list;
  DBuf<int32_t> seeds;
  int grid = 0;
};

Selection::Selection(const DevGraph& g, cudaStream_t graph_stream) : g_(g), s_(nullptr) {
  if (g.G != 1) throw Error(GD_EINVAL, "selections need a single graph (not a batch)");
  // own stream: the selection may outlive the caller's streams
  GD_CUDA(cudaStreamSynchronize(graph_stream));
  GD_CUDA(cudaStreamCreateWithFlags(&s_, cudaStreamNonBlocking));
  p_ = new Impl;
  cudaStream_t s = s_;
  Impl& P = *p_;
  P.active.alloc(g.n, s);
  P.active.zero();
  P.excluded.alloc(g.m + 4, s);
  P.excluded.zero();
  P.selected.alloc(g.m + 4, s);
  P.selected.zero();
  P.cand.alloc(g.m + 4, s);
  P.cand.zero();
  P.tup.alloc((size_t)g.m * 5, s);
  P.mom.alloc(kMoments * 2, s);
  P.mom.zero();
  P.count.alloc(1, s);
  P.list.alloc(g.m + 1, s);
  P.seeds.alloc(2, s);
  P.grid = std::max(1, std::min(2 * num_sms(), (int)std::max<int64_t>(1, g.m)));
  P.marks.alloc((size_t)P.grid * std::max<int64_t>(1, g.n), s);
  P.marks.zero();
  GD_CUDA(cudaStreamSynchronize(s));
}

Selection::~Selection() {
  if (s_) cudaStreamSynchronize(s_);
  delete p_;  // stream-ordered frees on s_
  if (s_) {
    cudaStreamSynchronize(s_);
    cudaStreamDestroy(s_);
  }
}

void Selection::apply(int action, int64_t a, uint64_t* moments) {
  Impl& P = *p_;
  const DevGraph& g = g_;
  cudaStream_t s = s_;
  int32_t seeds[2];
  int nseeds = 0;
  if (action == 0 || action == 1) {
    if (a < 0 || a >= g.n) throw Error(GD_EINVAL, "vertex out of range");
    int32_t r = 0;
    GD_CUDA(cudaMemcpyAsync(&r, g.d2r.p + a, 4, cudaMemcpyDeviceToHost, s));
    GD_CUDA(cudaStreamSynchronize(s));
    const unsigned char flag = action == 0 ? 1 : 0;
    GD_CUDA(cudaMemcpyAsync(P.active.p + r, &flag, 1, cudaMemcpyHostToDevice, s));
    seeds[nseeds++] = r;
  } else if (action == 2 || action == 3) {
    if (a < 0 || a >= g.m) throw Error(GD_EINVAL, "edge out of range");
    int32_t ends[2];
    GD_CUDA(cudaMemcpyAsync(&ends[0], g.eu.p + a, 4, cudaMemcpyDeviceToHost, s));
    GD_CUDA(cudaMemcpyAsync(&ends[1], g.ev.p + a, 4, cudaMemcpyDeviceToHost, s));
    GD_CUDA(cudaStreamSynchronize(s));
    for (int k = 0; k < 2; k++) {
      GD_CUDA(cudaMemcpyAsync(&seeds[k], g.d2r.p + ends[k], 4, cudaMemcpyDeviceToHost, s));
    }
    GD_CUDA(cudaStreamSynchronize(s));
    nseeds = 2;
    const unsigned char flag = action == 3 ? 1 : 0;
    GD_CUDA(cudaMemcpyAsync(P.excluded.p + a, &flag, 1, cudaMemcpyHostToDevice, s));
  } else {
    throw Error(GD_EINVAL, "unknown selection action");
  }
  SelView S{g.n, g.m, g.rp.p, g.col.p, g.seid.p, g.eu.p, g.ev.p, g.d2r.p, P.active.p,
            P.excluded.p, P.selected.p, P.cand.p, P.tup.p, P.mom.p};
  GD_CUDA(cudaMemcpyAsync(P.seeds.p, seeds, 4 * nseeds, cudaMemcpyHostToDevice, s));
  GD_CUDA(cudaMemsetAsync(P.count.p, 0, 8, s));
  k_collect<<<std::max(1, 4 * num_sms()), 256, 0, s>>>(S, P.seeds.p, nseeds, P.list.p,
                                                        P.count.p);
  GD_LAUNCH_CHECK("selection_collect");
  unsigned long long nl = 0;
  GD_CUDA(cudaMemcpyAsync(&nl, P.count.p, 8, cudaMemcpyDeviceToHost, s));
  GD_CUDA(cudaStreamSynchronize(s));
  if (nl) {
    k_refresh<256><<<(int)std::min<unsigned long long>(nl, (unsigned long long)P.grid), 256, 0,
                     s>>>(S, P.list.p, (int64_t)nl, P.marks.p);
    GD_LAUNCH_CHECK("selection_refresh");
  }
  if (moments)
    GD_CUDA(cudaMemcpyAsync(moments, P.mom.p, kMoments * 16, cudaMemcpyDeviceToHost, s));
  GD_CUDA(cudaStreamSynchronize(s));
}

}  // namespace gd
