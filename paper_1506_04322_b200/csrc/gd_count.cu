// Counting kernels of the B200 graphlet census (sm_100a).
//
// The reference computes, for every edge (u, v), the mark-based sweep of
// _micro_edge (census.py:190-256) / _count_edge (census.py:259-303): cost
// sum_e (d(lo) + sum_{w in N(lo)} d(w)) adjacency entries (1.4e13 at R-MAT-20).
// Here the same per-edge quantities are assembled from three enumerations in
// the degree-ordered rank space (rank = ascending (degree, id), so every
// "higher-priority" neighbour list is a contiguous row suffix/prefix):
//
//   pass A  triangle frames: for each vertex a, the local graph L(a) induced on
//           its higher-rank neighbours N+(a) as bitmaps.  Every triangle
//           {a<x<y} is one local edge; every 4-clique {a<x<y<z} one local
//           triangle.  Gives per-edge t(e) = |Tri_e| and cl(e) = 4-cliques
//           through e (packed in one 64-bit counter), and K4 totals.
//   pass B  triangle frames again (per-edge mode): per-edge
//           sum_{w in Tri_e} t(u,w), sum t(v,w), sum d(w)  -> ts, uu, vv, ti.
//   pass C  vertex-priority wedges s-w-x with w, x < s: cnt_s[x] common
//           lower neighbours; every 4-cycle is counted once at its top vertex
//           (2*C4 total = sum_wedges (cnt-1)), and per-edge 4-cycle counts
//           C4(e) = (A^3)_uv - d(u) - d(v) + 1 by wedge attribution.
//   finalize  per canonical edge: the 10 RAW_MICRO_FIELDS through the
//           identities of DESIGN.md (uu = T(u) - sumU + cl, ...), plus the
//           13 CensusSums in 128-bit (census.py:449-462).
#include <algorithm>
#include <functional>

#include <cub/cub.cuh>

#include "gd_count.cuh"

namespace gd {

namespace {

struct View {
  int64_t n, m;
  const int64_t* rp;
  const int32_t* col;
  const int32_t* seid;
  const int64_t* osplit;
  const int32_t* deg;
  const int32_t* r2d;
  const int32_t* vgraph;  // may be null (G == 1)
};

__device__ __forceinline__ int graph_of(const View& g, int v) {
  return g.vgraph ? g.vgraph[v] : 0;
}

__device__ __forceinline__ int pow2_at_least(int x) {
  int h = 32;
  while (h < x) h <<= 1;
  return h;
}

// ------------------------------------------------------------------------
// Per-frame scratch layout (shared memory for bounded frames, a global slab
// per CTA for the largest ones).  All offsets are in bytes.
// ------------------------------------------------------------------------
struct FrameLayout {
  int cap;        // max frame size D
  int hcap;       // hash capacity (pow2 >= 2*cap)
  int wcap;       // row words = ceil(cap/32)
  int rows;       // 1 if bitmap rows are used (pass A)
  int accum;      // 1 if pass-B accumulators are used
  size_t o_lv, o_le, o_p, o_hk, o_hv, o_rows, o_tri2, o_tl, o_dl, o_dn, o_acc;
  size_t bytes;
};

FrameLayout make_layout(int cap, bool rows, bool accum) {
  FrameLayout L{};
  L.cap = cap;
  int h = 32;
  while (h < 2 * cap) h <<= 1;
  L.hcap = h;
  L.wcap = (cap + 31) / 32;
  L.rows = rows;
  L.accum = accum;
  size_t o = 0;
  auto take = [&](size_t b) {
    size_t r = o;
    o += (b + 15) & ~size_t(15);
    return r;
  };
  if (accum) L.o_acc = take(sizeof(unsigned long long) * 3 * cap);
  L.o_lv = take(4 * cap);
  L.o_le = take(4 * cap);
  L.o_p = take(4 * (cap + 1));
  L.o_hk = take(4 * h);
  L.o_hv = take(4 * h);
  if (rows) {
    L.o_rows = take(4ull * cap * L.wcap);
    L.o_tri2 = take(4 * cap);
  }
  if (accum) {
    L.o_tl = take(4 * cap);
    L.o_dl = take(4 * cap);
    L.o_dn = take(4 * cap);
  }
  L.bytes = o;
  return L;
}

__device__ __forceinline__ void hash_insert(int* hk, int* hv, int hmask, int key, int val) {
  unsigned h = hash32((unsigned)key) & hmask;
  while (true) {
    int old = atomicCAS(&hk[h], -1, key);
    if (old == -1 || old == key) {
      hv[h] = val;
      return;
    }
    h = (h + 1) & hmask;
  }
}

__device__ __forceinline__ int hash_find(const int* hk, const int* hv, int hmask, int key) {
  unsigned h = hash32((unsigned)key) & hmask;
  while (true) {
    int k = hk[h];
    if (k == key) return hv[h];
    if (k == -1) return -1;
    h = (h + 1) & hmask;
  }
}

// Load N+(a) of frame a into Lv/Le, the item prefix P (from the global
// out-item prefix OP) and the hash of Lv.  Returns D; total items in P[D].
template <int NT>
__device__ int frame_load(const View& g, int a, char* mem, const FrameLayout& L,
                          const int64_t* __restrict__ OP, int& hmask) {
  const int64_t base = g.osplit[a];
  const int D = (int)(g.rp[a + 1] - base);
  int* Lv = (int*)(mem + L.o_lv);
  int* Le = (int*)(mem + L.o_le);
  int* P = (int*)(mem + L.o_p);
  int* hk = (int*)(mem + L.o_hk);
  int* hv = (int*)(mem + L.o_hv);
  int H = pow2_at_least(2 * D);
  if (H > L.hcap) H = L.hcap;
  hmask = H - 1;
  const int64_t p0 = OP[base];
  for (int j = threadIdx.x; j < D; j += NT) {
    Lv[j] = g.col[base + j];
    Le[j] = g.seid[base + j];
    P[j] = (int)(OP[base + j] - p0);
  }
  if (threadIdx.x == 0) P[D] = (int)(OP[base + D] - p0);
  for (int h = threadIdx.x; h < H; h += NT) hk[h] = -1;
  __syncthreads();
  for (int j = threadIdx.x; j < D; j += NT) hash_insert(hk, hv, hmask, Lv[j], j);
  return D;
}

// ------------------------------------------------------------------------
// pass A
// ------------------------------------------------------------------------
template <int NT>
__device__ void tri_frame(const View& g, int a, char* mem, const FrameLayout& L,
                          const int64_t* __restrict__ OP,
                          unsigned long long* __restrict__ tc,
                          unsigned long long* __restrict__ k4tot) {
  int hmask;
  const int D = frame_load<NT>(g, a, mem, L, OP, hmask);
  int* Lv = (int*)(mem + L.o_lv);
  int* Le = (int*)(mem + L.o_le);
  int* P = (int*)(mem + L.o_p);
  int* hk = (int*)(mem + L.o_hk);
  int* hv = (int*)(mem + L.o_hv);
  unsigned* rows = (unsigned*)(mem + L.o_rows);
  unsigned* tri2 = (unsigned*)(mem + L.o_tri2);
  const int W = (D + 31) >> 5;
  for (int i = threadIdx.x; i < D * W; i += NT) rows[i] = 0u;
  for (int j = threadIdx.x; j < D; j += NT) tri2[j] = 0u;
  __syncthreads();
  const int total = P[D];
  // sweep 1: local adjacency bitmaps (undirected)
  for (int i = threadIdx.x; i < total; i += NT) {
    int j = find_segment(P, D, i);
    int x = Lv[j];
    int y = g.col[g.osplit[x] + (i - P[j])];
    int k = hash_find(hk, hv, hmask, y);
    if (k >= 0) {
      atomicOr(&rows[j * W + (k >> 5)], 1u << (k & 31));
      atomicOr(&rows[k * W + (j >> 5)], 1u << (j & 31));
    }
  }
  __syncthreads();
  // sweep 2: per local edge (x_j, x_k) = triangle {a, x_j, x_k}
  for (int i = threadIdx.x; i < total; i += NT) {
    int j = find_segment(P, D, i);
    int x = Lv[j];
    int64_t q = g.osplit[x] + (i - P[j]);
    int y = g.col[q];
    int k = hash_find(hk, hv, hmask, y);
    if (k >= 0) {
      unsigned c = 0;
      const unsigned* rj = rows + j * W;
      const unsigned* rk = rows + k * W;
      for (int w = 0; w < W; w++) c += __popc(rj[w] & rk[w]);
      atomicAdd(&tc[g.seid[q]], (1ull << kTriShift) + c);
      if (c) {
        atomicAdd(&tri2[j], c);
        atomicAdd(&tri2[k], c);
      }
    }
  }
  __syncthreads();
  unsigned long long local = 0;
  for (int j = threadIdx.x; j < D; j += NT) {
    unsigned dl = 0;
    const unsigned* rj = rows + j * W;
    for (int w = 0; w < W; w++) dl += __popc(rj[w]);
    unsigned t2 = tri2[j];
    if (dl) atomicAdd(&tc[Le[j]], ((unsigned long long)dl << kTriShift) + (t2 >> 1));
    local += t2;
  }
  typedef cub::BlockReduce<unsigned long long, NT> BR;
  __shared__ typename BR::TempStorage tmp;
  unsigned long long s = BR(tmp).Sum(local);
  if (threadIdx.x == 0 && s) atomic_add_u128(k4tot + 2 * graph_of(g, a), s / 6);
  __syncthreads();
}

template <int NT>
__global__ void __launch_bounds__(NT)
k_tri_frames(View g, const int* __restrict__ frames, int nframes, FrameLayout L,
             char* gslab, const int64_t* __restrict__ OP,
             unsigned long long* __restrict__ tc, unsigned long long* __restrict__ k4tot) {
  extern __shared__ __align__(16) char smem[];
  char* mem = gslab ? gslab + (size_t)blockIdx.x * L.bytes : smem;
  for (int f = blockIdx.x; f < nframes; f += gridDim.x)
    tri_frame<NT>(g, frames[f], mem, L, OP, tc, k4tot);
}

// ------------------------------------------------------------------------
// pass B
// ------------------------------------------------------------------------
template <int NT>
__device__ void trisum_frame(const View& g, int a, char* mem, const FrameLayout& L,
                             const int64_t* __restrict__ OP,
                             const unsigned long long* __restrict__ tc,
                             unsigned long long* __restrict__ tsum) {
  int hmask;
  const int D = frame_load<NT>(g, a, mem, L, OP, hmask);
  int* Lv = (int*)(mem + L.o_lv);
  int* Le = (int*)(mem + L.o_le);
  int* P = (int*)(mem + L.o_p);
  int* hk = (int*)(mem + L.o_hk);
  int* hv = (int*)(mem + L.o_hv);
  int* tL = (int*)(mem + L.o_tl);
  int* dL = (int*)(mem + L.o_dl);
  int* nL = (int*)(mem + L.o_dn);
  unsigned long long* acc = (unsigned long long*)(mem + L.o_acc);
  for (int j = threadIdx.x; j < D; j += NT) {
    tL[j] = (int)(tc[Le[j]] >> kTriShift);
    dL[j] = g.deg[Lv[j]];
    nL[j] = g.r2d[Lv[j]];
    acc[3 * j] = 0;
    acc[3 * j + 1] = 0;
    acc[3 * j + 2] = 0;
  }
  __syncthreads();
  const int total = P[D];
  const unsigned long long deg_a = (unsigned long long)g.deg[a];
  for (int i = threadIdx.x; i < total; i += NT) {
    int j = find_segment(P, D, i);
    int x = Lv[j];
    int64_t q = g.osplit[x] + (i - P[j]);
    int y = g.col[q];
    int k = hash_find(hk, hv, hmask, y);
    if (k < 0) continue;
    int e = g.seid[q];
    unsigned long long t_jk = tc[e] >> kTriShift;
    // edge (x_j, x_k): third vertex a
    unsigned long long* te = tsum + 3 * (size_t)e;
    bool j_is_u = nL[j] < nL[k];
    atomicAdd(te + (j_is_u ? 0 : 1), (unsigned long long)tL[j]);
    atomicAdd(te + (j_is_u ? 1 : 0), (unsigned long long)tL[k]);
    atomicAdd(te + 2, deg_a);
    // edge (a, x_j): third vertex x_k; edge (a, x_k): third vertex x_j
    atomicAdd(&acc[3 * j], (unsigned long long)tL[k]);
    atomicAdd(&acc[3 * j + 1], t_jk);
    atomicAdd(&acc[3 * j + 2], (unsigned long long)dL[k]);
    atomicAdd(&acc[3 * k], (unsigned long long)tL[j]);
    atomicAdd(&acc[3 * k + 1], t_jk);
    atomicAdd(&acc[3 * k + 2], (unsigned long long)dL[j]);
  }
  __syncthreads();
  const int na = g.r2d[a];
  for (int j = threadIdx.x; j < D; j += NT) {
    if (acc[3 * j + 2] == 0) continue;  // no triangle on edge (a, x_j)
    unsigned long long* te = tsum + 3 * (size_t)Le[j];
    bool a_is_u = na < nL[j];
    atomicAdd(te + (a_is_u ? 0 : 1), acc[3 * j]);
    atomicAdd(te + (a_is_u ? 1 : 0), acc[3 * j + 1]);
    atomicAdd(te + 2, acc[3 * j + 2]);
  }
  __syncthreads();
}

template <int NT>
__global__ void __launch_bounds__(NT)
k_trisum_frames(View g, const int* __restrict__ frames, int nframes, FrameLayout L,
                char* gslab, const int64_t* __restrict__ OP,
                const unsigned long long* __restrict__ tc,
                unsigned long long* __restrict__ tsum) {
  extern __shared__ __align__(16) char smem[];
  char* mem = gslab ? gslab + (size_t)blockIdx.x * L.bytes : smem;
  for (int f = blockIdx.x; f < nframes; f += gridDim.x)
    trisum_frame<NT>(g, frames[f], mem, L, OP, tc, tsum);
}

// ------------------------------------------------------------------------
// frame work keys and item prefixes
// ------------------------------------------------------------------------
// out-item count of every slot: d+(col[q]) for out-slots (col[q] > row), else 0
__global__ void k_out_items(View g, int64_t* __restrict__ items) {
  // warp per row
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < g.n; r += warps) {
    const int64_t b = g.rp[r], s = g.osplit[r], e = g.rp[r + 1];
    for (int64_t q = b + lane_id(); q < e; q += 32) {
      int64_t v = 0;
      if (q >= s) {
        int x = g.col[q];
        v = g.rp[x + 1] - g.osplit[x];
      }
      items[q] = v;
    }
  }
}

// wedge prefix lengths: for lower slots (w = col[q] < s = row), the number of
// x in N(w) with x < s; 0 for upper slots.  Also per-frame wedge totals.
__global__ void k_wedge_items(View g, int64_t* __restrict__ items,
                              unsigned long long* __restrict__ wedges) {
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; s < g.n; s += warps) {
    const int64_t b = g.rp[s], o = g.osplit[s], e = g.rp[s + 1];
    unsigned long long sum = 0;
    for (int64_t q = b + lane_id(); q < e; q += 32) {
      int64_t v = 0;
      if (q < o) {
        int w = g.col[q];
        v = lower_bound_dev(g.col, g.rp[w], g.rp[w + 1], (int32_t)s) - g.rp[w];
      }
      items[q] = v;
      sum += v;
    }
    for (int off = 16; off; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
    if (lane_id() == 0) wedges[s] = sum;
  }
}

__global__ void k_frame_keys_tri(View g, unsigned long long* __restrict__ keys,
                                 int* __restrict__ ids) {
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < g.n;
       a += (int64_t)gridDim.x * blockDim.x) {
    int64_t D = g.rp[a + 1] - g.osplit[a];
    keys[a] = ~(unsigned long long)D;  // descending
    ids[a] = (int)a;
  }
}

__global__ void k_frame_keys_wedge(int64_t n, const unsigned long long* __restrict__ wedges,
                                   unsigned long long* __restrict__ keys,
                                   int* __restrict__ ids) {
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < n;
       a += (int64_t)gridDim.x * blockDim.x) {
    keys[a] = ~wedges[a];
    ids[a] = (int)a;
  }
}

// ------------------------------------------------------------------------
// pass C: vertex-priority wedges
// ------------------------------------------------------------------------
struct WedgeView {
  const int64_t* WP;  // [2m+1] exclusive prefix of wedge items per slot
};

// item i of frame s -> (slot p of w in row s, pos in row w)
__device__ __forceinline__ int64_t wedge_slot(const int64_t* __restrict__ WP, int64_t lo,
                                              int64_t hi, int64_t i) {
  // last p in [lo, hi) with WP[p] <= i
  while (lo < hi - 1) {
    int64_t mid = (lo + hi) >> 1;
    if (WP[mid] <= i) lo = mid; else hi = mid;
  }
  return lo;
}

// Wedge iteration.  The items of one frame (or chunk) are split in warp
// chunks of 32*K consecutive items; lane l handles items c0+l, c0+l+32, ...
// so lanes of a warp read consecutive entries of the same row w (coalesced)
// and the slot p of an item is found by one binary search per lane per chunk
// followed by forward steps (no per-item search).
constexpr int kWedgeK = 16;

enum WedgeMode { kCount = 0, kUse = 1, kZero = 2, kTake = 3 };

struct SlabCounter {
  unsigned* cnt;
  __device__ __forceinline__ void inc(int x) const { atomicAdd(&cnt[x], 1u); }
  __device__ __forceinline__ unsigned get(int x) const { return cnt[x]; }
  __device__ __forceinline__ unsigned take(int x) const { return atomicExch(&cnt[x], 0u); }
  __device__ __forceinline__ void zero(int x) const { cnt[x] = 0u; }
};

struct HashCounter {
  int* hk;
  int* hv;
  int hmask;
  __device__ __forceinline__ void inc(int x) const {
    unsigned h = hash32((unsigned)x) & hmask;
    while (true) {
      int old = atomicCAS(&hk[h], -1, x);
      if (old == -1 || old == x) {
        atomicAdd(&hv[h], 1);
        return;
      }
      h = (h + 1) & hmask;
    }
  }
  __device__ __forceinline__ unsigned get(int x) const {
    unsigned h = hash32((unsigned)x) & hmask;
    while (hk[h] != x) h = (h + 1) & hmask;
    return (unsigned)hv[h];
  }
  __device__ __forceinline__ unsigned take(int x) const { return get(x); }  // unused
  __device__ __forceinline__ void zero(int) const {}
};

// Runs one sweep of `mode` over items [i0, i1) of frame s (lower slots
// [b, o)).  Returns this thread's partial sum (kUse: sum of cnt-1 over its
// wedges; kTake: sum of c*(c-1) over taken counters).
template <int NT, int MODE, typename C>
__device__ unsigned long long wedge_sweep(const View& g, const int64_t* __restrict__ WP,
                                          int64_t b, int64_t o, int64_t i0, int64_t i1,
                                          const C& ctr, bool per_edge,
                                          unsigned long long* __restrict__ c4e) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int nw = NT / 32;
  constexpr int64_t CH = 32 * kWedgeK;
  unsigned long long local = 0;
  for (int64_t c0 = i0 + (int64_t)warp * CH; c0 < i1; c0 += (int64_t)nw * CH) {
    const int64_t c1 = c0 + CH < i1 ? c0 + CH : i1;
    int64_t i = c0 + lane;
    if (i >= c1) continue;
    int64_t p = wedge_slot(WP, b, o, i);
    int64_t wp1 = WP[p + 1];
    int64_t base = g.rp[g.col[p]] - WP[p];  // q = base + i
    unsigned long long top = 0;             // per-edge: pending sum for edge (s, w_p)
    for (; i < c1; i += 32) {
      if (wp1 <= i) {
        if (MODE == kUse && per_edge && top) {
          atomicAdd(&c4e[g.seid[p]], top);
          top = 0;
        }
        do {
          p++;
          wp1 = WP[p + 1];
        } while (wp1 <= i);
        base = g.rp[g.col[p]] - WP[p];
      }
      const int64_t q = base + i;
      const int x = g.col[q];
      if (MODE == kCount) {
        ctr.inc(x);
      } else if (MODE == kZero) {
        ctr.zero(x);
      } else if (MODE == kTake) {
        unsigned long long c = ctr.take(x);
        local += c * (c - (c > 0));
      } else {
        unsigned long long c = ctr.get(x) - 1u;
        if (c) {
          local += c;
          if (per_edge) {
            atomicAdd(&c4e[g.seid[q]], c);
            top += c;
          }
        }
      }
    }
    if (MODE == kUse && per_edge && top) atomicAdd(&c4e[g.seid[p]], top);
  }
  return local;
}

// Small frames: counters in a shared-memory hash.
template <int NT>
__global__ void __launch_bounds__(NT)
k_c4_frames_smem(View g, const int64_t* __restrict__ WP, const int* __restrict__ frames,
                 int nframes, int hcap, int per_edge,
                 unsigned long long* __restrict__ c4e,
                 unsigned long long* __restrict__ c4tot2) {
  extern __shared__ __align__(16) char smem[];
  int* hk = (int*)smem;
  int* hv = hk + hcap;
  typedef cub::BlockReduce<unsigned long long, NT> BR;
  __shared__ typename BR::TempStorage tmp;
  for (int f = blockIdx.x; f < nframes; f += gridDim.x) {
    const int s = frames[f];
    const int64_t b = g.rp[s], o = g.osplit[s];
    const int64_t i0 = WP[b], i1 = WP[o];
    const int64_t total = i1 - i0;
    int H = pow2_at_least((int)(2 * total < (int64_t)hcap ? 2 * total : (int64_t)hcap));
    if (H > hcap) H = hcap;
    HashCounter ctr{hk, hv, H - 1};
    for (int h = threadIdx.x; h < H; h += NT) {
      hk[h] = -1;
      hv[h] = 0;
    }
    __syncthreads();
    wedge_sweep<NT, kCount>(g, WP, b, o, i0, i1, ctr, false, c4e);
    __syncthreads();
    unsigned long long local = 0;
    if (!per_edge) {
      for (int h = threadIdx.x; h < H; h += NT) {
        unsigned long long c = (unsigned)hv[h];
        local += c * (c - (c > 0));  // 2 * C(c, 2)
      }
    } else {
      local = wedge_sweep<NT, kUse>(g, WP, b, o, i0, i1, ctr, true, c4e);
    }
    unsigned long long sum = BR(tmp).Sum(local);
    if (threadIdx.x == 0 && sum) atomic_add_u128(c4tot2 + 2 * graph_of(g, s), sum);
    __syncthreads();
  }
}

// Large frames: counters in a dense per-CTA global slab (n u32, zero on entry
// and restored to zero on exit).
template <int NT>
__global__ void __launch_bounds__(NT)
k_c4_frames_slab(View g, const int64_t* __restrict__ WP, const int* __restrict__ frames,
                 int nframes, unsigned* __restrict__ slabs, int64_t slab_stride, int per_edge,
                 unsigned long long* __restrict__ c4e, unsigned long long* __restrict__ c4tot2) {
  typedef cub::BlockReduce<unsigned long long, NT> BR;
  __shared__ typename BR::TempStorage tmp;
  SlabCounter ctr{slabs + (size_t)blockIdx.x * slab_stride};
  for (int f = blockIdx.x; f < nframes; f += gridDim.x) {
    const int s = frames[f];
    const int64_t b = g.rp[s], o = g.osplit[s];
    const int64_t i0 = WP[b], i1 = WP[o];
    wedge_sweep<NT, kCount>(g, WP, b, o, i0, i1, ctr, false, c4e);
    __syncthreads();
    unsigned long long local;
    if (!per_edge) {
      local = wedge_sweep<NT, kTake>(g, WP, b, o, i0, i1, ctr, false, c4e);
    } else {
      local = wedge_sweep<NT, kUse>(g, WP, b, o, i0, i1, ctr, true, c4e);
      __syncthreads();
      wedge_sweep<NT, kZero>(g, WP, b, o, i0, i1, ctr, false, c4e);
    }
    unsigned long long sum = BR(tmp).Sum(local);
    if (threadIdx.x == 0 && sum) atomic_add_u128(c4tot2 + 2 * graph_of(g, s), sum);
    __syncthreads();
  }
}

// Hub frames: each (frame, chunk) is one CTA; frame h uses slab h.  The
// sweeps are separate launches (phase 0 count, 1 use, 2 zero).
struct HubChunk {
  int frame;       // rank id s
  int slab;        // slab index
  int64_t i0, i1;  // item range
};

template <int NT>
__global__ void __launch_bounds__(NT)
k_c4_hub(View g, const int64_t* __restrict__ WP, const HubChunk* __restrict__ chunks,
         unsigned* __restrict__ slabs, int64_t slab_stride, int phase, int per_edge,
         unsigned long long* __restrict__ c4e, unsigned long long* __restrict__ c4tot2) {
  typedef cub::BlockReduce<unsigned long long, NT> BR;
  __shared__ typename BR::TempStorage tmp;
  const HubChunk ch = chunks[blockIdx.x];
  SlabCounter ctr{slabs + (size_t)ch.slab * slab_stride};
  const int s = ch.frame;
  const int64_t b = g.rp[s], o = g.osplit[s];
  if (phase == 0) {
    wedge_sweep<NT, kCount>(g, WP, b, o, ch.i0, ch.i1, ctr, false, c4e);
  } else if (phase == 1) {
    unsigned long long local =
        wedge_sweep<NT, kUse>(g, WP, b, o, ch.i0, ch.i1, ctr, per_edge != 0, c4e);
    unsigned long long sum = BR(tmp).Sum(local);
    if (threadIdx.x == 0 && sum) atomic_add_u128(c4tot2 + 2 * graph_of(g, s), sum);
  } else {
    wedge_sweep<NT, kZero>(g, WP, b, o, ch.i0, ch.i1, ctr, false, c4e);
  }
}

// Cooperative rounds for the heavy frames.  All CTAs are co-resident
// (cooperative launch) and walk the same round schedule: a round is up to F
// frames whose u16 counter slabs (n/2 words each) stay L2-resident; its
// items are cut into chunks of CH items spread over the whole grid.
//   step r:  count(round r) + zero(round r-1)  | barrier |  use(round r) | barrier
// Two slab sets alternate so zeroing round r-1 overlaps counting round r.
struct U16Counter {
  unsigned* w;  // 2 counters per 32-bit word
  __device__ __forceinline__ void inc(int x) const {
    atomicAdd(&w[x >> 1], 1u << ((x & 1) << 4));
  }
  __device__ __forceinline__ unsigned get(int x) const {
    return ((const unsigned short*)w)[x];
  }
  __device__ __forceinline__ unsigned take(int x) const { return get(x); }  // unused
  __device__ __forceinline__ void zero(int x) const { ((unsigned short*)w)[x] = 0; }
};

struct RoundPlan {
  const int* frames;    // heavy frames (rank ids), descending wedges
  const int64_t* cpre;  // [nf+1] chunk prefix
  const int* rf;        // [R+1] round -> first frame index
  int R;                // rounds
  int F;                // max frames per round (slabs per set)
  int64_t CH;           // items per chunk
  int64_t slab_words;   // 32-bit words per slab
};

__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned g = gen;
    const unsigned arrived = atomicAdd(&bar[0], 1u) + 1u;
    if (arrived == gridDim.x) {
      bar[0] = 0u;
      __threadfence();
      atomicAdd(&bar[1], 1u);
    } else {
      while (*(volatile unsigned*)&bar[1] == g) __nanosleep(64);
    }
    __threadfence();
  }
  gen++;
  __syncthreads();
}

template <int NT, int MODE>
__device__ void round_chunks(const View& g, const int64_t* __restrict__ WP, const RoundPlan& P,
                             int r, unsigned* __restrict__ slabs, bool per_edge,
                             unsigned long long* __restrict__ c4e,
                             unsigned long long* __restrict__ c4tot2) {
  typedef cub::BlockReduce<unsigned long long, NT> BR;
  __shared__ typename BR::TempStorage tmp;
  const int f0 = P.rf[r], f1 = P.rf[r + 1];
  const int64_t k0 = P.cpre[f0], k1 = P.cpre[f1];
  unsigned* set = slabs + (size_t)(r & 1) * P.F * P.slab_words;
  for (int64_t k = k0 + blockIdx.x; k < k1; k += gridDim.x) {
    // frame of chunk k: last j in [f0, f1) with cpre[j] <= k
    int lo = f0, hi = f1;
    while (lo < hi - 1) {
      int mid = (lo + hi) >> 1;
      if (P.cpre[mid] <= k) lo = mid; else hi = mid;
    }
    const int j = lo;
    const int s = P.frames[j];
    const int64_t b = g.rp[s], o = g.osplit[s];
    const int64_t fi0 = WP[b], fi1 = WP[o];
    const int64_t i0 = fi0 + (k - P.cpre[j]) * P.CH;
    const int64_t i1 = i0 + P.CH < fi1 ? i0 + P.CH : fi1;
    U16Counter ctr{set + (size_t)(j - f0) * P.slab_words};
    unsigned long long local = wedge_sweep<NT, MODE>(g, WP, b, o, i0, i1, ctr, per_edge, c4e);
    if (MODE == kUse) {
      unsigned long long sum = BR(tmp).Sum(local);
      if (threadIdx.x == 0 && sum) atomic_add_u128(c4tot2 + 2 * graph_of(g, s), sum);
      __syncthreads();
    }
  }
}

template <int NT>
__global__ void __launch_bounds__(NT)
k_c4_rounds(View g, const int64_t* __restrict__ WP, RoundPlan P, unsigned* __restrict__ slabs,
            int per_edge, unsigned long long* __restrict__ c4e,
            unsigned long long* __restrict__ c4tot2, unsigned* __restrict__ bar) {
  unsigned gen = 0;
  for (int r = 0; r <= P.R; r++) {
    if (r < P.R) round_chunks<NT, kCount>(g, WP, P, r, slabs, false, c4e, c4tot2);
    if (r > 0) round_chunks<NT, kZero>(g, WP, P, r - 1, slabs, false, c4e, c4tot2);
    if (r == P.R) break;
    grid_barrier(bar, gen);
    round_chunks<NT, kUse>(g, WP, P, r, slabs, per_edge != 0, c4e, c4tot2);
    grid_barrier(bar, gen);
  }
}

// ------------------------------------------------------------------------
// per-vertex T(x) (triangles at x) and S(x) = sum of neighbour degrees
// ------------------------------------------------------------------------
__global__ void k_vertex_stats(View g, const unsigned long long* __restrict__ tc,
                               unsigned long long* __restrict__ vT,
                               unsigned long long* __restrict__ vS) {
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < g.n; r += warps) {
    unsigned long long t = 0, sd = 0;
    for (int64_t q = g.rp[r] + lane_id(); q < g.rp[r + 1]; q += 32) {
      t += tc[g.seid[q]] >> kTriShift;
      sd += (unsigned long long)g.deg[g.col[q]];
    }
    for (int off = 16; off; off >>= 1) {
      t += __shfl_xor_sync(0xffffffffu, t, off);
      sd += __shfl_xor_sync(0xffffffffu, sd, off);
    }
    if (lane_id() == 0) {
      vT[r] = t >> 1;
      vS[r] = sd;
    }
  }
}

// ------------------------------------------------------------------------
// finalize
// ------------------------------------------------------------------------
struct EdgeIn {
  const int32_t* eu;
  const int32_t* ev;
  const int32_t* d2r;
  const int32_t* deg;
  const unsigned long long* tc;
  const unsigned long long* tsum;  // null in global mode
  const unsigned long long* c4e;   // null in global mode
  const unsigned long long* vT;
  const unsigned long long* vS;
};

typedef unsigned __int128 u128;

// per-edge contribution to the 13 CensusSums (census.py:449-462)
__device__ __forceinline__ void add_sums(u128* acc, long long t, long long su, long long sv,
                                         long long cl, long long cy, long long n, long long m) {
  long long i3 = n - 2 - t - su - sv;
  acc[0] += (u128)t;
  acc[1] += (u128)(su + sv);
  acc[2] += (u128)i3;
  acc[3] += (u128)cl;
  acc[4] += (u128)cy;
  acc[5] += (u128)((unsigned long long)t * (unsigned long long)(t - 1) / 2);
  acc[6] += (u128)((unsigned long long)su * (unsigned long long)sv);
  acc[7] += (u128)((unsigned long long)t * (unsigned long long)(su + sv));
  acc[8] += (u128)((unsigned long long)su * (unsigned long long)(su - 1) / 2 +
                   (unsigned long long)sv * (unsigned long long)(sv - 1) / 2);
  acc[9] += (u128)((unsigned long long)t * (unsigned long long)i3);
  acc[10] += (u128)((unsigned long long)(su + sv) * (unsigned long long)i3);
  acc[11] += (u128)((unsigned long long)i3 * (unsigned long long)(i3 - 1) / 2);
  acc[12] += (u128)(m + 1 - (t + su + 1) - (t + sv + 1));
}

// Compute the 10 raw per-edge fields of edge e (RAW_MICRO_FIELDS order).
__device__ __forceinline__ void edge_row(const EdgeIn& in, int64_t e, long long* row) {
  const int ru = in.d2r[in.eu[e]], rv = in.d2r[in.ev[e]];
  const unsigned long long pk = in.tc[e];
  const long long t = (long long)(pk >> kTriShift);
  const long long cl = (long long)(pk & kClMask);
  const long long du = in.deg[ru], dv = in.deg[rv];
  const long long su = du - 1 - t, sv = dv - 1 - t;
  row[0] = t;
  row[1] = su;
  row[2] = sv;
  row[3] = cl;
  if (!in.tsum) return;
  const long long sumU = (long long)in.tsum[3 * e], sumV = (long long)in.tsum[3 * e + 1];
  const long long tdeg = (long long)in.tsum[3 * e + 2];
  const long long tsu = sumU - 2 * cl - t, tsv = sumV - 2 * cl - t, ts = tsu + tsv;
  const long long uu = (long long)in.vT[ru] - t - cl - tsu;
  const long long vv = (long long)in.vT[rv] - t - cl - tsv;
  const long long cy = (long long)in.c4e[e] - ts - 2 * cl;
  const long long sdeg = (long long)in.vS[ru] - dv + (long long)in.vS[rv] - du - 2 * tdeg;
  const long long ti = tdeg - 2 * t - 2 * cl - ts;
  const long long si = sdeg - su - sv - ts - 2 * (uu + vv) - 2 * cy;
  row[4] = cy;
  row[5] = uu;
  row[6] = vv;
  row[7] = ts;
  row[8] = ti;
  row[9] = si;
}

template <int NT>
__device__ void block_flush_sums(u128* acc, unsigned long long* out) {
  // reduce 13 u128 accumulators across the block (as lo/hi pairs) and add
  typedef cub::BlockReduce<unsigned long long, NT> BR;
  __shared__ typename BR::TempStorage tmp;
  for (int k = 0; k < kNumSums; k++) {
    // split into 3 x 43-bit limbs so limb sums cannot overflow 64 bits
    const unsigned long long mask = (1ull << 43) - 1;
    unsigned long long l0 = (unsigned long long)(acc[k]) & mask;
    unsigned long long l1 = (unsigned long long)(acc[k] >> 43) & mask;
    unsigned long long l2 = (unsigned long long)(acc[k] >> 86);
    unsigned long long s0 = BR(tmp).Sum(l0);
    __syncthreads();
    unsigned long long s1 = BR(tmp).Sum(l1);
    __syncthreads();
    unsigned long long s2 = BR(tmp).Sum(l2);
    __syncthreads();
    if (threadIdx.x == 0) {
      u128 v = (u128)s0 + ((u128)s1 << 43) + ((u128)s2 << 86);
      atomic_add_u128(out + 2 * k, v);
    }
  }
}

// G == 1 (or a chunk of one graph): grid-stride over edges [e0, e1)
template <int NT>
__global__ void __launch_bounds__(NT)
k_finalize_single(EdgeIn in, int64_t e0, int64_t e1, long long n, long long m,
                  long long* __restrict__ table, unsigned long long* __restrict__ sums,
                  unsigned long long* __restrict__ seen) {
  u128 acc[kNumSums];
  for (int k = 0; k < kNumSums; k++) acc[k] = 0;
  unsigned long long cnt = 0;
  long long row[kNumMicro];
  for (int64_t e = e0 + blockIdx.x * (int64_t)NT + threadIdx.x; e < e1;
       e += (int64_t)gridDim.x * NT) {
    edge_row(in, e, row);
    const long long cy = in.tsum ? row[4] : 0;
    add_sums(acc, row[0], row[1], row[2], row[3], cy, n, m);
    cnt++;
    if (table) {
      long long* out = table + (size_t)e * kNumMicro;
#pragma unroll
      for (int c = 0; c < kNumMicro; c++) out[c] = row[c];
    }
  }
  block_flush_sums<NT>(acc, sums);
  typedef cub::BlockReduce<unsigned long long, NT> BR;
  __shared__ typename BR::TempStorage tmp2;
  unsigned long long c = BR(tmp2).Sum(cnt);
  if (threadIdx.x == 0 && c) atomicAdd(seen, c);
}

// G > 1: one CTA per graph
template <int NT>
__global__ void __launch_bounds__(NT)
k_finalize_batch(EdgeIn in, const int64_t* __restrict__ eoff, const int64_t* __restrict__ gn,
                 long long* __restrict__ table, unsigned long long* __restrict__ sums,
                 unsigned long long* __restrict__ seen) {
  const int gi = blockIdx.x;
  const int64_t e0 = eoff[gi], e1 = eoff[gi + 1];
  const long long n = gn[gi], m = e1 - e0;
  u128 acc[kNumSums];
  for (int k = 0; k < kNumSums; k++) acc[k] = 0;
  unsigned long long cnt = 0;
  long long row[kNumMicro];
  for (int64_t e = e0 + threadIdx.x; e < e1; e += NT) {
    edge_row(in, e, row);
    const long long cy = in.tsum ? row[4] : 0;
    add_sums(acc, row[0], row[1], row[2], row[3], cy, n, m);
    cnt++;
    if (table) {
      long long* out = table + (size_t)e * kNumMicro;
#pragma unroll
      for (int c = 0; c < kNumMicro; c++) out[c] = row[c];
    }
  }
  block_flush_sums<NT>(acc, sums + (size_t)gi * 2 * kNumSums);
  typedef cub::BlockReduce<unsigned long long, NT> BR;
  __shared__ typename BR::TempStorage tmp2;
  unsigned long long c = BR(tmp2).Sum(cnt);
  if (threadIdx.x == 0) seen[gi] = c;
}

// dual route: sums from a given per-edge table (frequencies_from_micro)
template <int NT>
__global__ void __launch_bounds__(NT)
k_sums_from_table(const long long* __restrict__ table, int64_t m, long long n,
                  unsigned long long* __restrict__ sums) {
  u128 acc[kNumSums];
  for (int k = 0; k < kNumSums; k++) acc[k] = 0;
  for (int64_t e = blockIdx.x * (int64_t)NT + threadIdx.x; e < m; e += (int64_t)gridDim.x * NT) {
    const long long* r = table + (size_t)e * kNumMicro;
    add_sums(acc, r[0], r[1], r[2], r[3], r[4], n, m);
  }
  block_flush_sums<NT>(acc, sums);
}

View make_view(const DevGraph& g) {
  View v;
  v.n = g.n;
  v.m = g.m;
  v.rp = g.rp.p;
  v.col = g.col.p;
  v.seid = g.seid.p;
  v.osplit = g.osplit.p;
  v.deg = g.deg.p;
  v.r2d = g.r2d.p;
  v.vgraph = g.G > 1 ? g.vgraph.p : nullptr;
  return v;
}

int grid_cap(int64_t work, int threads, int per_sm = 16) {
  int64_t g = (work + threads - 1) / threads;
  int64_t cap = (int64_t)num_sms() * per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

void exclusive_scan(const int64_t* in, int64_t* out, int64_t n, cudaStream_t s) {
  size_t tb = 0;
  GD_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n, s));
  DBuf<char> tmp;
  tmp.alloc(tb, s);
  GD_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, in, out, n, s));
}

void sort_frames(unsigned long long* keys, int* ids, int64_t n, DBuf<int>& sorted_ids,
                 DBuf<unsigned long long>& sorted_keys, cudaStream_t s) {
  sorted_ids.alloc(n, s);
  sorted_keys.alloc(n, s);
  size_t tb = 0;
  GD_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, sorted_keys.p, ids, sorted_ids.p,
                                          n, 0, 64, s));
  DBuf<char> tmp;
  tmp.alloc(tb, s);
  GD_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys, sorted_keys.p, ids, sorted_ids.p, n,
                                          0, 64, s));
}

// Count frames per bin: bins are [lo_b, hi_b] on the (descending) key.
std::vector<int64_t> host_keys(const DBuf<unsigned long long>& k, cudaStream_t s) {
  std::vector<int64_t> h(k.n);
  std::vector<unsigned long long> raw(k.n);
  if (k.n)
    GD_CUDA(cudaMemcpyAsync(raw.data(), k.p, k.n * 8, cudaMemcpyDeviceToHost, s));
  GD_CUDA(cudaStreamSynchronize(s));
  for (size_t i = 0; i < k.n; i++) h[i] = (int64_t)(~raw[i]);
  return h;
}

struct Timer {
  cudaStream_t s;
  std::vector<cudaEvent_t> ev;
  std::vector<std::string> names;
  explicit Timer(cudaStream_t st) : s(st) { mark("start"); }
  void mark(const std::string& name) {
    cudaEvent_t e;
    GD_CUDA(cudaEventCreate(&e));
    GD_CUDA(cudaEventRecord(e, s));
    ev.push_back(e);
    names.push_back(name);
  }
  void collect(std::vector<float>& ms, std::vector<std::string>& out_names) {
    GD_CUDA(cudaStreamSynchronize(s));
    ms.clear();
    out_names.clear();
    for (size_t i = 1; i < ev.size(); i++) {
      float t = 0;
      GD_CUDA(cudaEventElapsedTime(&t, ev[i - 1], ev[i]));
      ms.push_back(t);
      out_names.push_back(names[i]);
    }
  }
  ~Timer() {
    for (auto e : ev) cudaEventDestroy(e);
  }
};

// bins for the triangle frames (by D = |N+(a)|)
struct TriBin {
  int lo, hi;  // D in [lo, hi]
  int nt;      // threads
};

template <int NT>
void launch_tri(const View& v, const int* frames, int nf, const FrameLayout& L, char* slab,
                int grid, const int64_t* OP, unsigned long long* tc, unsigned long long* k4,
                cudaStream_t s) {
  size_t sm = slab ? 0 : L.bytes;
  if (sm > 48 * 1024)
    GD_CUDA(cudaFuncSetAttribute(k_tri_frames<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sm));
  k_tri_frames<NT><<<grid, NT, sm, s>>>(v, frames, nf, L, slab, OP, tc, k4);
  GD_LAUNCH_CHECK("tri_frames");
}

template <int NT>
void launch_trisum(const View& v, const int* frames, int nf, const FrameLayout& L, char* slab,
                   int grid, const int64_t* OP, const unsigned long long* tc,
                   unsigned long long* tsum, cudaStream_t s) {
  size_t sm = slab ? 0 : L.bytes;
  if (sm > 48 * 1024)
    GD_CUDA(cudaFuncSetAttribute(k_trisum_frames<NT>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  k_trisum_frames<NT><<<grid, NT, sm, s>>>(v, frames, nf, L, slab, OP, tc, tsum);
  GD_LAUNCH_CHECK("trisum_frames");
}

}  // namespace

// ---------------------------------------------------------------------------
// Host orchestration
// ---------------------------------------------------------------------------
// Test-only schedule overrides (GD_FORCE_PATH=tri_gmem,c4_slab,...): route
// every frame through one kernel variant so each variant can be checked
// against the oracle on small graphs.  Results never depend on the path.
struct ForcePaths {
  bool tri_gmem = false, tri_small = false, c4_slab = false, c4_coop = false,
       c4_hub32 = false, c4_smem = false;
};

static ForcePaths read_force() {
  ForcePaths f;
  const char* e = getenv("GD_FORCE_PATH");
  if (!e) return f;
  std::string v(e);
  f.tri_gmem = v.find("tri_gmem") != std::string::npos;
  f.tri_small = v.find("tri_small") != std::string::npos;
  f.c4_slab = v.find("c4_slab") != std::string::npos;
  f.c4_coop = v.find("c4_coop") != std::string::npos;
  f.c4_hub32 = v.find("c4_hub32") != std::string::npos;
  f.c4_smem = v.find("c4_smem") != std::string::npos;
  return f;
}

void run_census(DevGraph& g, bool per_edge, long long* table_dev, unsigned long long* sums_dev,
                unsigned long long* seen_dev, CensusExtras& ex, cudaStream_t s) {
  const ForcePaths force = read_force();
  const long long launches0 = g_launches;
  const int64_t n = g.n, m = g.m, G = g.G;
  const View v = make_view(g);
  Timer timer(s);
  ex.k4tot.assign(G, 0);
  ex.c4tot2.assign(G, 0);

  DBuf<unsigned long long> tc, tsum, c4e, vT, vS, k4tot, c4tot2;
  tc.alloc(m, s);
  tc.zero();
  k4tot.alloc(2 * G, s);
  k4tot.zero();
  c4tot2.alloc(2 * G, s);
  c4tot2.zero();
  if (per_edge) {
    tsum.alloc(3 * m, s);
    tsum.zero();
    c4e.alloc(m, s);
    c4e.zero();
  }
  vT.alloc(n, s);
  vS.alloc(n, s);

  // ---- scheduling: item prefixes and frame orders -----------------------
  DBuf<int64_t> items, OP, WP;
  items.alloc(2 * m + 1, s);
  OP.alloc(2 * m + 1, s);
  WP.alloc(2 * m + 1, s);
  DBuf<unsigned long long> wedges;
  wedges.alloc(n, s);
  if (n) {
    k_out_items<<<grid_cap(n * 32, 256), 256, 0, s>>>(v, items.p);
    GD_LAUNCH_CHECK("out_items");
  }
  GD_CUDA(cudaMemsetAsync(items.p + 2 * m, 0, 8, s));
  exclusive_scan(items.p, OP.p, 2 * m + 1, s);
  if (n) {
    k_wedge_items<<<grid_cap(n * 32, 256), 256, 0, s>>>(v, items.p, wedges.p);
    GD_LAUNCH_CHECK("wedge_items");
  }
  GD_CUDA(cudaMemsetAsync(items.p + 2 * m, 0, 8, s));
  exclusive_scan(items.p, WP.p, 2 * m + 1, s);
  items.release();
  timer.mark("sched_prefix");

  DBuf<unsigned long long> fk, fk_sorted, wk_sorted;
  DBuf<int> fid, tri_frames, c4_frames;
  fk.alloc(n, s);
  fid.alloc(n, s);
  if (n) {
    k_frame_keys_tri<<<grid_cap(n, 256), 256, 0, s>>>(v, fk.p, fid.p);
    GD_LAUNCH_CHECK("frame_keys_tri");
  }
  if (n) sort_frames(fk.p, fid.p, n, tri_frames, fk_sorted, s);
  if (n) {
    k_frame_keys_wedge<<<grid_cap(n, 256), 256, 0, s>>>(n, wedges.p, fk.p, fid.p);
    GD_LAUNCH_CHECK("frame_keys_wedge");
  }
  if (n) sort_frames(fk.p, fid.p, n, c4_frames, wk_sorted, s);
  std::vector<int64_t> dkeys = host_keys(fk_sorted, s);  // descending D
  std::vector<int64_t> wkeys = host_keys(wk_sorted, s);  // descending wedges
  timer.mark("schedule");

  // ---- pass A -------------------------------------------------------------
  // frames with D >= 2, descending D.  Bins: (1024,inf) global slab,
  // (512,1024], (128,512], (32,128], [2,32].
  auto count_range = [&](const std::vector<int64_t>& keys, int64_t lo, int64_t hi) {
    // keys descending; return [begin, end) of entries with lo <= key <= hi
    auto b = std::lower_bound(keys.begin(), keys.end(), hi, std::greater<int64_t>());
    auto e = std::upper_bound(keys.begin(), keys.end(), lo, std::greater<int64_t>());
    return std::make_pair((int64_t)(b - keys.begin()), (int64_t)(e - keys.begin()));
  };
  ex.stats.clear();
  ex.stats_names.clear();
  auto run_tri_like = [&](bool trisum) {
    const bool rows = !trisum;
    const int64_t maxD = dkeys.empty() ? 0 : dkeys[0];
    struct B { int64_t lo, hi; int nt; bool gmem; };
    std::vector<B> bins = {{1025, INT64_MAX, 512, true}, {513, 1024, 512, false},
                           {129, 512, 256, false}, {33, 128, 128, false}, {2, 32, 32, false}};
    if (force.tri_gmem) bins = {{2, INT64_MAX, 512, true}};
    if (force.tri_small) bins = {{2, INT64_MAX, 32, false}};
    for (const B& bn : bins) {
      auto r = count_range(dkeys, bn.lo, bn.hi);
      const int64_t nf = r.second - r.first;
      if (nf <= 0) continue;
      const int cap = (int)std::min<int64_t>(bn.hi, maxD);
      FrameLayout L = make_layout(cap, rows, trisum);
      const int* fr = tri_frames.p + r.first;
      DBuf<char> slab;
      int grid;
      if (bn.gmem) {
        grid = (int)std::min<int64_t>(nf, 2 * num_sms());
        slab.alloc((size_t)grid * L.bytes, s);
      } else {
        grid = (int)std::min<int64_t>(nf, (int64_t)num_sms() * 64);
      }
      char* sp = bn.gmem ? slab.p : nullptr;
      if (!trisum) {
        switch (bn.nt) {
          case 512: launch_tri<512>(v, fr, (int)nf, L, sp, grid, OP.p, tc.p, k4tot.p, s); break;
          case 256: launch_tri<256>(v, fr, (int)nf, L, sp, grid, OP.p, tc.p, k4tot.p, s); break;
          case 128: launch_tri<128>(v, fr, (int)nf, L, sp, grid, OP.p, tc.p, k4tot.p, s); break;
          default: launch_tri<32>(v, fr, (int)nf, L, sp, grid, OP.p, tc.p, k4tot.p, s); break;
        }
      } else {
        switch (bn.nt) {
          case 512: launch_trisum<512>(v, fr, (int)nf, L, sp, grid, OP.p, tc.p, tsum.p, s); break;
          case 256: launch_trisum<256>(v, fr, (int)nf, L, sp, grid, OP.p, tc.p, tsum.p, s); break;
          case 128: launch_trisum<128>(v, fr, (int)nf, L, sp, grid, OP.p, tc.p, tsum.p, s); break;
          default: launch_trisum<32>(v, fr, (int)nf, L, sp, grid, OP.p, tc.p, tsum.p, s); break;
        }
      }
    }
  };
  run_tri_like(false);
  timer.mark("tri_frames");

  if (n) {
    k_vertex_stats<<<grid_cap(n * 32, 256), 256, 0, s>>>(v, tc.p, vT.p, vS.p);
    GD_LAUNCH_CHECK("vertex_stats");
  }
  timer.mark("vertex_stats");

  // ---- pass B -------------------------------------------------------------
  if (per_edge) {
    run_tri_like(true);
    timer.mark("trisum_frames");
  }

  // ---- pass C -------------------------------------------------------------
  {
    int64_t total_w = 0;
    for (int64_t w : wkeys) total_w += w;
    ex.stats.push_back(total_w);
    ex.stats_names.push_back("wedges");
    // Bins by wedges: (coop_t, inf) cooperative rounds with L2-resident u16
    // slabs (frames whose lower degree < 65536), (slab_t, coop_t] per-CTA
    // u32 slabs, (256, slab_t] and [1, 256] shared-memory hashes.  Frames
    // whose counters may exceed 16 bits go through the u32 hub path.
    int64_t slab_t = 4096, coop_t = 1 << 17, small_t = 256;
    if (force.c4_slab) small_t = slab_t = 0, coop_t = INT64_MAX - 1;
    if (force.c4_coop || force.c4_hub32) small_t = slab_t = coop_t = 0;
    if (force.c4_smem) small_t = 0, slab_t = 8192;
    auto rh = count_range(wkeys, coop_t + 1, INT64_MAX);
    auto rl = count_range(wkeys, slab_t + 1, coop_t);
    auto rs1 = count_range(wkeys, small_t + 1, slab_t);
    auto rs0 = count_range(wkeys, 1, small_t);
    const int64_t slab_stride = (n + 31) & ~int64_t(31);
    const int64_t nh = rh.second - rh.first;
    int64_t n_u32_hubs = 0;
    if (nh > 0) {
      // heavy frames: split into u16-safe (lower degree < 65536) and u32 hubs
      std::vector<int> hf(nh);
      GD_CUDA(cudaMemcpyAsync(hf.data(), c4_frames.p + rh.first, nh * 4, cudaMemcpyDeviceToHost,
                              s));
      std::vector<int64_t> hb(nh), ho(nh);
      GD_CUDA(cudaStreamSynchronize(s));
      std::vector<int64_t> hrp(n + 1), hos(n);
      GD_CUDA(cudaMemcpyAsync(hrp.data(), g.rp.p, (n + 1) * 8, cudaMemcpyDeviceToHost, s));
      GD_CUDA(cudaMemcpyAsync(hos.data(), g.osplit.p, n * 8, cudaMemcpyDeviceToHost, s));
      GD_CUDA(cudaStreamSynchronize(s));
      std::vector<int> f16, f32;
      std::vector<int64_t> w16, w32;
      for (int64_t h = 0; h < nh; h++) {
        const int sf = hf[h];
        if (hos[sf] - hrp[sf] < 65536 && !force.c4_hub32) {
          f16.push_back(sf);
          w16.push_back(wkeys[rh.first + h]);
        } else {
          f32.push_back(sf);
          w32.push_back(wkeys[rh.first + h]);
        }
      }
      n_u32_hubs = (int64_t)f32.size();
      if (!f16.empty()) {
        const int64_t CH = 8192;
        const int64_t slab_words = (slab_stride / 2 + 31) & ~int64_t(31);
        const int64_t l2_budget = 48ll << 20;
        const int F = (int)std::max<int64_t>(1, std::min<int64_t>(64, l2_budget / (slab_words * 4)));
        std::vector<int64_t> cpre(f16.size() + 1, 0);
        for (size_t j = 0; j < f16.size(); j++) cpre[j + 1] = cpre[j] + (w16[j] + CH - 1) / CH;
        std::vector<int> rf;
        for (size_t j = 0; j < f16.size(); j += F) rf.push_back((int)j);
        rf.push_back((int)f16.size());
        DBuf<int> dfr, drf;
        DBuf<int64_t> dcp;
        DBuf<unsigned> slabs, bar;
        dfr.alloc(f16.size(), s);
        drf.alloc(rf.size(), s);
        dcp.alloc(cpre.size(), s);
        slabs.alloc((size_t)2 * F * slab_words, s);
        slabs.zero();
        bar.alloc(2, s);
        bar.zero();
        GD_CUDA(cudaMemcpyAsync(dfr.p, f16.data(), f16.size() * 4, cudaMemcpyHostToDevice, s));
        GD_CUDA(cudaMemcpyAsync(drf.p, rf.data(), rf.size() * 4, cudaMemcpyHostToDevice, s));
        GD_CUDA(cudaMemcpyAsync(dcp.p, cpre.data(), cpre.size() * 8, cudaMemcpyHostToDevice, s));
        RoundPlan P{dfr.p, dcp.p, drf.p, (int)rf.size() - 1, F, CH, slab_words};
        constexpr int NT = 512;
        int per_sm = 0;
        GD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_c4_rounds<NT>, NT, 0));
        if (per_sm < 1) throw Error(GD_ECUDA, "c4 rounds kernel cannot be resident");
        const int grid = per_sm * num_sms();
        int pe = per_edge ? 1 : 0;
        unsigned long long* c4e_p = c4e.p;
        unsigned long long* c4t_p = c4tot2.p;
        unsigned* slabs_p = slabs.p;
        unsigned* bar_p = bar.p;
        const int64_t* WP_p = WP.p;
        void* args[] = {(void*)&v, (void*)&WP_p, (void*)&P, (void*)&slabs_p, (void*)&pe,
                        (void*)&c4e_p, (void*)&c4t_p, (void*)&bar_p};
        GD_CUDA(cudaLaunchCooperativeKernel((void*)k_c4_rounds<NT>, dim3(grid), dim3(NT), args, 0,
                                            s));
        GD_LAUNCH_CHECK("c4_rounds");
        ex.stats.push_back((int64_t)rf.size() - 1);
        ex.stats_names.push_back("c4_rounds");
      }
      timer.mark("c4_coop");
      if (!f32.empty()) {
        const int64_t max_slabs = std::max<int64_t>(
            1, std::min<int64_t>((int64_t)f32.size(), (int64_t)(2ll << 30) / (slab_stride * 4)));
        DBuf<unsigned> slabs;
        slabs.alloc((size_t)max_slabs * slab_stride, s);
        slabs.zero();
        const int64_t chunk_items = 1 << 16;
        for (size_t g0 = 0; g0 < f32.size(); g0 += max_slabs) {
          const size_t g1 = std::min(f32.size(), (size_t)(g0 + max_slabs));
          std::vector<HubChunk> chunks;
          for (size_t h = g0; h < g1; h++) {
            const int sframe = f32[h];
            int64_t i0 = 0, i1 = 0;
            GD_CUDA(cudaMemcpyAsync(&i0, WP.p + hrp[sframe], 8, cudaMemcpyDeviceToHost, s));
            GD_CUDA(cudaMemcpyAsync(&i1, WP.p + hos[sframe], 8, cudaMemcpyDeviceToHost, s));
            GD_CUDA(cudaStreamSynchronize(s));
            for (int64_t c = i0; c < i1; c += chunk_items)
              chunks.push_back({sframe, (int)(h - g0), c, std::min(i1, c + chunk_items)});
          }
          DBuf<HubChunk> dch;
          dch.alloc(chunks.size(), s);
          GD_CUDA(cudaMemcpyAsync(dch.p, chunks.data(), chunks.size() * sizeof(HubChunk),
                                  cudaMemcpyHostToDevice, s));
          for (int phase = 0; phase < 3; phase++) {
            k_c4_hub<512><<<(int)chunks.size(), 512, 0, s>>>(
                v, WP.p, dch.p, slabs.p, slab_stride, phase, per_edge ? 1 : 0, c4e.p, c4tot2.p);
            GD_LAUNCH_CHECK("c4_hub");
          }
          GD_CUDA(cudaStreamSynchronize(s));
        }
      }
      timer.mark("c4_hubs32");
    }
    const int64_t nl = rl.second - rl.first;
    if (nl > 0) {
      const int grid = (int)std::min<int64_t>(nl, 2 * num_sms());
      DBuf<unsigned> slabs;
      slabs.alloc((size_t)grid * slab_stride, s);
      slabs.zero();
      k_c4_frames_slab<512><<<grid, 512, 0, s>>>(v, WP.p, c4_frames.p + rl.first, (int)nl, slabs.p,
                                            slab_stride, per_edge ? 1 : 0, c4e.p, c4tot2.p);
      GD_LAUNCH_CHECK("c4_frames_slab");
      timer.mark("c4_slab");
    }
    const int64_t ns1 = rs1.second - rs1.first;
    if (ns1 > 0) {
      int hcap = 512;
      while (hcap < 2 * wkeys[rs1.first]) hcap <<= 1;
      const size_t sm = (size_t)hcap * 8;
      if (sm > 200 * 1024) throw Error(GD_EINVAL, "forced smem path: frame too large");
      GD_CUDA(cudaFuncSetAttribute(k_c4_frames_smem<256>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      const int grid = (int)std::min<int64_t>(ns1, (int64_t)num_sms() * 8);
      k_c4_frames_smem<256><<<grid, 256, sm, s>>>(v, WP.p, c4_frames.p + rs1.first, (int)ns1,
                                                  hcap, per_edge ? 1 : 0, c4e.p, c4tot2.p);
      GD_LAUNCH_CHECK("c4_frames_smem256");
      timer.mark("c4_smem256");
    }
    const int64_t ns0 = rs0.second - rs0.first;
    if (ns0 > 0) {
      const int hcap = 512;
      const size_t sm = (size_t)hcap * 8;
      const int grid = (int)std::min<int64_t>(ns0, (int64_t)num_sms() * 32);
      k_c4_frames_smem<64><<<grid, 64, sm, s>>>(v, WP.p, c4_frames.p + rs0.first, (int)ns0, hcap,
                                                per_edge ? 1 : 0, c4e.p, c4tot2.p);
      GD_LAUNCH_CHECK("c4_frames_smem64");
    }
    ex.stats.push_back(nh);
    ex.stats_names.push_back("coop_frames");
    ex.stats.push_back(n_u32_hubs);
    ex.stats_names.push_back("u32_hub_frames");
    ex.stats.push_back(nl);
    ex.stats_names.push_back("slab_frames");
  }
  timer.mark("c4_wedges");

  // ---- finalize -------------------------------------------------------------
  EdgeIn in;
  in.eu = g.eu.p;
  in.ev = g.ev.p;
  in.d2r = g.d2r.p;
  in.deg = g.deg.p;
  in.tc = tc.p;
  in.tsum = per_edge ? tsum.p : nullptr;
  in.c4e = per_edge ? c4e.p : nullptr;
  in.vT = vT.p;
  in.vS = vS.p;
  GD_CUDA(cudaMemsetAsync(sums_dev, 0, (size_t)G * 2 * kNumSums * 8, s));
  GD_CUDA(cudaMemsetAsync(seen_dev, 0, (size_t)G * 8, s));
  if (G == 1) {
    if (m) {
      k_finalize_single<256><<<grid_cap(m, 256, 4), 256, 0, s>>>(in, 0, m, n, m, table_dev,
                                                                 sums_dev, seen_dev);
      GD_LAUNCH_CHECK("finalize_single");
    }
  } else {
    k_finalize_batch<128><<<(int)G, 128, 0, s>>>(in, g.eoff.p, g.gn.p, table_dev, sums_dev,
                                                 seen_dev);
    GD_LAUNCH_CHECK("finalize_batch");
  }
  timer.mark("finalize");

  // totals for the host-side closure of global mode and the consistency checks
  std::vector<unsigned long long> hk4(2 * G), hc4(2 * G);
  GD_CUDA(cudaMemcpyAsync(hk4.data(), k4tot.p, 2 * G * 8, cudaMemcpyDeviceToHost, s));
  GD_CUDA(cudaMemcpyAsync(hc4.data(), c4tot2.p, 2 * G * 8, cudaMemcpyDeviceToHost, s));
  timer.collect(ex.ms, ex.names);
  ex.stats.push_back(g_launches - launches0);
  ex.stats_names.push_back("launches");
  for (int64_t i = 0; i < G; i++) {
    ex.k4tot[i] = ((unsigned __int128)hk4[2 * i + 1] << 64) | hk4[2 * i];
    ex.c4tot2[i] = ((unsigned __int128)hc4[2 * i + 1] << 64) | hc4[2 * i];
  }
}

void sums_from_table(const long long* table_dev, int64_t m, int64_t n,
                     unsigned long long* sums_dev, cudaStream_t s) {
  GD_CUDA(cudaMemsetAsync(sums_dev, 0, 2 * kNumSums * 8, s));
  if (m) {
    k_sums_from_table<256><<<grid_cap(m, 256, 4), 256, 0, s>>>(table_dev, m, n, sums_dev);
    GD_LAUNCH_CHECK("sums_from_table");
  }
}

}  // namespace gd
