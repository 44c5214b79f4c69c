// Counting kernels of the B200 graphlet census (sm_100a).
//
// The reference computes, for every edge (u, v), the mark-based sweep of
// _micro_edge (census.py:190-256) / _count_edge (census.py:259-303): cost
// sum_e (d(lo) + sum_{w in N(lo)} d(w)) adjacency entries (1.4e13 at R-MAT-20).
// Here the same per-edge quantities are assembled from three enumerations in
// the degree-ordered rank space (rank = ascending (degree, id), so every
// higher-priority neighbour list is a contiguous row suffix, every
// lower-priority one a prefix):
//
//   pass A  triangle frames: for each vertex a, the local graph L(a) induced on
//           its higher-rank neighbours N+(a) as bitmap rows.  Every triangle
//           {a<x<y} is one local edge; every 4-clique {a<x<y<z} one local
//           triangle.  Per edge t(e) = |Tri_e| and cl(e) (4-cliques through e)
//           packed in one 64-bit counter; per vertex T(x); K4 totals.
//   pass B  triangle frames again (per-edge mode): per edge
//           sum_{w in Tri_e} t(lo,w), sum t(hi,w), sum d(w).
//   pass C  vertex-priority wedges s-w-x with w, x < s: counters cnt_s[x];
//           every 4-cycle is counted once at its top vertex
//           (2*C4 = sum_wedges (cnt-1)) and per edge
//           C4(e) = (A^3)_uv - d(u) - d(v) + 1 by wedge attribution.
//   finalize  per canonical edge: the 10 RAW_MICRO_FIELDS and
//           the 13 CensusSums (census.py:449-462) in 128-bit.
//
// Per-edge accumulators are indexed by CSR SLOT, not by edge id: the
// contributions of one frame land on consecutive slots of one row, so the
// atomics of a warp coalesce.  Passes A/B write the edge's "out-slot" (slot in
// the row of its lower-rank endpoint, e2o); pass C writes either slot and the
// finalize adds both (e2o + e2i).
#include <algorithm>
#include <climits>
#include <functional>
#include <type_traits>
#include <map>
#include <mutex>

#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include "gd_count.cuh"

namespace cg = cooperative_groups;

namespace gd {

namespace {

struct View {
  int64_t n, m;
  const int64_t* rp;
  const int32_t* col;
  const int64_t* osplit;
  const int64_t* e2o;
  const int32_t* seid;
  const int32_t* deg;
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

typedef unsigned long long u64;
typedef unsigned __int128 u128;

// ------------------------------------------------------------------------
// Per-frame scratch layout (shared memory for bounded frames, a global slab
// per CTA for the largest ones).  Bitmap rows are 64-bit words with an odd
// row stride (conflict-free across rows).
// ------------------------------------------------------------------------
struct FrameLayout {
  int cap;     // max frame size D
  int hcap;    // hash capacity (pow2 >= 2*cap)
  int wb;      // 64-bit words per bitmap row block (column blocking of big frames)
  int rows;    // 1: pass-A bitmap rows
  int accum;   // 1: pass-B accumulators
  size_t o_qb, o_lv, o_p, o_hk, o_hv, o_bf, o_rows, o_tri2, o_dla, o_tl, o_dl, o_acc;
  size_t bytes;
};

__host__ __device__ __forceinline__ int row_stride64(int W) { return W | 1; }

// Membership filter of a frame's hash: one bit per (multiplicative) hash
// value at 32 bits per key, so ~97% of the probes of non-members (about 90%
// of all probes) end after one shared-memory word instead of a probe chain.
__host__ __device__ __forceinline__ int filter_bits(int D) {
  int b = 1024;
  while (b < 32 * D) b <<= 1;
  return b;
}

FrameLayout make_layout(int cap, bool rows, bool accum, int wb = 0) {
  FrameLayout L{};
  L.cap = cap;
  L.wb = wb > 0 ? wb : (cap + 63) / 64;
  int h = 32;
  while (h < 2 * cap) h <<= 1;
  L.hcap = h;
  L.rows = rows;
  L.accum = accum;
  size_t o = 0;
  auto take = [&](size_t b) {
    size_t r = o;
    o += (b + 15) & ~size_t(15);
    return r;
  };
  L.o_qb = take(8 * (size_t)cap);
  if (accum) L.o_acc = take(sizeof(u64) * 3 * cap);
  if (rows) L.o_rows = take(8ull * cap * row_stride64(L.wb));
  L.o_lv = take(4 * (size_t)cap);
  L.o_p = take(4 * (size_t)(cap + 1));
  L.o_hk = take(4 * (size_t)h);
  L.o_hv = take(4 * (size_t)h);
  L.o_bf = take(filter_bits(cap) / 8);
  if (rows) {
    L.o_tri2 = take(4 * (size_t)cap);
    L.o_dla = take(4 * (size_t)cap);
  }
  if (accum) {
    L.o_tl = take(4 * (size_t)cap);
    L.o_dl = take(4 * (size_t)cap);
  }
  L.bytes = o;
  return L;
}

// Multiplicative hashing into a power-of-two table (top bits), linear probing.
__device__ __forceinline__ unsigned mhash(unsigned x, int shift) {
  return (x * 2654435761u) >> shift;
}

struct LocalHash {
  int* hk;
  int* hv;
  unsigned* bf;  // membership filter
  int hmask, hshift, fshift;
  __device__ __forceinline__ void insert(int key, int val) const {
    const unsigned fb = mhash((unsigned)key, fshift);
    atomicOr(&bf[fb >> 5], 1u << (fb & 31));
    unsigned h = mhash((unsigned)key, hshift);
    while (true) {
      const int old = atomicCAS(&hk[h], -1, key);
      if (old == -1 || old == key) {
        hv[h] = val;
        return;
      }
      h = (h + 1) & hmask;
    }
  }
  __device__ __forceinline__ bool maybe(int key) const {  // the filter alone
    const unsigned fb = mhash((unsigned)key, fshift);
    return (bf[fb >> 5] >> (fb & 31)) & 1u;
  }
  __device__ __forceinline__ int find_exact(int key) const {  // the hash alone
    unsigned h = mhash((unsigned)key, hshift);
    int k = hk[h];
    while (k != key) {
      if (k == -1) return -1;
      h = (h + 1) & hmask;
      k = hk[h];
    }
    return hv[h];
  }
  __device__ __forceinline__ int find(int key) const {
    const unsigned fb = mhash((unsigned)key, fshift);
    if (!((bf[fb >> 5] >> (fb & 31)) & 1u)) return -1;
    unsigned h = mhash((unsigned)key, hshift);
    int k = hk[h];
    while (k != key) {
      if (k == -1) return -1;
      h = (h + 1) & hmask;
      k = hk[h];
    }
    return hv[h];
  }
};

// Load N+(a) into Lv, QB[j] = osplit[x_j] - P[j] (so item i of segment j
// lives at slot QB[j] + i), the item prefix P (from the global out-item
// prefix OP) and the hash of Lv.  Returns D; total items in P[D].
template <int NT>
__device__ int frame_load(const View& g, int a, char* mem, const FrameLayout& L,
                          const int64_t* __restrict__ OP, LocalHash& H) {
  const int64_t base = g.osplit[a];
  const int D = (int)(g.rp[a + 1] - base);
  int* Lv = (int*)(mem + L.o_lv);
  int* P = (int*)(mem + L.o_p);
  int64_t* QB = (int64_t*)(mem + L.o_qb);
  int hsize = pow2_at_least(2 * D);
  if (hsize > L.hcap) hsize = L.hcap;
  H.hk = (int*)(mem + L.o_hk);
  H.hv = (int*)(mem + L.o_hv);
  H.bf = (unsigned*)(mem + L.o_bf);
  H.hmask = hsize - 1;
  H.hshift = 32 - (31 - __clz(hsize));
  const int fbits = filter_bits(D);
  H.fshift = 32 - (31 - __clz(fbits));
  const int64_t p0 = OP[base];
  for (int j = threadIdx.x; j < D; j += NT) {
    const int x = g.col[base + j];
    const int pj = (int)(OP[base + j] - p0);
    Lv[j] = x;
    P[j] = pj;
    QB[j] = g.osplit[x] - pj;
  }
  if (threadIdx.x == 0) P[D] = (int)(OP[base + D] - p0);
  for (int h = threadIdx.x; h < hsize; h += NT) H.hk[h] = -1;
  for (int w = threadIdx.x; w < fbits / 32; w += NT) H.bf[w] = 0u;
  __syncthreads();
  for (int j = threadIdx.x; j < D; j += NT) H.insert(Lv[j], j);
  return D;
}

// Items [0, total) of a frame, item i -> segment j with P[j] <= i < P[j+1]:
// warp chunks of 32*K items, lane-interleaved (consecutive lanes read
// consecutive entries of one row), one binary search per lane per chunk, and
// U items per lane in flight (their col[] loads are issued back to back).
// f(j, i, q, y) receives the slot q = QB[j] + i and the neighbour y = col[q].
#ifndef GD_TRI_K
#define GD_TRI_K 32
#endif
#ifndef GD_TRI_U
#define GD_TRI_U 1
#endif
template <int NT, typename F>
__device__ __forceinline__ void for_frame_items(const View& g, const int* P, const int64_t* QB,
                                                int D, int total, F&& f) {
  constexpr int K = GD_TRI_K, U = GD_TRI_U;
  constexpr int NW = NT / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifndef GD_TRI_NO_PREFETCH
  // rolling prefetch: the col[] load of the lane's next item is issued
  // before the current item is processed (one load in flight while the
  // hash probe of the previous one runs; 3 extra registers)
  for (int c0 = warp * 32 * K; c0 < total; c0 += NW * 32 * K) {
    const int c1 = min(c0 + 32 * K, total);
    int i = c0 + lane;
    if (i >= c1) continue;
    int j = find_segment(P, D, i);
    int pj1 = P[j + 1];
    int64_t q = QB[j] + i;
    int y = __ldg(g.col + q);
    for (; i < c1; i += 32) {
      const int ni = i + 32;
      int jn = j;
      int64_t qn = 0;
      int yn = 0;
      if (ni < c1) {
        while (pj1 <= ni) pj1 = P[++jn + 1];
        qn = QB[jn] + ni;
        yn = __ldg(g.col + qn);
      }
      f(j, i, q, y);
      j = jn;
      q = qn;
      y = yn;
    }
  }
#else
  for (int c0 = warp * 32 * K; c0 < total; c0 += NW * 32 * K) {
    const int c1 = min(c0 + 32 * K, total);
    int i = c0 + lane;
    if (i >= c1) continue;
    int j = find_segment(P, D, i);
    int pj1 = P[j + 1];
    for (; i < c1; i += 32 * U) {
      int jj[U];
      int64_t qq[U];
      int yy[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int ii = i + 32 * u;
        if (ii < c1) {
          while (pj1 <= ii) pj1 = P[++j + 1];
          jj[u] = j;
          qq[u] = QB[j] + ii;
        }
      }
#pragma unroll
      for (int u = 0; u < U; u++)
        if (i + 32 * u < c1) yy[u] = __ldg(g.col + qq[u]);
#pragma unroll
      for (int u = 0; u < U; u++)
        if (i + 32 * u < c1) f(jj[u], i + 32 * u, qq[u], yy[u]);
    }
  }
#endif
}

// Sweep 1 of a triangle frame with the hit path compacted.  About one item
// in ten is a local edge, so nearly every 32-item step holds one, and running
// the hash probe, the bitmap updates and the list append inside the item loop
// executed half of the kernel's instructions with a few lanes active (ncu:
// 14-17 active lanes per instruction).  Here the item loop only tests the
// membership filter; the lanes that pass push (j, i) onto a per-warp queue in
// shared memory, and whenever 32 entries are queued the whole warp takes one
// each: exact hash lookup, then hit(j, k, i, is_hit) with all lanes converged
// (hit() may use full-mask warp collectives).
#ifndef GD_TRI_NO_COMPACT
#define GD_TRI_COMPACT 1
#endif
template <int NT, typename F>
__device__ __forceinline__ void frame_items_compact(const View& g, const int* P,
                                                    const int64_t* QB, int D, int total,
                                                    const LocalHash& H, u64* wq, F&& hit) {
  constexpr int K = GD_TRI_K;
  constexpr int NW = NT / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  u64* q64 = wq + warp * 64;
  int qn = 0, head = 0;  // queued entries and the ring's first one (warp-uniform)
  // entries leave in arrival order (the hit lists stay in item order, which
  // keeps the slot atomics of sweep 2 and pass B coalesced)
  auto drain = [&](int base, int cnt) {
    int j = 0, i = 0, k = -1;
    if (lane < cnt) {
      const u64 e = q64[(base + lane) & 63];
      j = (int)(e >> 32);
      i = (int)(unsigned)e;
      k = H.find_exact(__ldg(g.col + QB[j] + i));
    }
    hit(j, k, i, k >= 0);
  };
  for (int c0 = warp * 32 * K; c0 < total; c0 += NW * 32 * K) {
    const int c1 = min(c0 + 32 * K, total);
    int i = c0 + lane;
    bool valid = i < c1;
    int j = 0, pj1 = 0, y = 0;
    if (valid) {
      j = find_segment(P, D, i);
      pj1 = P[j + 1];
      y = __ldg(g.col + QB[j] + i);
    }
    for (int base = c0; base < c1; base += 32) {
      // the col[] load of the lane's next item is issued before this one is tested
      const int ni = i + 32;
      const bool nvalid = ni < c1;
      int jn = j, yn = 0;
      if (nvalid) {
        while (pj1 <= ni) pj1 = P[++jn + 1];
        yn = __ldg(g.col + QB[jn] + ni);
      }
      const bool pass = valid && H.maybe(y);
      const unsigned m = __ballot_sync(0xffffffffu, pass);
      if (m) {
        if (pass)
          q64[(head + qn + __popc(m & lt)) & 63] = ((u64)(unsigned)j << 32) | (u64)(unsigned)i;
        qn += __popc(m);
        if (qn >= 32) {
          __syncwarp();
          drain(head, 32);
          head = (head + 32) & 63;
          qn -= 32;
          __syncwarp();
        }
      }
      i = ni;
      valid = nvalid;
      j = jn;
      y = yn;
    }
  }
  __syncwarp();
  if (qn) drain(head, qn);
}

// The same sweep walked row by row.  The item-space loop above spends ~50
// SASS instructions per 32-item step on the per-lane segment walk (P[] loop,
// QB[] load, 64-bit slot address) before the filter test.  A frame's rows
// average hundreds of items, so here a warp's chunk [c0, c1) is cut at the
// row boundaries inside it and every piece is scanned with warp-uniform
// bounds and one uniform row pointer: no per-lane search, U loads in flight
// per lane, and at most one partly filled step per piece.
#ifndef GD_TRI_RU
#define GD_TRI_RU 4
#endif
template <int NT, typename F>
__device__ __forceinline__ void frame_items_rows(const View& g, const int* P, const int64_t* QB,
                                                 int D, int total, const LocalHash& H, u64* wq,
                                                 F&& hit) {
  constexpr int K = GD_TRI_K, U = GD_TRI_RU;
  constexpr int NW = NT / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  u64* q64 = wq + warp * 64;
  // the queue through a 32-bit shared-window address (see smem_u32 below: the
  // generic form rebuilds the window base before every store)
  const unsigned sQ = (unsigned)__cvta_generic_to_shared(q64);
  int qn = 0, head = 0;  // queued entries and the ring's first one (warp-uniform)
  auto drain = [&](int base, int cnt) {
    int j = 0, i = 0, k = -1;
    if (lane < cnt) {
      const u64 e = q64[(base + lane) & 63];
      j = (int)(e >> 32);
      i = (int)(unsigned)e;
      k = H.find_exact(__ldg(g.col + QB[j] + i));
    }
    hit(j, k, i, k >= 0);
  };
  for (int c0 = warp * 32 * K; c0 < total; c0 += NW * 32 * K) {
    const int c1 = min(c0 + 32 * K, total);
    int j = find_segment(P, D, c0);
    int lo = c0;
    while (lo < c1) {
      const int hi = min(P[j + 1], c1);
      if (hi > lo) {
        // item i of this row lives at rowl[i - lane]
        const int* __restrict__ rowl = g.col + (QB[j] + lane);
        for (int base = lo; base < hi; base += 32 * U) {
          const int* __restrict__ p = rowl + base;
          const int rem = hi - base - lane;  // this lane's items left in the row: (rem + 31) / 32
          int y[U];
#pragma unroll
          for (int u = 0; u < U; u++) y[u] = rem > 32 * u ? __ldg(p + 32 * u) : 0;
#pragma unroll
          for (int u = 0; u < U; u++) {
            if (base + 32 * u < hi) {
              const bool pass = rem > 32 * u && H.maybe(y[u]);
              const unsigned m = __ballot_sync(0xffffffffu, pass);
              if (m) {
                if (pass) {
                  const unsigned a = sQ + 8u * ((unsigned)(head + qn + __popc(m & lt)) & 63u);
                  asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(a),
                               "r"((unsigned)(base + 32 * u + lane)), "r"((unsigned)j)
                               : "memory");
                }
                qn += __popc(m);
                if (qn >= 32) {
                  __syncwarp();
                  drain(head, 32);
                  head = (head + 32) & 63;
                  qn -= 32;
                  __syncwarp();
                }
              }
            }
          }
        }
      }
      lo = hi;
      j++;
    }
  }
  __syncwarp();
  if (qn) drain(head, qn);
}
#ifndef GD_TRI_NO_ROWS
#define GD_TRI_SWEEP1 frame_items_rows
#else
#define GD_TRI_SWEEP1 frame_items_compact
#endif

// Set bit b of a 64-bit-word bitmap row with a native 32-bit atomicOr (a
// 64-bit shared-memory atomicOr compiles to a CAS loop).
__device__ __forceinline__ void set_bit(u64* row, int b) {
  atomicOr((unsigned*)row + (b >> 5), 1u << (b & 31));
}

__device__ __forceinline__ u64 pack_hit(int j, int k, int i) {
  return ((u64)(unsigned)j << 48) | ((u64)(unsigned)k << 32) | (u64)(unsigned)i;
}

// Local-edge (hit) lists.  Sweep 1 of a triangle frame appends every local
// edge (j, k, item i) to a per-CTA staging list in global memory (L2-hot);
// sweep 2 then walks the list instead of probing every item again.  In
// per-edge mode the list is copied to an exact-size slice of a graph-wide
// hit buffer (bump allocated) so pass B needs no probing at all.  A frame
// whose list overflows staging or the hit buffer falls back to probing.
struct HitLists {
  u64* stage;          // [grid][stage_cap] staging lists
  int stage_cap;       // entries per CTA (0: no lists)
  u64* buf;            // graph-wide hit buffer (null: do not persist)
  u64* top;            // bump pointer into buf
  u64 cap;             // entries in buf
  int64_t* hoff;       // [n] frame -> first entry in buf
  int* hcnt;           // [n] frame -> entries, -1 = not persisted
};

// Walk a hit list, 32 consecutive entries per warp step; the entry of the
// lane's next step is loaded before this one is processed.  The entries of a
// step are consecutive local edges in item order, so most of them share their
// row j: `grp` is the mask of the lanes with this lane's j (lanes past the end
// stand alone), for one shared-memory atomic per distinct j instead of up to 32
// serialised on one address.  f(valid, e, h, grp).
template <int NT, typename F>
__device__ __forceinline__ void for_hits(const u64* list, int nh, F&& f) {
  const int lane = threadIdx.x & 31;
  int h = threadIdx.x;
  u64 e = h < nh ? list[h] : 0ull;
  for (int h0 = threadIdx.x & ~31; h0 < nh; h0 += NT, h += NT) {
    const u64 en = h + NT < nh ? list[h + NT] : 0ull;
    const bool valid = h < nh;
    const int key = valid ? (int)(e >> 48) : 0x10000 + lane;
#ifndef GD_NO_GROUPED
    const unsigned grp = __match_any_sync(0xffffffffu, key);
#else
    const unsigned grp = 1u << lane;
#endif
    f(valid, e, h, grp);
    e = en;
  }
}
// Sum of v over the lanes of grp (every lane of the warp calls it with its own
// group mask).  The 64-bit form takes values below 2^32.
__device__ __forceinline__ unsigned group_sum(unsigned grp, unsigned v) {
#ifndef GD_NO_GROUPED
  return __reduce_add_sync(grp, v);
#else
  return v;
#endif
}
__device__ __forceinline__ u64 group_sum(unsigned grp, u64 v) {
#ifndef GD_NO_GROUPED
  const unsigned lo = __reduce_add_sync(grp, (unsigned)v & 0xffffu);
  const unsigned hi = __reduce_add_sync(grp, (unsigned)(v >> 16));
  return ((u64)hi << 16) + lo;
#else
  return v;
#endif
}
__device__ __forceinline__ bool group_leader(unsigned grp) {
  return (int)(threadIdx.x & 31) == __ffs(grp) - 1;
}

// ------------------------------------------------------------------------
// pass A
// ------------------------------------------------------------------------
// Frames whose bitmap rows fit in one block (all but the largest).
template <int NT>
__device__ void tri_frame_single(const View& g, int a, char* mem, const FrameLayout& L,
                          const int64_t* __restrict__ OP, u64* __restrict__ tcs,
                          u64* __restrict__ vT, u64* __restrict__ k4tot, const HitLists& HL,
                          u64* wq) {
  __shared__ int nhits;
  __shared__ u64 s_off;
  LocalHash H;
  const int D = frame_load<NT>(g, a, mem, L, OP, H);
  const int* Lv = (const int*)(mem + L.o_lv);
  const int* P = (const int*)(mem + L.o_p);
  const int64_t* QB = (const int64_t*)(mem + L.o_qb);
  u64* rows = (u64*)(mem + L.o_rows);
  unsigned* tri2 = (unsigned*)(mem + L.o_tri2);
  u64* hits = HL.stage ? HL.stage + (size_t)blockIdx.x * HL.stage_cap : nullptr;
  const int W = (D + 63) >> 6;
  const int RS = row_stride64(W);
  for (int i = threadIdx.x; i < D * RS; i += NT) rows[i] = 0ull;
  for (int j = threadIdx.x; j < D; j += NT) tri2[j] = 0u;
  if (threadIdx.x == 0) nhits = 0;
  __syncthreads();
  const int total = P[D];
  const int hitcap = (hits && D < 65536) ? HL.stage_cap : 0;
  // sweep 1: local adjacency bitmaps (undirected) + the list of local edges
#ifdef GD_TRI_COMPACT
  GD_TRI_SWEEP1<NT>(g, P, QB, D, total, H, wq, [&](int j, int k, int i, bool is_hit) {
    const unsigned hm = __ballot_sync(0xffffffffu, is_hit);
    if (!hm) return;
    if (is_hit) {
      set_bit(rows + j * RS, k);
      set_bit(rows + k * RS, j);
    }
    if (hitcap) {  // warp-aggregated append
      int h0 = 0;
      if (lane_id() == 0) h0 = atomicAdd(&nhits, __popc(hm));
      const int h = __shfl_sync(0xffffffffu, h0, 0) + __popc(hm & ((1u << lane_id()) - 1u));
      if (is_hit && h < hitcap) hits[h] = pack_hit(j, k, i);
    }
  });
#else
  for_frame_items<NT>(g, P, QB, D, total, [&](int j, int i, int64_t, int y) {
    const int k = H.find(y);
    if (k >= 0) {
      set_bit(rows + j * RS, k);
      set_bit(rows + k * RS, j);
      if (hitcap) {  // warp-aggregated append
        const unsigned act = __activemask();
        const int leader = __ffs(act) - 1;
        int h0 = 0;
        if ((int)lane_id() == leader) h0 = atomicAdd(&nhits, __popc(act));
        const int h = __shfl_sync(act, h0, leader) + __popc(act & ((1u << lane_id()) - 1u));
        if (h < hitcap) hits[h] = pack_hit(j, k, i);
      }
    }
  });
#endif
  __syncthreads();
  const int nh = nhits;
  const bool listed = hitcap > 0 && nh <= hitcap;
  // persist the list for pass B (exact-size bump allocation)
  if (HL.buf && threadIdx.x == 0) {
    u64 off = ~0ull;
    if (listed && nh > 0) {
      off = atomicAdd(HL.top, (u64)nh);
      if (off + (u64)nh > HL.cap) off = ~0ull;
    }
    s_off = off;
    HL.hoff[a] = (int64_t)off;
    HL.hcnt[a] = (listed && (nh == 0 || off != ~0ull)) ? nh : -1;
  }
  // sweep 2: each local edge (x_j, x_k) is the triangle {a, x_j, x_k}; its
  // common local neighbours are the 4-cliques {a, x_j, x_k, z}
  auto local_edge = [&](int j, int k, int64_t q) {
    unsigned c = 0;
    const u64* rj = rows + j * RS;
    const u64* rk = rows + k * RS;
    for (int w = 0; w < W; w++) c += __popcll(rj[w] & rk[w]);
    atomicAdd(&tcs[q], (1ull << kTriShift) + c);
    if (c) {
      atomicAdd(&tri2[j], c);
      atomicAdd(&tri2[k], c);
    }
  };
  if (listed) {
    __syncthreads();
    const u64 off = HL.buf ? s_off : ~0ull;
    u64* dst = off != ~0ull ? HL.buf + off : nullptr;
    for_hits<NT>(hits, nh, [&](bool valid, u64 e, int h, unsigned grp) {
      const int j = (int)(e >> 48), k = (int)((e >> 32) & 0xffff), i = (int)(unsigned)e;
      unsigned c = 0;
      if (valid) {
        if (dst) dst[h] = e;
        const u64* rj = rows + j * RS;
        const u64* rk = rows + k * RS;
        for (int w = 0; w < W; w++) c += __popcll(rj[w] & rk[w]);
        atomicAdd(&tcs[QB[j] + i], (1ull << kTriShift) + c);
        if (c) atomicAdd(&tri2[k], c);
      }
      const unsigned cs = group_sum(grp, c);
      if (cs && group_leader(grp)) atomicAdd(&tri2[j], cs);
    });
  } else {
    for_frame_items<NT>(g, P, QB, D, total, [&](int j, int, int64_t q, int y) {
      const int k = H.find(y);
      if (k >= 0) local_edge(j, k, q);
    });
  }
  __syncthreads();
  const int64_t base = g.osplit[a];
  u64 t2sum = 0, dlsum = 0;
  for (int j = threadIdx.x; j < D; j += NT) {
    unsigned dl = 0;
    const u64* rj = rows + j * RS;
    for (int w = 0; w < W; w++) dl += __popcll(rj[w]);
    if (dl) {
      atomicAdd(&tcs[base + j], ((u64)dl << kTriShift) + (tri2[j] >> 1));
      atomicAdd(&vT[Lv[j]], (u64)dl);
    }
    t2sum += tri2[j];
    dlsum += dl;
  }
  typedef cub::BlockReduce<u64, NT> BR;
  __shared__ typename BR::TempStorage tmp;
  const u64 s1 = BR(tmp).Sum(t2sum);
  __syncthreads();
  const u64 s2 = BR(tmp).Sum(dlsum);
  if (threadIdx.x == 0) {
    if (s1) atomic_add_u128(k4tot + 2 * graph_of(g, a), s1 / 6);
    if (s2) atomicAdd(&vT[a], s2 >> 1);
  }
  __syncthreads();
}

// Frames whose bitmap rows are split into column blocks (the largest).
template <int NT>
__device__ void tri_frame(const View& g, int a, char* mem, const FrameLayout& L,
                          const int64_t* __restrict__ OP, u64* __restrict__ tcs,
                          u64* __restrict__ vT, u64* __restrict__ k4tot, const HitLists& HL,
                          u64* wq) {
  __shared__ int nhits;
  __shared__ u64 s_off;
  LocalHash H;
  const int D = frame_load<NT>(g, a, mem, L, OP, H);
  const int* Lv = (const int*)(mem + L.o_lv);
  const int* P = (const int*)(mem + L.o_p);
  const int64_t* QB = (const int64_t*)(mem + L.o_qb);
  u64* rows = (u64*)(mem + L.o_rows);
  unsigned* tri2 = (unsigned*)(mem + L.o_tri2);
  unsigned* dla = (unsigned*)(mem + L.o_dla);
  u64* hits = HL.stage ? HL.stage + (size_t)blockIdx.x * HL.stage_cap : nullptr;
  // bitmap rows in column blocks of WB words (one block unless D is large)
  const int W = (D + 63) >> 6;
  const int WB = W < L.wb ? W : L.wb;
  const int NB = (W + WB - 1) / WB;
  const int RS = row_stride64(WB);
  for (int j = threadIdx.x; j < D; j += NT) {
    tri2[j] = 0u;
    dla[j] = 0u;
  }
  if (threadIdx.x == 0) nhits = 0;
  const int total = P[D];
  const int hitcap = (hits && D < 65536) ? HL.stage_cap : 0;
  // set the bits of local edge (j, k) that fall in column block [c0, c1)
  auto set_bits = [&](int j, int k, int c0, int c1) {
    if (k >= c0 && k < c1) set_bit(rows + j * RS, k - c0);
    if (j >= c0 && j < c1) set_bit(rows + k * RS, j - c0);
  };
  auto local_edge = [&](int j, int k, int64_t q, bool first) {
    unsigned c = 0;
    const u64* rj = rows + j * RS;
    const u64* rk = rows + k * RS;
    for (int w = 0; w < WB; w++) c += __popcll(rj[w] & rk[w]);
    const u64 add = (first ? (1ull << kTriShift) : 0ull) + c;
    if (add) atomicAdd(&tcs[q], add);
    if (c) {
      atomicAdd(&tri2[j], c);
      atomicAdd(&tri2[k], c);
    }
  };
  bool listed = false;
  int nh = 0;
  for (int blk = 0; blk < NB; blk++) {
    const int c0 = blk * WB * 64, c1 = min(D, c0 + WB * 64);
    const int wcnt = (c1 - c0 + 63) >> 6;  // words used in this block
    for (int i = threadIdx.x; i < D * RS; i += NT) rows[i] = 0ull;
    __syncthreads();
#ifdef GD_TRI_COMPACT
    if (blk == 0) {
      // sweep 1 (probing, hit path compacted): bitmap bits + the list of local edges
      GD_TRI_SWEEP1<NT>(g, P, QB, D, total, H, wq, [&](int j, int k, int i, bool is_hit) {
        const unsigned hm = __ballot_sync(0xffffffffu, is_hit);
        if (!hm) return;
        if (is_hit) set_bits(j, k, c0, c1);
        if (hitcap) {  // warp-aggregated append
          int h0 = 0;
          if (lane_id() == 0) h0 = atomicAdd(&nhits, __popc(hm));
          const int h = __shfl_sync(0xffffffffu, h0, 0) + __popc(hm & ((1u << lane_id()) - 1u));
          if (is_hit && h < hitcap) hits[h] = pack_hit(j, k, i);
        }
      });
      __syncthreads();
      nh = nhits;
      listed = hitcap > 0 && nh <= hitcap;
      // persist the list for pass B (exact-size bump allocation)
      if (HL.buf && threadIdx.x == 0) {
        u64 off = ~0ull;
        if (listed && nh > 0) {
          off = atomicAdd(HL.top, (u64)nh);
          if (off + (u64)nh > HL.cap) off = ~0ull;
        }
        s_off = off;
        HL.hoff[a] = (int64_t)off;
        HL.hcnt[a] = (listed && (nh == 0 || off != ~0ull)) ? nh : -1;
      }
      __syncthreads();
    } else
#endif
    if (blk == 0 || !listed) {
      // sweep 1 (probing): bitmap bits + the list of local edges
      for_frame_items<NT>(g, P, QB, D, total, [&](int j, int i, int64_t, int y) {
        const int k = H.find(y);
        if (k >= 0) {
          set_bits(j, k, c0, c1);
          if (blk == 0 && hitcap) {  // warp-aggregated append
            const unsigned act = __activemask();
            const int leader = __ffs(act) - 1;
            int h0 = 0;
            if ((int)lane_id() == leader) h0 = atomicAdd(&nhits, __popc(act));
            const int h = __shfl_sync(act, h0, leader) + __popc(act & ((1u << lane_id()) - 1u));
            if (h < hitcap) hits[h] = pack_hit(j, k, i);
          }
        }
      });
      __syncthreads();
      if (blk == 0) {
        nh = nhits;
        listed = hitcap > 0 && nh <= hitcap;
        // persist the list for pass B (exact-size bump allocation)
        if (HL.buf && threadIdx.x == 0) {
          u64 off = ~0ull;
          if (listed && nh > 0) {
            off = atomicAdd(HL.top, (u64)nh);
            if (off + (u64)nh > HL.cap) off = ~0ull;
          }
          s_off = off;
          HL.hoff[a] = (int64_t)off;
          HL.hcnt[a] = (listed && (nh == 0 || off != ~0ull)) ? nh : -1;
        }
        __syncthreads();
      }
    } else {
      for (int h = threadIdx.x; h < nh; h += NT) {
        const u64 e = hits[h];
        set_bits((int)(e >> 48), (int)((e >> 32) & 0xffff), c0, c1);
      }
      __syncthreads();
    }
    // sweep 2: each local edge (x_j, x_k) is the triangle {a, x_j, x_k}; its
    // common local neighbours are the 4-cliques {a, x_j, x_k, z}
    if (listed) {
      u64* dst = (blk == 0 && HL.buf && s_off != ~0ull) ? HL.buf + s_off : nullptr;
      for_hits<NT>(hits, nh, [&](bool valid, u64 e, int h, unsigned grp) {
        const int j = (int)(e >> 48), k = (int)((e >> 32) & 0xffff), i = (int)(unsigned)e;
        unsigned c = 0;
        if (valid) {
          if (dst) dst[h] = e;
          const u64* rj = rows + j * RS;
          const u64* rk = rows + k * RS;
          for (int w = 0; w < WB; w++) c += __popcll(rj[w] & rk[w]);
          const u64 add = (blk == 0 ? (1ull << kTriShift) : 0ull) + c;
          if (add) atomicAdd(&tcs[QB[j] + i], add);
          if (c) atomicAdd(&tri2[k], c);
        }
        const unsigned cs = group_sum(grp, c);
        if (cs && group_leader(grp)) atomicAdd(&tri2[j], cs);
      });
    } else {
      for_frame_items<NT>(g, P, QB, D, total, [&](int j, int, int64_t q, int y) {
        const int k = H.find(y);
        if (k >= 0) local_edge(j, k, q, blk == 0);
      });
    }
    __syncthreads();
    for (int j = threadIdx.x; j < D; j += NT) {
      unsigned dl = 0;
      const u64* rj = rows + j * RS;
      for (int w = 0; w < wcnt; w++) dl += __popcll(rj[w]);
      dla[j] += dl;
    }
    __syncthreads();
  }
  const int64_t base = g.osplit[a];
  u64 t2sum = 0, dlsum = 0;
  for (int j = threadIdx.x; j < D; j += NT) {
    const unsigned dl = dla[j];
    if (dl) {
      atomicAdd(&tcs[base + j], ((u64)dl << kTriShift) + (tri2[j] >> 1));
      atomicAdd(&vT[Lv[j]], (u64)dl);
    }
    t2sum += tri2[j];
    dlsum += dl;
  }
  typedef cub::BlockReduce<u64, NT> BR;
  __shared__ typename BR::TempStorage tmp;
  const u64 s1 = BR(tmp).Sum(t2sum);
  __syncthreads();
  const u64 s2 = BR(tmp).Sum(dlsum);
  if (threadIdx.x == 0) {
    if (s1) atomic_add_u128(k4tot + 2 * graph_of(g, a), s1 / 6);
    if (s2) atomicAdd(&vT[a], s2 >> 1);
  }
  __syncthreads();
}

// Next frame of this CTA: the c-th claim of rank r is frame r + world * c.
// (The frame bodies end with a block barrier, so s_claim is free again.)
__device__ __forceinline__ int claim_frame(unsigned* claim, int* s_claim, int rank, int world) {
  if (threadIdx.x == 0) *s_claim = (int)atomicAdd(claim, 1u);
  __syncthreads();
  const int c = *s_claim;
  __syncthreads();
  return rank + world * c;
}

// GM: frame scratch in a global slab (largest frames); otherwise in shared
// memory, where keeping the pointer's provenance static lets the compiler
// emit LDS/STS/ATOMS instead of generic loads.
#if defined(GD_TRI_FULL_OCC) && GD_TRI_FULL_OCC
#define GD_TRI_BOUNDS(NT) __launch_bounds__(NT, (NT) >= 64 ? 2048 / (NT) : 32)
#else
#define GD_TRI_BOUNDS(NT) __launch_bounds__(NT)
#endif
template <int NT, bool BLOCKED, bool GM>
__global__ void GD_TRI_BOUNDS(NT)
k_tri_frames(View g, const int* __restrict__ frames, int nframes, int rank, int world,
             FrameLayout L, char* gslab, const int64_t* __restrict__ OP, u64* __restrict__ tcs,
             u64* __restrict__ vT, u64* __restrict__ k4tot, HitLists HL,
             unsigned* __restrict__ claim) {
  extern __shared__ __align__(16) char smem[];
  __shared__ u64 wq[(NT / 32) * 64];  // per-warp queues of filter passes (frame_items_compact)
  __shared__ int s_claim;
  char* mem = GM ? gslab + (size_t)blockIdx.x * L.bytes : smem;
  // frames are claimed in descending-D order (a static round-robin gives the
  // first CTAs the largest frame of every round)
  while (true) {
    const int f = claim_frame(claim, &s_claim, rank, world);
    if (f >= nframes) break;
    if (BLOCKED)
      tri_frame<NT>(g, frames[f], mem, L, OP, tcs, vT, k4tot, HL, wq);
    else
      tri_frame_single<NT>(g, frames[f], mem, L, OP, tcs, vT, k4tot, HL, wq);
  }
}

// ------------------------------------------------------------------------
// pass B: per out-slot sums over the triangle set, by rank side
//   tsl: sum t(lo, w)   tsh: sum t(hi, w)   tsd: sum d(w)   (w in Tri_e)
// Frames with a persisted hit list walk it; the others probe again.
// ------------------------------------------------------------------------
// AccT: the per-base-edge accumulators in shared memory; u32 when
// D * max_degree < 2^32 (native shared atomics; a 64-bit shared atomicAdd is
// a CAS loop), u64 otherwise.
template <int NT, typename AccT, typename ST>
__device__ void trisum_frame(const View& g, int a, char* mem, const FrameLayout& L,
                             const int64_t* __restrict__ OP, const u64* __restrict__ tcs,
                             ST* __restrict__ tsl, ST* __restrict__ tsh,
                             ST* __restrict__ tsd, const HitLists& HL) {
  LocalHash H;
  const int D = frame_load<NT>(g, a, mem, L, OP, H);
  const int* Lv = (const int*)(mem + L.o_lv);
  const int* P = (const int*)(mem + L.o_p);
  const int64_t* QB = (const int64_t*)(mem + L.o_qb);
  int* tL = (int*)(mem + L.o_tl);
  int* dL = (int*)(mem + L.o_dl);
  AccT* acc = (AccT*)(mem + L.o_acc);
  const int64_t base = g.osplit[a];
  for (int j = threadIdx.x; j < D; j += NT) {
    tL[j] = (int)(tcs[base + j] >> kTriShift);
    dL[j] = g.deg[Lv[j]];
    acc[3 * j] = 0;
    acc[3 * j + 1] = 0;
    acc[3 * j + 2] = 0;
  }
  __syncthreads();
  const int total = P[D];
  const u64 deg_a = (u64)g.deg[a];
  auto local_edge = [&](int j, int k, int64_t q) {
    const u64 t_jk = tcs[q] >> kTriShift;
    // edge (x_j, x_k), lo side x_j, third vertex a
    atomicAdd(&tsl[q], (ST)tL[j]);
    atomicAdd(&tsh[q], (ST)tL[k]);
    atomicAdd(&tsd[q], (ST)deg_a);
    // edge (a, x_j): third vertex x_k; edge (a, x_k): third vertex x_j
    atomicAdd(&acc[3 * j], (AccT)tL[k]);
    atomicAdd(&acc[3 * j + 1], (AccT)t_jk);
    atomicAdd(&acc[3 * j + 2], (AccT)dL[k]);
    atomicAdd(&acc[3 * k], (AccT)tL[j]);
    atomicAdd(&acc[3 * k + 1], (AccT)t_jk);
    atomicAdd(&acc[3 * k + 2], (AccT)dL[j]);
  };
  const int nh = HL.hcnt ? HL.hcnt[a] : -1;
  if (nh >= 0) {
    const u64* src = HL.buf + HL.hoff[a];
    for_hits<NT>(src, nh, [&](bool valid, u64 e, int, unsigned grp) {
      const int j = (int)(e >> 48), k = (int)((e >> 32) & 0xffff), i = (int)(unsigned)e;
      AccT v0 = 0, v1 = 0, v2 = 0;
      if (valid) {
        const int64_t q = QB[j] + i;
        const u64 t_jk = tcs[q] >> kTriShift;
        const int tj = tL[j], tk = tL[k];
        atomicAdd(&tsl[q], (ST)tj);
        atomicAdd(&tsh[q], (ST)tk);
        atomicAdd(&tsd[q], (ST)deg_a);
        atomicAdd(&acc[3 * k], (AccT)tj);
        atomicAdd(&acc[3 * k + 1], (AccT)t_jk);
        atomicAdd(&acc[3 * k + 2], (AccT)dL[j]);
        v0 = (AccT)tk;
        v1 = (AccT)t_jk;
        v2 = (AccT)dL[k];
      }
      // the row side (a, x_j): one atomic per distinct j of the step
      v0 = group_sum(grp, v0);
      v1 = group_sum(grp, v1);
      v2 = group_sum(grp, v2);
      if (v2 && group_leader(grp)) {
        atomicAdd(&acc[3 * j], v0);
        atomicAdd(&acc[3 * j + 1], v1);
        atomicAdd(&acc[3 * j + 2], v2);
      }
    });
  } else {
    for_frame_items<NT>(g, P, QB, D, total, [&](int j, int, int64_t q, int y) {
      const int k = H.find(y);
      if (k >= 0) local_edge(j, k, q);
    });
  }
  __syncthreads();
  for (int j = threadIdx.x; j < D; j += NT) {
    if (acc[3 * j + 2] == 0) continue;  // no triangle on edge (a, x_j)
    atomicAdd(&tsl[base + j], (ST)acc[3 * j]);
    atomicAdd(&tsh[base + j], (ST)acc[3 * j + 1]);
    atomicAdd(&tsd[base + j], (ST)acc[3 * j + 2]);
  }
  __syncthreads();
}

template <int NT, bool GM, typename AccT, typename ST>
__global__ void __launch_bounds__(NT)
k_trisum_frames(View g, const int* __restrict__ frames, int nframes, int rank, int world,
                FrameLayout L, char* gslab, const int64_t* __restrict__ OP,
                const u64* __restrict__ tcs, ST* __restrict__ tsl, ST* __restrict__ tsh,
                ST* __restrict__ tsd, HitLists HL, unsigned* __restrict__ claim) {
  extern __shared__ __align__(16) char smem[];
  __shared__ int s_claim;
  char* mem = GM ? gslab + (size_t)blockIdx.x * L.bytes : smem;
  while (true) {
    const int f = claim_frame(claim, &s_claim, rank, world);
    if (f >= nframes) break;
    trisum_frame<NT, AccT, ST>(g, frames[f], mem, L, OP, tcs, tsl, tsh, tsd, HL);
  }
}

// Upper bound of the local-edge count of all frames: sum_a min(items_a, C(D_a, 2)).
__global__ void k_hit_bound(View g, const int64_t* __restrict__ OP, u64* __restrict__ out) {
  u64 acc = 0;
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < g.n;
       a += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = g.osplit[a], e = g.rp[a + 1];
    const u64 D = (u64)(e - b), items = (u64)(OP[e] - OP[b]);
    const u64 c2 = D * (D - (D > 0)) / 2;
    acc += items < c2 ? items : c2;
  }
  for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

// ------------------------------------------------------------------------
// schedule: item counts per slot and frame keys (warp per row)
//   out-slot q (col[q] > row):   d+(col[q])            (pass A/B items)
//   lower slot q (w = col[q] < s): position of s in row w = #x in N(w), x < s
//                                  (pass C items; e2o of the edge is that slot)
// ------------------------------------------------------------------------
__global__ void k_slot_items(View g, int64_t S, int64_t* __restrict__ oitems,
                             int64_t* __restrict__ witems) {
  // one thread per slot: q is the out-slot of its edge iff e2o[edge] == q
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= S) return;
  const int x = g.col[q];
  const int64_t eo = g.e2o[g.seid[q]];
  int64_t oi = 0, wi = 0;
  if (eo == q)
    oi = g.rp[x + 1] - g.osplit[x];  // out-items: the higher-rank neighbours of x
  else
    wi = eo - g.rp[x];  // wedges s-x-*: the entries of row x below s
  oitems[q] = oi;
  witems[q] = wi;
}

// Frame sort keys from the scanned prefixes, one thread per row.
__global__ void k_frame_keys(View g, const int64_t* __restrict__ WP, u64* __restrict__ tri_key,
                             u64* __restrict__ wedge_key, int* __restrict__ ids_a,
                             int* __restrict__ ids_b) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= g.n) return;
  const int64_t b = g.rp[r], o = g.osplit[r], e = g.rp[r + 1];
  const u64 wsum = (u64)(WP[o] - WP[b]);  // (wedge items sit on the lower slots [b, o))
  const u64 D = (u64)(e - o);
  tri_key[r] = ~D;  // descending
  // wedges, with the lowest bit set when counters may exceed 16 bits
  const u64 big = (o - b) >= 65536 ? 1ull : 0ull;
  wedge_key[r] = ~((wsum << 1) | big);
  ids_a[r] = (int)r;
  ids_b[r] = (int)r;
}

// ------------------------------------------------------------------------
// pass C: vertex-priority wedges
// ------------------------------------------------------------------------
// item i of frame s -> lower slot p of w in row s: last p in [lo, hi) with
// WP[p] <= i
__device__ __forceinline__ int64_t wedge_slot(const int64_t* __restrict__ WP, int64_t lo,
                                              int64_t hi, int64_t i) {
  while (lo < hi - 1) {
    int64_t mid = (lo + hi) >> 1;
    if (WP[mid] <= i) lo = mid; else hi = mid;
  }
  return lo;
}

enum WedgeMode { kCount = 0, kUse = 1, kZero = 2, kTake = 3 };

// Fire-and-forget global reductions as PTX `red`.  Written as atomicAdd, a
// reduction whose result is unused becomes REDG, except in kernels that also
// hold a fence (the flow kernel's release of a finished task): there ptxas
// keeps every one of them an ATOMG that tracks its response.  `red` carries
// the PTX memory-model semantics the fence + barrier protocol relies on.
__device__ __forceinline__ void red_add(unsigned* a, unsigned v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void red_add(unsigned long long* a, unsigned long long v) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}

// red when v != 0, predicated inside the asm (a C++ `if` around an asm
// volatile becomes a branch with its own reconvergence point)
__device__ __forceinline__ void red_add_nz(unsigned* a, unsigned v) {
  asm volatile("{ .reg .pred p; setp.ne.u32 p, %1, 0; @p red.relaxed.gpu.global.add.u32 [%0], %1; }"
               ::"l"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void red_add_nz(unsigned long long* a, unsigned long long v) {
  asm volatile("{ .reg .pred p; setp.ne.u64 p, %1, 0; @p red.relaxed.gpu.global.add.u64 [%0], %1; }"
               ::"l"(a), "l"(v) : "memory");
}

struct SlabCounter {  // dense u32 counters in global memory
  unsigned* cnt;
  __device__ __forceinline__ void inc(int x) const { red_add(&cnt[x], 1u); }
  __device__ __forceinline__ unsigned get(int x) const { return cnt[x]; }
  __device__ __forceinline__ unsigned take(int x) const { return atomicExch(&cnt[x], 0u); }
  __device__ __forceinline__ void zero(int x) const { cnt[x] = 0u; }
};

struct U16Counter {  // dense u16 counters, two per 32-bit word
  unsigned* w;
  __device__ __forceinline__ void inc(int x) const {
    red_add(&w[x >> 1], 1u << ((x & 1) << 4));
  }
  __device__ __forceinline__ unsigned get(int x) const {
#ifdef GD_CNT_CG  // experiment: counter reads bypass L1
    return __ldcg((const unsigned short*)w + x);
#else
    return ((const unsigned short*)w)[x];
#endif
  }
  __device__ __forceinline__ unsigned take(int x) const { return get(x); }  // unused
  __device__ __forceinline__ void zero(int x) const { ((unsigned short*)w)[x] = 0; }
};

template <bool C16>
struct HashCounter {  // shared-memory open-addressing hash, u32 or u16 counts
  int* hk;
  unsigned* hv;  // C16: two counts per word
  int hmask, hshift;
  __device__ __forceinline__ int slot(int x) const {
    unsigned h = mhash((unsigned)x, hshift);
    while (hk[h] != x) h = (h + 1) & hmask;
    return (int)h;
  }
  __device__ __forceinline__ void inc(int x) const {
    unsigned h = mhash((unsigned)x, hshift);
    while (true) {
      int old = atomicCAS(&hk[h], -1, x);
      if (old == -1 || old == x) break;
      h = (h + 1) & hmask;
    }
    if (C16) atomicAdd(&hv[h >> 1], 1u << ((h & 1) << 4));
    else atomicAdd(&hv[h], 1u);
  }
  __device__ __forceinline__ unsigned count_at(int h) const {
    return C16 ? (unsigned)((const unsigned short*)hv)[h] : hv[h];
  }
  __device__ __forceinline__ unsigned get(int x) const { return count_at(slot(x)); }
  __device__ __forceinline__ unsigned take(int x) const { return get(x); }  // unused
  __device__ __forceinline__ void zero(int) const {}
};

// One sweep of `mode` over items [i0, i1) of frame s (lower slots [b, o)).
// Each warp takes one contiguous piece (a multiple of 32 items); lane l
// handles c0+l, c0+l+32, ..., so lanes read consecutive entries of one row w
// (coalesced).  The slot of the first item is found by one binary search per
// lane per piece; later rows follow by advancing p (measured: per-512-item
// searches spent ~40% of the heavy-frame kernel's stalls on that chain).
// Steps whose U items all lie in the current row (the common case: a
// wedge-weighted row holds ~360 items at config 3) take a fast path with no
// per-item slot state: all U col[] loads, then all U counter loads, then the
// updates, so the dependent counter reads of the use sweep overlap instead of
// alternating with the per-edge atomics.  Steps that cross a row boundary
// walk their items one at a time.
// Returns the thread's partial (kUse: sum of cnt-1; kTake: sum of c*(c-1)).
template <int NT, int MODE, typename C, int U = 1, typename CT = u64, int PIECES = 1>
__device__ __forceinline__ u64 wedge_sweep(const View& g, const int64_t* __restrict__ WP,
                                           int64_t b, int64_t o, int64_t i0, int64_t i1,
                                           const C& ctr, bool per_edge, CT* __restrict__ c4s,
                                           int* piece_ctr = nullptr) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int nw = NT / 32;
  // PIECES > 1: nw * PIECES pieces claimed dynamically from a CTA counter
  const int npieces = nw * PIECES;
  const int64_t per = (((i1 - i0) + npieces - 1) / npieces + 31) & ~int64_t(31);
  auto claim = [&]() {
    int v = 0;
    if (lane == 0) v = atomicAdd(piece_ctr, 1);
    return __shfl_sync(0xffffffffu, v, 0);
  };
  u64 local = 0;
  for (int pc = PIECES == 1 ? warp : claim(); pc < npieces; pc = PIECES == 1 ? npieces : claim()) {
  const int64_t c0 = i0 + (int64_t)pc * per;
  const int64_t c1 = c0 + per < i1 ? c0 + per : i1;
  int64_t i = c0 + lane;
  if (i >= c1) continue;
  int64_t p = wedge_slot(WP, b, o, i);
  int64_t wp1 = WP[p + 1];
  int64_t base = g.rp[g.col[p]] - WP[p];  // slot of item i in row w: base + i
  int64_t ptop = p;                       // per-edge: pending sum for slot ptop (edge s-w)
  u64 top = 0;
  // one item: x = col[q], q its slot, pr its row
  auto one = [&](int x, int64_t q, int64_t pr, unsigned cnt) {
    if (MODE == kCount) {
      ctr.inc(x);
    } else if (MODE == kZero) {
      ctr.zero(x);
    } else if (MODE == kTake) {
      const u64 c = ctr.take(x);
      local += c * (c - (c > 0));
    } else {
      const u64 c = cnt - 1u;
      if (c) {
        local += c;
        if (per_edge) {
#ifndef GD_EXP_NO_C4S  // timing experiment only (tools/build_variant.py)
          red_add(&c4s[q], (CT)c);  // edge w-x
#endif
          if (pr != ptop) {
            if (top) red_add(&c4s[ptop], (CT)top);
            top = 0;
            ptop = pr;
          }
          top += c;
        }
      }
    }
  };
  for (; i < c1; i += 32 * U) {
    const int64_t ilast = i + 32 * (U - 1);
    if (ilast < c1 && ilast < wp1) {  // all U items in row p
      const int64_t q0 = base + i;
      int xx[U];
#pragma unroll
      for (int u = 0; u < U; u++) xx[u] = __ldg(g.col + q0 + 32 * u);
      unsigned cc[U];
#pragma unroll
      for (int u = 0; u < U; u++) cc[u] = MODE == kUse ? ctr.get(xx[u]) : 0u;
#pragma unroll
      for (int u = 0; u < U; u++) one(xx[u], q0 + 32 * u, p, cc[u]);
    } else {
#pragma unroll 1
      for (int u = 0; u < U; u++) {
        const int64_t ii = i + 32 * u;
        if (ii >= c1) break;
        if (wp1 <= ii) {
          do {
            p++;
            wp1 = WP[p + 1];
          } while (wp1 <= ii);
          base = g.rp[g.col[p]] - WP[p];
        }
        const int x = __ldg(g.col + base + ii);
        one(x, base + ii, p, MODE == kUse ? ctr.get(x) : 0u);
      }
    }
  }
  if (MODE == kUse && per_edge && top) red_add(&c4s[ptop], (CT)top);
  }
  return local;
}

// Small and medium frames: counters in a shared-memory hash.
template <int NT, bool C16, typename CT>
__global__ void __launch_bounds__(NT)
k_c4_frames_smem(View g, const int64_t* __restrict__ WP, const int* __restrict__ frames,
                 int nframes, int rank, int world, int hcap, int per_edge, CT* __restrict__ c4s,
                 u64* __restrict__ c4tot2) {
  extern __shared__ __align__(16) char smem[];
  int* hk = (int*)smem;
  unsigned* hv = (unsigned*)(hk + hcap);
  typedef cub::BlockReduce<u64, NT> BR;
  __shared__ typename BR::TempStorage tmp;
  for (int f = rank + world * blockIdx.x; f < nframes; f += world * gridDim.x) {
    const int s = frames[f];
    const int64_t b = g.rp[s], o = g.osplit[s];
    const int64_t i0 = WP[b], i1 = WP[o];
    const int64_t total = i1 - i0;
    int H = pow2_at_least((int)(2 * total < (int64_t)hcap ? 2 * total : (int64_t)hcap));
    if (H > hcap) H = hcap;
    HashCounter<C16> ctr{hk, hv, H - 1, 32 - (31 - __clz(H))};
    for (int h = threadIdx.x; h < H; h += NT) hk[h] = -1;
    for (int h = threadIdx.x; h < (C16 ? H / 2 : H); h += NT) hv[h] = 0u;
    __syncthreads();
    wedge_sweep<NT, kCount, HashCounter<C16>, 1, CT>(g, WP, b, o, i0, i1, ctr, false, c4s);
    __syncthreads();
    u64 local = 0;
    if (!per_edge) {
      for (int h = threadIdx.x; h < H; h += NT) {
        const u64 c = ctr.count_at(h);
        local += c * (c - (c > 0));  // 2 * C(c, 2)
      }
    } else {
      local = wedge_sweep<NT, kUse, HashCounter<C16>, 1, CT>(g, WP, b, o, i0, i1, ctr, true, c4s);
    }
    const u64 sum = BR(tmp).Sum(local);
    if (threadIdx.x == 0 && sum) atomic_add_u128(c4tot2 + 2 * graph_of(g, s), sum);
    __syncthreads();
  }
}

// Hub frames whose counters may exceed 16 bits: each (frame, chunk) is one
// CTA, frame h uses u32 slab h; the sweeps are separate launches (phase 0
// count, 1 use, 2 zero).
struct HubChunk {
  int frame;       // rank id s
  int slab;        // slab index
  int64_t i0, i1;  // item range
};

template <int NT, typename CT>
__global__ void __launch_bounds__(NT)
k_c4_hub(View g, const int64_t* __restrict__ WP, const HubChunk* __restrict__ chunks,
         unsigned* __restrict__ slabs, int64_t slab_stride, int phase, int per_edge,
         CT* __restrict__ c4s, u64* __restrict__ c4tot2) {
  typedef cub::BlockReduce<u64, NT> BR;
  __shared__ typename BR::TempStorage tmp;
  const HubChunk ch = chunks[blockIdx.x];
  SlabCounter ctr{slabs + (size_t)ch.slab * slab_stride};
  const int s = ch.frame;
  const int64_t b = g.rp[s], o = g.osplit[s];
  if (phase == 0) {
    wedge_sweep<NT, kCount, SlabCounter, 1, CT>(g, WP, b, o, ch.i0, ch.i1, ctr, false, c4s);
  } else if (phase == 1) {
    const u64 local =
        wedge_sweep<NT, kUse, SlabCounter, 1, CT>(g, WP, b, o, ch.i0, ch.i1, ctr, per_edge != 0, c4s);
    const u64 sum = BR(tmp).Sum(local);
    if (threadIdx.x == 0 && sum) atomic_add_u128(c4tot2 + 2 * graph_of(g, s), sum);
  } else {
    wedge_sweep<NT, kZero, SlabCounter, 1, CT>(g, WP, b, o, ch.i0, ch.i1, ctr, false, c4s);
  }
}

// Heavy frames on thread-block clusters: the dense u16 counter array of one
// frame (one counter per rank id < n) is spread over the distributed shared
// memory of a cluster of `csize` CTAs (counter x lives in CTA x / per).  The
// count sweep is remote shared-memory atomics, the use sweep remote reads;
// no counter ever touches L2/HBM, which stays free for the adjacency rows.
// Each cluster takes frames (descending work) from a global queue.
struct DsmemCounter {
  unsigned* base;  // this CTA's slab (same offset in every CTA of the cluster)
  int per;         // counters per CTA (even)
  __device__ __forceinline__ void inc(int x) const {
    const int owner = x / per, off = x - owner * per;
    unsigned* w = cg::this_cluster().map_shared_rank(base, owner) + (off >> 1);
    atomicAdd(w, 1u << ((off & 1) << 4));
  }
  __device__ __forceinline__ unsigned get(int x) const {
    const int owner = x / per, off = x - owner * per;
    const unsigned short* c =
        (const unsigned short*)cg::this_cluster().map_shared_rank(base, owner);
    return c[off];
  }
  __device__ __forceinline__ unsigned take(int x) const { return get(x); }  // unused
  __device__ __forceinline__ void zero(int) const {}
};

template <int NT, typename CT>
__global__ void __launch_bounds__(NT, 1)
k_c4_cluster(View g, const int64_t* __restrict__ WP, const int* __restrict__ frames,
             int nframes, int rank, int world, int* __restrict__ queue, int per, int per_edge,
             CT* __restrict__ c4s, u64* __restrict__ c4tot2) {
  extern __shared__ __align__(16) unsigned slab[];
  __shared__ int s_frame;
  typedef cub::BlockReduce<u64, NT> BR;
  __shared__ typename BR::TempStorage tmp;
  cg::cluster_group cluster = cg::this_cluster();
  const int crank = (int)cluster.block_rank(), csize = (int)cluster.num_blocks();
  const int words = per >> 1;
  uint4* z4 = (uint4*)slab;
  for (int i = threadIdx.x; i < words / 4; i += NT) z4[i] = make_uint4(0u, 0u, 0u, 0u);
  DsmemCounter ctr{slab, per};
  while (true) {
    if (crank == 0 && threadIdx.x == 0) {
      const int q = atomicAdd(queue, 1);
      s_frame = rank + world * q;  // this shard's frames: every world-th
    }
    cluster.sync();  // counters zeroed everywhere, frame published
    const int f = *cluster.map_shared_rank(&s_frame, 0);
    // no CTA may exit (or rank 0 republish) while another still reads s_frame
    cluster.sync();
    if (f >= nframes) break;
    const int s = frames[f];
    const int64_t b = g.rp[s], o = g.osplit[s];
    const int64_t fi0 = WP[b], fi1 = WP[o];
    const int64_t len = (fi1 - fi0 + csize - 1) / csize;
    const int64_t i0 = fi0 + len * crank;
    const int64_t i1 = i0 + len < fi1 ? i0 + len : fi1;
    if (i0 < i1) wedge_sweep<NT, kCount, DsmemCounter, 1, CT>(g, WP, b, o, i0, i1, ctr, false, c4s);
    cluster.sync();
    const u64 local =
        i0 < i1 ? wedge_sweep<NT, kUse, DsmemCounter, 1, CT>(g, WP, b, o, i0, i1, ctr, per_edge != 0,
                                                             c4s)
                : 0;
    const u64 sum = BR(tmp).Sum(local);
    if (threadIdx.x == 0 && sum) atomic_add_u128(c4tot2 + 2 * graph_of(g, s), sum);
    cluster.sync();  // every remote read of this frame done
    for (int i = threadIdx.x; i < words / 4; i += NT) z4[i] = make_uint4(0u, 0u, 0u, 0u);
  }
}

// Heavy frames (more than 24576 wedges, n too large for cluster shared
// memory) as a dataflow of tasks with no grid barrier.  Frames are grouped in
// rounds of F frames (one dense u16 counter slab each, ranks [x0, n)); a
// round's wedge items are cut into chunks.  One task sequence is handed out in
// order by a global counter:
//   step t:  C(t) count chunks of round t | U(t-LU) use chunks (or S(t-LU)
//            slab scans in global mode) | Z(t-LU-1) zeroing of that round's slabs
// with NS >= LU + 2 slab sets (round r uses set r % NS; default LU = 1,
// NS = 4: a fourth set gives the count tasks of round t a step of slack
// behind the zeroing they wait for, measured 72.3 -> 65.3 ms at config 3 and
// 774 -> 692 ms at config 5, per-edge).  A task waits (spins) only
// on a segment handed out earlier: U(r), S(r) on C(r); Z(r) on U(r); C(t) on
// the segment that freed its set (Z(t-NS) or S(t-NS)).  Every awaited task is
// therefore already running on a resident CTA, so the kernel needs neither a
// cooperative launch nor co-residency, and a CTA that finishes early takes
// the next task instead of idling at a barrier.
enum FlowType { kFlowCount = 0, kFlowUse = 1, kFlowScan = 2, kFlowZeroSweep = 3, kFlowZeroFill = 4 };

struct FlowSeg {
  int type, round;
  int64_t task0, ntasks;  // global task range [task0, task0 + ntasks)
  int dep;                // segment awaited (-1: none); needs all its tasks done
};

struct FlowPlan {
  const int* frames;    // heavy frames (rank ids), descending wedges
  const int64_t* cpre;  // [nf+1] chunk prefix
  const int* rf;        // [R+1] round -> first frame index
  const int64_t* rch;   // [R] items per chunk of each round
  const FlowSeg* segs;  // [nseg]
  int nseg;
  int F;                // slabs per set
  int64_t slab_words;   // 32-bit words per slab
  int x0;               // first counter (even): counters cover ranks [x0, n)
  int64_t pieces;       // uint4 per fill / scan piece
  int nsets;            // slab sets (round r uses set r % nsets)
};

#ifndef GD_FLOW_PIECES
#define GD_FLOW_PIECES 2
#endif
template <int NT, int MODE, int U, typename CT>
__device__ __forceinline__ u64 flow_chunk(const View& g, const int64_t* __restrict__ WP, const FlowPlan& P, int r,
                          int64_t k, unsigned* __restrict__ set, bool per_edge, CT* __restrict__ c4s,
                          int& s_out, int* piece_ctr) {
  const int f0 = P.rf[r], f1 = P.rf[r + 1];
  k += P.cpre[f0];
  int lo = f0, hi = f1;  // frame of chunk k: last j with cpre[j] <= k
  while (lo < hi - 1) {
    int mid = (lo + hi) >> 1;
    if (P.cpre[mid] <= k) lo = mid; else hi = mid;
  }
  const int j = lo;
  const int s = P.frames[j];
  s_out = s;
  const int64_t b = g.rp[s], o = g.osplit[s];
  const int64_t fi0 = WP[b], fi1 = WP[o];
  const int64_t CH = P.rch[r];
  const int64_t i0 = fi0 + (k - P.cpre[j]) * CH;
  const int64_t i1 = i0 + CH < fi1 ? i0 + CH : fi1;
  U16Counter ctr{set + (size_t)(j - f0) * P.slab_words - (P.x0 >> 1)};
  // count sweeps claim pieces dynamically (their warps finish unevenly);
  // use sweeps keep one contiguous piece per warp (a piece boundary costs a
  // slot search and a pending per-edge flush)
  constexpr int PC = MODE == kCount ? GD_FLOW_PIECES : 1;
  return wedge_sweep<NT, MODE, U16Counter, U, CT, PC>(g, WP, b, o, i0, i1, ctr, per_edge, c4s,
                                                      piece_ctr);
}

#ifndef GD_FLOW_MINB
#define GD_FLOW_MINB 4
#endif
#ifndef GD_FLOW_U
#define GD_FLOW_U 1
#endif
#ifndef GD_FLOW_UU
#define GD_FLOW_UU 2
#endif
template <int NT, int MINB, int U, int UU, typename CT>
__global__ void __launch_bounds__(NT, MINB)
k_c4_flow(View g, const int64_t* __restrict__ WP, FlowPlan P, unsigned* __restrict__ slabs,
          int per_edge, CT* __restrict__ c4s, u64* __restrict__ c4tot2,
          unsigned long long* __restrict__ next_task, int* __restrict__ done) {
  typedef cub::BlockReduce<u64, NT> BR;
  __shared__ typename BR::TempStorage tmp;
  __shared__ long long s_task;
  __shared__ int s_piece;  // dynamic piece counter of the current task
  const int64_t total = P.segs[P.nseg - 1].task0 + P.segs[P.nseg - 1].ntasks;
  const size_t set_words = (size_t)P.F * P.slab_words;
  if (threadIdx.x == 0) s_task = (long long)atomicAdd(next_task, 1ull);
  while (true) {
    __syncthreads();
    const int64_t task = s_task;
    if (task >= total) break;
    // the next task is claimed now (its latency overlaps this one); it can
    // only wait on tasks handed out before it, so holding it is safe
    long long nxt = 0;
    if (threadIdx.x == 0) nxt = (long long)atomicAdd(next_task, 1ull);
    int lo = 0, hi = P.nseg;  // segment of the task: last with task0 <= task
    while (lo < hi - 1) {
      int mid = (lo + hi) >> 1;
      if (P.segs[mid].task0 <= task) lo = mid; else hi = mid;
    }
    const FlowSeg sg = P.segs[lo];
    if (threadIdx.x == 0) s_piece = 0;  // published by the barrier below
    if (threadIdx.x == 0 && sg.dep >= 0) {
      const int need = (int)P.segs[sg.dep].ntasks;
      while (*(volatile int*)&done[sg.dep] < need) __nanosleep(128);
      __threadfence();  // acquire: later loads see the awaited tasks' writes
    }
    __syncthreads();
    const int64_t k = task - sg.task0;
    const int r = sg.round;
    unsigned* set = slabs + (size_t)(r % P.nsets) * set_words;
    if (sg.type == kFlowCount) {
      int s;
      flow_chunk<NT, kCount, U, CT>(g, WP, P, r, k, set, false, c4s, s, &s_piece);
    } else if (sg.type == kFlowUse) {
      int s;
      const u64 local =
          flow_chunk<NT, kUse, UU, CT>(g, WP, P, r, k, set, per_edge != 0, c4s, s, &s_piece);
      const u64 sum = BR(tmp).Sum(local);
      if (threadIdx.x == 0 && sum) atomic_add_u128(c4tot2 + 2 * graph_of(g, s), sum);
    } else if (sg.type == kFlowZeroSweep) {
      int s;
      flow_chunk<NT, kZero, U, CT>(g, WP, P, r, k, set, false, c4s, s, &s_piece);
    } else {
      // piece k of the round's used slabs: fill with zeros, or (global mode)
      // sum 2*C(c,2) of its counters and zero them
      const int64_t per_slab = (P.slab_words / 4 + P.pieces - 1) / P.pieces;
      const int64_t fj = k / per_slab, pc = k - fj * per_slab;
      uint4* z = (uint4*)(set + (size_t)fj * P.slab_words);
      const int64_t e0 = pc * P.pieces;
      const int64_t e1 = e0 + P.pieces < P.slab_words / 4 ? e0 + P.pieces : P.slab_words / 4;
      const uint4 zero4 = make_uint4(0u, 0u, 0u, 0u);
      if (sg.type == kFlowZeroFill) {
        for (int64_t i = e0 + threadIdx.x; i < e1; i += NT) z[i] = zero4;
      } else {
        u64 local = 0;
        for (int64_t i = e0 + threadIdx.x; i < e1; i += NT) {
          const uint4 w4 = z[i];
          const unsigned wv[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
          for (int t = 0; t < 4; t++) {
            const u64 c0 = wv[t] & 0xffffu, c1 = wv[t] >> 16;
            local += c0 * (c0 - (c0 > 0)) + c1 * (c1 - (c1 > 0));
          }
          if (wv[0] | wv[1] | wv[2] | wv[3]) z[i] = zero4;
        }
        const u64 sum = BR(tmp).Sum(local);
        if (threadIdx.x == 0 && sum)
          atomic_add_u128(c4tot2 + 2 * graph_of(g, P.frames[P.rf[r] + fj]), sum);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();  // release: this task's writes before its completion
      atomicAdd(&done[lo], 1);
      s_task = nxt;
    }
  }
}

// ------------------------------------------------------------------------
// Heavy frames on x-tiles in shared memory.  The dense u16 counter array of
// frame s over ranks [x0, s) is cut into tiles of T counters; job (s, p)
// counts, on one CTA, only the wedges s-w-x with x in tile p, whose items are
// the sub-range [TS[w][p], TS[w][p+1]) of every lower row w (TS: per-row tile
// split slots, k_tile_splits).  Both sweeps then run on shared-memory atomics
// and loads (measured on B200: >= 1.5 T random u16 atomics/s in shared
// memory against 0.19 T/s as L2-resident and 0.03 T/s as DRAM-resident global
// reductions), and no counter ever reaches L2 or HBM.  Per job the CTA's
// warps claim batches of 32 consecutive lower slots q_s of row s (segments
// (w, [a, b))), prefix their lengths with a warp scan and walk the items
// lane-interleaved (consecutive lanes read consecutive slots of one row w).
// ------------------------------------------------------------------------
// Tiles have degree-aware widths: a counter of x never exceeds deg(x) (its
// wedges s-w-x need w in N(x)), and ranks ascend by degree, so a tile whose
// highest rank has degree < 2^b packs b-bit counters (b = 2, 4, 8, 16) and
// spans 16/b times the ranks of a 16-bit tile in the same shared memory.  Tiles
// of one width form a run of equal spans (the last one cut at the degree
// limit); at most four runs, ascending widths.
struct TileRuns {
  int R[4];  // first rank of the run (INT_MAX: unused)
  int T[4];  // ranks per tile
  int I[4];  // index of the run's first tile
  __host__ __device__ __forceinline__ int tile_of(int x) const {
    const int r = (x >= R[1]) + (x >= R[2]) + (x >= R[3]);
    const int R0 = r == 0 ? R[0] : r == 1 ? R[1] : r == 2 ? R[2] : R[3];
    const int T0 = r == 0 ? T[0] : r == 1 ? T[1] : r == 2 ? T[2] : T[3];
    const int I0 = r == 0 ? I[0] : r == 1 ? I[1] : r == 2 ? I[2] : I[3];
    return I0 + (x - R0) / T0;
  }
};

struct TilePlan {
  const int* frames;    // heavy frames (rank ids), descending wedges
  const int64_t* jpre;  // [nf+1] job prefix: frame j owns jobs [jpre[j], jpre[j+1])
  const int* jframe;    // [njobs] frame of each job
  int nf;
  int64_t njobs;
  int cap16;            // shared-memory tile capacity in 16-bit units (multiple of 8)
  int P1;               // split entries per row (tiles + 1)
  const int64_t* TS;    // [n][P1] absolute slot of the first entry >= tb[p]
  const int* tb;        // [P1] first rank of tile p (tb[P1-1] = n)
  const int* tlg;       // [P1-1] log2 of the counter bits of tile p (1..4)
  int piece_min;        // chunks averaging >= this many items per segment take the piece walk
  const int2* jobs;     // [njobs] (frame index, tile | last << 16) in processing order
};

// first rank whose degree exceeds 0, 1, 3, 15, 255 (ranks ascend by degree)
__global__ void k_degree_ranks(View g, int* __restrict__ out) {
  const int lim[5] = {0, 1, 3, 15, 255};
  if (threadIdx.x < 5) {
    int64_t lo = 0, hi = g.n;  // first r in [0, n] with deg[r] > lim
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (g.deg[mid] > lim[threadIdx.x]) hi = mid; else lo = mid + 1;
    }
    out[threadIdx.x] = (int)lo;
  }
}

// TS[w][p] = rp[w] + #(entries of row w with rank < tb[p]), warp per row:
// lane j marks the tiles that start at entry j (tile(x_{j-1}) < p <= tile(x_j)).
// GS lanes per row: 8 for the rows below degree 256 (most rows hold a few
// entries; a warp per row ran at 1-2 active lanes), 32 above.
// Long rows are cut into segments of kSplitSeg entries (blockIdx.y): a segment
// needs only the tile of the entry before it, so a hub row of 60,000 entries
// is not one warp's serial walk.
constexpr int kSplitSeg = 1024;
template <int GS>
__global__ void k_tile_splits(View g, TileRuns RN, int P1, int64_t* __restrict__ TS, int64_t w0,
                              int64_t w1) {
  const auto grp = cg::tiled_partition<GS>(cg::this_thread_block());
  const int64_t groups = (int64_t)gridDim.x * (blockDim.x / GS);
  const int lane = (int)grp.thread_rank();
  const bool segmented = gridDim.y > 1;
  for (int64_t w = w0 + (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / GS; w < w1; w += groups) {
    const int64_t b = g.rp[w], e = g.rp[w + 1];
    const int64_t cb = segmented ? b + (int64_t)blockIdx.y * kSplitSeg : b;
    const int64_t ce = segmented ? (cb + kSplitSeg < e ? cb + kSplitSeg : e) : e;
    if (cb >= e && (cb > b || blockIdx.y > 0)) continue;  // no such segment
    int64_t* ts = TS + w * P1;
    int last = -1;  // tile of the last entry seen (all lanes)
    if (cb > b) {
      const int x = g.col[cb - 1];
      last = x < RN.R[0] ? -1 : RN.tile_of(x);
    }
    for (int64_t c = cb; c < ce; c += GS) {
      const int64_t q = c + lane;
      int t = INT_MAX;
      if (q < ce) {  // entries below the first tile (leaves) count as tile -1
        const int x = g.col[q];
        t = x < RN.R[0] ? -1 : RN.tile_of(x);
      }
      int prev = grp.shfl_up(t, 1);
      if (lane == 0) prev = last;
      if (q < ce)
        for (int p = prev + 1; p <= t && p < P1; p++) ts[p] = q;
      last = grp.shfl(t, GS - 1);
      if (last == INT_MAX) {  // the segment ended inside this chunk: its last tile
        const unsigned valid = grp.ballot(q < ce);
        last = grp.shfl(t, 31 - __clz(valid));
      }
    }
    if (ce == e)  // the row's last segment: the tiles past its last entry
      for (int p = last + 1 + lane; p < P1; p += GS) ts[p] = e;
  }
}

// Items of one chunk of a job's nonempty segments (k: items seg_pre[k] ..
// seg_pre[k+1] at slots seg_off[k] + item), walked by a warp over the item
// range [r0, r1) in steps of 32 consecutive items.  The segments after the
// current one start at distinct items (empty segments are compacted away),
// so at most 32 of them start inside a step: lane l tests segment kc+1+l, a
// warp OR collects the start bits M, and lane j's segment is
// kc + popc(M & bits <= j) -- no search, one shared load per lane.  U steps
// are resolved before their col[] loads are issued.  f(k, q, x, M, j) gets
// the segment k (-1 past r1), slot q, x = col[q] and the step's start bits.
#ifndef GD_TILE_U
#define GD_TILE_U 4  // measured U = 1 / 2 / 3 / 4 / 6 / 8: C3 per-edge 45.6 / 37.7 / 36.0 / 34.8 / 36.2 / 36.8 ms
#endif
#ifndef GD_TILE_NT
#define GD_TILE_NT 1024
#endif
#ifndef GD_TILE_CLAIMS
#define GD_TILE_CLAIMS 1  // item ranges per warp and chunk (8 / 4 / 2 / 1: C3 per-edge pass C 21.6 / 19.6 / 18.7 / 18.4 ms)
#endif
template <int U, typename QT, typename F>
__device__ __forceinline__ void tile_range_items(const View& g, const int* seg_pre,
                                                 const QT* seg_off, int cnt,
                                                 int r0, int r1, F&& f) {
  const int lane = threadIdx.x & 31;
  const unsigned le = 0xffffffffu >> (31 - lane);  // bits 0..lane
  // current segment: last k with seg_pre[k] <= r0 (seg_pre ascends, seg_pre[0]
  // = 0 <= r0).  A warp search: the lanes test 32 spread entries, then the 32
  // entries of the block found (cnt <= 1024): two shared loads and two
  // ballots instead of a ten-step dependent binary search per claimed range.
#ifndef GD_TILE_BSEARCH
  int kc;
  {
    const int b = lane << 5;
    const unsigned m1 = __ballot_sync(0xffffffffu, b < cnt && seg_pre[b] <= r0);
    const int blk = (__popc(m1) - 1) << 5;  // m1 has bit 0 set
    const unsigned m2 = __ballot_sync(0xffffffffu, blk + lane < cnt && seg_pre[blk + lane] <= r0);
    kc = blk + __popc(m2) - 1;
  }
#else
  int lo = 0, hi = cnt;
  while (lo < hi - 1) {
    const int mid = (lo + hi) >> 1;
    if (seg_pre[mid] <= r0) lo = mid; else hi = mid;
  }
  int kc = lo;
#endif
#ifndef GD_TILE_NOFAST
  // start of the segment after kc (uniform): steps that end before it lie in
  // segment kc and need no resolution
  int nb = kc + 1 < cnt ? seg_pre[kc + 1] : INT_MAX;
  QT off_kc = seg_off[kc];
#endif
  for (int base = r0; base < r1; base += 32 * U) {
    int kk[U];
    QT qq[U];
    unsigned mm[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int wb = base + 32 * u;
#ifndef GD_TILE_NOFAST
      if (wb + 32 <= nb) {  // the whole step inside segment kc
        kk[u] = wb + lane < r1 ? kc : -1;
        qq[u] = off_kc + wb + lane;
        mm[u] = 0u;
        continue;
      }
#endif
      const int k = kc + 1 + lane;
      const int sp = k < cnt ? seg_pre[k] : INT_MAX;
      const int r = sp - wb;
      const unsigned M = __reduce_or_sync(0xffffffffu, r < 32 ? 1u << r : 0u);
      const int ks = kc + __popc(M & le);
      const int adv = __popc(M);
      kc += adv;
      kk[u] = wb + lane < r1 ? ks : -1;
      qq[u] = seg_off[ks] + wb + lane;
      mm[u] = M;
#ifndef GD_TILE_NOFAST
      // lane adv loaded seg_pre[kc_new + 1] (re-read when all 32 lanes' segments
      // started in this step); lane 31's slot gives seg_off[kc_new]
      nb =__shfl_sync(0xffffffffu, sp, adv & 31);
      if (adv == 32) nb = kc + 1 < cnt ? seg_pre[kc + 1] : INT_MAX;
      off_kc = __shfl_sync(0xffffffffu, qq[u], 31) - (wb + 31);
#endif
    }
    int xx[U];
#pragma unroll
    for (int u = 0; u < U; u++) xx[u] = kk[u] >= 0 ? __ldg(g.col + qq[u]) : 0;
#pragma unroll
    for (int u = 0; u < U; u++) f(kk[u], qq[u], xx[u], mm[u]);
  }
}

// Indexed variant for chunks of at most kTileIdxCap items: the chunk setup
// leaves, per 32-item word w of the chunk, the start bits B[w] of the segments
// beginning inside it and C[w] = number of segments beginning before item
// 32w.  A step then needs no search, no warp collective and no state carried
// from the previous step: lane l of word w is in segment C[w] - 1 +
// popc(B[w] & bits <= l) (two broadcast shared loads).  Invalid lanes (past
// r1) get k = -1 and slot 0.  f(k, q, x).
constexpr int kTileIdxCap = 32768;
constexpr int kTileIdxWords = kTileIdxCap / 32 + 8;  // + padding read by the last steps

// Shared memory through explicit 32-bit shared-window addresses held in
// registers: inside these loops the compiler otherwise rebuilds the window
// base (S2R SR_CgaCtaId + LEA) before every access (SASS of the first
// version: 8 of a step's 44 instructions).
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ unsigned lds_u32(unsigned a) {
  unsigned v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ long long lds_off(unsigned base, int k, int) {
  return (long long)(int)lds_u32(base + 4u * (unsigned)k);
}
__device__ __forceinline__ long long lds_off(unsigned base, int k, long long) {
  long long v;
  asm volatile("ld.shared.s64 %0, [%1];" : "=l"(v) : "r"(base + 8u * (unsigned)k));
  return v;
}
__device__ __forceinline__ void reds_add(unsigned a, unsigned v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void reds_add(unsigned a, unsigned long long v) {
  asm volatile("red.shared.add.u64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}

template <int U, typename QT, typename F>
__device__ __forceinline__ void tile_items_indexed(const View& g, unsigned sB, unsigned sC,
                                                   unsigned sOff, int r0, int r1, F&& f) {
  const int lane = threadIdx.x & 31;
  const unsigned le = 0xffffffffu >> (31 - lane);  // bits 0..lane
  int base = r0;
#ifndef GD_TILE_IDX_NOSPLIT
  // full groups (every range but a window's last is a multiple of 32 items):
  // no validity selects; f(valid, k, q, x) folds its own on the literal
  for (; base + 32 * U <= r1; base += 32 * U) {
    int kk[U];
    QT qq[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int wb = base + 32 * u;
      const unsigned w4 = ((unsigned)wb >> 5) << 2;
      kk[u] = (int)lds_u32(sC + w4) - 1 + __popc(lds_u32(sB + w4) & le);
      qq[u] = (QT)((QT)lds_off(sOff, kk[u], QT()) + wb + lane);
    }
    int xx[U];
#pragma unroll
    for (int u = 0; u < U; u++) xx[u] = __ldg(g.col + qq[u]);
#pragma unroll
    for (int u = 0; u < U; u++) f(true, kk[u], qq[u], xx[u]);
  }
#endif
  for (; base < r1; base += 32 * U) {  // the ragged last group
    int kk[U];
    QT qq[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int wb = base + 32 * u;
      const unsigned w4 = ((unsigned)wb >> 5) << 2;
      const bool valid = wb + lane < r1;
      int ks = (int)lds_u32(sC + w4) - 1 + __popc(lds_u32(sB + w4) & le);
      ks = valid ? ks : 0;  // (past the chunk's last word the index arrays hold stale values)
      const QT off = (QT)lds_off(sOff, ks, QT());
      kk[u] = valid ? ks : -1;
      qq[u] = valid ? (QT)(off + wb + lane) : (QT)0;
    }
    int xx[U];
#pragma unroll
    for (int u = 0; u < U; u++) xx[u] = __ldg(g.col + qq[u]);
#pragma unroll
    for (int u = 0; u < U; u++) f(kk[u] >= 0, kk[u], qq[u], xx[u]);
  }
}

// Piece walk for chunks whose segments are long: the claimed item range
// [r0, r1) is cut at the segment boundaries inside it and every piece is
// scanned with warp-uniform bounds and one row pointer (no per-lane segment
// resolution at all; at most one partly filled step per piece).
// item(valid, q, x) per lane and step (lanes past the piece get x = xd);
// piece_end(k) once per piece, converged.
#ifndef GD_TILE_PU
#define GD_TILE_PU 8  // col[] loads in flight per lane in the piece walk (4 / 6 / 8: C5 per-edge pass C 203 / 194 / 190 ms)
#endif
#ifndef GD_TILE_PIECE_MIN
#define GD_TILE_PIECE_MIN 192  // average items per segment of a chunk from which pieces are used
// (measured 16 / 48 / 64 / 128 / 256 / 512: C3 per-edge pass C 33.2 / 28.9 / 27.5 / 25.0 / 23.7 / 25.5 ms,
// indexed only 28.6; a two-stage pipeline across pieces was slower: 27.9 ms)
#endif
template <int U, typename QT, typename FI, typename FE>
__device__ __forceinline__ void tile_items_pieces(const View& g, unsigned sPre, unsigned sOff,
                                                  int cnt, int r0, int r1, int xd, FI&& item,
                                                  FE&& piece_end) {
  const int lane = threadIdx.x & 31;
  int kc;  // last k with seg_pre[k] <= r0 (warp search, see tile_range_items)
  {
    const int b = lane << 5;
    const unsigned m1 =
        __ballot_sync(0xffffffffu, b < cnt && (int)lds_u32(sPre + 4u * (unsigned)b) <= r0);
    const int blk = (__popc(m1) - 1) << 5;
    const unsigned m2 = __ballot_sync(
        0xffffffffu, blk + lane < cnt && (int)lds_u32(sPre + 4u * (unsigned)(blk + lane)) <= r0);
    kc = blk + __popc(m2) - 1;
  }
  int lo = r0;
  // the bounds of the next piece are loaded while this one is walked (the
  // arrays have a spare entry past the chunk's last segment)
  int npre = (int)lds_u32(sPre + 4u * (unsigned)(kc + 1));
  QT noff = (QT)lds_off(sOff, kc, QT());
  while (lo < r1) {
    const int hi = min(npre, r1);
    const QT off = noff;
    npre = (int)lds_u32(sPre + 4u * (unsigned)(kc + 2));
    noff = (QT)lds_off(sOff, kc + 1, QT());
    const QT ql = off + (QT)lane;  // item i of the segment lives at slot ql + i - lane
    const int* __restrict__ rowl = g.col + ql;
    for (int base = lo; base < hi; base += 32 * U) {
      const int* __restrict__ pp = rowl + base;
      const int rem = hi - base - lane;
      int xx[U];
#pragma unroll
      for (int u = 0; u < U; u++) xx[u] = rem > 32 * u ? __ldg(pp + 32 * u) : xd;
#pragma unroll
      for (int u = 0; u < U; u++)
        if (base + 32 * u < hi) item(rem > 32 * u, (QT)(ql + base + 32 * u), xx[u]);
    }
    piece_end(kc);
    lo = hi;
    kc++;
  }
}

__device__ __forceinline__ unsigned warp_sum(unsigned v) { return __reduce_add_sync(0xffffffffu, v); }
__device__ __forceinline__ u64 warp_sum(u64 v) {
  for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// QT: slot index type (int when every slot index fits 31 bits: one IMAD.WIDE
// per address instead of 64-bit adds)
template <int NT, typename CT, typename QT>
__global__ void __launch_bounds__(NT, 1024 / NT)
k_c4_tiles(View g, const int64_t* __restrict__ WP, TilePlan P, int per_edge,
           CT* __restrict__ c4s, u64* __restrict__ c4tot2,
           unsigned long long* __restrict__ next_job) {
  constexpr int NW = NT / 32;
  constexpr int U = GD_TILE_U;
  constexpr int C = NT;  // segments per chunk (one per thread)
  // per-edge segment sums: below degree 2^16 a segment's sum is < dmax^2 < 2^32
  typedef typename std::conditional<std::is_same<CT, unsigned>::value, unsigned, u64>::type SumT;
  extern __shared__ __align__(16) unsigned tile[];  // T u16 counters
  __shared__ long long s_job, s_next;
  __shared__ int s_range;
  __shared__ QT seg_off[C + 1];
  __shared__ int seg_pre[C + 2];
  __shared__ SumT seg_sum[C];
  __shared__ int seg_slot[C];
  __shared__ unsigned segB[kTileIdxWords];  // indexed chunks: segment start bits per word
  __shared__ int segC[kTileIdxWords];       // indexed chunks: segments before each word
  typedef cub::BlockScan<long long, NT> BS;
  typedef cub::BlockReduce<u64, NT> BR;
  __shared__ union {
    typename BS::TempStorage scan;
    typename BR::TempStorage red;
  } tmp;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned sTile = smem_u32(tile), sB = smem_u32(segB), sC = smem_u32(segC);
  unsigned sOff = smem_u32(seg_off), sSum = smem_u32(seg_sum), sPre = smem_u32(seg_pre);
  unsigned sTileP = sTile;  // opaque copies for the piece walk: kept in registers, not rebuilt
  asm volatile("" : "+r"(sTileP), "+r"(sOff), "+r"(sSum), "+r"(sPre));
  if (threadIdx.x == 0) s_next = (long long)atomicAdd(next_job, 1ull);
  while (true) {
    __syncthreads();
    if (threadIdx.x == 0) s_job = s_next;
    __syncthreads();
    const int64_t job = s_job;
    if (job >= P.njobs) break;
    // the next job is claimed now: its latency overlaps this one
    if (threadIdx.x == 0) s_next = (long long)atomicAdd(next_job, 1ull);
    const int2 jb = P.jobs[job];
    const int fj = jb.x;
    const int s = P.frames[fj];
    const int p = jb.y & 0xffff;
    const bool last = (jb.y >> 16) != 0;  // tile holding rank s - 1: items capped at s
    const int X = P.tb[p];
    // counter width of this tile: 2^lgb bits, 2^csh counters per 32-bit word
    const int lgb = P.tlg[p], csh = 5 - lgb;
    const unsigned cmask = (1u << csh) - 1u, vmask = 0xffffffffu >> (32 - (1 << lgb));
    const int64_t b = g.rp[s], nseg = g.osplit[s] - b;
    uint4* t4 = (uint4*)tile;
    for (int i = threadIdx.x; i < P.cap16 / 8; i += NT) t4[i] = make_uint4(0u, 0u, 0u, 0u);
    // the word after the counters serves the piece walk's idle lanes: every
    // counter in it reads 1 (they add 0 to it, and a count of 1 closes no cycle)
    const int XD = X + ((P.cap16 / 2) << csh);
    if (threadIdx.x == 0) tile[P.cap16 / 2] = 0xffffffffu / vmask;
    u64 local = 0;
    for (int sweep = 0; sweep < (per_edge ? 2 : 1); sweep++) {
      for (int64_t c0 = 0; c0 < nseg; c0 += C) {
        // chunk setup: segment of thread t = lower slot q_s = b + c0 + t
        const int cnt = (int)(nseg - c0 < C ? nseg - c0 : C);
        const int64_t qs = b + c0 + threadIdx.x;
        int64_t a = 0, e = 0;
        if (threadIdx.x < cnt) {
          const int w = __ldg(g.col + qs);
          const int64_t* ts = P.TS + (int64_t)w * P.P1 + p;
          a = ts[0];
          e = ts[1];
          if (last) e = min(e, g.rp[w] + (WP[qs + 1] - WP[qs]));
        }
        const int len = e > a ? (int)(e - a) : 0;
#ifdef GD_TILE_PREFETCH
        // bulk L2 prefetch of the segment's items before the warps walk them
        // (experiment: measured 1-4 % slower at C3 and C5, so opt-in)
        if (len > 0 && sweep == 0) {
          const uintptr_t lo = (uintptr_t)(g.col + a) & ~uintptr_t(15);
          const uintptr_t hi = ((uintptr_t)(g.col + e) + 15) & ~uintptr_t(15);
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"((unsigned)(hi - lo))
                       : "memory");
        }
#endif
        // exclusive prefix of (nonempty flag, length) in one scan: nonempty
        // segments get dense indices (a step of 32 items then meets at most
        // 32 segment starts)
        long long pk, tot;
        BS(tmp.scan).ExclusiveSum(((long long)(len > 0) << 32) | len, pk, tot);
        const int pre = (int)(pk & 0xffffffffll), ci = (int)(pk >> 32);
        const int total = (int)(tot & 0xffffffffll), ncomp = (int)(tot >> 32);
        // long segments: piece walk; short ones: the per-word segment index
#ifndef GD_TILE_NOPIECES
        const bool pieces = (long long)total >= (long long)P.piece_min * ncomp;
#else
        const bool pieces = false;
#endif
#ifndef GD_TILE_NOINDEX
        const bool indexed = !pieces;
#else
        const bool indexed = false;
#endif
        if (len > 0) {
          seg_off[ci] = (QT)(a - pre);
          seg_pre[ci] = pre;
          seg_slot[ci] = (int)(c0 + threadIdx.x);
        }
        if (threadIdx.x == 0) seg_pre[ncomp] = total;
        if (sweep) seg_sum[threadIdx.x] = 0;
        // the chunk's items in windows of kTileIdxCap: each window gets its own
        // word index (segB / segC, relative to the window's first item)
        for (int v0 = 0; v0 < (indexed ? total : 1); v0 += kTileIdxCap) {
        const int vl = indexed ? min(total - v0, kTileIdxCap) : total;
        if (indexed) {
          if (v0) __syncthreads();
          for (int w = threadIdx.x; w < kTileIdxWords; w += NT) segB[w] = 0u;
          __syncthreads();
        }
        if (indexed && len > 0) {
          const int p = pre - v0, e = p + len;  // the segment's items relative to the window
          if (e >= 0 && p < vl) {
            if (p >= 0) atomicOr(&segB[p >> 5], 1u << (p & 31));
            // words w with 32w in (p, e]: ci + 1 segments begin before item 32w
            const int wmax = min(e >> 5, (vl - 1) >> 5);
            for (int w = p < 0 ? 0 : (p >> 5) + 1; w <= wmax; w++) segC[w] = ci + 1;
          }
        }
        if (threadIdx.x == 0) {
          s_range = v0;
          if (v0 == 0) segC[0] = 0;
        }
        __syncthreads();
        const unsigned sBw = sB - (((unsigned)v0 >> 5) << 2), sCw = sC - (((unsigned)v0 >> 5) << 2);
        // item ranges claimed dynamically: long segments spread over warps
        // GD_TILE_CLAIMS ranges per warp on average (each claim costs a
        // shared atomic and a segment search)
        const int R = max(64, ((vl / (GD_TILE_CLAIMS * NW)) + 31) & ~31);
        while (true) {
          int r0 = 0;
          if (lane == 0) r0 = atomicAdd(&s_range, R);
          r0 = __shfl_sync(0xffffffffu, r0, 0);
          if (r0 >= v0 + vl) break;
          const int r1 = min(v0 + vl, r0 + R);
          if (sweep == 0 && pieces) {
            tile_items_pieces<GD_TILE_PU, QT>(g, sPre, sOff, ncomp, r0, r1, XD, [&](bool valid, QT, int x) {
              const unsigned xr = (unsigned)(x - X);
              reds_add(sTileP + ((xr >> csh) << 2), (valid ? 1u : 0u) << ((xr & cmask) << lgb));
            }, [](int) {});
          } else if (pieces) {
            SumT acc = 0;
            tile_items_pieces<GD_TILE_PU, QT>(g, sPre, sOff, ncomp, r0, r1, XD, [&](bool, QT q, int x) {
              const unsigned xr = (unsigned)(x - X);
              const unsigned cnt = (lds_u32(sTileP + ((xr >> csh) << 2)) >> ((xr & cmask) << lgb)) & vmask;
              const SumT c = (SumT)(cnt - 1u);  // 0 on idle lanes (the spare word)
              red_add_nz(&c4s[q], (CT)c);  // edge w-x
              acc += c;
            }, [&](int k) {
              const SumT sm = warp_sum(acc);
              if (sm && lane == 0) reds_add(sSum + (unsigned)sizeof(SumT) * (unsigned)k, sm);
              acc = 0;
            });
          } else if (sweep == 0 && indexed) {
            // invalid lanes add 0 to word 0: no branch around the atomic
            tile_items_indexed<U, QT>(g, sBw, sCw, sOff, r0, r1, [&](bool valid, int, QT, int x) {
              const unsigned xr = valid ? (unsigned)(x - X) : 0u;
              reds_add(sTileP + ((xr >> csh) << 2), (valid ? 1u : 0u) << ((xr & cmask) << lgb));
            });
          } else if (sweep == 0) {
            tile_range_items<U>(g, seg_pre, seg_off, ncomp, r0, r1,
                                [&](int k, QT, int x, unsigned) {
                                  if (k >= 0) {
                                    const unsigned xr = (unsigned)(x - X);
                                    atomicAdd(&tile[xr >> csh], 1u << ((xr & cmask) << lgb));
                                  }
                                });
          } else if (indexed) {
            int cur_k = -1;
            SumT cur = 0;
            tile_items_indexed<U, QT>(g, sBw, sCw, sOff, r0, r1, [&](bool valid, int k, QT q, int x) {
              const unsigned xr = valid ? (unsigned)(x - X) : 0u;
              const unsigned cnt = (lds_u32(sTileP + ((xr >> csh) << 2)) >> ((xr & cmask) << lgb)) & vmask;
              const SumT c = valid ? (SumT)(cnt - 1u) : (SumT)0;
              if (c) red_add(&c4s[q], (CT)c);  // edge w-x
              if (k != cur_k) {
                if (cur) reds_add(sSum + (unsigned)sizeof(SumT) * (unsigned)cur_k, cur);
                cur_k = k;
                cur = 0;
              }
              cur += c;
            });
            if (cur) reds_add(sSum + (unsigned)sizeof(SumT) * (unsigned)cur_k, cur);
          } else {
#ifndef GD_TILE_RUNSCAN
            // per-lane running sum of its current segment, flushed to the
            // segment's shared slot sum when the lane moves on (lanes of a
            // long segment flush once per segment; no cross-lane scan)
            int cur_k = -1;
            SumT cur = 0;
            tile_range_items<U>(g, seg_pre, seg_off, ncomp, r0, r1,
                                [&](int k, QT q, int x, unsigned) {
              if (k < 0) return;
              const unsigned xr = (unsigned)(x - X);
              const SumT c = (SumT)(((tile[xr >> csh] >> ((xr & cmask) << lgb)) & vmask) - 1u);
              if (c) red_add(&c4s[q], (CT)c);  // edge w-x
              if (k != cur_k) {
                if (cur) atomicAdd(&seg_sum[cur_k], cur);
                cur_k = k;
                cur = 0;
              }
              cur += c;
            });
            if (cur) atomicAdd(&seg_sum[cur_k], cur);
#else
            tile_range_items<U>(g, seg_pre, seg_off, ncomp, r0, r1,
                                [&](int k, QT q, int x, unsigned M) {
              SumT c = 0;
              if (k >= 0) {
                const unsigned xr = (unsigned)(x - X);
                c = (SumT)(((tile[xr >> csh] >> ((xr & cmask) << lgb)) & vmask) - 1u);
                if (c) red_add(&c4s[q], (CT)c);  // edge w-x
              }
              // per-run sums of the step (runs of one segment end where the
              // next lane starts a segment): inclusive warp scan, minus the
              // scan value just before the run; the run's last lane adds it
              SumT incl = c;
#pragma unroll
              for (int off = 1; off < 32; off <<= 1) {
                const SumT v = __shfl_up_sync(0xffffffffu, incl, off);
                if (lane >= off) incl += v;
              }
              const unsigned start = M & (0xffffffffu >> (31 - lane));  // run start <= lane
              const int rs = start ? 31 - __clz(start) : 0;
              const SumT before = __shfl_sync(0xffffffffu, incl, rs > 0 ? rs - 1 : 0);
              const SumT run = incl - (rs > 0 ? before : (SumT)0);
              const int kn = __shfl_down_sync(0xffffffffu, k, 1);
              const bool end = lane == 31 || ((M >> (lane + 1)) & 1u) || kn != k;
              if (k >= 0 && end && run) atomicAdd(&seg_sum[k], run);
            });
#endif
          }
        }
        }  // windows
        __syncthreads();
        if (sweep && threadIdx.x < ncomp) {
          const SumT sm = seg_sum[threadIdx.x];
          if (sm) {
            red_add(&c4s[b + seg_slot[threadIdx.x]], (CT)sm);  // edge s-w
            local += (u64)sm;
          }
        }
      }
    }
    if (!per_edge) {  // 2*C(c,2) over the tile's counters
      const int bits = 1 << lgb;
      for (int i = threadIdx.x; i < P.cap16 / 8; i += NT) {
        const uint4 w4 = t4[i];
        const unsigned wv[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
        for (int t = 0; t < 4; t++) {
          if (!wv[t]) continue;
          for (int k = 0; k < 32; k += bits) {
            const u64 c = (wv[t] >> k) & vmask;
            local += c * (c - (c > 0));
          }
        }
      }
    }
    __syncthreads();
    const u64 sum = BR(tmp.red).Sum(local);
    if (threadIdx.x == 0 && sum) atomic_add_u128(c4tot2 + 2 * graph_of(g, s), sum);
  }
}

// ------------------------------------------------------------------------
// per-vertex S(x) = sum of neighbour degrees (warp per row)
// ------------------------------------------------------------------------
__global__ void k_vertex_s(View g, u64* __restrict__ vS) {
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < g.n; r += warps) {
    u64 sd = 0;
    for (int64_t q = g.rp[r] + lane_id(); q < g.rp[r + 1]; q += 32)
      sd += (u64)g.deg[g.col[q]];
    for (int off = 16; off; off >>= 1) sd += __shfl_xor_sync(0xffffffffu, sd, off);
    if (lane_id() == 0) vS[r] = sd;
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
  const int64_t* e2o;
  const int64_t* e2i;
  const u64* tcs;
  const void* tsl;  // null in global mode
  const void* tsh;
  const void* tsd;
  const void* c4s;
  bool narrow;      // per-slot sums held as u32 (max degree < 65536)
  const u64* vT;
  const u64* vS;
  const uint4* vrec;  // [n][2] by dense id: {rank, degree, T lo, T hi} {S lo, S hi, -, -}
};

// Per-vertex record of the finalize, indexed by DENSE id: one 32-byte sector
// per endpoint instead of four scattered gathers (d2r, deg, T, S).
__global__ void k_vertex_records(int64_t n, const int32_t* __restrict__ d2r,
                                 const int32_t* __restrict__ deg, const u64* __restrict__ vT,
                                 const u64* __restrict__ vS, uint4* __restrict__ vrec) {
  const int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (d >= n) return;
  const int r = d2r[d];
  const u64 T = vT[r], S = vS[r];
  vrec[2 * d] = make_uint4((unsigned)r, (unsigned)deg[r], (unsigned)T, (unsigned)(T >> 32));
  vrec[2 * d + 1] = make_uint4((unsigned)S, (unsigned)(S >> 32), 0u, 0u);
}

__device__ __forceinline__ long long slot_val(const void* p, int64_t q, bool narrow) {
  return narrow ? (long long)((const unsigned*)p)[q] : (long long)((const u64*)p)[q];
}

// per-edge contribution to the 13 CensusSums (census.py:449-462)
__device__ __forceinline__ void add_sums(u128* acc, long long t, long long su, long long sv,
                                         long long cl, long long cy, long long n, long long m) {
  const long long i3 = n - 2 - t - su - sv;
  acc[0] += (u128)t;
  acc[1] += (u128)(su + sv);
  acc[2] += (u128)i3;
  acc[3] += (u128)cl;
  acc[4] += (u128)cy;
  acc[5] += (u128)((u64)t * (u64)(t - 1) / 2);
  acc[6] += (u128)((u64)su * (u64)sv);
  acc[7] += (u128)((u64)t * (u64)(su + sv));
  acc[8] += (u128)((u64)su * (u64)(su - 1) / 2 + (u64)sv * (u64)(sv - 1) / 2);
  acc[9] += (u128)((u64)t * (u64)i3);
  acc[10] += (u128)((u64)(su + sv) * (u64)i3);
  acc[11] += (u128)((u64)i3 * (u64)(i3 - 1) / 2);
  acc[12] += (u128)(m + 1 - (t + su + 1) - (t + sv + 1));
}

// The 10 raw per-edge fields of edge e (RAW_MICRO_FIELDS order).
__device__ __forceinline__ void edge_row(const EdgeIn& in, int64_t e, long long* row) {
  const int64_t du_ = in.eu[e], dv_ = in.ev[e];
  const uint4 ua = __ldg(in.vrec + 2 * du_), ub = __ldg(in.vrec + 2 * du_ + 1);
  const uint4 va = __ldg(in.vrec + 2 * dv_), vb = __ldg(in.vrec + 2 * dv_ + 1);
  const int ru = (int)ua.x, rv = (int)va.x;
  const int64_t qo = in.e2o[e];
  const u64 pk = in.tcs[qo];
  const long long t = (long long)(pk >> kTriShift);
  const long long cl = (long long)(pk & kClMask);
  const long long du = (long long)ua.y, dv = (long long)va.y;
  const long long su = du - 1 - t, sv = dv - 1 - t;
  row[0] = t;
  row[1] = su;
  row[2] = sv;
  row[3] = cl;
  if (!in.tsl) return;
  // out-slot sums are by rank side: lo = lower-rank endpoint
  const long long slo = slot_val(in.tsl, qo, in.narrow), shi = slot_val(in.tsh, qo, in.narrow);
  const long long sumU = ru < rv ? slo : shi, sumV = ru < rv ? shi : slo;
  const long long tdeg = slot_val(in.tsd, qo, in.narrow);
  const long long tsu = sumU - 2 * cl - t, tsv = sumV - 2 * cl - t, ts = tsu + tsv;
  const long long Tu = (long long)(((u64)ua.w << 32) | ua.z), Tv = (long long)(((u64)va.w << 32) | va.z);
  const long long Su = (long long)(((u64)ub.y << 32) | ub.x), Sv = (long long)(((u64)vb.y << 32) | vb.x);
  const long long uu = Tu - t - cl - tsu;
  const long long vv = Tv - t - cl - tsv;
  const long long c4 = slot_val(in.c4s, qo, in.narrow) + slot_val(in.c4s, in.e2i[e], in.narrow);
  const long long cy = c4 - ts - 2 * cl;
  const long long sdeg = Su - dv + Sv - du - 2 * tdeg;
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
__device__ void block_flush_sums(u128* acc, u64* out) {
  // reduce 13 u128 accumulators across the block as 3 x 43-bit limbs (limb
  // sums cannot overflow 64 bits) and add with carry
  typedef cub::BlockReduce<u64, NT> BR;
  __shared__ typename BR::TempStorage tmp;
  const u64 mask = (1ull << 43) - 1;
#pragma unroll  // static indices keep the 13 accumulators in registers (208 B of stack otherwise)
  for (int k = 0; k < kNumSums; k++) {
    const u64 l0 = (u64)(acc[k]) & mask;
    const u64 l1 = (u64)(acc[k] >> 43) & mask;
    const u64 l2 = (u64)(acc[k] >> 86);
    const u64 s0 = BR(tmp).Sum(l0);
    __syncthreads();
    const u64 s1 = BR(tmp).Sum(l1);
    __syncthreads();
    const u64 s2 = BR(tmp).Sum(l2);
    __syncthreads();
    if (threadIdx.x == 0) {
      const u128 v = (u128)s0 + ((u128)s1 << 43) + ((u128)s2 << 86);
      atomic_add_u128(out + 2 * k, v);
    }
  }
}

__device__ __forceinline__ void store_row(long long* __restrict__ table, int64_t e,
                                          const long long* row) {
  long long* out = table + (size_t)e * kNumMicro;
#pragma unroll
  for (int c = 0; c < kNumMicro; c += 2) {
    longlong2 v;
    v.x = row[c];
    v.y = row[c + 1];
    *(longlong2*)(out + c) = v;
  }
}

// G == 1: grid-stride over the edges [e0, e1); row e is written at table
// row e - e0 (a rank's shard of the table in a multi-GPU census)
template <int NT>
__global__ void __launch_bounds__(NT)
k_finalize_single(EdgeIn in, int64_t e0, int64_t e1, long long n, long long m,
                  long long* __restrict__ table, u64* __restrict__ sums, u64* __restrict__ seen) {
  u128 acc[kNumSums];
#pragma unroll
  for (int k = 0; k < kNumSums; k++) acc[k] = 0;
  u64 cnt = 0;
  long long row[kNumMicro];
  for (int64_t e = e0 + blockIdx.x * (int64_t)NT + threadIdx.x; e < e1;
       e += (int64_t)gridDim.x * NT) {
    edge_row(in, e, row);
    add_sums(acc, row[0], row[1], row[2], row[3], in.tsl ? row[4] : 0, n, m);
    cnt++;
    if (table) store_row(table, e - e0, row);
  }
  block_flush_sums<NT>(acc, sums);
  typedef cub::BlockReduce<u64, NT> BR;
  __shared__ typename BR::TempStorage tmp2;
  const u64 c = BR(tmp2).Sum(cnt);
  if (threadIdx.x == 0 && c) atomicAdd(seen, c);
}

// ---- small graphs: the reference's marks protocol, one kernel ------------
// Graphs (or batches of graphs) whose adjacency fits in shared memory are
// counted by a direct restatement of _micro_edge (census.py:190-256) on the
// device: the CTA stages its graph's CSR in local dense ids, each warp takes
// edges and keeps a private n-byte marks array (1 = N(u) only, 2 = Tri,
// 3 = N(v) only), and the ten per-edge fields and 13 sums come out of one
// launch -- no schedule, no passes, no host round trips (config 1: 10,000
// edges; config 4: 4,096 graphs, one CTA each).
struct SmallIn {
  const int64_t* rp;    // rank CSR
  const int32_t* col;
  const int32_t* eu;    // canonical edges (dense ids)
  const int32_t* ev;
  const int32_t* d2r;
  const int32_t* r2d;
  const int64_t* voff;  // [G+1] dense vertex offset of each graph (batch)
  const int64_t* eoff;  // [G+1] canonical edge offset of each graph (batch)
  int64_t n1, m1;       // one graph: vertex and edge count
};

// 2-bit marks, private to one thread, laid out word-major / lane-minor so the
// 32 lanes of a warp always hit 32 different banks
struct LaneMarks {
  unsigned* w;  // word i of this thread at w[i * NT]
  int stride;
  __device__ __forceinline__ unsigned get(int x) const {
    return (w[(x >> 4) * stride] >> ((x & 15) << 1)) & 3u;
  }
  __device__ __forceinline__ void set(int x, unsigned v) const {
    unsigned* p = w + (x >> 4) * stride;
    const int sh = (x & 15) << 1;
    *p = (*p & ~(3u << sh)) | (v << sh);
  }
};

// Adjacency of a small-graph census: rank-space rows in global memory (one
// graph) or local dense rows staged in shared memory (a batch, whose
// graphs' vertices are scattered over the rank space).
struct GlobalRows {
  const int64_t* rp;
  const int32_t* col;
  __device__ __forceinline__ int deg(int x) const { return (int)(rp[x + 1] - rp[x]); }
  __device__ __forceinline__ const int32_t* row(int x) const { return col + rp[x]; }
};
struct SharedRows {
  const int* off;
  const int* adj;
  __device__ __forceinline__ int deg(int x) const { return off[x + 1] - off[x]; }
  __device__ __forceinline__ const int* row(int x) const { return adj + off[x]; }
};

template <int NT, bool BATCH, bool STAGE>
__global__ void __launch_bounds__(NT)
k_small_census(SmallIn in, int G, int words, long long* __restrict__ table,
               u64* __restrict__ sums, u64* __restrict__ seen) {
  extern __shared__ __align__(16) int sm_i[];
  const int gi = BATCH ? blockIdx.x : 0;
  const int64_t v0 = BATCH ? in.voff[gi] : 0, e0 = BATCH ? in.eoff[gi] : 0;
  const int64_t e1 = BATCH ? in.eoff[gi + 1] : in.m1;
  const int nv = (int)(BATCH ? in.voff[gi + 1] - v0 : in.n1);
  unsigned* marks = (unsigned*)sm_i;  // [words][NT]
  for (int i = threadIdx.x; i < words * NT; i += NT) marks[i] = 0u;
  typename std::conditional<BATCH || STAGE, SharedRows, GlobalRows>::type R;
  if constexpr (BATCH) {
    // stage the graph in local dense ids: degrees, offsets (block scan),
    // rows (thread per vertex, its row converted rank -> local dense)
    int* off = (int*)(marks + (size_t)words * NT);  // [nv + 1]
    int* adj = off + nv + 1;                        // [2 m_g]
    typedef cub::BlockScan<int, NT> BS;
    __shared__ typename BS::TempStorage scan_tmp;
    const int per = (nv + NT - 1) / NT;
    int local = 0;
    int64_t rb[8];
    for (int i = 0; i < per && i < 8; i++) {
      const int d = threadIdx.x * per + i;
      if (d < nv) {
        const int r = in.d2r[v0 + d];
        rb[i] = in.rp[r];
        local += (int)(in.rp[r + 1] - rb[i]);
      }
    }
    for (int i = 8; i < per; i++) {
      const int d = threadIdx.x * per + i;
      if (d < nv) {
        const int r = in.d2r[v0 + d];
        local += (int)(in.rp[r + 1] - in.rp[r]);
      }
    }
    int base;
    BS(scan_tmp).ExclusiveSum(local, base);
    for (int i = 0; i < per; i++) {
      const int d = threadIdx.x * per + i;
      if (d >= nv) break;
      int64_t b;
      int dd;
      if (i < 8) {
        b = rb[i];
        dd = (int)(in.rp[in.d2r[v0 + d] + 1] - b);
      } else {
        const int r = in.d2r[v0 + d];
        b = in.rp[r];
        dd = (int)(in.rp[r + 1] - b);
      }
      off[d] = base;
      for (int j = 0; j < dd; j++) adj[base + j] = in.r2d[in.col[b + j]] - (int)v0;
      base += dd;
    }
    if (threadIdx.x == NT - 1) off[nv] = base;
    R.off = off;
    R.adj = adj;
  } else if constexpr (STAGE) {
    // one graph that fits: its rank CSR copied as is (coalesced) -- every
    // later access is a shared-memory load
    int* off = (int*)(marks + (size_t)words * NT);  // [n + 1]
    int* adj = off + nv + 1;                        // [2 m]
    for (int i = threadIdx.x; i <= nv; i += NT) off[i] = (int)in.rp[i];
    const int two_m = (int)(2 * (e1 - e0));
    for (int i = threadIdx.x; i < two_m; i += NT) adj[i] = in.col[i];
    R.off = off;
    R.adj = adj;
  } else {
    R.rp = in.rp;
    R.col = in.col;
  }
  __syncthreads();
  // --- the marks protocol, one edge per thread: _micro_edge (census.py:
  // 190-256) for the per-edge table, _count_edge (259-303: d(lo) <= d(hi),
  // half the sweeps) for the global census.  Vertex labels: local dense ids
  // (batch) or rank ids (one graph); the w < y tests only need some fixed
  // total order to count each edge once.  The graph is small (n <= 8192), so
  // per-edge counts fit 32 bits and the 13 sums of a CTA fit 64 bits.
  const LaneMarks mk{marks + threadIdx.x, NT};
  const long long n = nv, m = e1 - e0;
  u64 acc[kNumSums];
  for (int k = 0; k < kNumSums; k++) acc[k] = 0;
  u64 cnt = 0;
  const int64_t first = e0 + (BATCH ? 0 : (int64_t)blockIdx.x * NT) + threadIdx.x;
  const int64_t step = BATCH ? NT : (int64_t)gridDim.x * NT;
  for (int64_t e = first; e < e1; e += step) {
    int u = BATCH ? in.eu[e] - (int)v0 : in.d2r[in.eu[e]];
    int v = BATCH ? in.ev[e] - (int)v0 : in.d2r[in.ev[e]];
    const bool flip = !table && R.deg(u) > R.deg(v);  // _count_edge orientation
    if (flip) {
      const int x = u;
      u = v;
      v = x;
    }
    const auto* au = R.row(u);
    const auto* av = R.row(v);
    const int du = R.deg(u), dv = R.deg(v);
    for (int i = 0; i < du; i++) mk.set(au[i], 1);
    mk.set(v, 0);
    int t = 0, su = 0, sv = 0;
    for (int i = 0; i < dv; i++) {
      const int w = av[i];
      if (mk.get(w) == 1) {
        mk.set(w, 2);
        t++;
      } else if (w != u) {
        mk.set(w, 3);
        sv++;
      }
    }
    for (int i = 0; i < du; i++) su += mk.get(au[i]) == 1;
    int cl = 0, ts = 0, tdeg = 0, cy = 0, uu = 0, vv = 0, sdeg = 0;
    for (int i = 0; i < dv; i++) {  // Tri sweep (census.py:215-225 / 286-291)
      const int w = av[i];
      if (mk.get(w) != 2) continue;
      const auto* aw = R.row(w);
      const int dw = R.deg(w);
      tdeg += dw;
      for (int k = 0; k < dw; k++) {
        const int y = aw[k];
        const unsigned mr = mk.get(y);
        if (mr == 2) cl += w < y;
        else if (mr) ts++;
      }
    }
    for (int i = 0; i < du; i++) {  // Star_u sweep (census.py:227-236 / 292-299)
      const int w = au[i];
      if (mk.get(w) != 1) continue;
      const auto* aw = R.row(w);
      const int dw = R.deg(w);
      sdeg += dw;
      for (int k = 0; k < dw; k++) {
        const int y = aw[k];
        const unsigned mr = mk.get(y);
        if (mr == 3) cy++;
        else if (mr == 1 && w < y) uu++;
      }
    }
    if (table) {
      for (int i = 0; i < dv; i++) {  // Star_v sweep (census.py:238-244)
        const int w = av[i];
        if (mk.get(w) != 3) continue;
        const auto* aw = R.row(w);
        const int dw = R.deg(w);
        sdeg += dw;
        for (int k = 0; k < dw; k++) {
          const int y = aw[k];
          vv += mk.get(y) == 3 && w < y;
        }
      }
    }
    for (int i = 0; i < du; i++) mk.set(au[i], 0);  // census.py:252-255
    for (int i = 0; i < dv; i++) mk.set(av[i], 0);
    if (flip) {  // back to the canonical (u, v) sides
      const int x = su;
      su = sv;
      sv = x;
    }
    // _census_batch (census.py:449-462) in 64 bits (small graph)
    const u64 i3 = (u64)(n - 2 - t - su - sv);
    acc[0] += t;
    acc[1] += su + sv;
    acc[2] += i3;
    acc[3] += cl;
    acc[4] += cy;
    acc[5] += (u64)t * (t - 1) / 2;
    acc[6] += (u64)su * sv;
    acc[7] += (u64)t * (su + sv);
    acc[8] += (u64)su * (su - 1) / 2 + (u64)sv * (sv - 1) / 2;
    acc[9] += (u64)t * i3;
    acc[10] += (u64)(su + sv) * i3;
    acc[11] += i3 * (i3 - 1) / 2;
    acc[12] += (u64)(m + 1 - (t + su + 1) - (t + sv + 1));
    cnt++;
    if (table) {
      const long long ti = (long long)tdeg - 2 * t - 2 * cl - ts;                      // 246-247
      const long long si = (long long)sdeg - su - sv - ts - 2 * (uu + vv) - 2 * cy;  // 248-250
      const long long row[kNumMicro] = {t, su, sv, cl, cy, uu, vv, ts, ti, si};
      store_row(table, e, row);
    }
  }
  typedef cub::BlockReduce<u64, NT> BR;
  __shared__ typename BR::TempStorage tmp2;
  u64* out = sums + (size_t)gi * 2 * kNumSums;
  for (int k = 0; k < kNumSums; k++) {
    const u64 v = BR(tmp2).Sum(acc[k]);
    if (threadIdx.x == 0 && v) atomic_add_u128(out + 2 * k, (u128)v);
    __syncthreads();
  }
  const u64 c = BR(tmp2).Sum(cnt);
  if (threadIdx.x == 0 && c) atomicAdd(seen + gi, c);
}

// ---- multi-GPU ownership (gd_count.cuh: Shard) ----------------------------
// per-edge partials of passes B and C in rank-major blocks [W][4][M]: the
// block of rank r holds the 4 fields of its owned edges [r*M, (r+1)*M)
template <typename ST>
__global__ void k_pack_edge_partials(int64_t m, int64_t M, const int64_t* __restrict__ e2o,
                                     const int64_t* __restrict__ e2i, const ST* __restrict__ tsl,
                                     const ST* __restrict__ tsh, const ST* __restrict__ tsd,
                                     const ST* __restrict__ c4s, ST* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / M, i = e - r * M, q = e2o[e];
    ST* b = out + r * 4 * M;
    b[i] = tsl[q];
    b[M + i] = tsh[q];
    b[2 * M + i] = tsd[q];
    b[3 * M + i] = c4s[q] + c4s[e2i[e]];
  }
}

// an owner's reduced block back into the slot-indexed arrays the finalize reads
template <typename ST>
__global__ void k_unpack_owned(int64_t e0, int64_t e1, int64_t M, const int64_t* __restrict__ e2o,
                               const int64_t* __restrict__ e2i, const ST* __restrict__ in,
                               ST* __restrict__ tsl, ST* __restrict__ tsh, ST* __restrict__ tsd,
                               ST* __restrict__ c4s) {
  for (int64_t e = e0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < e1;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e - e0, q = e2o[e];
    tsl[q] = in[i];
    tsh[q] = in[M + i];
    tsd[q] = in[2 * M + i];
    c4s[q] = in[3 * M + i];
    c4s[e2i[e]] = 0;
  }
}

// pass-A counters: slot-indexed (out-slots only) <-> edge-indexed
__global__ void k_gather_edges(int64_t m, const int64_t* __restrict__ e2o,
                               const u64* __restrict__ slots, u64* __restrict__ edges) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x)
    edges[e] = slots[e2o[e]];
}

__global__ void k_scatter_edges(int64_t m, const int64_t* __restrict__ e2o,
                                const u64* __restrict__ edges, u64* __restrict__ slots) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x)
    slots[e2o[e]] = edges[e];
}

// 128-bit sums and edge counts of every rank (all-gathered) added exactly
__global__ void k_sum_shards(const u64* __restrict__ gsums, const u64* __restrict__ gseen, int W,
                             u64* __restrict__ sums, u64* __restrict__ seen) {
  const int k = threadIdx.x;
  if (k < kNumSums) {
    u128 t = 0;
    for (int r = 0; r < W; r++) {
      const u64* p = gsums + (size_t)r * 2 * kNumSums + 2 * k;
      t += ((u128)p[1] << 64) | p[0];
    }
    sums[2 * k] = (u64)t;
    sums[2 * k + 1] = (u64)(t >> 64);
  }
  if (k == 0) {
    u64 c = 0;
    for (int r = 0; r < W; r++) c += gseen[r];
    *seen = c;
  }
}

// G > 1: one CTA per graph
template <int NT>
__global__ void __launch_bounds__(NT)
k_finalize_batch(EdgeIn in, const int64_t* __restrict__ eoff, const int64_t* __restrict__ gn,
                 long long* __restrict__ table, u64* __restrict__ sums, u64* __restrict__ seen) {
  const int gi = blockIdx.x;
  const int64_t e0 = eoff[gi], e1 = eoff[gi + 1];
  const long long n = gn[gi], m = e1 - e0;
  u128 acc[kNumSums];
  for (int k = 0; k < kNumSums; k++) acc[k] = 0;
  u64 cnt = 0;
  long long row[kNumMicro];
  for (int64_t e = e0 + threadIdx.x; e < e1; e += NT) {
    edge_row(in, e, row);
    add_sums(acc, row[0], row[1], row[2], row[3], in.tsl ? row[4] : 0, n, m);
    cnt++;
    if (table) store_row(table, e, row);
  }
  block_flush_sums<NT>(acc, sums + (size_t)gi * 2 * kNumSums);
  typedef cub::BlockReduce<u64, NT> BR;
  __shared__ typename BR::TempStorage tmp2;
  const u64 c = BR(tmp2).Sum(cnt);
  if (threadIdx.x == 0) seen[gi] = c;
}

// dual route: sums from a given per-edge table (frequencies_from_micro)
template <int NT>
__global__ void __launch_bounds__(NT)
k_sums_from_table(const long long* __restrict__ table, int64_t m, long long n,
                  u64* __restrict__ sums) {
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
  v.osplit = g.osplit.p;
  v.e2o = g.e2o.p;
  v.seid = g.seid.p;
  v.deg = g.deg.p;
  v.vgraph = g.G > 1 ? g.vgraph.p : nullptr;
  return v;
}

int grid_cap(int64_t work, int threads, int per_sm = 16) {
  int64_t gsz = (work + threads - 1) / threads;
  const int64_t cap = (int64_t)num_sms() * per_sm;
  if (gsz > cap) gsz = cap;
  if (gsz < 1) gsz = 1;
  return (int)gsz;
}

void exclusive_scan(const int64_t* in, int64_t* out, int64_t n, cudaStream_t s) {
  size_t tb = 0;
  GD_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n, s));
  DBuf<char> tmp;
  tmp.alloc(tb, s);
  GD_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, in, out, n, s));
}

void sort_frames(u64* keys, int* ids, int64_t n, DBuf<int>& sorted_ids,
                 DBuf<u64>& sorted_keys, cudaStream_t s) {
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

// Bin boundaries of a descending key order without copying the keys: the
// keys are stored complemented (ascending); for each threshold t the number
// of frames with value >= t.
__global__ void k_count_ge(const u64* __restrict__ stored, int64_t n,
                           const u64* __restrict__ thr, int nthr, int64_t* __restrict__ out) {
  const int t = threadIdx.x;
  if (t >= nthr) return;
  const u64 key = ~thr[t];
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (stored[mid] <= key) lo = mid + 1; else hi = mid;
  }
  out[t] = lo;
}

struct DevKeys {
  const u64* stored = nullptr;  // complemented values, ascending
  int64_t n = 0;
  int shift = 0;                // value = key >> shift
  cudaStream_t s = 0;
  // [begin, end) of the frames with lo <= value >> shift <= hi, for all bins at once
  std::vector<std::pair<int64_t, int64_t>> ranges(
      const std::vector<std::pair<int64_t, int64_t>>& bins) const {
    std::vector<u64> thr;
    for (auto& b : bins) {
      thr.push_back((u64)b.first << shift);
      thr.push_back(b.second >= (INT64_MAX >> shift) ? ~0ull : (u64)(b.second + 1) << shift);
    }
    std::vector<int64_t> cnt(thr.size(), 0);
    if (n && !thr.empty()) {
      DBuf<u64> dthr;
      DBuf<int64_t> dcnt;
      dthr.alloc(thr.size(), s);
      dcnt.alloc(thr.size(), s);
      GD_CUDA(cudaMemcpyAsync(dthr.p, thr.data(), thr.size() * 8, cudaMemcpyHostToDevice, s));
      k_count_ge<<<1, 64, 0, s>>>(stored, n, dthr.p, (int)thr.size(), dcnt.p);
      GD_LAUNCH_CHECK("count_ge");
      GD_CUDA(cudaMemcpyAsync(cnt.data(), dcnt.p, cnt.size() * 8, cudaMemcpyDeviceToHost, s));
      GD_CUDA(cudaStreamSynchronize(s));
    }
    std::vector<std::pair<int64_t, int64_t>> out;
    for (size_t i = 0; i < bins.size(); i++) {
      const int64_t b = thr[2 * i + 1] == ~0ull ? 0 : cnt[2 * i + 1];
      out.push_back({b, std::max(b, cnt[2 * i])});
    }
    return out;
  }
  // raw keys (values << shift | flags) of frames [a, b)
  std::vector<u64> keys(int64_t a, int64_t b) const {
    std::vector<u64> h(std::max<int64_t>(0, b - a));
    if (!h.empty()) {
      GD_CUDA(cudaMemcpyAsync(h.data(), stored + a, h.size() * 8, cudaMemcpyDeviceToHost, s));
      GD_CUDA(cudaStreamSynchronize(s));
    }
    for (auto& x : h) x = ~x;
    return h;
  }
  int64_t value(int64_t i) const { return i < n ? (int64_t)(keys(i, i + 1)[0] >> shift) : 0; }
};


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

// Opt in to the dynamic shared memory a launch needs (static shared memory
// counts against the same 48 KB default, so always set it).  The attribute
// is process-wide per kernel while censuses may run on several host threads
// at once, so it only ever grows (under a lock): a launch never sees a
// smaller limit set by a concurrent census of a smaller graph.
template <typename K>
void set_smem(K kernel, size_t bytes) {
  static std::mutex mu;
  static std::map<const void*, size_t> cur;
  std::lock_guard<std::mutex> lock(mu);
  size_t& c = cur[(const void*)kernel];
  if (bytes <= c) return;
  GD_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)bytes));
  c = bytes;
}

// Test-only schedule overrides (GD_FORCE_PATH=tri_gmem,c4_coop,...): route
// every frame through one kernel variant so each variant can be checked
// against the oracle on small graphs.  Results never depend on the path.
struct ForcePaths {
  bool any = false;
  bool tri_gmem = false, tri_small = false, tri_blocks = false, c4_smem = false,
       c4_coop = false, c4_hub32 = false, c4_flow = false, c4_cluster = false,
       c4_tile64 = false;
};

ForcePaths read_force() {
  ForcePaths f;
  const char* e = getenv("GD_FORCE_PATH");
  if (!e) return f;
  const std::string v(e);
  f.any = !v.empty();
  f.tri_gmem = v.find("tri_gmem") != std::string::npos;
  f.tri_small = v.find("tri_small") != std::string::npos;
  f.tri_blocks = v.find("tri_blocks") != std::string::npos;
  f.c4_smem = v.find("c4_smem") != std::string::npos;
  f.c4_coop = v.find("c4_coop") != std::string::npos;
  f.c4_hub32 = v.find("c4_hub32") != std::string::npos;
  // heavy-frame schedulers on any graph size: cluster path off, two frames
  // per round (many rounds, every slab set reused)
  f.c4_flow = v.find("c4_flow") != std::string::npos;
  // heavy frames on the (older) DSMEM cluster kernel, or on x-tiles of 64
  // counters (every frame cut into many tiles)
  f.c4_cluster = v.find("c4_cluster") != std::string::npos;
  f.c4_tile64 = v.find("c4_tile64") != std::string::npos;
  return f;
}

int64_t env_int(const char* name, int64_t dflt) {
  const char* e = getenv(name);
  return e ? std::atoll(e) : dflt;
}

}  // namespace

// ---------------------------------------------------------------------------
// Host orchestration
// ---------------------------------------------------------------------------
void run_census(DevGraph& g, bool per_edge, long long* table_dev, unsigned long long* sums_dev,
                unsigned long long* seen_dev, CensusExtras& ex, cudaStream_t s, const Shard& sh) {
  const ForcePaths force = read_force();
  // shards executed by this process: its own (multi-GPU) or all (emulated)
  const int world = std::max(1, sh.world);
  std::vector<int> my_ranks;
  if (sh.real()) my_ranks.push_back(sh.rank);
  else for (int r = 0; r < world; r++) my_ranks.push_back(r);
  const long long launches0 = g_launches;
  const int64_t n = g.n, m = g.m, G = g.G, S = 2 * m;
  const View v = make_view(g);
  Timer timer(s);
  ex.k4tot.assign(G, 0);
  ex.c4tot2.assign(G, 0);
  ex.stats.clear();
  ex.stats_names.clear();
  auto stat = [&](const char* name, int64_t val) {
    ex.stats.push_back(val);
    ex.stats_names.push_back(name);
  };

  // ---- small graphs: one direct kernel (k_small_census) --------------------
  if (m > 0 && world == 1 && !force.any && env_int("GD_SMALL", 1) != 0) {
    std::vector<int64_t> voff(G + 1, 0), eoff(G + 1, 0);
    if (G == 1) {
      voff[1] = n;
      eoff[1] = m;
    } else {
      for (int64_t i = 0; i < G; i++) voff[i + 1] = voff[i] + g.h_gn[i];
      eoff = g.h_eoff;
    }
    int64_t nmax = 0, stage = 0;
    for (int64_t i = 0; i < G; i++) {
      const int64_t nv = voff[i + 1] - voff[i], mg = eoff[i + 1] - eoff[i];
      nmax = std::max(nmax, nv);
      stage = std::max(stage, 4 * (nv + 1) + 8 * mg);
    }
    // one thread per edge with 2-bit marks over the graph's vertices: the
    // graph must be small (counts then fit 32 bits) and fit shared memory
    const int NT = G > 1 ? 256 : 128;
    const int64_t words = (nmax + 15) / 16;
    // one graph: its CSR is staged too when it fits beside the marks
    const bool stage_one = G == 1 && 4 * words * NT + stage <= env_int("GD_SMALL_SMEM", 160 * 1024);
    const int64_t smem = 4 * words * NT + (G > 1 || stage_one ? stage : 0);
    const int64_t limit = env_int("GD_SMALL_SMEM", 160 * 1024);
    // (64-bit sums per CTA: m_g * C(n_g, 2) < 2^64 for n_g <= 8192)
    if (nmax <= 8192 && smem <= limit) {
      DBuf<int64_t> dvo;
      SmallIn in{g.rp.p, g.col.p, g.eu.p, g.ev.p, g.d2r.p, g.r2d.p, nullptr, nullptr, n, m};
      if (G > 1) {
        dvo.alloc(G + 1, s);
        GD_CUDA(cudaMemcpyAsync(dvo.p, voff.data(), (G + 1) * 8, cudaMemcpyHostToDevice, s));
        in.voff = dvo.p;
        in.eoff = g.eoff.p;
      }
      GD_CUDA(cudaMemsetAsync(sums_dev, 0, (size_t)G * 2 * kNumSums * 8, s));
      GD_CUDA(cudaMemsetAsync(seen_dev, 0, (size_t)G * 8, s));
#define GD_SMALL_LAUNCH(NTV, BATCH, STAGE)                                                    \
  {                                                                                           \
    auto kern = k_small_census<NTV, BATCH, STAGE>;                                            \
    set_smem(kern, (size_t)smem);                                                             \
    int occ = 1;                                                                              \
    GD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NTV, (size_t)smem));    \
    const int64_t grid = G > 1 ? G : std::min<int64_t>((m + NTV - 1) / NTV,                   \
                                                       (int64_t)std::max(occ, 1) * num_sms()); \
    kern<<<(int)grid, NTV, (size_t)smem, s>>>(in, (int)G, (int)words, table_dev, sums_dev,    \
                                              seen_dev);                                      \
  }
      if (G > 1) GD_SMALL_LAUNCH(256, true, false)
      else if (stage_one) GD_SMALL_LAUNCH(128, false, true)
      else GD_SMALL_LAUNCH(128, false, false)
#undef GD_SMALL_LAUNCH
      GD_LAUNCH_CHECK("small_census");
      timer.mark("small");
      timer.collect(ex.ms, ex.names);
      stat("small_graph_path", 1);
      stat("launches", g_launches - launches0);
      stat("shards", 1);
      ex.direct = true;
      return;
    }
  }

  // slot-indexed accumulators (workspace buffers, zeroed per call)
  struct WBuf { u64* p; };
  auto wz = [&](const char* name, size_t count) {
    u64* q = ws_get<u64>(g, name, count, s);
    if (count) GD_CUDA(cudaMemsetAsync(q, 0, count * 8, s));
    return WBuf{q};
  };
  WBuf tcs = wz("tcs", S), vT = wz("vT", n), k4tot = wz("k4tot", 2 * G),
       c4tot2 = wz("c4tot2", 2 * G);
  WBuf vS{ws_get<u64>(g, "vS", n, s)};
  // per-slot pass-B sums and 4-cycle partials: u32 when the maximum degree
  // is below 2^16 (every partial of slot q is bounded by a quantity of its
  // edge e = (u, v): C4(e) <= (d(u)-1)(d(v)-1), sum_{w in Tri_e} t(lo, w) and
  // sum d(w) <= (dmax-1) dmax < 2^32), halving the sectors of their coalesced
  // atomics; u64 otherwise and for real shards (64-bit NCCL sums)
  const bool narrow = per_edge && g.max_deg < 65536 &&
                      env_int("GD_WIDE_SLOTS", 0) == 0;
  const size_t slot_words = narrow ? (S + 1) / 2 : S;
  WBuf tsl{nullptr}, tsh{nullptr}, tsd{nullptr}, c4s{nullptr};
  if (per_edge) {
    tsl = wz("tsl", slot_words);
    tsh = wz("tsh", slot_words);
    tsd = wz("tsd", slot_words);
    c4s = wz("c4s", slot_words);
  }
  stat("narrow_slots", narrow ? 1 : 0);

  // ---- schedule: item prefixes and frame orders ---------------------------
  struct IBuf { int64_t* p; };
  IBuf oitems{ws_get<int64_t>(g, "oitems", S + 1, s)}, witems{ws_get<int64_t>(g, "witems", S + 1, s)};
  IBuf OP{ws_get<int64_t>(g, "OP", S + 1, s)}, WP{ws_get<int64_t>(g, "WP", S + 1, s)};
  DBuf<u64> tkey, wkey, tkey_s, wkey_s;
  DBuf<int> ida, idb, tri_frames, c4_frames;
  tkey.alloc(n, s);
  wkey.alloc(n, s);
  ida.alloc(n, s);
  idb.alloc(n, s);
  GD_CUDA(cudaMemsetAsync(oitems.p + S, 0, 8, s));
  GD_CUDA(cudaMemsetAsync(witems.p + S, 0, 8, s));
  if (S) {
    k_slot_items<<<(unsigned)((S + 255) / 256), 256, 0, s>>>(v, S, oitems.p, witems.p);
    GD_LAUNCH_CHECK("slot_items");
  }
  exclusive_scan(oitems.p, OP.p, S + 1, s);
  exclusive_scan(witems.p, WP.p, S + 1, s);
  if (n) {
    k_frame_keys<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(v, WP.p, tkey.p, wkey.p, ida.p, idb.p);
    GD_LAUNCH_CHECK("frame_keys");
  }
  int64_t tot_items = 0;
  if (S) GD_CUDA(cudaMemcpyAsync(&tot_items, OP.p + S, 8, cudaMemcpyDeviceToHost, s));
  DevKeys dk, wk;
  if (n) {
    sort_frames(tkey.p, ida.p, n, tri_frames, tkey_s, s);
    sort_frames(wkey.p, idb.p, n, c4_frames, wkey_s, s);
    dk = DevKeys{tkey_s.p, n, 0, s};
    wk = DevKeys{wkey_s.p, n, 1, s};
  }
  timer.mark("schedule");

  // ---- pass A / pass B: triangle frames by D = |N+(a)| ----------------------
  const int64_t maxD = n ? dk.value(0) : 0;
  // graph-wide hit buffer (per-edge mode): exact-size lists for pass B.
  // Capacity = min(sum_a min(items_a, C(D_a, 2)) -- cached per graph --, 60% of
  // the memory this census can get: device free memory, the unused reserve
  // of the stream-ordered pool and this thread's cached hit buffer).  The
  // buffer is kept in the per-thread workspace (a fresh 76 GB stream-ordered
  // allocation per census measured 0.4-0.8 s slower at config 5 once graph
  // builds and tables interleave with it; gd_trim_workspace releases it).
  // If the allocation fails -- e.g. concurrent censuses on several host
  // threads -- the capacity is halved, and at worst pass B re-probes every
  // frame (hit_cap = 0): slower, never wrong.
  const bool lists = env_int("GD_TRI_LISTS", 1) != 0;
  DBuf<u64> hitbuf_mem;
  u64* hitbuf = nullptr;
  u64* hittop = nullptr;
  int64_t* hoff = nullptr;
  int* hcnt = nullptr;
  u64 hit_cap = 0;
  if (per_edge && lists && n) {
    if (!g.hit_cap_known) {
      DBuf<u64> bound;
      bound.alloc(1, s);
      bound.zero();
      k_hit_bound<<<grid_cap(n, 256), 256, 0, s>>>(v, OP.p, bound.p);
      GD_LAUNCH_CHECK("hit_bound");
      u64 hb = 0;
      GD_CUDA(cudaMemcpyAsync(&hb, bound.p, 8, cudaMemcpyDeviceToHost, s));
      GD_CUDA(cudaStreamSynchronize(s));
      g.hit_cap = hb;
      g.hit_cap_known = true;
    }
    const auto it = thread_workspace().find("hitbuf");
    const u64 mine = it != thread_workspace().end() ? (u64)it->second.bytes : 0;
    if (env_int("GD_HIT_CAP", 0) == 0 && (mine >= g.hit_cap * 8 ||
                                           (g.hit_cap_used && mine >= g.hit_cap_used * 8))) {
      // this thread's cached buffer already holds every list of this graph
      // (or what its last census got): no memory queries inside the pipeline
      hit_cap = mine >= g.hit_cap * 8 ? g.hit_cap : g.hit_cap_used;
    } else {
      size_t fr = 0, tot = 0;
      GD_CUDA(cudaMemGetInfo(&fr, &tot));
      u64 spare = 0;
      int dev = 0;
      cudaMemPool_t pool;
      uint64_t res = 0, used = 0;
      if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess &&
          cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &res) == cudaSuccess &&
          cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used) == cudaSuccess &&
          res > used)
        spare = res - used;
      hit_cap = std::min<u64>(g.hit_cap, (u64)((fr + spare + mine) * 0.6) / 8);
      hit_cap = std::min<u64>(hit_cap, (u64)env_int("GD_HIT_CAP", INT64_MAX));  // tests
    }
    const bool cached = env_int("GD_HIT_WS", 1) != 0;
    while (hit_cap) {
      if (cached) {
        try {
          hitbuf = ws_get<u64>(g, "hitbuf", hit_cap, s);
          break;
        } catch (const Error&) {
          cudaGetLastError();
          thread_workspace().erase("hitbuf");
        }
      } else {
        void* p = nullptr;
        if (cudaMallocAsync(&p, hit_cap * 8, s) == cudaSuccess) {
          hitbuf_mem.p = (u64*)p;
          hitbuf_mem.n = hit_cap;
          hitbuf_mem.s = s;
          hitbuf = hitbuf_mem.p;
          break;
        }
        cudaGetLastError();  // out of memory: try half, then fall back to probing
      }
      hit_cap = hit_cap > (1u << 20) ? hit_cap / 2 : 0;
    }
    g.hit_cap_used = cached ? hit_cap : 0;
    if (hit_cap) {
      hittop = ws_get<u64>(g, "hittop", 1, s);
      GD_CUDA(cudaMemsetAsync(hittop, 0, 8, s));
      hoff = ws_get<int64_t>(g, "hoff", n, s);
      hcnt = ws_get<int>(g, "hcnt", n, s);
      GD_CUDA(cudaMemsetAsync(hcnt, 0xff, n * sizeof(int), s));  // -1: not persisted
    }
    stat("hit_buffer_entries", (int64_t)hit_cap);
  }
  // one claim counter per frame-kernel launch (frames are claimed dynamically)
  constexpr int kMaxClaims = 4096;
  DBuf<unsigned> claims;
  claims.alloc(kMaxClaims, s);
  claims.zero();
  int nclaims = 0;
  auto run_frames = [&](bool trisum) {
    struct B { int64_t lo, hi; int nt; bool gmem; };
    std::vector<B> bins = {{1025, INT64_MAX, 512, true}, {513, 1024, 512, false},
                           {129, 512, 256, false}, {33, 128, 128, false}, {2, 32, 32, false}};
    if (env_int("GD_TRI_SPLIT", 1) == 1)
      bins = {{1025, INT64_MAX, (int)env_int("GD_TRI_GM_NT", 1024), true},
              {513, 1024, (int)env_int("GD_TRI_B1024_NT", 1024), false},
              {257, 512, (int)env_int("GD_TRI_B512_NT", 512), false},
              {129, 256, (int)env_int("GD_TRI_B256_NT", 256), false}, {65, 128, 128, false}, {33, 64, 128, false},
              {2, 32, 32, false}};
    if (env_int("GD_TRI_SPLIT", 1) == 2)
      bins = {{1025, INT64_MAX, 512, true}, {513, 1024, 512, false},
              {257, 512, (int)env_int("GD_TRI_B512_NT", 256), false},
              {129, 256, 128, false}, {33, 128, 128, false}, {2, 32, 32, false}};
    int64_t stage_max = 1 << 20;
    if (force.tri_gmem) bins = {{2, INT64_MAX, 512, true}};
    if (force.tri_small) bins = {{2, INT64_MAX, 32, false}}, stage_max = 16;
    std::vector<std::pair<int64_t, int64_t>> bq;
    for (const B& bn : bins) bq.push_back({bn.lo, bn.hi});
    const auto brs = dk.ranges(bq);
    for (size_t bi = 0; bi < bins.size(); bi++) {
      B bn = bins[bi];
      const auto r = brs[bi];
      const int64_t nf = r.second - r.first;
      if (nf <= 0) continue;
      const int cap = (int)std::min<int64_t>(bn.hi, maxD);
      FrameLayout L = make_layout(cap, !trisum, trisum);
      // pass B keeps no bitmap rows: its largest frames fit shared memory;
      // pass A splits the bitmap rows of big frames into column blocks
      // (column blocking of pass A measured slower than global-memory rows at
      // config 5: 309 vs 176 ms, so it is opt-in: GD_TRI_BLOCKED=1)
      if (bn.gmem && !force.tri_gmem && (trisum || env_int("GD_TRI_BLOCKED", 1))) {
        const int W = (cap + 63) / 64;
        for (int nb = 1; nb <= W; nb++) {
          FrameLayout t = make_layout(cap, !trisum, trisum, (W + nb - 1) / nb);
          if (t.bytes <= 200 * 1024) {
            L = t;
            bn.gmem = false;
            break;
          }
        }
      }
      if (force.tri_blocks && !trisum) L = make_layout(cap, true, false, 1);
      const bool blocked = !trisum && L.wb < (cap + 63) / 64;
      const bool acc32 = (int64_t)cap * g.max_deg < (int64_t)UINT32_MAX;
      const int* fr = tri_frames.p + r.first;
      const int64_t per_rank = (nf + world - 1) / world;
      const size_t sm = bn.gmem ? 0 : L.bytes;
      // persistent grid: the resident CTAs (each owns a staging list)
      int occ = 1;
#define GD_OCC(NTV)                                                                         \
  {                                                                                          \
    if (!trisum) {                                                                           \
      set_smem(k_tri_frames<NTV, false, false>, sm);                                         \
      set_smem(k_tri_frames<NTV, true, false>, sm);                                          \
      GD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tri_frames<NTV, false, false>, NTV, sm)); \
    } else {                                                                                 \
      set_smem(k_trisum_frames<NTV, false, unsigned, u64>, sm);                              \
      set_smem(k_trisum_frames<NTV, false, u64, u64>, sm);                                   \
      set_smem(k_trisum_frames<NTV, false, unsigned, unsigned>, sm);                         \
      set_smem(k_trisum_frames<NTV, false, u64, unsigned>, sm);                              \
      GD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_trisum_frames<NTV, false, u64, u64>, NTV, sm)); \
    }                                                                                        \
  }
      switch (bn.nt) {
        case 1024: GD_OCC(1024) break;
        case 512: GD_OCC(512) break;
        case 256: GD_OCC(256) break;
        case 128: GD_OCC(128) break;
        default: GD_OCC(32) break;
      }
#undef GD_OCC
      occ = std::max(occ, 1);
      int grid = (int)std::min<int64_t>(per_rank, (int64_t)num_sms() * occ);
      if (bn.gmem) grid = (int)std::min<int64_t>(per_rank, 2 * num_sms());
      DBuf<char> slab;
      if (bn.gmem) slab.alloc((size_t)grid * L.bytes, s);
      char* sp = bn.gmem ? slab.p : nullptr;
      HitLists HL{};
      if (lists) {
        const int64_t c2 = (int64_t)cap * (cap - 1) / 2;
        HL.stage_cap = (int)std::max<int64_t>(1, std::min<int64_t>(c2, stage_max));
        if (!trisum) HL.stage = ws_get<u64>(g, "stage", (size_t)grid * HL.stage_cap, s);
        HL.buf = hit_cap ? hitbuf : nullptr;
        HL.top = hittop;
        HL.cap = hit_cap;
        HL.hoff = hit_cap ? hoff : nullptr;
        HL.hcnt = hit_cap ? hcnt : nullptr;
      }
      for (const int rk : my_ranks) {
      // claim counter of this launch (a slot of a zeroed per-census array)
      if (nclaims >= kMaxClaims) throw Error(GD_EINVAL, "too many frame launches in one census");
      unsigned* claim = claims.p + nclaims++;
#define GD_TRISUM_LAUNCH(NTV, ST)                                                            \
  {                                                                                          \
    ST* ql = (ST*)tsl.p;                                                                     \
    ST* qh = (ST*)tsh.p;                                                                     \
    ST* qd = (ST*)tsd.p;                                                                     \
    if (sp)                                                                                  \
      k_trisum_frames<NTV, true, u64, ST><<<grid, NTV, sm, s>>>(v, fr, (int)nf, rk, world, L, \
                                                                sp, OP.p, tcs.p, ql, qh, qd, HL, claim); \
    else if (acc32)                                                                          \
      k_trisum_frames<NTV, false, unsigned, ST><<<grid, NTV, sm, s>>>(                        \
          v, fr, (int)nf, rk, world, L, sp, OP.p, tcs.p, ql, qh, qd, HL, claim);             \
    else                                                                                     \
      k_trisum_frames<NTV, false, u64, ST><<<grid, NTV, sm, s>>>(                             \
          v, fr, (int)nf, rk, world, L, sp, OP.p, tcs.p, ql, qh, qd, HL, claim);             \
  }
#define GD_TRI_LAUNCH(NTV)                                                                   \
  if (!trisum && blocked) {                                                                  \
    if (sp)                                                                                  \
      k_tri_frames<NTV, true, true><<<grid, NTV, sm, s>>>(v, fr, (int)nf, rk, world, L, sp,   \
                                                          OP.p, tcs.p, vT.p, k4tot.p, HL, claim); \
    else                                                                                     \
      k_tri_frames<NTV, true, false><<<grid, NTV, sm, s>>>(v, fr, (int)nf, rk, world, L, sp,  \
                                                           OP.p, tcs.p, vT.p, k4tot.p, HL, claim); \
    GD_LAUNCH_CHECK("tri_frames_blocked");                                                   \
  } else if (!trisum) {                                                                      \
    if (sp)                                                                                  \
      k_tri_frames<NTV, false, true><<<grid, NTV, sm, s>>>(v, fr, (int)nf, rk, world, L, sp,  \
                                                           OP.p, tcs.p, vT.p, k4tot.p, HL, claim); \
    else                                                                                     \
      k_tri_frames<NTV, false, false><<<grid, NTV, sm, s>>>(v, fr, (int)nf, rk, world, L, sp, \
                                                            OP.p, tcs.p, vT.p, k4tot.p, HL, claim); \
    GD_LAUNCH_CHECK("tri_frames");                                                           \
  } else {                                                                                   \
    if (narrow)                                                                              \
      GD_TRISUM_LAUNCH(NTV, unsigned)                                                        \
    else                                                                                     \
      GD_TRISUM_LAUNCH(NTV, u64)                                                             \
    GD_LAUNCH_CHECK("trisum_frames");                                                        \
  }
      switch (bn.nt) {
        case 1024: GD_TRI_LAUNCH(1024) break;
        case 512: GD_TRI_LAUNCH(512) break;
        case 256: GD_TRI_LAUNCH(256) break;
        case 128: GD_TRI_LAUNCH(128) break;
        default: GD_TRI_LAUNCH(32) break;
      }
      }
#undef GD_TRI_LAUNCH
#undef GD_TRISUM_LAUNCH
    }
  };
  run_frames(false);
  timer.mark("tri_frames");
  // multi-GPU ownership (gd_count.cuh): G == 1 graphs split their rows
  const bool owned = (world > 1 || sh.real()) && G == 1 && m > 0;
  if (owned) {  // t / cl of every edge and T(x): all ranks need them in pass B
    u64* tce = ws_get<u64>(g, "tce", (size_t)m, s);
    k_gather_edges<<<grid_cap(m, 256), 256, 0, s>>>(m, g.e2o.p, tcs.p, tce);
    GD_LAUNCH_CHECK("gather_edges");
    if (sh.real()) {
      sh.allreduce(tce, (size_t)m);
      sh.allreduce(vT.p, (size_t)n);
    }
    k_scatter_edges<<<grid_cap(m, 256), 256, 0, s>>>(m, g.e2o.p, tce, tcs.p);
    GD_LAUNCH_CHECK("scatter_edges");
    timer.mark("allreduce_a");
  } else if (sh.real()) {  // batches: every slot of every shard
    sh.allreduce(tcs.p, (size_t)S);
    sh.allreduce(vT.p, (size_t)n);
    timer.mark("allreduce_a");
  }
  if (n) {
    k_vertex_s<<<grid_cap(n * 32, 256), 256, 0, s>>>(v, vS.p);
    GD_LAUNCH_CHECK("vertex_s");
  }
  if (per_edge) {
    run_frames(true);
    timer.mark("trisum_frames");
  }

  // ---- pass C: wedges ---------------------------------------------------------
  // Bins by wedges W: [1, 256] smem hash (u32), (256, 4096] smem hash (u32),
  // (4096, 24576] smem hash 32K entries (u16 counts), above: cooperative rounds
  // with L2-resident u16 slabs; frames whose counters could exceed 16 bits
  // (lower degree >= 65536) take the u32 hub path.
  int64_t total_w = 0;
  if (S) {
    GD_CUDA(cudaMemcpyAsync(&total_w, WP.p + S, 8, cudaMemcpyDeviceToHost, s));
    GD_CUDA(cudaStreamSynchronize(s));
  }
  stat("wedges", total_w);
  stat("tri_items", tot_items);
  int64_t t0 = 256, ta = 1024, t1 = 4096, tb = 12288, t2 = 24576;
  t2 = env_int("GD_C4_HEAVY_MIN", 12288);  // frames above t2 wedges take the heavy-frame path
  tb = std::min(tb, t2), t1 = std::min(t1, t2), ta = std::min(ta, t2), t0 = std::min(t0, t2);
  if (force.c4_coop || force.c4_hub32 || force.c4_flow) t0 = ta = t1 = tb = t2 = 0;
  if (force.c4_smem) t0 = ta = t1 = 0;  // every frame <= t2 through the u16 hashes
  const auto wr = wk.ranges({{1, t0}, {t0 + 1, ta}, {ta + 1, t1}, {t1 + 1, tb}, {tb + 1, t2},
                             {t2 + 1, INT64_MAX}});
  const auto rs0 = wr[0], rsa = wr[1], rs1 = wr[2], rsb = wr[3], rs2 = wr[4], rh = wr[5];
  const int pe = per_edge ? 1 : 0;
  u64* c4s_p = per_edge ? c4s.p : nullptr;
  const int64_t nh = rh.second - rh.first;
  int64_t n32 = 0, nrounds = 0, heavy_w = 0;
  bool tiles_used = false;
  if (nh > 0) {
    std::vector<int> hf(nh);
    GD_CUDA(cudaMemcpyAsync(hf.data(), c4_frames.p + rh.first, nh * 4, cudaMemcpyDeviceToHost, s));
    const std::vector<u64> hkeys = wk.keys(rh.first, rh.second);  // (W << 1) | big
    GD_CUDA(cudaStreamSynchronize(s));
    std::vector<int> f16_all, f32_all;
    std::vector<int64_t> w16_all, h16, h32;
    for (int64_t h = 0; h < nh; h++) {
      if ((hkeys[h] & 1) || force.c4_hub32) {
        f32_all.push_back(hf[h]);
        h32.push_back(h);
      } else {
        f16_all.push_back(hf[h]);
        w16_all.push_back((int64_t)(hkeys[h] >> 1));
        h16.push_back(h);
        heavy_w += (int64_t)(hkeys[h] >> 1);
      }
    }
    n32 = (int64_t)f32_all.size();
    // counters cover ranks [x0, n): isolated vertices (the lowest ranks)
    // never end a wedge
    int x0 = 0;
    int drank[5] = {0, 0, 0, 0, 0};  // first rank with degree > 0, 1, 3, 15, 255
    if (!f16_all.empty()) {
      int* d0 = ws_get<int>(g, "x0", 5, s);
      k_degree_ranks<<<1, 32, 0, s>>>(v, d0);
      GD_LAUNCH_CHECK("degree_ranks");
      GD_CUDA(cudaMemcpyAsync(drank, d0, 20, cudaMemcpyDeviceToHost, s));
      GD_CUDA(cudaStreamSynchronize(s));
      x0 = drank[0] & ~1;
    }
    // x-tiles in shared memory for every heavy frame (the dense-slab flow
    // kernel and the DSMEM cluster kernel stay selectable: GD_C4_TILES=0,
    // GD_FORCE_PATH=c4_flow / c4_cluster).  Measured: C3 per-edge 48.3 (flow)
    // -> 34.8 ms, C3 global 30.1 -> 18.6, C5 global 320 -> 236, C5 per-edge
    // 474 -> 470 ms (its ~22-item row pieces make the use sweep the costly half)
    const int64_t tile_mode = env_int("GD_C4_TILES", 1);
    const bool use_tiles = !force.c4_flow && !force.c4_cluster && tile_mode != 0;
    tiles_used = use_tiles && !f16_all.empty();
    for (const int rk : my_ranks) {
    // this shard's frames: every world-th heavy frame in descending-work order
    std::vector<int> f16, f32;
    std::vector<int64_t> w16;
    for (size_t i = 0; i < f16_all.size(); i++)
      if ((int)(h16[i] % world) == rk) {
        f16.push_back(f16_all[i]);
        w16.push_back(w16_all[i]);
      }
    for (size_t i = 0; i < f32_all.size(); i++)
      if ((int)(h32[i] % world) == rk) f32.push_back(f32_all[i]);
    // dense counters in cluster shared memory when n fits in <= 4 CTAs (wider
    // clusters measured slower than the L2 rounds: hot counters serialise
    // on one SM's shared memory and only 7 16-CTA clusters are resident)
    int csize = 0, per = 0;
    if (force.c4_cluster || (env_int("GD_C4_CLUSTER", 1) && !force.c4_flow && !use_tiles)) {
      const int64_t max_per = 98304;  // u16 counters per CTA (192 KB)
      const int cmax = (int)env_int("GD_C4_CLUSTER_MAX", 4);
      for (int c = 1; c <= cmax; c *= 2) {
        const int64_t p = (((n + c - 1) / c) + 7) & ~int64_t(7);
        if (p <= max_per) {
          csize = c;
          per = (int)p;
          break;
        }
      }
    }
    if (!f16.empty() && use_tiles) {
      constexpr int NT = GD_TILE_NT;
      // tile: the dynamic shared memory one CTA (1024 threads) or two (512
      // each) per SM can hold beside the kernel's static arrays
      const int T = force.c4_tile64 ? 64 : (int)(env_int("GD_C4_TILE", NT == 1024 ? 90112 : 45056) &
                                                 ~int64_t(7));
      // degree-aware tiles (TileRuns): from x0 upward, the counter width whose
      // tile reaches farthest; GD_C4_TILE_BITS=16 keeps uniform 16-bit tiles
      const int min_bits = (int)env_int("GD_C4_TILE_BITS", 2);
      TileRuns RN;
      for (int c = 0; c < 4; c++) RN.R[c] = INT_MAX, RN.T[c] = 1, RN.I[c] = 0;
      std::vector<int> tb, tlg;
      {
        const int64_t lim[4] = {drank[2], drank[3], drank[4], n};  // b = 2, 4, 8, 16
        // a wedge ending at a degree-1 vertex closes no 4-cycle (its counter
        // stays 1): the tiles start at the first rank of degree 2
        int64_t X = env_int("GD_C4_TILE_LEAVES", 0) ? x0 : drank[1];
        int run = -1, run_lg = 0;
        while (X < n) {
          int64_t best = -1;
          int best_lg = 4;
          for (int lg = 1; lg <= 4; lg++) {
            if ((1 << lg) < min_bits) continue;
            const int64_t end = std::min<int64_t>(X + (int64_t)T * (16 >> lg), lim[lg - 1]);
            if (end > best) best = end, best_lg = lg;
          }
          if (run < 0 || best_lg != run_lg) {
            run++;
            run_lg = best_lg;
            RN.R[run] = (int)X;
            RN.T[run] = T * (16 >> best_lg);
            RN.I[run] = (int)tb.size();
          }
          tb.push_back((int)X);
          tlg.push_back(best_lg);
          X = best;
        }
        tb.push_back((int)n);
      }
      const int64_t ptot = (int64_t)tlg.size();
      const int P1 = (int)ptot + 1;
      stat("c4_tile_count", ptot);
      int64_t* TS = ws_get<int64_t>(g, "c4_ts", (size_t)n * P1, s);
      {
        const int64_t wm = std::min<int64_t>(drank[4], n);  // first rank of degree >= 256
        const int64_t wz = std::min<int64_t>(drank[0], wm);  // isolated vertices: rows never read
        if (wm > wz)
          k_tile_splits<8><<<grid_cap((wm - wz) * 8, 256), 256, 0, s>>>(v, RN, P1, TS, wz, wm);
        if (n > wm) {
          const int nseg = (int)std::min<int64_t>(65535, (g.max_deg + kSplitSeg - 1) / kSplitSeg);
          const dim3 grid2(grid_cap((n - wm) * 32, 256), std::max(nseg, 1));
          k_tile_splits<32><<<grid2, 256, 0, s>>>(v, RN, P1, TS, wm, n);
        }
      }
      GD_LAUNCH_CHECK("tile_splits");
      std::vector<int64_t> jpre(f16.size() + 1, 0);
      for (size_t j = 0; j < f16.size(); j++)
        jpre[j + 1] = jpre[j] + (f16[j] - 1 < RN.R[0] ? 0 : (int64_t)(RN.tile_of(f16[j] - 1) + 1));
      std::vector<int> jframe(jpre.back());
      for (size_t j = 0; j < f16.size(); j++)
        std::fill(jframe.begin() + jpre[j], jframe.begin() + jpre[j + 1], (int)j);
      // Job order: tile-major, highest tile first.  The jobs in flight at any
      // time then read the same x-range of the lower rows -- col[] entries of
      // one tile, 1/4 (C3) to 1/13 (C5) of the array, which stays in L2 -- where
      // the frame-major order walked whole rows of unrelated frames (at C5
      // every col[] entry came from DRAM: 689 GB per census).  Within a tile
      // the frames keep their descending-work order.
      if (ptot >= 65536) throw Error(GD_EINVAL, "too many pass-C tiles");
      const int64_t job_order = env_int("GD_C4_JOB_ORDER", 1);
      std::vector<int2> jobs;
      jobs.reserve(jpre.back());
      if (job_order == 0) {
        for (size_t j = 0; j < f16.size(); j++)
          for (int64_t q = jpre[j]; q < jpre[j + 1]; q++)
            jobs.push_back(make_int2((int)j, (int)(q - jpre[j]) | (q + 1 == jpre[j + 1] ? 1 << 16 : 0)));
      } else {
        for (int64_t pp = 0; pp < ptot; pp++) {
          const int64_t tp = job_order == 1 ? ptot - 1 - pp : pp;
          for (size_t j = 0; j < f16.size(); j++) {
            const int64_t nt = jpre[j + 1] - jpre[j];
            if (nt > tp) jobs.push_back(make_int2((int)j, (int)tp | (tp + 1 == nt ? 1 << 16 : 0)));
          }
        }
      }
      DBuf<int2> djobs;
      djobs.alloc(jobs.size(), s);
      GD_CUDA(cudaMemcpyAsync(djobs.p, jobs.data(), jobs.size() * sizeof(int2), cudaMemcpyHostToDevice, s));
      DBuf<int> dfr, djf, dtb, dtl;
      DBuf<int64_t> djp;
      DBuf<unsigned long long> njob;
      dfr.alloc(f16.size(), s);
      djp.alloc(jpre.size(), s);
      djf.alloc(jframe.size(), s);
      dtb.alloc(tb.size(), s);
      dtl.alloc(tlg.size(), s);
      njob.alloc(1, s);
      njob.zero();
      GD_CUDA(cudaMemcpyAsync(dfr.p, f16.data(), f16.size() * 4, cudaMemcpyHostToDevice, s));
      GD_CUDA(cudaMemcpyAsync(djp.p, jpre.data(), jpre.size() * 8, cudaMemcpyHostToDevice, s));
      GD_CUDA(cudaMemcpyAsync(djf.p, jframe.data(), jframe.size() * 4, cudaMemcpyHostToDevice, s));
      GD_CUDA(cudaMemcpyAsync(dtb.p, tb.data(), tb.size() * 4, cudaMemcpyHostToDevice, s));
      GD_CUDA(cudaMemcpyAsync(dtl.p, tlg.data(), tlg.size() * 4, cudaMemcpyHostToDevice, s));
      TilePlan TP{dfr.p, djp.p, djf.p, (int)f16.size(), jpre.back(), T, P1, TS, dtb.p, dtl.p,
                  (int)std::max<int64_t>(1, env_int("GD_C4_PIECE_MIN", GD_TILE_PIECE_MIN)), djobs.p};
      const size_t sm = (size_t)T * 2 + 16;  // + the spare word of the piece walk
      // 32-bit slot indices when every slot fits 31 bits
      const bool idx32 = S < ((int64_t)1 << 31) && env_int("GD_TILE_IDX32", 1) != 0;
      auto tk = idx32 ? k_c4_tiles<NT, u64, int> : k_c4_tiles<NT, u64, long long>;
      auto tk32 = idx32 ? k_c4_tiles<NT, unsigned, int> : k_c4_tiles<NT, unsigned, long long>;
      set_smem(tk, sm);
      set_smem(tk32, sm);
      int occ = 0;
      GD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tk, NT, sm));
      if (occ < 1) throw Error(GD_ECUDA, "c4 tile kernel cannot be resident");
      const int grid = (int)std::min<int64_t>(jpre.back(), (int64_t)occ * num_sms());
      if (grid < 1) {  // every wedge of these frames ends at a leaf: nothing to count
      } else if (narrow)
        tk32<<<grid, NT, sm, s>>>(v, WP.p, TP, pe, (unsigned*)c4s_p, c4tot2.p, njob.p);
      else
        tk<<<grid, NT, sm, s>>>(v, WP.p, TP, pe, c4s_p, c4tot2.p, njob.p);
      GD_LAUNCH_CHECK("c4_tiles");
      nrounds += jpre.back();  // reported: tile jobs
    } else if (!f16.empty() && csize) {
      constexpr int NT = 512;
      const size_t sm = (size_t)per * 2;
      auto kern = k_c4_cluster<NT, u64>;
      auto kern32 = k_c4_cluster<NT, unsigned>;
      set_smem(kern, sm);
      set_smem(kern32, sm);
      if (csize > 8) {
        GD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        GD_CUDA(cudaFuncSetAttribute(kern32, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      }
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = csize;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.blockDim = dim3(NT);
      cfg.dynamicSmemBytes = sm;
      cfg.stream = s;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      cfg.gridDim = dim3(csize);
      int nclusters = 0;
      GD_CUDA(cudaOccupancyMaxActiveClusters(&nclusters, (void*)kern, &cfg));
      if (nclusters < 1) throw Error(GD_ECUDA, "cluster kernel cannot be resident");
      cfg.gridDim = dim3(nclusters * csize);
      DBuf<int> dfr, queue;
      // this shard's own frames (f16), walked as shard 0 of 1
      dfr.alloc(f16.size(), s);
      queue.alloc(1, s);
      queue.zero();
      GD_CUDA(cudaMemcpyAsync(dfr.p, f16.data(), f16.size() * 4, cudaMemcpyHostToDevice, s));
      if (narrow)
        GD_CUDA(cudaLaunchKernelEx(&cfg, kern32, v, (const int64_t*)WP.p, (const int*)dfr.p,
                                   (int)f16.size(), 0, 1, queue.p, per, pe,
                                   (unsigned*)c4s_p, c4tot2.p));
      else
        GD_CUDA(cudaLaunchKernelEx(&cfg, kern, v, (const int64_t*)WP.p, (const int*)dfr.p,
                                   (int)f16.size(), 0, 1, queue.p, per, pe, c4s_p,
                                   c4tot2.p));
      GD_LAUNCH_CHECK("c4_cluster");
      nrounds = -csize;  // reported as the cluster size
    } else if (!f16.empty()) {
      constexpr int NT = 512;
      int per_sm = 0;
      // 4 CTAs/SM (32 registers) and 2 items per lane in flight: measured
      // 72.6 ms vs 87.6 (3 CTAs, 1 item) on config 3; the use sweep's
      // dependent counter reads are latency-bound
      auto fk = k_c4_flow<NT, GD_FLOW_MINB, GD_FLOW_U, GD_FLOW_UU, u64>;
      auto fk32 = k_c4_flow<NT, GD_FLOW_MINB, GD_FLOW_U, GD_FLOW_UU, unsigned>;
      const int fnt = NT;
      GD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fk, fnt, 0));
      if (per_sm < 1) throw Error(GD_ECUDA, "c4 flow kernel cannot be resident");
      const int grid = per_sm * num_sms();
      const int64_t slab_words = ((((int64_t)n - x0) + 1) / 2 + 31) & ~int64_t(31);
      const int64_t l2_budget = env_int("GD_C4_FLOW_MB", 640) << 20;  // all slab sets
      // a round's use (or scan) tasks are handed out LU steps after its count
      // tasks and its zeroing one step later; a count task waits for the
      // zeroing of the set it reuses, NS rounds back
      const int LU = (int)std::max<int64_t>(1, env_int("GD_C4_ULAG", 1));
      const int NS = (int)std::max<int64_t>(LU + 2, env_int("GD_C4_SETS", 4));
      const int F = force.c4_flow ? 2 : (int)std::max<int64_t>(
          1, std::min<int64_t>(256, l2_budget / (NS * slab_words * 4)));
      const int64_t pieces = force.c4_flow ? 8 : 16384;  // uint4 per fill / scan task
      const int64_t per_slab = (slab_words / 4 + pieces - 1) / pieces;
      const int64_t min_ch = force.c4_flow ? 1 : env_int("GD_C4_MIN_CHUNK", 8192);
      // chunk = a round's wedges / (4 x grid), in [8192, 262144]: each task
      // boundary costs a CTA barrier, a block reduction and a dependency
      // check, while too few tasks per round leave CTAs idle at the round's
      // tail (measured max 65536 -> 262144 and 2 -> 4 tasks per CTA: C5
      // per-edge flow 599 -> 493 ms, C3 51.3 -> 49.3 ms)
      const int64_t max_ch = std::max(min_ch, env_int("GD_C4_MAX_CHUNK", 262144));
      const int64_t per_cta = std::max<int64_t>(1, env_int("GD_C4_TASKS_PER_CTA", 4));
      std::vector<int> rf, rzs, rscan;
      std::vector<int64_t> rch, cpre(f16.size() + 1, 0);
      for (size_t j0 = 0; j0 < f16.size(); j0 += F) {
        const size_t j1 = std::min(f16.size(), j0 + (size_t)F);
        int64_t wr = 0;
        for (size_t j = j0; j < j1; j++) wr += w16[j];
        rzs.push_back(wr * 32 < (int64_t)(j1 - j0) * slab_words * 4 ? 1 : 0);
        rscan.push_back(!per_edge && wr * 32 > (int64_t)(j1 - j0) * slab_words * 4 * 2 ? 1 : 0);
        int64_t ch = wr / (per_cta * (int64_t)grid);
        ch = std::max<int64_t>(min_ch, std::min<int64_t>(max_ch, (ch + 511) & ~int64_t(511)));
        if (force.c4_flow) ch = 64;  // many small tasks
        rf.push_back((int)j0);
        rch.push_back(ch);
        for (size_t j = j0; j < j1; j++) cpre[j + 1] = cpre[j] + (w16[j] + ch - 1) / ch;
      }
      rf.push_back((int)f16.size());
      const int R = (int)rf.size() - 1;
      std::vector<FlowSeg> segs;
      std::vector<int> freed(R, -1), cseg(R, -1), useg(R, -1);
      int64_t task0 = 0;
      auto add = [&](int type, int r, int64_t nt, int dep) {
        segs.push_back(FlowSeg{type, r, task0, nt, dep});
        task0 += nt;
        return (int)segs.size() - 1;
      };
      for (int t = 0; t <= R + LU; t++) {
        if (t < R)
          cseg[t] = add(kFlowCount, t, cpre[rf[t + 1]] - cpre[rf[t]], t >= NS ? freed[t - NS] : -1);
        const int r1 = t - LU;
        if (r1 >= 0 && r1 < R) {
          const int64_t used = rf[r1 + 1] - rf[r1];
          if (rscan[r1]) freed[r1] = add(kFlowScan, r1, used * per_slab, cseg[r1]);
          else useg[r1] = add(kFlowUse, r1, cpre[rf[r1 + 1]] - cpre[rf[r1]], cseg[r1]);
        }
        const int r2 = t - LU - 1;
        if (r2 >= 0 && r2 < R && !rscan[r2] && r2 + NS < R) {
          const int64_t used = rf[r2 + 1] - rf[r2];
          freed[r2] = rzs[r2] ? add(kFlowZeroSweep, r2, cpre[rf[r2 + 1]] - cpre[rf[r2]], useg[r2])
                              : add(kFlowZeroFill, r2, used * per_slab, useg[r2]);
        }
      }
      DBuf<int> dfr, drf, done;
      DBuf<int64_t> dcp, drch;
      DBuf<FlowSeg> dseg;
      DBuf<unsigned long long> ntask;
      dfr.alloc(f16.size(), s);
      drf.alloc(rf.size(), s);
      dcp.alloc(cpre.size(), s);
      drch.alloc(rch.size(), s);
      dseg.alloc(segs.size(), s);
      done.alloc(segs.size(), s);
      done.zero();
      ntask.alloc(1, s);
      ntask.zero();
      GD_CUDA(cudaMemcpyAsync(dfr.p, f16.data(), f16.size() * 4, cudaMemcpyHostToDevice, s));
      GD_CUDA(cudaMemcpyAsync(drf.p, rf.data(), rf.size() * 4, cudaMemcpyHostToDevice, s));
      GD_CUDA(cudaMemcpyAsync(dcp.p, cpre.data(), cpre.size() * 8, cudaMemcpyHostToDevice, s));
      GD_CUDA(cudaMemcpyAsync(drch.p, rch.data(), rch.size() * 8, cudaMemcpyHostToDevice, s));
      GD_CUDA(cudaMemcpyAsync(dseg.p, segs.data(), segs.size() * sizeof(FlowSeg),
                              cudaMemcpyHostToDevice, s));
      const size_t slab_total = (size_t)NS * F * slab_words;
      unsigned* slabs = ws_get<unsigned>(g, "c4_slabs", slab_total, s);
      GD_CUDA(cudaMemsetAsync(slabs, 0, slab_total * 4, s));
      FlowPlan P{dfr.p, dcp.p, drf.p, drch.p, dseg.p, (int)segs.size(), F, slab_words, x0,
                 pieces, NS};
      nrounds += R;
      if (narrow)
        fk32<<<grid, fnt, 0, s>>>(v, WP.p, P, slabs, pe, (unsigned*)c4s_p, c4tot2.p, ntask.p,
                                  done.p);
      else
        fk<<<grid, fnt, 0, s>>>(v, WP.p, P, slabs, pe, c4s_p, c4tot2.p, ntask.p, done.p);
      GD_LAUNCH_CHECK("c4_flow");
    }
    timer.mark("c4_coop");
    if (!f32.empty()) {
      std::vector<int64_t> b32(f32.size()), o32(f32.size()), i0v(f32.size()), i1v(f32.size());
      for (size_t h = 0; h < f32.size(); h++) {
        GD_CUDA(cudaMemcpyAsync(&b32[h], g.rp.p + f32[h], 8, cudaMemcpyDeviceToHost, s));
        GD_CUDA(cudaMemcpyAsync(&o32[h], g.osplit.p + f32[h], 8, cudaMemcpyDeviceToHost, s));
      }
      GD_CUDA(cudaStreamSynchronize(s));
      for (size_t h = 0; h < f32.size(); h++) {
        GD_CUDA(cudaMemcpyAsync(&i0v[h], WP.p + b32[h], 8, cudaMemcpyDeviceToHost, s));
        GD_CUDA(cudaMemcpyAsync(&i1v[h], WP.p + o32[h], 8, cudaMemcpyDeviceToHost, s));
      }
      GD_CUDA(cudaStreamSynchronize(s));
      const int64_t slab_stride = (n + 31) & ~int64_t(31);
      const int64_t max_slabs = std::max<int64_t>(
          1, std::min<int64_t>((int64_t)f32.size(), (int64_t)(2ll << 30) / (slab_stride * 4)));
      DBuf<unsigned> slabs;
      slabs.alloc((size_t)max_slabs * slab_stride, s);
      slabs.zero();
      const int64_t chunk_items = 1 << 16;
      for (size_t g0 = 0; g0 < f32.size(); g0 += max_slabs) {
        const size_t g1 = std::min(f32.size(), (size_t)(g0 + max_slabs));
        std::vector<HubChunk> chunks;
        for (size_t h = g0; h < g1; h++)
          for (int64_t c = i0v[h]; c < i1v[h]; c += chunk_items)
            chunks.push_back({f32[h], (int)(h - g0), c, std::min(i1v[h], c + chunk_items)});
        if (chunks.empty()) continue;
        DBuf<HubChunk> dch;
        dch.alloc(chunks.size(), s);
        GD_CUDA(cudaMemcpyAsync(dch.p, chunks.data(), chunks.size() * sizeof(HubChunk),
                                cudaMemcpyHostToDevice, s));
        for (int phase = 0; phase < 3; phase++) {
          if (narrow)
            k_c4_hub<512, unsigned><<<(int)chunks.size(), 512, 0, s>>>(
                v, WP.p, dch.p, slabs.p, slab_stride, phase, pe, (unsigned*)c4s_p, c4tot2.p);
          else
            k_c4_hub<512, u64><<<(int)chunks.size(), 512, 0, s>>>(
                v, WP.p, dch.p, slabs.p, slab_stride, phase, pe, c4s_p, c4tot2.p);
          GD_LAUNCH_CHECK("c4_hub");
        }
        GD_CUDA(cudaStreamSynchronize(s));
      }
      timer.mark("c4_hub32");
    }
    }  // shards
  }
  auto smem_bin = [&](std::pair<int64_t, int64_t> r, auto kernel, auto kernel32, int nt, bool c16,
                      int per_sm) {
    const int64_t nf = r.second - r.first;
    if (nf <= 0) return;
    // capacity > max distinct counters (<= wedges): load <= 1/2 (u32 bins)
    // or <= 3/4 (u16 bin)
    int hcap = 512;
    const int64_t wmax = wk.value(r.first);
    while ((c16 ? 3 * (int64_t)hcap / 4 : (int64_t)hcap / 2) < wmax) hcap <<= 1;
    const size_t sm = (size_t)hcap * 4 + (size_t)hcap * (c16 ? 2 : 4);
    if (sm > 200 * 1024) throw Error(GD_EINVAL, "wedge frame too large for the shared hash");
    set_smem(kernel, sm);
    set_smem(kernel32, sm);
    const int grid =
        (int)std::min<int64_t>((nf + world - 1) / world, (int64_t)num_sms() * per_sm);
    for (const int rk : my_ranks) {
      if (narrow)
        kernel32<<<grid, nt, sm, s>>>(v, WP.p, c4_frames.p + r.first, (int)nf, rk, world, hcap,
                                      pe, (unsigned*)c4s_p, c4tot2.p);
      else
        kernel<<<grid, nt, sm, s>>>(v, WP.p, c4_frames.p + r.first, (int)nf, rk, world, hcap, pe,
                                    c4s_p, c4tot2.p);
      GD_LAUNCH_CHECK("c4_frames_smem");
    }
  };
#define GD_SMK(NT_, C16_) k_c4_frames_smem<NT_, C16_, u64>, k_c4_frames_smem<NT_, C16_, unsigned>
  // hash capacity grows with the bin's largest frame: finer bins keep more
  // CTAs resident per SM (u16 counts above 4096 wedges)
  if (env_int("GD_C4_TOP_NT", 1024) == 1024)
    smem_bin(rs2, GD_SMK(1024, true), 1024, true, 1);
  else
    smem_bin(rs2, GD_SMK(512, true), 512, true, 1);
  if (env_int("GD_C4_MID_NT", 1024) == 1024)
    smem_bin(rsb, GD_SMK(1024, true), 1024, true, 2);
  else
    smem_bin(rsb, GD_SMK(512, true), 512, true, 2);
  smem_bin(rs1, GD_SMK(256, false), 256, false, 3);
  smem_bin(rsa, GD_SMK(128, false), 128, false, 12);
  smem_bin(rs0, GD_SMK(64, false), 64, false, 32);
#undef GD_SMK
  timer.mark("c4_smem");
  // owned edge ranges: per-edge partials reduce-scattered onto their owners
  const int64_t M = owned ? (m + world - 1) / world : m;
  if (owned && per_edge) {
    const int esz = narrow ? 4 : 8;
    char* packed = ws_get<char>(g, "packed", (size_t)world * 4 * M * esz, s);
    char* mine = ws_get<char>(g, "owned", (size_t)4 * M * esz, s);
#define GD_PACK(ST)                                                                               \
    k_pack_edge_partials<ST><<<grid_cap(m, 256), 256, 0, s>>>(m, M, g.e2o.p, g.e2i.p, (ST*)tsl.p, \
        (ST*)tsh.p, (ST*)tsd.p, (ST*)c4s.p, (ST*)packed)
    if (narrow) GD_PACK(unsigned); else GD_PACK(u64);
#undef GD_PACK
    GD_LAUNCH_CHECK("pack_edge_partials");
    if (sh.real()) sh.reduce_scatter(packed, mine, (size_t)4 * M, esz);
    for (const int rk : my_ranks) {
      int64_t e0, e1;
      shard_rows(m, rk, world, &e0, &e1);
      if (e1 <= e0) continue;
      const char* src = sh.real() ? mine : packed + (size_t)rk * 4 * M * esz;
#define GD_UNPACK(ST)                                                                             \
      k_unpack_owned<ST><<<grid_cap(e1 - e0, 256), 256, 0, s>>>(e0, e1, M, g.e2o.p, g.e2i.p,       \
          (const ST*)src, (ST*)tsl.p, (ST*)tsh.p, (ST*)tsd.p, (ST*)c4s.p)
      if (narrow) GD_UNPACK(unsigned); else GD_UNPACK(u64);
#undef GD_UNPACK
      GD_LAUNCH_CHECK("unpack_owned");
    }
    timer.mark("reduce_scatter_bc");
  } else if (sh.real() && per_edge) {  // batches: every slot of every shard
    sh.allreduce(tsl.p, (size_t)S);
    sh.allreduce(tsh.p, (size_t)S);
    sh.allreduce(tsd.p, (size_t)S);
    sh.allreduce(c4s.p, (size_t)S);
    timer.mark("allreduce_bc");
  }
  stat("c4_coop_frames", nh - n32);
  stat("c4_heavy_wedges", heavy_w);
  stat("c4_tiles", tiles_used ? 1 : 0);
  stat("c4_rounds", nrounds);
  stat("c4_u32_hub_frames", n32);
  stat("c4_smem_frames", (rs0.second - rs0.first) + (rsa.second - rsa.first) +
                             (rs1.second - rs1.first) + (rsb.second - rsb.first) +
                             (rs2.second - rs2.first));

  // ---- finalize -----------------------------------------------------------
  EdgeIn in;
  in.eu = g.eu.p;
  in.ev = g.ev.p;
  in.d2r = g.d2r.p;
  in.deg = g.deg.p;
  in.e2o = g.e2o.p;
  in.e2i = g.e2i.p;
  in.tcs = tcs.p;
  in.narrow = narrow;
  in.tsl = per_edge ? tsl.p : nullptr;
  in.tsh = per_edge ? tsh.p : nullptr;
  in.tsd = per_edge ? tsd.p : nullptr;
  in.c4s = per_edge ? c4s.p : nullptr;
  in.vT = vT.p;
  in.vS = vS.p;
  DBuf<uint4> vrec;
  vrec.alloc((size_t)std::max<int64_t>(2 * n, 1), s);
  if (n) {
    k_vertex_records<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, g.d2r.p, g.deg.p, vT.p, vS.p, vrec.p);
    GD_LAUNCH_CHECK("vertex_records");
  }
  in.vrec = vrec.p;
  GD_CUDA(cudaMemsetAsync(sums_dev, 0, (size_t)G * 2 * kNumSums * 8, s));
  GD_CUDA(cudaMemsetAsync(seen_dev, 0, (size_t)G * 8, s));
  cudaStream_t copy_stream = nullptr;  // set when the table's D2H was started here
  if (G == 1 && owned) {
    // real: this rank's rows into its table shard, then all ranks' sums
    // added; emulated: every rank's range at its offset of the full table
    for (const int rk : my_ranks) {
      int64_t e0, e1;
      shard_rows(m, rk, world, &e0, &e1);
      if (rk == sh.rank || !sh.real()) {
        ex.row0 = sh.real() ? e0 : 0;
        ex.rows = sh.real() ? e1 - e0 : m;
      }
      if (e1 <= e0) continue;
      long long* tp = table_dev ? table_dev + (sh.real() ? 0 : e0 * kNumMicro) : nullptr;
      k_finalize_single<256><<<grid_cap(e1 - e0, 256, 4), 256, 0, s>>>(in, e0, e1, n, m, tp,
                                                                       sums_dev, seen_dev);
      GD_LAUNCH_CHECK("finalize_single");
    }
    if (sh.real()) {
      DBuf<u64> gs, gn;
      gs.alloc((size_t)world * 2 * kNumSums, s);
      gn.alloc((size_t)world, s);
      sh.allgather(sums_dev, gs.p, (size_t)(2 * kNumSums));
      sh.allgather(seen_dev, gn.p, 1);
      k_sum_shards<<<1, 32, 0, s>>>(gs.p, gn.p, world, sums_dev, seen_dev);
      GD_LAUNCH_CHECK("sum_shards");
    }
  } else if (G == 1 && ex.host_table && table_dev && m >= (1 << 20) &&
             env_int("GD_D2H_OVERLAP", 1)) {
    // rows finalized in chunks; each chunk's D2H runs on the copy stream
    // while the next chunk is finalized (the table's copy is PCIe-bound:
    // it starts ~1.3 ms earlier at R-MAT-20)
    constexpr int K = 8;
    static thread_local cudaStream_t cs = nullptr;
    static thread_local cudaEvent_t ev[K] = {};
    if (!cs) {
      GD_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
      for (int c = 0; c < K; c++) GD_CUDA(cudaEventCreateWithFlags(&ev[c], cudaEventDisableTiming));
    }
    for (int c = 0; c < K; c++) {
      const int64_t e0 = m * c / K, e1 = m * (c + 1) / K;
      if (e1 <= e0) continue;
      k_finalize_single<256><<<grid_cap(e1 - e0, 256, 4), 256, 0, s>>>(
          in, e0, e1, n, m, table_dev + e0 * kNumMicro, sums_dev, seen_dev);
      GD_LAUNCH_CHECK("finalize_single");
      GD_CUDA(cudaEventRecord(ev[c], s));
      GD_CUDA(cudaStreamWaitEvent(cs, ev[c], 0));
      GD_CUDA(cudaMemcpyAsync((char*)ex.host_table + (size_t)e0 * kNumMicro * 8,
                              table_dev + e0 * kNumMicro, (size_t)(e1 - e0) * kNumMicro * 8,
                              cudaMemcpyDeviceToHost, cs));
    }
    copy_stream = cs;
  } else if (G == 1) {
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

  // per-shard 128-bit totals: gathered (not summed) so carries stay exact
  const int nranks = sh.real() ? world : 1;
  std::vector<u64> hk4(2 * G * nranks), hc4(2 * G * nranks);
  if (sh.real()) {
    DBuf<u64> gk4, gc4;
    gk4.alloc(2 * G * nranks, s);
    gc4.alloc(2 * G * nranks, s);
    sh.allgather(k4tot.p, gk4.p, (size_t)(2 * G));
    sh.allgather(c4tot2.p, gc4.p, (size_t)(2 * G));
    GD_CUDA(cudaMemcpyAsync(hk4.data(), gk4.p, hk4.size() * 8, cudaMemcpyDeviceToHost, s));
    GD_CUDA(cudaMemcpyAsync(hc4.data(), gc4.p, hc4.size() * 8, cudaMemcpyDeviceToHost, s));
    GD_CUDA(cudaStreamSynchronize(s));
  } else {
    GD_CUDA(cudaMemcpyAsync(hk4.data(), k4tot.p, 2 * G * 8, cudaMemcpyDeviceToHost, s));
    GD_CUDA(cudaMemcpyAsync(hc4.data(), c4tot2.p, 2 * G * 8, cudaMemcpyDeviceToHost, s));
  }
  timer.collect(ex.ms, ex.names);
  if (copy_stream) {
    GD_CUDA(cudaStreamSynchronize(copy_stream));
    ex.table_copied = true;
  }
  stat("launches", g_launches - launches0);
  stat("shards", world);
  for (int r = 0; r < nranks; r++) {
    const u64* a = hk4.data() + 2 * G * r;
    const u64* c = hc4.data() + 2 * G * r;
    for (int64_t i = 0; i < G; i++) {
      ex.k4tot[i] += ((u128)a[2 * i + 1] << 64) | a[2 * i];
      ex.c4tot2[i] += ((u128)c[2 * i + 1] << 64) | c[2 * i];
    }
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
