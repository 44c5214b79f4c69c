// On-device graph construction: the sanitising CSR build of the reference
// (Graph.from_edges graph.py:118-157 + Graph.__init__ graph.py:68-114) and
// the degree-ordered ("rank") relabelled CSR the counting kernels run on.
//
// Pipeline (all on the library stream):
//   pairs --(drop loops, canonicalise, range checks)--> 64-bit edge keys
//         --radix sort + unique--> canonical edges (lexicographic u<v)
//         --degrees, sort vertices by (degree, id)--> rank relabel
//         --2m slot keys (rank(u), rank(v)) sorted--> rank CSR + slot edge ids
#include <cub/cub.cuh>

#include "gd_build.cuh"

namespace gd {

namespace {

constexpr unsigned long long kSentinel = ~0ull;

__device__ __forceinline__ unsigned long long ordered_u64(long long x) {
  return (unsigned long long)x ^ 0x8000000000000000ull;
}
__device__ __forceinline__ long long from_ordered_u64(unsigned long long x) {
  return (long long)(x ^ 0x8000000000000000ull);
}

struct BuildFlags {
  unsigned long long loops;      // number of self-loop pairs
  long long max_id;              // max endpoint over non-loop pairs
  long long min_id;              // min endpoint over non-loop pairs
  unsigned long long bad_graph;  // batch: pairs outside their graph's [0, n_g)
};

__device__ __forceinline__ void atomic_max_ll(long long* p, long long v) {
  atomicMax((long long*)p, v);
}
__device__ __forceinline__ void atomic_min_ll(long long* p, long long v) {
  atomicMin((long long*)p, v);
}

// Pass 1 over raw pairs: self-loop count and id range of non-loop pairs.
__global__ void k_scan_pairs(const long long* __restrict__ pairs, int64_t k,
                             BuildFlags* flags) {
  long long lmax = LLONG_MIN, lmin = LLONG_MAX;
  unsigned long long loops = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k;
       i += (int64_t)gridDim.x * blockDim.x) {
    long long a = pairs[2 * i], b = pairs[2 * i + 1];
    if (a == b) { loops++; continue; }
    lmax = max(lmax, max(a, b));
    lmin = min(lmin, min(a, b));
  }
  // warp reduce then one atomic per warp
  for (int o = 16; o; o >>= 1) {
    lmax = max(lmax, (long long)__shfl_xor_sync(0xffffffffu, lmax, o));
    lmin = min(lmin, (long long)__shfl_xor_sync(0xffffffffu, lmin, o));
    loops += __shfl_xor_sync(0xffffffffu, loops, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (loops) atomicAdd(&flags->loops, loops);
    atomic_max_ll(&flags->max_id, lmax);
    atomic_min_ll(&flags->min_id, lmin);
  }
}

// Edge keys pack (min << kb) | max with kb = bits of the vertex count, so the
// radix sorts run over 2 kb + 1 bits (the sentinel, all ones, sorts last)
// instead of 64: 3 passes instead of 8 at config 1, 6 at config 3.
// Dense ids already: loops -> sentinel.
__global__ void k_pair_keys_dense(const long long* __restrict__ pairs, int64_t k, int kb,
                                  unsigned long long* __restrict__ keys) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k;
       i += (int64_t)gridDim.x * blockDim.x) {
    long long a = pairs[2 * i], b = pairs[2 * i + 1];
    if (a == b) { keys[i] = kSentinel; continue; }
    unsigned long long lo = (unsigned long long)min(a, b);
    unsigned long long hi = (unsigned long long)max(a, b);
    keys[i] = (lo << kb) | hi;
  }
}

// Remap mode: endpoints of non-loop pairs as order-preserving u64.
__global__ void k_endpoint_ids(const long long* __restrict__ pairs, int64_t k,
                               unsigned long long* __restrict__ ids) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k;
       i += (int64_t)gridDim.x * blockDim.x) {
    long long a = pairs[2 * i], b = pairs[2 * i + 1];
    if (a == b) {
      ids[2 * i] = kSentinel;
      ids[2 * i + 1] = kSentinel;
    } else {
      ids[2 * i] = ordered_u64(a);
      ids[2 * i + 1] = ordered_u64(b);
    }
  }
}

// Remap mode: dense ids by binary search into the sorted unique originals.
__global__ void k_pair_keys_remap(const long long* __restrict__ pairs, int64_t k,
                                  const unsigned long long* __restrict__ uniq,
                                  int64_t n, int kb, unsigned long long* __restrict__ keys) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k;
       i += (int64_t)gridDim.x * blockDim.x) {
    long long a = pairs[2 * i], b = pairs[2 * i + 1];
    if (a == b) { keys[i] = kSentinel; continue; }
    unsigned long long da = (unsigned long long)lower_bound_dev(uniq, 0, n, ordered_u64(a));
    unsigned long long db = (unsigned long long)lower_bound_dev(uniq, 0, n, ordered_u64(b));
    unsigned long long lo = min(da, db), hi = max(da, db);
    keys[i] = (lo << kb) | hi;
  }
}

__global__ void k_orig_from_ordered(const unsigned long long* __restrict__ uniq,
                                    int64_t n, long long* __restrict__ orig) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    orig[i] = from_ordered_u64(uniq[i]);
}

// Batch: per pair, add its graph's vertex offset; ids must be in [0, n_g).
__global__ void k_batch_keys(const long long* __restrict__ pairs, int64_t k,
                             const int64_t* __restrict__ poff, int64_t G,
                             const int64_t* __restrict__ gn,
                             const int64_t* __restrict__ voff, int kb,
                             unsigned long long* __restrict__ keys,
                             BuildFlags* flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k;
       i += (int64_t)gridDim.x * blockDim.x) {
    // graph of pair i: last g with poff[g] <= i
    int64_t lo = 0, hi = G - 1;
    while (lo < hi) {
      int64_t mid = (lo + hi + 1) >> 1;
      if (poff[mid] <= i) lo = mid; else hi = mid - 1;
    }
    long long a = pairs[2 * i], b = pairs[2 * i + 1];
    if (a == b) { keys[i] = kSentinel; continue; }
    if (a < 0 || b < 0 || a >= gn[lo] || b >= gn[lo]) {
      atomicAdd(&flags->bad_graph, 1ull);
      keys[i] = kSentinel;
      continue;
    }
    unsigned long long x = (unsigned long long)(min(a, b) + voff[lo]);
    unsigned long long y = (unsigned long long)(max(a, b) + voff[lo]);
    keys[i] = (x << kb) | y;
  }
}

__global__ void k_split_keys(const unsigned long long* __restrict__ keys, int64_t m, int kb,
                             int32_t* __restrict__ eu, int32_t* __restrict__ ev,
                             int32_t* __restrict__ deg) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long key = keys[i];
    int u = (int)(key >> kb), v = (int)(key & ((1ull << kb) - 1));
    eu[i] = u;
    ev[i] = v;
    atomicAdd(&deg[u], 1);
    atomicAdd(&deg[v], 1);
  }
}

__global__ void k_iota(int32_t* __restrict__ a, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    a[i] = (int32_t)i;
}

__global__ void k_deg_keys(const int32_t* __restrict__ d, unsigned long long* __restrict__ k,
                           int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    k[i] = (unsigned long long)d[i];
}

__global__ void k_rank_tables(const int32_t* __restrict__ r2d, int64_t n,
                              const int32_t* __restrict__ deg_dense,
                              int32_t* __restrict__ d2r, int32_t* __restrict__ deg_rank,
                              int64_t* __restrict__ deg64) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    int d = r2d[r];
    d2r[d] = (int32_t)r;
    int dg = deg_dense[d];
    deg_rank[r] = dg;
    deg64[r] = dg;
  }
}

__global__ void k_slot_keys(const int32_t* __restrict__ eu, const int32_t* __restrict__ ev,
                            const int32_t* __restrict__ d2r, int64_t m, int kb,
                            unsigned long long* __restrict__ keys,
                            int32_t* __restrict__ vals) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long ru = (unsigned)d2r[eu[e]], rv = (unsigned)d2r[ev[e]];
    keys[2 * e] = (ru << kb) | rv;
    keys[2 * e + 1] = (rv << kb) | ru;
    vals[2 * e] = (int32_t)e;
    vals[2 * e + 1] = (int32_t)e;
  }
}

// Sorted slot keys (row rank << kb | neighbour rank) -> col[], and the two
// slots of every edge: the out-slot lies in the row of the lower rank.
__global__ void k_slot_cols(const unsigned long long* __restrict__ keys, int64_t s, int kb,
                            const int32_t* __restrict__ seid, int32_t* __restrict__ col,
                            int64_t* __restrict__ e2o, int64_t* __restrict__ e2i) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < s;
       i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long key = keys[i];
    const int32_t c = (int32_t)(key & ((1ull << kb) - 1));
    const int32_t r = (int32_t)(key >> kb);
    col[i] = c;
    const int e = seid[i];
    if (c > r) e2o[e] = i; else e2i[e] = i;
  }
}

__global__ void k_osplit(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                         int64_t n, int64_t* __restrict__ osplit) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x)
    osplit[r] = lower_bound_dev(col, rp[r], rp[r + 1], (int32_t)(r + 1));
}

__global__ void k_vgraph(const int32_t* __restrict__ r2d, int64_t n,
                         const int64_t* __restrict__ voff, int64_t G,
                         int32_t* __restrict__ vgraph) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    int64_t d = r2d[r];
    int64_t lo = 0, hi = G - 1;
    while (lo < hi) {
      int64_t mid = (lo + hi + 1) >> 1;
      if (voff[mid] <= d) lo = mid; else hi = mid - 1;
    }
    vgraph[r] = (int32_t)lo;
  }
}

// eoff[g] = first canonical edge of graph g: edges ascend by their lower dense
// id and the graphs own contiguous id ranges, so it is a lower bound over eu.
__global__ void k_edge_offsets(const int32_t* __restrict__ eu, int64_t m,
                               const int64_t* __restrict__ voff, int64_t G,
                               int64_t* __restrict__ eoff) {
  const int64_t gi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (gi > G) return;
  int64_t lo = 0, hi = m;
  if (gi == G) lo = m;
  const int64_t v0 = gi < G ? voff[gi] : 0;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)eu[mid] < v0) lo = mid + 1; else hi = mid;
  }
  eoff[gi] = lo;
}

__global__ void k_max_int(const int32_t* __restrict__ a, int64_t n, int* out) {
  int v = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    v = max(v, a[i]);
  for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, v);
}

int bits_for(uint64_t x) {  // number of bits to represent values in [0, x]
  int b = 1;
  while (b < 64 && (x >> b)) b++;
  return b;
}

int grid_for(int64_t n, int threads = 256) {
  int64_t g = (n + threads - 1) / threads;
  int64_t cap = (int64_t)num_sms() * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

// --- thin CUB wrappers (temp storage from the stream-ordered pool) ---------
void sort_keys(unsigned long long* in, unsigned long long* out, int64_t n,
               int end_bit, cudaStream_t s) {
  size_t tb = 0;
  GD_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, in, out, n, 0, end_bit, s));
  DBuf<char> tmp;
  tmp.alloc(tb, s);
  GD_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tb, in, out, n, 0, end_bit, s));
}

template <typename V>
void sort_pairs(unsigned long long* kin, unsigned long long* kout, V* vin, V* vout,
                int64_t n, int end_bit, cudaStream_t s) {
  size_t tb = 0;
  GD_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, kin, kout, vin, vout, n, 0,
                                          end_bit, s));
  DBuf<char> tmp;
  tmp.alloc(tb, s);
  GD_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, kin, kout, vin, vout, n, 0,
                                          end_bit, s));
}

int64_t unique_keys(unsigned long long* in, unsigned long long* out, int64_t n,
                    cudaStream_t s) {
  DBuf<int64_t> cnt;
  cnt.alloc(1, s);
  size_t tb = 0;
  GD_CUDA(cub::DeviceSelect::Unique(nullptr, tb, in, out, cnt.p, n, s));
  DBuf<char> tmp;
  tmp.alloc(tb, s);
  GD_CUDA(cub::DeviceSelect::Unique(tmp.p, tb, in, out, cnt.p, n, s));
  int64_t h = 0;
  GD_CUDA(cudaMemcpyAsync(&h, cnt.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  GD_CUDA(cudaStreamSynchronize(s));
  return h;
}

void exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, cudaStream_t s) {
  size_t tb = 0;
  GD_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n, s));
  DBuf<char> tmp;
  tmp.alloc(tb, s);
  GD_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, in, out, n, s));
}

// Shared tail: canonical unique keys (sentinel already removed) -> DevGraph.
void finish_graph(DevGraph& g, DBuf<unsigned long long>& ukeys, int64_t m, int64_t n,
                  cudaStream_t s) {
  if (n > INT32_MAX - 1) throw Error(GD_ECAPACITY, "vertex count exceeds int32 ids");
  if (2 * m > (int64_t)INT32_MAX * 2)
    throw Error(GD_ECAPACITY, "edge count exceeds int32 edge ids");
  g.n = n;
  g.m = m;
  g.eu.alloc(m, s);
  g.ev.alloc(m, s);
  DBuf<int32_t> deg_dense;
  deg_dense.alloc(n, s);
  deg_dense.zero();
  if (m) {
    k_split_keys<<<grid_for(m), 256, 0, s>>>(ukeys.p, m, bits_for((uint64_t)n), g.eu.p, g.ev.p,
                                             deg_dense.p);
    GD_LAUNCH_CHECK("split_keys");
  }
  ukeys.release();

  // rank relabel: ascending (degree, dense id); radix sort is stable and the
  // values start in id order.
  g.r2d.alloc(n, s);
  g.d2r.alloc(n, s);
  g.deg.alloc(n, s);
  g.rp.alloc(n + 1, s);
  g.max_deg = 0;
  if (n) {
    DBuf<unsigned long long> dk, dk2;
    DBuf<int32_t> ids;
    dk.alloc(n, s);
    dk2.alloc(n, s);
    ids.alloc(n, s);
    k_iota<<<grid_for(n), 256, 0, s>>>(ids.p, n);
    k_deg_keys<<<grid_for(n), 256, 0, s>>>(deg_dense.p, dk.p, n);
    GD_LAUNCH_CHECK("deg_keys");
    sort_pairs<int32_t>(dk.p, dk2.p, ids.p, g.r2d.p, n, bits_for((uint64_t)n), s);
    DBuf<int64_t> deg64;
    deg64.alloc(n, s);
    k_rank_tables<<<grid_for(n), 256, 0, s>>>(g.r2d.p, n, deg_dense.p, g.d2r.p, g.deg.p,
                                              deg64.p);
    GD_LAUNCH_CHECK("rank_tables");
    exclusive_scan_i64(deg64.p, g.rp.p, n, s);
    int64_t two_m = 2 * m;
    GD_CUDA(cudaMemcpyAsync(g.rp.p + n, &two_m, sizeof(int64_t), cudaMemcpyHostToDevice, s));
    DBuf<int> mx;
    mx.alloc(1, s);
    mx.zero();
    k_max_int<<<grid_for(n), 256, 0, s>>>(g.deg.p, n, mx.p);
    GD_CUDA(cudaMemcpyAsync(&g.max_deg, mx.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  } else {
    int64_t zero = 0;
    GD_CUDA(cudaMemcpyAsync(g.rp.p, &zero, sizeof(int64_t), cudaMemcpyHostToDevice, s));
  }

  // rank CSR: 2m slot keys sorted by (rank(row), rank(col)), payload edge id
  g.col.alloc(2 * m, s);
  g.seid.alloc(2 * m, s);
  g.osplit.alloc(n, s);
  if (m) {
    DBuf<unsigned long long> sk, sk2;
    DBuf<int32_t> sv;
    sk.alloc(2 * m, s);
    sk2.alloc(2 * m, s);
    sv.alloc(2 * m, s);
    const int kb = bits_for((uint64_t)n);
    k_slot_keys<<<grid_for(m), 256, 0, s>>>(g.eu.p, g.ev.p, g.d2r.p, m, kb, sk.p, sv.p);
    GD_LAUNCH_CHECK("slot_keys");
    sort_pairs<int32_t>(sk.p, sk2.p, sv.p, g.seid.p, 2 * m, 2 * kb, s);
    g.e2o.alloc(m, s);
    g.e2i.alloc(m, s);
    k_slot_cols<<<grid_for(2 * m), 256, 0, s>>>(sk2.p, 2 * m, kb, g.seid.p, g.col.p, g.e2o.p,
                                                g.e2i.p);
    GD_LAUNCH_CHECK("slot_cols");
  } else {
    g.e2o.alloc(m, s);
    g.e2i.alloc(m, s);
  }
  if (n) {
    k_osplit<<<grid_for(n), 256, 0, s>>>(g.rp.p, g.col.p, n, g.osplit.p);
    GD_LAUNCH_CHECK("osplit");
  }
  GD_CUDA(cudaStreamSynchronize(s));
  if (g.max_deg >= (1 << 24) - 1)
    throw Error(GD_ECAPACITY, "max degree beyond the packed 24-bit triangle counter");
}

}  // namespace

// ---------------------------------------------------------------------------
void build_graph(DevGraph& g, const int64_t* pairs_in, int64_t k, int64_t n_decl,
                 int mode, int flags, cudaStream_t s) {
  if (k < 0) throw Error(GD_EINVAL, "negative pair count");
  if (mode < GD_IDS_REMAP || mode > GD_IDS_SANITIZED) throw Error(GD_EINVAL, "bad ids mode");
  if ((mode == GD_IDS_DECLARED || mode == GD_IDS_SANITIZED) && n_decl < 0)
    throw Error(GD_EINVAL, "declared vertex count must be >= 0");
  if (k > ((int64_t)1 << 31)) throw Error(GD_ECAPACITY, "more than 2^31 input pairs");

  DBuf<long long> pairs;
  const long long* dp = (const long long*)pairs_in;
  if (!(flags & GD_INPUT_DEVICE) && k) {
    pairs.alloc(2 * k, s);
    copy_h2d(pairs.p, pairs_in, 2 * k * sizeof(int64_t), s);
    dp = pairs.p;
  }

  BuildFlags hf{0, LLONG_MIN, LLONG_MAX, 0};
  DBuf<BuildFlags> df;
  df.alloc(1, s);
  GD_CUDA(cudaMemcpyAsync(df.p, &hf, sizeof(hf), cudaMemcpyHostToDevice, s));
  if (k) {
    k_scan_pairs<<<grid_for(k), 256, 0, s>>>(dp, k, df.p);
    GD_LAUNCH_CHECK("scan_pairs");
  }
  GD_CUDA(cudaMemcpyAsync(&hf, df.p, sizeof(hf), cudaMemcpyDeviceToHost, s));
  GD_CUDA(cudaStreamSynchronize(s));
  const bool any_edge = (int64_t)hf.loops < k;

  int64_t n = 0;
  DBuf<unsigned long long> keys, ukeys;
  keys.alloc(k, s);
  if (mode == GD_IDS_SANITIZED) {
    // Graph.__init__ (graph.py:70-81): range, loops and duplicates are errors.
    if (k && (hf.min_id < 0 || hf.max_id >= n_decl || (hf.loops && n_decl <= 0)))
      throw Error(GD_EINVAL, "edge endpoints out of range [0, n)");
    if (hf.loops) {
      // a loop (a, a) with a out of range is also a range error in the reference
      throw Error(GD_EINVAL, "self-loops are not allowed in a sanitized Graph");
    }
    n = n_decl;
  } else if (mode == GD_IDS_DECLARED) {
    // Graph.from_edges declared-n branch (graph.py:139-147)
    n = n_decl;
    if (any_edge && hf.max_id >= n)
      throw Error(GD_EPARSE, "vertex id " + std::to_string(hf.max_id) +
                                 " out of declared range [0, " + std::to_string(n) + ")");
    if (any_edge && hf.min_id < 0) throw Error(GD_EPARSE, "negative vertex id");
  } else if (mode == GD_IDS_MAX_ID) {
    // use_max_id branch (graph.py:148-152)
    if (any_edge && hf.min_id < 0) throw Error(GD_EPARSE, "negative vertex id");
    n = any_edge ? hf.max_id + 1 : 0;
  }
  if (mode != GD_IDS_REMAP && n > (int64_t)INT32_MAX - 1)
    throw Error(GD_ECAPACITY, "vertex count exceeds int32 ids");

  if (mode == GD_IDS_REMAP) {
    // ids = unique endpoints of the non-loop pairs (graph.py:154-157)
    DBuf<unsigned long long> ids, sids;
    ids.alloc(2 * k, s);
    sids.alloc(2 * k, s);
    if (k) {
      k_endpoint_ids<<<grid_for(k), 256, 0, s>>>(dp, k, ids.p);
      GD_LAUNCH_CHECK("endpoint_ids");
      sort_keys(ids.p, sids.p, 2 * k, 64, s);
    }
    DBuf<unsigned long long> uniq;
    uniq.alloc(2 * k, s);
    int64_t nu = k ? unique_keys(sids.p, uniq.p, 2 * k, s) : 0;
    if (hf.loops && nu) nu -= 1;  // sentinel
    n = nu;
    if (n > (int64_t)INT32_MAX - 1) throw Error(GD_ECAPACITY, "vertex count exceeds int32 ids");
    g.orig.alloc(n, s);
    if (n) {
      k_orig_from_ordered<<<grid_for(n), 256, 0, s>>>(uniq.p, n, (long long*)g.orig.p);
      GD_LAUNCH_CHECK("orig_ids");
    }
    if (k) {
      k_pair_keys_remap<<<grid_for(k), 256, 0, s>>>(dp, k, uniq.p, n, bits_for((uint64_t)n),
                                                    keys.p);
      GD_LAUNCH_CHECK("pair_keys_remap");
    }
  } else if (k) {
    k_pair_keys_dense<<<grid_for(k), 256, 0, s>>>(dp, k, bits_for((uint64_t)n), keys.p);
    GD_LAUNCH_CHECK("pair_keys");
  }
  pairs.release();

  int64_t m = 0;
  if (k) {
    DBuf<unsigned long long> sorted;
    sorted.alloc(k, s);
    sort_keys(keys.p, sorted.p, k, std::min(64, 2 * bits_for((uint64_t)n) + 1), s);
    keys.release();
    ukeys.alloc(k, s);
    m = unique_keys(sorted.p, ukeys.p, k, s);
    if (hf.loops && m) m -= 1;  // drop the sentinel at the end
    if (mode == GD_IDS_SANITIZED && m != k)
      throw Error(GD_EINVAL, "duplicate edges are not allowed in a sanitized Graph");
  }
  g.G = 1;
  g.h_eoff = {0, m};
  g.h_gn = {n};
  g.eoff.alloc(2, s);
  g.gn.alloc(1, s);
  GD_CUDA(cudaMemcpyAsync(g.eoff.p, g.h_eoff.data(), 2 * sizeof(int64_t),
                          cudaMemcpyHostToDevice, s));
  GD_CUDA(cudaMemcpyAsync(g.gn.p, g.h_gn.data(), sizeof(int64_t), cudaMemcpyHostToDevice, s));
  finish_graph(g, ukeys, m, n, s);
}

void build_graph_batch(DevGraph& g, const int64_t* pairs_in, const int64_t* poff_h,
                       const int64_t* gn_h, int64_t G, int flags, cudaStream_t s) {
  if (G <= 0) throw Error(GD_EINVAL, "batch needs at least one graph");
  int64_t k = poff_h[G] - poff_h[0];
  if (poff_h[0] != 0) throw Error(GD_EINVAL, "pair_offsets[0] must be 0");
  std::vector<int64_t> voff(G + 1, 0);
  for (int64_t i = 0; i < G; i++) {
    if (gn_h[i] < 0) throw Error(GD_EINVAL, "negative vertex count");
    if (poff_h[i + 1] < poff_h[i]) throw Error(GD_EINVAL, "pair_offsets must be nondecreasing");
    voff[i + 1] = voff[i] + gn_h[i];
  }
  int64_t n = voff[G];
  if (n > (int64_t)INT32_MAX - 1) throw Error(GD_ECAPACITY, "vertex count exceeds int32 ids");

  DBuf<long long> pairs;
  const long long* dp = (const long long*)pairs_in;
  if (!(flags & GD_INPUT_DEVICE) && k) {
    pairs.alloc(2 * k, s);
    copy_h2d(pairs.p, pairs_in, 2 * k * sizeof(int64_t), s);
    dp = pairs.p;
  }
  DBuf<int64_t> d_poff, d_gn, d_voff;
  d_poff.alloc(G + 1, s);
  d_gn.alloc(G, s);
  d_voff.alloc(G + 1, s);
  GD_CUDA(cudaMemcpyAsync(d_poff.p, poff_h, (G + 1) * 8, cudaMemcpyHostToDevice, s));
  GD_CUDA(cudaMemcpyAsync(d_gn.p, gn_h, G * 8, cudaMemcpyHostToDevice, s));
  GD_CUDA(cudaMemcpyAsync(d_voff.p, voff.data(), (G + 1) * 8, cudaMemcpyHostToDevice, s));

  BuildFlags hf{0, LLONG_MIN, LLONG_MAX, 0};
  DBuf<BuildFlags> df;
  df.alloc(1, s);
  GD_CUDA(cudaMemcpyAsync(df.p, &hf, sizeof(hf), cudaMemcpyHostToDevice, s));
  DBuf<unsigned long long> keys, ukeys;
  keys.alloc(k, s);
  if (k) {
    k_scan_pairs<<<grid_for(k), 256, 0, s>>>(dp, k, df.p);
    k_batch_keys<<<grid_for(k), 256, 0, s>>>(dp, k, d_poff.p, G, d_gn.p, d_voff.p,
                                             bits_for((uint64_t)n), keys.p, df.p);
    GD_LAUNCH_CHECK("batch_keys");
  }
  GD_CUDA(cudaMemcpyAsync(&hf, df.p, sizeof(hf), cudaMemcpyDeviceToHost, s));
  GD_CUDA(cudaStreamSynchronize(s));
  if (hf.bad_graph) throw Error(GD_EPARSE, "vertex id out of its graph's declared range");
  pairs.release();
  int64_t m = 0;
  if (k) {
    DBuf<unsigned long long> sorted;
    sorted.alloc(k, s);
    sort_keys(keys.p, sorted.p, k, std::min(64, 2 * bits_for((uint64_t)n) + 1), s);
    keys.release();
    ukeys.alloc(k, s);
    m = unique_keys(sorted.p, ukeys.p, k, s);
    if (hf.loops && m) m -= 1;
  }
  g.G = G;
  finish_graph(g, ukeys, m, n, s);

  // per-graph bookkeeping
  g.vgraph.alloc(n, s);
  if (n) {
    k_vgraph<<<grid_for(n), 256, 0, s>>>(g.r2d.p, n, d_voff.p, G, g.vgraph.p);
    GD_LAUNCH_CHECK("vgraph");
  }
  g.eoff.alloc(G + 1, s);
  g.gn.alloc(G, s);
  k_edge_offsets<<<grid_for(G + 1), 256, 0, s>>>(g.eu.p, m, d_voff.p, G, g.eoff.p);
  GD_LAUNCH_CHECK("edge_offsets");
  g.h_eoff.assign(G + 1, 0);
  g.h_gn.assign(gn_h, gn_h + G);
  GD_CUDA(cudaMemcpyAsync(g.h_eoff.data(), g.eoff.p, (G + 1) * 8, cudaMemcpyDeviceToHost, s));
  GD_CUDA(cudaMemcpyAsync(g.gn.p, g.h_gn.data(), G * 8, cudaMemcpyHostToDevice, s));
  GD_CUDA(cudaStreamSynchronize(s));
}

// ---------------------------------------------------------------------------
// Export of the reference Graph arrays (dense-id CSR) to host memory.
// ---------------------------------------------------------------------------
namespace {
__global__ void k_dense_slot_keys(const int32_t* __restrict__ eu, const int32_t* __restrict__ ev,
                                  int64_t m, unsigned long long* __restrict__ keys,
                                  int64_t* __restrict__ vals) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long u = (unsigned)eu[e], v = (unsigned)ev[e];
    keys[2 * e] = (u << 32) | v;
    keys[2 * e + 1] = (v << 32) | u;
    vals[2 * e] = e;
    vals[2 * e + 1] = e;
  }
}
__global__ void k_dense_cols(const unsigned long long* __restrict__ keys, int64_t s,
                             int64_t* __restrict__ col) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < s;
       i += (int64_t)gridDim.x * blockDim.x)
    col[i] = (int64_t)(keys[i] & 0xffffffffu);
}
__global__ void k_edges_i64(const int32_t* __restrict__ eu, const int32_t* __restrict__ ev,
                            int64_t m, int64_t* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    out[2 * e] = eu[e];
    out[2 * e + 1] = ev[e];
  }
}
__global__ void k_dense_degrees(const int32_t* __restrict__ deg_rank,
                                const int32_t* __restrict__ d2r, int64_t n,
                                int64_t* __restrict__ out) {
  for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d < n;
       d += (int64_t)gridDim.x * blockDim.x)
    out[d] = deg_rank[d2r[d]];
}
}  // namespace

void export_graph(const DevGraph& g, int64_t* edges, int64_t* orig_ids, int64_t* indptr,
                  int64_t* indices, int64_t* slot_ids, int64_t* degrees, cudaStream_t s) {
  const int64_t n = g.n, m = g.m;
  if (edges && m) {
    DBuf<int64_t> t;
    t.alloc(2 * m, s);
    k_edges_i64<<<grid_for(m), 256, 0, s>>>(g.eu.p, g.ev.p, m, t.p);
    GD_CUDA(cudaMemcpyAsync(edges, t.p, 2 * m * 8, cudaMemcpyDeviceToHost, s));
    GD_CUDA(cudaStreamSynchronize(s));
  }
  if (orig_ids) {
    if (g.orig.n) {
      GD_CUDA(cudaMemcpyAsync(orig_ids, g.orig.p, n * 8, cudaMemcpyDeviceToHost, s));
    } else {
      for (int64_t i = 0; i < n; i++) orig_ids[i] = i;
    }
  }
  DBuf<int64_t> degd;
  if ((degrees || indptr) && n) {
    degd.alloc(n, s);
    k_dense_degrees<<<grid_for(n), 256, 0, s>>>(g.deg.p, g.d2r.p, n, degd.p);
    GD_LAUNCH_CHECK("dense_degrees");
  }
  if (degrees && n)
    GD_CUDA(cudaMemcpyAsync(degrees, degd.p, n * 8, cudaMemcpyDeviceToHost, s));
  if (indptr) {
    DBuf<int64_t> ip;
    ip.alloc(n + 1, s);
    if (n) exclusive_scan_i64(degd.p, ip.p, n, s);
    int64_t two_m = 2 * m;
    GD_CUDA(cudaMemcpyAsync(ip.p + n, &two_m, 8, cudaMemcpyHostToDevice, s));
    GD_CUDA(cudaMemcpyAsync(indptr, ip.p, (n + 1) * 8, cudaMemcpyDeviceToHost, s));
    GD_CUDA(cudaStreamSynchronize(s));
  }
  if ((indices || slot_ids) && m) {
    DBuf<unsigned long long> k1, k2;
    DBuf<int64_t> v1, v2;
    k1.alloc(2 * m, s);
    k2.alloc(2 * m, s);
    v1.alloc(2 * m, s);
    v2.alloc(2 * m, s);
    k_dense_slot_keys<<<grid_for(m), 256, 0, s>>>(g.eu.p, g.ev.p, m, k1.p, v1.p);
    sort_pairs<int64_t>(k1.p, k2.p, v1.p, v2.p, 2 * m, 64, s);
    if (indices) {
      k_dense_cols<<<grid_for(2 * m), 256, 0, s>>>(k2.p, 2 * m, v1.p);
      GD_CUDA(cudaMemcpyAsync(indices, v1.p, 2 * m * 8, cudaMemcpyDeviceToHost, s));
    }
    if (slot_ids) GD_CUDA(cudaMemcpyAsync(slot_ids, v2.p, 2 * m * 8, cudaMemcpyDeviceToHost, s));
    GD_CUDA(cudaStreamSynchronize(s));
  }
  GD_CUDA(cudaStreamSynchronize(s));
}

}  // namespace gd
