// extern "C" boundary of libgdgpu.so (declared in include/gd_api.h).
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <algorithm>
#include <mutex>
#include <vector>

#include "gd_build.cuh"
#include "gd_count.cuh"
#include "gd_parse.cuh"
#include "gd_derive.cuh"
#include "gd_rank.cuh"
#include "gd_select.cuh"

struct gd_graph {
  gd::DevGraph g;
  cudaStream_t s = nullptr;
  // censuses of one graph from several host threads run one at a time (the
  // graph's stream, cached schedule sizes and last timings / stats are
  // per graph); read-only calls (export, derive, rank) need no lock
  mutable std::mutex mu;
  std::vector<float> ms;
  std::string names;
  std::vector<int64_t> stats;
  std::string stats_names;
};

// NCCL is resolved at gd_comm_init (dlopen), so the library loads on hosts
// and in processes without it; the data-path collectives are ncclAllReduce
// (sum of per-slot uint64 counters) and ncclAllGather (128-bit totals).
struct NcclApi {
  ncclResult_t (*getUniqueId)(ncclUniqueId*);
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t);
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t);
  ncclResult_t (*reduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                                ncclComm_t, cudaStream_t);
  ncclResult_t (*commDestroy)(ncclComm_t);
  const char* (*getErrorString)(ncclResult_t);
};

struct gd_comm {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
};

namespace gd {

static thread_local std::string t_last_error;

static const NcclApi& nccl() {
  static NcclApi api{};
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = "cannot dlopen libnccl.so.2";
      return;
    }
    api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
    api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
    api.allReduce = (decltype(api.allReduce))dlsym(h, "ncclAllReduce");
    api.allGather = (decltype(api.allGather))dlsym(h, "ncclAllGather");
    api.reduceScatter = (decltype(api.reduceScatter))dlsym(h, "ncclReduceScatter");
    api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
    api.getErrorString = (decltype(api.getErrorString))dlsym(h, "ncclGetErrorString");
  });
  if (!api.allReduce || !api.reduceScatter)
    throw Error(GD_ECUDA, err.empty() ? "NCCL symbols missing" : err);
  return api;
}

#define GD_NCCL(call)                                                             \
  do {                                                                            \
    ncclResult_t _r = (call);                                                     \
    if (_r != ncclSuccess)                                                        \
      throw ::gd::Error(GD_ECUDA, std::string(#call) + ": " + nccl().getErrorString(_r)); \
  } while (0)
thread_local long long g_launches = 0;

int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
        sms <= 0)
      sms = 148;
  }
  return sms;
}

static void init_pool_once() {
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;  // keep freed blocks cached across calls
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);

    }
  });
}

// Headroom in the stream-ordered pool.  The census workspace stays allocated
// between calls, so with the pool reserved only up to its high-water mark the
// transient buffers of the next graph build and census (sort temporaries,
// the device table) must fit in the few GB left beside it; measured: the
// build of a fresh R-MAT-20 graph then stalls for 150-480 ms in every few
// calls, and never once the pool holds spare reserve.  After a census the
// pool is grown (once per new high-water mark) to used_high + min(used_high
// / 2, 16 GiB); gd_trim_workspace() gives everything back.
static void ensure_pool_headroom(cudaStream_t s) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) return;
  uint64_t used_high = 0, reserved = 0;
  cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &used_high);
  cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
  const uint64_t target = used_high + std::min<uint64_t>(used_high / 2, 16ull << 30);
  if (reserved >= target) return;
  void* p = nullptr;
  if (cudaMallocAsync(&p, target - reserved, s) == cudaSuccess) {
    cudaFreeAsync(p, s);
    cudaStreamSynchronize(s);
  } else {
    cudaGetLastError();  // not enough free memory for the headroom: run without it
  }
  // the padding allocation is not real use: reset the high-water mark (to
  // the current use) so the next target follows the censuses, not this padding
  uint64_t zero = 0;
  if (cudaMemPoolSetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &zero) != cudaSuccess)
    cudaGetLastError();
}

std::map<std::string, WsBuf>& thread_workspace() {
  static thread_local std::map<std::string, WsBuf> w;
  return w;
}

// Graph streams are recycled through a small process-wide pool instead of
// being created and destroyed with every graph (a fresh graph per call is the
// common service pattern; stream creation / destruction is driver work on the
// host path of every call).
static std::mutex g_stream_mu;
static std::vector<cudaStream_t> g_stream_pool;

static cudaStream_t acquire_stream() {
  {
    std::lock_guard<std::mutex> lock(g_stream_mu);
    if (!g_stream_pool.empty()) {
      cudaStream_t s = g_stream_pool.back();
      g_stream_pool.pop_back();
      return s;
    }
  }
  cudaStream_t s = nullptr;
  GD_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  return s;
}

static void release_stream(cudaStream_t s) {  // s is idle (synchronized)
  std::lock_guard<std::mutex> lock(g_stream_mu);
  if (g_stream_pool.size() < 64) g_stream_pool.push_back(s);
  else cudaStreamDestroy(s);
}

static cudaStream_t thread_stream() {
  static thread_local cudaStream_t s = nullptr;
  if (!s) GD_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  return s;
}

template <typename F>
static int guarded(F&& f) {
  try {
    init_pool_once();
    f();
    return GD_OK;
  } catch (const Error& e) {
    t_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    t_last_error = "host allocation failed";
    return GD_ECAPACITY;
  } catch (const std::exception& e) {
    t_last_error = e.what();
    return GD_ECUDA;
  }
}

typedef unsigned __int128 u128;

static u128 get128(const unsigned long long* p) { return ((u128)p[1] << 64) | p[0]; }
static void put128(uint64_t* p, u128 v) {
  p[0] = (uint64_t)v;
  p[1] = (uint64_t)(v >> 64);
}

// Fill in / check the 4-clique and 4-cycle fields from the device totals.
//   sum_e cl(e) = 6 K4;  sum_e cy(e) = 4 * (#4-cycles - sum_e C(t,2) + 3 K4)
// (each 4-clique holds 3 four-cycles, each diamond one; diamonds =
// sum_e C(t,2) - 6 K4, close_quads census.py:399-403).
static void close_cycles(uint64_t* sums, const CensusExtras& ex, int64_t G, bool per_edge) {
  for (int64_t i = 0; i < G; i++) {
    uint64_t* s = sums + i * 2 * kNumSums;
    const u128 k4 = ex.k4tot[i];
    const u128 c4x2 = ex.c4tot2[i];
    if (c4x2 & 1) throw Error(GD_ECONSISTENCY, "odd 4-cycle wedge-pair total");
    const u128 c4 = c4x2 >> 1;
    const u128 ntt = get128((const unsigned long long*)(s + 2 * 5));
    if (get128((const unsigned long long*)(s + 2 * 3)) != 6 * k4)
      throw Error(GD_ECONSISTENCY, "per-edge 4-clique sum != 6 x enumerated 4-cliques");
    if (c4 + 3 * k4 < ntt) throw Error(GD_ECONSISTENCY, "negative induced 4-cycle count");
    const u128 cy = 4 * (c4 + 3 * k4 - ntt);
    if (per_edge) {
      if (get128((const unsigned long long*)(s + 2 * 4)) != cy)
        throw Error(GD_ECONSISTENCY, "per-edge 4-cycle sum != 4 x enumerated 4-cycles");
    } else {
      put128(s + 2 * 4, cy);
    }
  }
}

static void store_timings(gd_graph* h, CensusExtras& ex) {
  h->ms = ex.ms;
  h->names.clear();
  for (auto& n : ex.names) h->names += n + "\n";
  h->stats = ex.stats;
  h->stats_names.clear();
  for (auto& n : ex.stats_names) h->stats_names += n + "\n";
}

static void census(gd_graph* h, bool per_edge, int64_t* table, int flags, uint64_t* sums,
                   int64_t* seen, const Shard& shard = Shard()) {
  std::lock_guard<std::mutex> lock(h->mu);
  static const bool prof = getenv("GD_HOST_PROFILE") != nullptr;
  std::vector<std::pair<const char*, std::chrono::steady_clock::time_point>> tp;
  auto mark = [&](const char* w) {
    if (prof) tp.push_back({w, std::chrono::steady_clock::now()});
  };
  mark("start");
  DevGraph& g = h->g;
  cudaStream_t s = h->s;
  const int64_t G = g.G;
  DBuf<unsigned long long> dsums, dseen;
  dsums.alloc(G * 2 * kNumSums, s);
  dseen.alloc(G, s);
  DBuf<long long> dtable;
  long long* tptr = nullptr;
  // a real multi-GPU census writes only this rank's rows (shard_rows)
  int64_t r0 = 0, r1 = g.m;
  if (shard.real() && G == 1) shard_rows(g.m, shard.rank, shard.world, &r0, &r1);
  if (per_edge && table) {
    if (flags & GD_OUTPUT_DEVICE) {
      tptr = (long long*)table;
    } else {
      dtable.alloc((size_t)std::max<int64_t>(r1 - r0, 1) * kNumMicro, s);
      tptr = dtable.p;
    }
  }
  CensusExtras ex;
  // a page-locked host table (the default path's pooled blocks) is filled
  // chunk by chunk from inside the census, overlapped with the finalize
  if (dtable.p && r0 == 0 && r1 == g.m && G == 1 && !shard.real() && host_is_pinned(table))
    ex.host_table = table;
  mark("alloc");
  run_census(g, per_edge, tptr, dsums.p, dseen.p, ex, s, shard);
  mark("run_census");
  if (ex.rows >= 0 && (ex.row0 != r0 || ex.rows != r1 - r0))
    throw Error(GD_ECUDA, "shard row range mismatch");
  // sums and counts through this thread's page-locked result block
  const size_t ns = (size_t)G * 2 * kNumSums;
  uint64_t* pin = (uint64_t*)host_results((ns + G) * 8);
  GD_CUDA(cudaMemcpyAsync(pin, dsums.p, ns * 8, cudaMemcpyDeviceToHost, s));
  GD_CUDA(cudaMemcpyAsync(pin + ns, dseen.p, G * 8, cudaMemcpyDeviceToHost, s));
  if (dtable.p && r1 > r0 && !ex.table_copied)
    copy_d2h(table, dtable.p, (size_t)(r1 - r0) * kNumMicro * 8, s);
  GD_CUDA(cudaStreamSynchronize(s));
  mark("d2h");
  store_timings(h, ex);
  ensure_pool_headroom(s);
  mark("headroom");
  if (!ex.direct) close_cycles(pin, ex, G, per_edge);
  if (sums) std::memcpy(sums, pin, ns * 8);
  if (seen) std::memcpy(seen, pin + ns, G * 8);
  if (prof) {
    for (size_t i = 1; i < tp.size(); i++)
      fprintf(stderr, "%s %.1f us  ", tp[i].first,
              std::chrono::duration<double, std::micro>(tp[i].second - tp[i - 1].second).count());
    fprintf(stderr, "\n");
  }
}

}  // namespace gd

using namespace gd;

extern "C" {

const char* gd_last_error(void) { return t_last_error.c_str(); }

int gd_version(void) { return 1; }

int gd_device_ok(void) {
  int c = 0;
  return (cudaGetDeviceCount(&c) == cudaSuccess && c > 0) ? 1 : 0;
}

int gd_graph_create(const int64_t* pairs, int64_t k, int64_t n, int ids_mode, int flags,
                    gd_graph** out) {
  if (!out) {
    t_last_error = "out is NULL";
    return GD_EINVAL;
  }
  *out = nullptr;
  if (k > 0 && !pairs) {
    t_last_error = "pairs is NULL";
    return GD_EINVAL;
  }
  gd_graph* h = new gd_graph();
  int rc = guarded([&] {
    h->s = acquire_stream();
    build_graph(h->g, pairs, k, n, ids_mode, flags, h->s);
  });
  if (rc != GD_OK) {
    gd_graph_free(h);
    return rc;
  }
  *out = h;
  return GD_OK;
}

int gd_graph_create_batch(const int64_t* pairs, const int64_t* pair_offsets,
                          const int64_t* n_per_graph, int64_t num_graphs, int flags,
                          gd_graph** out) {
  if (!out || !pair_offsets || !n_per_graph) {
    t_last_error = "NULL argument";
    return GD_EINVAL;
  }
  *out = nullptr;
  gd_graph* h = new gd_graph();
  int rc = guarded([&] {
    h->s = acquire_stream();
    build_graph_batch(h->g, pairs, pair_offsets, n_per_graph, num_graphs, flags, h->s);
  });
  if (rc != GD_OK) {
    gd_graph_free(h);
    return rc;
  }
  *out = h;
  return GD_OK;
}

int gd_graph_create_batch_list(const int64_t* const* lists, const int64_t* pair_offsets,
                               const int64_t* n_per_graph, int64_t num_graphs, int flags,
                               gd_graph** out) {
  if (!out || !pair_offsets || !n_per_graph || (num_graphs > 0 && !lists)) {
    t_last_error = "NULL argument";
    return GD_EINVAL;
  }
  *out = nullptr;
  gd_graph* h = new gd_graph();
  int rc = guarded([&] {
    h->s = acquire_stream();
    const int64_t k = num_graphs > 0 ? pair_offsets[num_graphs] - pair_offsets[0] : 0;
    if (k < 0 || (num_graphs > 0 && pair_offsets[0] != 0))
      throw Error(GD_EINVAL, "bad pair_offsets");
    for (int64_t i = 0; i < num_graphs; i++)
      if (pair_offsets[i + 1] < pair_offsets[i]) throw Error(GD_EINVAL, "bad pair_offsets");
    // the per-graph arrays are gathered into page-locked staging by all host
    // cores in blocks of ~8 MB; the DMA of a block runs while the next is gathered
    static const bool prof = getenv("GD_HOST_PROFILE") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    int64_t* flat = (int64_t*)host_staging((size_t)std::max<int64_t>(k, 1) * 16);
    DBuf<long long> dpairs;
    dpairs.alloc((size_t)std::max<int64_t>(2 * k, 2), h->s);
    for (int64_t g0 = 0; g0 < num_graphs;) {
      int64_t g1 = g0 + 1;
      while (g1 < num_graphs && pair_offsets[g1] - pair_offsets[g0] < (int64_t)(8 << 20) / 16) g1++;
      gather_pairs(lists, pair_offsets, g0, g1, flat);
      const int64_t a = pair_offsets[g0], b = pair_offsets[g1];
      if (b > a)
        GD_CUDA(cudaMemcpyAsync(dpairs.p + 2 * a, flat + 2 * a, (size_t)(b - a) * 16,
                                cudaMemcpyHostToDevice, h->s));
      g0 = g1;
    }
    const auto t1 = std::chrono::steady_clock::now();
    if (prof) GD_CUDA(cudaStreamSynchronize(h->s));
    const auto t2 = std::chrono::steady_clock::now();
    build_graph_batch(h->g, (const int64_t*)dpairs.p, pair_offsets, n_per_graph, num_graphs,
                      flags | GD_INPUT_DEVICE, h->s);
    if (prof) {
      const auto t3 = std::chrono::steady_clock::now();
      auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
      fprintf(stderr, "batch_list: gather+issue %.0f us  h2d drain %.0f us  build %.0f us\n",
              us(t0, t1), us(t1, t2), us(t2, t3));
    }
  });
  if (rc != GD_OK) {
    gd_graph_free(h);
    return rc;
  }
  *out = h;
  return GD_OK;
}

int gd_graph_info(const gd_graph* h, int64_t* n, int64_t* m, int64_t* num_graphs) {
  if (!h) {
    t_last_error = "NULL graph";
    return GD_EINVAL;
  }
  if (n) *n = h->g.n;
  if (m) *m = h->g.m;
  if (num_graphs) *num_graphs = h->g.G;
  return GD_OK;
}

int gd_graph_sizes(const gd_graph* h, int64_t* n_per_graph, int64_t* m_per_graph) {
  if (!h) {
    t_last_error = "NULL graph";
    return GD_EINVAL;
  }
  for (int64_t i = 0; i < h->g.G; i++) {
    if (n_per_graph) n_per_graph[i] = h->g.h_gn[i];
    if (m_per_graph) m_per_graph[i] = h->g.h_eoff[i + 1] - h->g.h_eoff[i];
  }
  return GD_OK;
}

int gd_graph_export(const gd_graph* h, int64_t* edges, int64_t* orig_ids, int64_t* indptr,
                    int64_t* indices, int64_t* edge_slot_ids, int64_t* degrees) {
  if (!h) {
    t_last_error = "NULL graph";
    return GD_EINVAL;
  }
  return guarded([&] {
    export_graph(h->g, edges, orig_ids, indptr, indices, edge_slot_ids, degrees, h->s);
  });
}

void gd_graph_free(gd_graph* h) {
  if (!h) return;
  if (h->s) cudaStreamSynchronize(h->s);
  {
    // release device buffers before the stream goes away
    gd::DevGraph empty;
    std::swap(h->g, empty);
  }
  if (h->s) {
    cudaStreamSynchronize(h->s);
    release_stream(h->s);
  }
  delete h;
}

int gd_census_global(gd_graph* h, uint64_t* sums, int64_t* edges_seen) {
  if (!h) {
    t_last_error = "NULL graph";
    return GD_EINVAL;
  }
  return guarded([&] { census(h, false, nullptr, 0, sums, edges_seen); });
}

int gd_census_per_edge(gd_graph* h, int64_t* table, int flags, uint64_t* sums,
                       int64_t* edges_seen) {
  if (!h) {
    t_last_error = "NULL graph";
    return GD_EINVAL;
  }
  return guarded([&] { census(h, true, table, flags, sums, edges_seen); });
}

int gd_sums_from_table(const int64_t* table, int64_t m, int64_t n, int flags, uint64_t* sums) {
  if ((m > 0 && !table) || !sums || m < 0) {
    t_last_error = "bad argument";
    return GD_EINVAL;
  }
  return guarded([&] {
    cudaStream_t s = thread_stream();
    DBuf<long long> dt;
    const long long* tp = (const long long*)table;
    if (!(flags & GD_INPUT_DEVICE) && m) {
      dt.alloc((size_t)m * kNumMicro, s);
      GD_CUDA(cudaMemcpyAsync(dt.p, table, (size_t)m * kNumMicro * 8, cudaMemcpyHostToDevice, s));
      tp = dt.p;
    }
    DBuf<unsigned long long> ds;
    ds.alloc(2 * kNumSums, s);
    sums_from_table(tp, m, n, ds.p, s);
    GD_CUDA(cudaMemcpyAsync(sums, ds.p, 2 * kNumSums * 8, cudaMemcpyDeviceToHost, s));
    GD_CUDA(cudaStreamSynchronize(s));
  });
}

int gd_census_global_edges(const int64_t* edges, int64_t m, int64_t n, int flags, uint64_t* sums,
                           int64_t* edges_seen) {
  gd_graph* h = nullptr;
  int rc = gd_graph_create(edges, m, n, GD_IDS_SANITIZED, flags & GD_INPUT_DEVICE, &h);
  if (rc != GD_OK) return rc;
  rc = gd_census_global(h, sums, edges_seen);
  gd_graph_free(h);
  return rc;
}

int gd_census_per_edge_edges(const int64_t* edges, int64_t m, int64_t n, int flags,
                             int64_t* table, uint64_t* sums, int64_t* edges_seen) {
  gd_graph* h = nullptr;
  int rc = gd_graph_create(edges, m, n, GD_IDS_SANITIZED, flags & GD_INPUT_DEVICE, &h);
  if (rc != GD_OK) return rc;
  rc = gd_census_per_edge(h, table, flags & GD_OUTPUT_DEVICE, sums, edges_seen);
  gd_graph_free(h);
  return rc;
}

int gd_comm_unique_id(unsigned char* id_out) {
  if (!id_out) {
    t_last_error = "id_out is NULL";
    return GD_EINVAL;
  }
  return guarded([&] {
    ncclUniqueId id;
    GD_NCCL(nccl().getUniqueId(&id));
    std::memcpy(id_out, id.internal, NCCL_UNIQUE_ID_BYTES);
  });
}

int gd_comm_init(const unsigned char* id_in, int rank, int world, gd_comm** out) {
  if (!id_in || !out || world < 1 || rank < 0 || rank >= world) {
    t_last_error = "bad communicator arguments";
    return GD_EINVAL;
  }
  *out = nullptr;
  gd_comm* c = new gd_comm();
  int rc = guarded([&] {
    ncclUniqueId id;
    std::memcpy(id.internal, id_in, NCCL_UNIQUE_ID_BYTES);
    GD_NCCL(nccl().commInitRank(&c->comm, world, id, rank));
    c->rank = rank;
    c->world = world;
  });
  if (rc != GD_OK) {
    delete c;
    return rc;
  }
  *out = c;
  return GD_OK;
}

void gd_comm_free(gd_comm* c) {
  if (!c) return;
  if (c->comm) {
    try {
      nccl().commDestroy(c->comm);
    } catch (...) {
    }
  }
  delete c;
}

int gd_census_sharded(gd_graph* h, gd_comm* c, int virtual_ranks, int per_edge, int64_t* table,
                      int flags, uint64_t* sums, int64_t* edges_seen) {
  if (!h || (!c && virtual_ranks < 1)) {
    t_last_error = "bad sharding arguments";
    return GD_EINVAL;
  }
  return guarded([&] {
    Shard sh;
    if (c) {
      sh.rank = c->rank;
      sh.world = c->world;
      cudaStream_t s = h->s;
      ncclComm_t comm = c->comm;
      sh.allreduce = [s, comm](unsigned long long* p, size_t count) {
        GD_NCCL(nccl().allReduce(p, p, count, ncclUint64, ncclSum, comm, s));
      };
      sh.allgather = [s, comm](const unsigned long long* in, unsigned long long* out,
                               size_t count) {
        GD_NCCL(nccl().allGather(in, out, count, ncclUint64, comm, s));
      };
      sh.reduce_scatter = [s, comm](const void* in, void* out, size_t count, int esz) {
        GD_NCCL(nccl().reduceScatter(in, out, count, esz == 4 ? ncclUint32 : ncclUint64,
                                     ncclSum, comm, s));
      };
    } else {
      sh.world = virtual_ranks;
    }
    census(h, per_edge != 0, table, flags, sums, edges_seen, sh);
  });
}

int gd_shard_rows(int64_t m, int rank, int world, int64_t* e0, int64_t* e1) {
  if (!e0 || !e1 || world < 1 || rank < 0 || rank >= world || m < 0) {
    t_last_error = "bad shard arguments";
    return GD_EINVAL;
  }
  shard_rows(m, rank, world, e0, e1);
  return GD_OK;
}

// Closures of census.py:388-430 in exact 128-bit integers, for many graphs
// at once (the batched feature path).  Each status is 0, or 1 + the index of
// the first failing identity (a ConsistencyError in the reference).
int gd_close_counts(const uint64_t* sums, const int64_t* n_per_graph, const int64_t* m_per_graph,
                    int64_t num_graphs, int64_t* counts, int* status) {
  if (!sums || !n_per_graph || !m_per_graph || !counts || !status || num_graphs < 0) {
    t_last_error = "bad argument";
    return GD_EINVAL;
  }
  typedef __int128 i128;
  auto comb = [](i128 n, int k) -> i128 {
    if (n < k) return 0;
    i128 r = 1;
    for (int i = 0; i < k; i++) r = r * (n - i) / (i + 1);
    return r;
  };
  for (int64_t gi = 0; gi < num_graphs; gi++) {
    const uint64_t* sp = sums + gi * 2 * kNumSums;
    i128 v[kNumSums];
    for (int k = 0; k < kNumSums; k++) v[k] = (i128)(((unsigned __int128)sp[2 * k + 1] << 64) | sp[2 * k]);
    const i128 n = n_per_graph[gi], m = m_per_graph[gi];
    int st = 0, step = 0;
    auto div = [&](i128 x, int d) -> i128 {
      step++;
      if (st) return 0;
      if (x % d != 0 || x < 0) st = step;
      return x / d;
    };
    auto nn = [&](i128 x) -> i128 {
      step++;
      if (!st && x < 0) st = step;
      return x;
    };
    // CensusSums.FIELDS: tri star indep3 clique4 cycle4 n_tt n_susv n_ts n_ss_same n_ti n_si n_ii outside
    const i128 f31 = div(v[0], 3), f32 = div(v[1], 2), f33 = nn(v[2]);
    const i128 f34 = nn(comb(n, 3) - f31 - f32 - f33);
    const i128 f41 = div(v[3], 6);
    const i128 f42 = nn(v[5] - 6 * f41);
    const i128 f44 = div(v[4], 4);
    const i128 f46 = nn(v[6] - 4 * f44);
    const i128 f43 = div(v[7] - 4 * f42, 2);
    const i128 f45 = div(v[8] - f43, 3);
    const i128 f47 = div(v[9] - f43, 3);
    const i128 f48 = div(v[10] - 2 * f46, 2);
    const i128 f49 = div(v[12] - 6 * f41 - 4 * f42 - 2 * f43 - 4 * f44 - 2 * f46, 2);
    const i128 f410 = nn(v[11] - 2 * f49);
    const i128 f411 =
        nn(comb(n, 4) - (f41 + f42 + f43 + f44 + f45 + f46 + f47 + f48 + f49 + f410));
    const i128 out[17] = {m, comb(n, 2) - m, f31, f32, f33, f34, f41, f42, f43,
                          f44, f45, f46, f47, f48, f49, f410, f411};
    for (int c = 0; c < 17; c++) {
      counts[gi * 34 + 2 * c] = (int64_t)(uint64_t)out[c];
      counts[gi * 34 + 2 * c + 1] = (int64_t)(out[c] >> 64);
    }
    status[gi] = st;
  }
  return GD_OK;
}

int gd_graph_timings(const gd_graph* h, float* ms, int capacity, const char** names) {
  if (!h) return 0;
  std::lock_guard<std::mutex> lock(h->mu);
  int k = (int)std::min<size_t>(h->ms.size(), (size_t)std::max(capacity, 0));
  for (int i = 0; i < k; i++) ms[i] = h->ms[i];
  if (names) *names = h->names.c_str();
  return k;
}

int gd_graph_stats(const gd_graph* h, int64_t* values, int capacity, const char** names) {
  if (!h) return 0;
  std::lock_guard<std::mutex> lock(h->mu);
  int k = (int)std::min<size_t>(h->stats.size(), (size_t)std::max(capacity, 0));
  for (int i = 0; i < k; i++) values[i] = h->stats[i];
  if (names) *names = h->stats_names.c_str();
  return k;
}

int gd_set_device(int device) {
  return guarded([&] { GD_CUDA(cudaSetDevice(device)); });
}

void* gd_device_alloc(int64_t bytes) {
  void* p = nullptr;
  if (bytes <= 0) return nullptr;
  if (cudaMalloc(&p, (size_t)bytes) != cudaSuccess) {
    t_last_error = "cudaMalloc failed";
    return nullptr;
  }
  return p;
}

void gd_device_free(void* p) {
  if (p) cudaFree(p);
}

void* gd_host_alloc(int64_t bytes) {
  void* p = nullptr;
  if (bytes <= 0) return nullptr;
  if (cudaHostAlloc(&p, (size_t)bytes, cudaHostAllocDefault) != cudaSuccess) {
    t_last_error = "cudaHostAlloc failed";
    return nullptr;
  }
  return p;
}

void gd_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int gd_flush_l2(void) {
  return guarded([&] {
    static void* buf = nullptr;
    const size_t bytes = 256ull << 20;  // 2x the 126 MB L2
    cudaStream_t s = thread_stream();
    if (!buf) GD_CUDA(cudaMalloc(&buf, bytes));
    GD_CUDA(cudaMemsetAsync(buf, (int)(rand() & 0xff), bytes, s));
    GD_CUDA(cudaStreamSynchronize(s));
  });
}

struct gd_parsed {
  gd::ParseOut out;
};

int gd_parse_edge_list(const char* text, int64_t len, const char* const* prefixes,
                       int nprefixes, int flags, gd_parsed** out) {
  if (!out || (len > 0 && !text) || (nprefixes > 0 && !prefixes)) {
    t_last_error = "NULL argument";
    return GD_EINVAL;
  }
  *out = nullptr;
  gd_parsed* p = new gd_parsed();
  const int rc = guarded([&] {
    cudaStream_t s = thread_stream();
    parse_edge_list(text, len, prefixes, nprefixes, (flags & GD_PARSE_CR_NEWLINE) ? 1 : 0,
                    (flags & GD_PARSE_MM_SHIFT) ? 1 : 0, p->out, s);
  });
  if (rc != GD_OK) {
    delete p;
    return rc;
  }
  *out = p;
  return GD_OK;
}

int gd_parsed_info(const gd_parsed* p, int64_t* info) {
  if (!p || !info) {
    t_last_error = "NULL argument";
    return GD_EINVAL;
  }
  for (int k = 0; k < 12; k++) info[k] = p->out.info[k];
  return GD_OK;
}

const int64_t* gd_parsed_pairs(const gd_parsed* p) { return p ? p->out.pairs.p : nullptr; }

void gd_parsed_free(gd_parsed* p) {
  if (!p) return;
  if (p->out.pairs.p) cudaStreamSynchronize(p->out.pairs.s);
  delete p;
}

static const char* kNegNames[10] = {"tt0", "susv0", "ts0", "ss0", "ti0",
                                    "ti1", "si0", "si1", "ii0", "ii1"};

static void set_bad(int64_t hb, int64_t* bad) {
  if (bad) *bad = hb;
  if (hb >= 0)
    throw Error(GD_ECONSISTENCY, std::string("negative micro count ") + kNegNames[hb & 15] +
                                     " on edge " + std::to_string(hb >> 4));
}

int gd_micro_roles(const gd_graph* h, const int64_t* table, int flags, const int64_t* orig_ids,
                   int64_t* roles, int64_t* bad) {
  if (!h || (h->g.m && (!table || !roles)) || (h->g.n && !orig_ids)) {
    t_last_error = "NULL argument";
    return GD_EINVAL;
  }
  return guarded([&] {
    const int64_t hb = micro_roles(h->g, (const long long*)table, (flags & GD_INPUT_DEVICE) != 0,
                                   orig_ids, (long long*)roles, thread_stream());
    set_bad(hb, bad);
  });
}

struct gd_text {
  gd::CsvText csv;
};

int gd_micro_csv(const gd_graph* h, const int64_t* table, int flags, const int64_t* orig_ids,
                 gd_text** out, int64_t* bad) {
  if (!h || !out || (h->g.m && !table) || (h->g.n && !orig_ids)) {
    t_last_error = "NULL argument";
    return GD_EINVAL;
  }
  *out = nullptr;
  gd_text* t = new gd_text();
  const int rc = guarded([&] {
    const int64_t hb = micro_csv(h->g, (const long long*)table, (flags & GD_INPUT_DEVICE) != 0,
                                 orig_ids, t->csv, thread_stream());
    set_bad(hb, bad);
  });
  if (rc != GD_OK) {
    delete t;
    return rc;
  }
  *out = t;
  return GD_OK;
}

int64_t gd_text_size(const gd_text* t) { return t ? t->csv.bytes : 0; }

int gd_text_copy(const gd_text* t, int64_t offset, int64_t len, char* host) {
  if (!t || offset < 0 || len < 0 || offset + len > t->csv.bytes || (len && !host)) {
    t_last_error = "bad text range";
    return GD_EINVAL;
  }
  return guarded([&] {
    if (len) GD_CUDA(cudaMemcpy(host, t->csv.text.p + offset, len, cudaMemcpyDeviceToHost));
  });
}

void gd_text_free(gd_text* t) {
  if (!t) return;
  if (t->csv.text.p) cudaStreamSynchronize(t->csv.text.s);
  delete t;
}

static bool check_table_args(const gd_graph* h, const int64_t* table, int pattern) {
  if (!h || (h->g.m && !table)) {
    t_last_error = "NULL argument";
    return false;
  }
  if (pattern < 0 || pattern > 3) {
    t_last_error = "unknown pattern";
    return false;
  }
  return true;
}

int gd_edge_weights(const gd_graph* h, const int64_t* table, int flags, int pattern,
                    int64_t* weights) {
  if (!check_table_args(h, table, pattern) || (h->g.m && !weights)) return GD_EINVAL;
  return guarded([&] {
    edge_weights(h->g, (const long long*)table, (flags & GD_INPUT_DEVICE) != 0, pattern, weights,
                 thread_stream());
  });
}

int gd_rank_edges(const gd_graph* h, const int64_t* table, int flags, int pattern, int64_t k,
                  int64_t* index, int64_t* u, int64_t* v, int64_t* weight) {
  if (!check_table_args(h, table, pattern)) return GD_EINVAL;
  const int64_t kk = (k < 0 || k > h->g.m) ? h->g.m : k;
  if (kk && (!index || !u || !v || !weight)) {
    t_last_error = "NULL output";
    return GD_EINVAL;
  }
  return guarded([&] {
    rank_edges(h->g, (const long long*)table, (flags & GD_INPUT_DEVICE) != 0, pattern, kk, index,
               u, v, weight, thread_stream());
  });
}

int gd_vertex_triangles(const gd_graph* h, const int64_t* table, int flags, int64_t* per_vertex) {
  if (!check_table_args(h, table, 0) || (h->g.n && !per_vertex)) return GD_EINVAL;
  return guarded([&] {
    vertex_triangles(h->g, (const long long*)table, (flags & GD_INPUT_DEVICE) != 0, per_vertex,
                     thread_stream());
  });
}

struct gd_selection {
  gd::Selection* sel = nullptr;
};

int gd_selection_create(const gd_graph* h, gd_selection** out) {
  if (!h || !out) {
    t_last_error = "NULL argument";
    return GD_EINVAL;
  }
  *out = nullptr;
  gd_selection* p = new gd_selection();
  const int rc = guarded([&] { p->sel = new gd::Selection(h->g, h->s); });
  if (rc != GD_OK) {
    delete p;
    return rc;
  }
  *out = p;
  return GD_OK;
}

int gd_selection_apply(gd_selection* p, int action, int64_t a, uint64_t* moments) {
  if (!p || !p->sel) {
    t_last_error = "NULL selection";
    return GD_EINVAL;
  }
  return guarded([&] { p->sel->apply(action, a, moments); });
}

void gd_selection_free(gd_selection* p) {
  if (!p) return;
  delete p->sel;
  delete p;
}

int gd_trim_workspace(void) {
  return guarded([&] {
    cudaStream_t s = thread_stream();
    GD_CUDA(cudaStreamSynchronize(s));
    GD_CUDA(cudaDeviceSynchronize());
    thread_workspace().clear();
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess)
      cudaMemPoolTrimTo(pool, 0);  // and the pool's spare reserve
  });
}

// Device memory pool of the library's allocations: [0] reserved bytes,
// [1] reserved high-water mark, [2] used bytes, [3] used high-water mark.
int gd_pool_stats(uint64_t* out) {
  if (!out) {
    t_last_error = "out is NULL";
    return GD_EINVAL;
  }
  return guarded([&] {
    int dev = 0;
    GD_CUDA(cudaGetDevice(&dev));
    cudaMemPool_t pool;
    GD_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    const cudaMemPoolAttr attrs[4] = {cudaMemPoolAttrReservedMemCurrent,
                                      cudaMemPoolAttrReservedMemHigh,
                                      cudaMemPoolAttrUsedMemCurrent, cudaMemPoolAttrUsedMemHigh};
    for (int i = 0; i < 4; i++) GD_CUDA(cudaMemPoolGetAttribute(pool, attrs[i], &out[i]));
  });
}

}  // extern "C"
