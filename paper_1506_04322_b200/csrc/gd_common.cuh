// Shared definitions of the B200 graphlet census library (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/gd_api.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libgdgpu targets sm_100a (B200) only"
#endif

namespace gd {

// ---------------------------------------------------------------------------
// Errors: C++ exceptions inside the library, mapped to status codes at the
// C-ABI boundary (gd_api.cu).
// ---------------------------------------------------------------------------
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& msg) : std::runtime_error(msg), code(c) {}
};

#define GD_CUDA(call)                                                        \
  do {                                                                       \
    cudaError_t _e = (call);                                                 \
    if (_e != cudaSuccess)                                                   \
      throw ::gd::Error(GD_ECUDA, std::string(#call) + ": " +                \
                                      cudaGetErrorString(_e));               \
  } while (0)

// Every launch of one of our kernels goes through GD_LAUNCH_CHECK, which
// also counts it (reported as the "launches" statistic of a census).
extern thread_local long long g_launches;

#define GD_LAUNCH_CHECK(what)                                                \
  do {                                                                       \
    ::gd::g_launches++;                                                      \
    cudaError_t _e = cudaGetLastError();                                     \
    if (_e != cudaSuccess)                                                   \
      throw ::gd::Error(GD_ECUDA, std::string("launch ") + (what) + ": " +   \
                                      cudaGetErrorString(_e));               \
  } while (0)

// ---------------------------------------------------------------------------
// Device buffers (stream-ordered allocations from the default pool).
// ---------------------------------------------------------------------------
template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept { *this = std::move(o); }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p; n = o.n; s = o.s;
      o.p = nullptr; o.n = 0;
    }
    return *this;
  }
  ~DBuf() { release(); }
  void alloc(size_t count, cudaStream_t stream) {
    release();
    s = stream;
    n = count;
    if (count) GD_CUDA(cudaMallocAsync((void**)&p, count * sizeof(T), stream));
  }
  void zero() {
    if (n) GD_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  size_t bytes() const { return n * sizeof(T); }
};

// Number of fields of CensusSums (census.py:359-378) and per-edge columns
// (census.py:95-97).
constexpr int kNumSums = GD_NUM_SUMS;
constexpr int kNumMicro = GD_NUM_MICRO;

// Packed per-edge triangle / 4-clique counter: t in bits [40, 64), cl in
// bits [0, 40).  One 64-bit atomic per enumerated triangle carries both.
constexpr int kTriShift = 40;
constexpr unsigned long long kClMask = (1ull << kTriShift) - 1ull;

// ---------------------------------------------------------------------------
// Device graph.  Two vertex spaces:
//   dense ids   : the reference's ids (graph.py:154-157), canonical edge order
//   rank ids    : vertices relabelled by ascending (degree, dense id); the
//                 counting kernels run here so "higher priority" == larger id
//                 and every oriented / prefix list is a contiguous row range.
// ---------------------------------------------------------------------------
struct DevGraph {
  int64_t n = 0, m = 0, G = 1;
  int max_deg = 0;
  // canonical edges (dense ids), edge e = (eu[e], ev[e]), eu < ev
  DBuf<int32_t> eu, ev;
  // rank-space symmetric CSR
  DBuf<int64_t> rp;     // [n+1]
  DBuf<int32_t> col;    // [2m] neighbour rank ids, rows strictly ascending
  DBuf<int32_t> seid;   // [2m] canonical edge id of each slot
  DBuf<int64_t> osplit; // [n] absolute slot index of the first neighbour > row
  DBuf<int64_t> e2o;    // [m] slot of edge e in the row of its lower-rank endpoint
  DBuf<int64_t> e2i;    // [m] slot of edge e in the row of its higher-rank endpoint
  DBuf<int32_t> deg;    // [n] degree by rank id
  DBuf<int32_t> r2d;    // [n] rank id -> dense id
  DBuf<int32_t> d2r;    // [n] dense id -> rank id
  DBuf<int64_t> orig;   // [n] dense id -> original id (remap mode), else empty
  // batch bookkeeping (G graphs as one disjoint union)
  DBuf<int32_t> vgraph; // [n] rank id -> graph id (empty when G == 1)
  DBuf<int64_t> eoff;   // [G+1] canonical edge offsets per graph
  DBuf<int64_t> gn;     // [G] vertex count per graph
  std::vector<int64_t> h_eoff, h_gn;
  uint64_t hit_cap = 0;      // entries of the persisted hit-list buffer
  bool hit_cap_known = false;
  uint64_t hit_cap_used = 0; // capacity the last census of this graph got
};

// Census workspace: large scratch buffers (slot accumulators, item prefixes,
// hit buffer, counter slabs) cached per host thread and reused by every
// census of every graph on that thread, so a fresh graph of the same size
// never re-allocates.  Calls are synchronous, so one thread's buffers are
// idle between calls.  Grown with stream-ordered free + alloc on the calling
// census stream; released by gd_trim_workspace() or at thread exit.
struct WsBuf {
  void* p = nullptr;
  size_t bytes = 0;
  WsBuf() = default;
  WsBuf(const WsBuf&) = delete;
  WsBuf& operator=(const WsBuf&) = delete;
  ~WsBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
};
std::map<std::string, WsBuf>& thread_workspace();

template <typename T>
T* ws_get(DevGraph&, const char* name, size_t count, cudaStream_t s) {
  WsBuf& b = thread_workspace()[name];
  const size_t bytes = count * sizeof(T);
  if (b.bytes < bytes) {
    if (b.p) GD_CUDA(cudaFreeAsync(b.p, s));
    b.p = nullptr;
    b.bytes = 0;
    GD_CUDA(cudaMallocAsync(&b.p, bytes, s));
    b.bytes = bytes;
  }
  return (T*)b.p;
}

// Host <-> device copies of caller buffers that may be pageable: large
// pageable copies are staged through page-locked blocks by all host cores
// (gd_copy.cu).  copy_d2h returns when the host buffer holds the data.
void copy_h2d(void* dst, const void* src, size_t bytes, cudaStream_t s);
void copy_d2h(void* dst, const void* src, size_t bytes, cudaStream_t s);
bool host_is_pinned(const void* p);  // page-locked (or managed) host memory
// This thread's page-locked host staging block of at least `bytes` (grown,
// never shrunk; valid until the next call on the same thread), and the
// parallel gather of per-graph pair arrays into it.
void* host_staging(size_t bytes);
// A second per-thread page-locked block for small per-call results (sums).
void* host_results(size_t bytes);
void gather_pairs(const int64_t* const* lists, const int64_t* offs, int64_t g0, int64_t g1,
                  int64_t* flat);

// ---------------------------------------------------------------------------
// small device helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ unsigned hash32(unsigned x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

// 128-bit atomic accumulation as (lo, hi) uint64 words with carry.
__device__ __forceinline__ void atomic_add_u128(unsigned long long* lohi,
                                                unsigned __int128 v) {
  unsigned long long lo = (unsigned long long)v;
  unsigned long long hi = (unsigned long long)(v >> 64);
  if (lo) {
    unsigned long long old = atomicAdd(lohi, lo);
    if (old + lo < old) hi += 1ull;
  }
  if (hi) atomicAdd(lohi + 1, hi);
}

template <typename T>
__device__ __forceinline__ int64_t lower_bound_dev(const T* a, int64_t lo,
                                                   int64_t hi, T key) {
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// upper_bound over a small shared-memory prefix array: largest j with
// P[j] <= x, P[0] = 0, P nondecreasing, j in [0, cnt).
__device__ __forceinline__ int find_segment(const int* P, int cnt, int x) {
  int lo = 0, hi = cnt - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (P[mid] <= x) lo = mid; else hi = mid - 1;
  }
  return lo;
}

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

int num_sms();

}  // namespace gd
