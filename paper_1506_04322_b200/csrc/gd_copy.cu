// Host <-> device copies of caller buffers that may be pageable.
//
// cudaMemcpyAsync from / to pageable host memory runs through the driver's
// own single-threaded staging (measured at C3: the 268 MB pair array takes
// ~24 ms pageable against ~5 ms page-locked).  Here large pageable copies go
// through a ring of page-locked staging blocks owned by the calling thread:
// the host side of every chunk is copied by all cores (OpenMP) while the DMA
// of the previous chunk runs.  Page-locked caller buffers are copied directly.
#include <omp.h>

#include <cstring>

#include "gd_common.cuh"

namespace gd {

namespace {

constexpr size_t kChunk = 32u << 20;  // bytes per staging block
constexpr int kSlots = 4;
constexpr size_t kDirect = 8u << 20;  // below this, one plain cudaMemcpyAsync

struct Staging {
  char* buf[kSlots] = {};
  cudaEvent_t ev[kSlots] = {};
  bool used[kSlots] = {};
  bool ok = false;
  Staging() {
    for (int i = 0; i < kSlots; i++) {
      if (cudaHostAlloc((void**)&buf[i], kChunk, cudaHostAllocDefault) != cudaSuccess ||
          cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        return;
      }
    }
    ok = true;
  }
  ~Staging() {
    for (int i = 0; i < kSlots; i++) {
      if (buf[i]) cudaFreeHost(buf[i]);
      if (ev[i]) cudaEventDestroy(ev[i]);
    }
  }
};

Staging& staging() {
  static thread_local Staging st;
  return st;
}

bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}

void par_memcpy(char* dst, const char* src, size_t len) {
  const int nt = std::min(8, std::max(1, omp_get_max_threads()));
  const size_t per = ((len + nt - 1) / nt + 4095) & ~size_t(4095);
#pragma omp parallel for num_threads(nt) schedule(static, 1)
  for (int t = 0; t < nt; t++) {
    const size_t a = (size_t)t * per;
    if (a < len) std::memcpy(dst + a, src + a, std::min(per, len - a));
  }
}

}  // namespace

void copy_h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  Staging& st = staging();
  if (bytes < kDirect || is_pinned(src) || !st.ok) {
    GD_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    return;
  }
  for (size_t off = 0, c = 0; off < bytes; off += kChunk, c++) {
    const int k = (int)(c % kSlots);
    const size_t len = std::min(kChunk, bytes - off);
    if (st.used[k]) GD_CUDA(cudaEventSynchronize(st.ev[k]));  // the slot's previous DMA
    par_memcpy(st.buf[k], (const char*)src + off, len);
    GD_CUDA(cudaMemcpyAsync((char*)dst + off, st.buf[k], len, cudaMemcpyHostToDevice, s));
    GD_CUDA(cudaEventRecord(st.ev[k], s));
    st.used[k] = true;
  }
}

bool host_is_pinned(const void* p) { return is_pinned(p); }

void copy_d2h(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  Staging& st = staging();
  if (bytes < kDirect || is_pinned(dst) || !st.ok) {
    GD_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
    GD_CUDA(cudaStreamSynchronize(s));
    return;
  }
  const size_t nchunks = (bytes + kChunk - 1) / kChunk;
  // keep kSlots DMAs in flight; drain chunk c - kSlots + 1 after issuing c
  auto drain = [&](size_t c) {
    const int k = (int)(c % kSlots);
    GD_CUDA(cudaEventSynchronize(st.ev[k]));
    const size_t off = c * kChunk;
    par_memcpy((char*)dst + off, st.buf[k], std::min(kChunk, bytes - off));
  };
  for (size_t c = 0; c < nchunks; c++) {
    if (c >= (size_t)kSlots) drain(c - kSlots);
    const int k = (int)(c % kSlots);
    const size_t off = c * kChunk;
    GD_CUDA(cudaMemcpyAsync(st.buf[k], (const char*)src + off, std::min(kChunk, bytes - off),
                            cudaMemcpyDeviceToHost, s));
    GD_CUDA(cudaEventRecord(st.ev[k], s));
    st.used[k] = true;
  }
  for (size_t c = nchunks > (size_t)kSlots ? nchunks - kSlots : 0; c < nchunks; c++) drain(c);
}

namespace {
struct Block {
  void* p = nullptr;
  size_t n = 0;
  ~Block() {
    if (p) cudaFreeHost(p);
  }
  void* get(size_t bytes) {
    if (n < bytes) {
      const size_t want = std::max(bytes, n * 2);
      if (p) cudaFreeHost(p);
      p = nullptr;
      n = 0;
      GD_CUDA(cudaHostAlloc(&p, want, cudaHostAllocDefault));
      n = want;
    }
    return p;
  }
};
}  // namespace

void* host_results(size_t bytes) {
  static thread_local Block b;
  return b.get(bytes);
}

void* host_staging(size_t bytes) {
  struct Block {
    void* p = nullptr;
    size_t n = 0;
    ~Block() {
      if (p) cudaFreeHost(p);
    }
  };
  static thread_local Block b;
  if (b.n < bytes) {
    const size_t want = std::max(bytes, b.n * 2);
    if (b.p) cudaFreeHost(b.p);
    b.p = nullptr;
    b.n = 0;
    GD_CUDA(cudaHostAlloc(&b.p, want, cudaHostAllocDefault));
    b.n = want;
  }
  return b.p;
}

void gather_pairs(const int64_t* const* lists, const int64_t* offs, int64_t g0, int64_t g1,
                  int64_t* flat) {
  const int nt = std::min(16, std::max(1, omp_get_max_threads()));
#pragma omp parallel for num_threads(nt) schedule(dynamic, 32)
  for (int64_t g = g0; g < g1; g++) {
    const int64_t k = offs[g + 1] - offs[g];
    if (k > 0) std::memcpy(flat + 2 * offs[g], lists[g], (size_t)k * 16);
  }
}

}  // namespace gd
