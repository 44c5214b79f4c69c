// Edge-list text parser on the B200: the reference's
// load_edge_list (graph.py:223-285) for ASCII input, producing the raw int64
// pairs directly in device memory, where gd_graph_create (GD_INPUT_DEVICE)
// sanitises them -- the text crosses PCIe once and no host array of pairs is
// built.
//
// Line semantics (graph.py:245-275): each line is stripped; empty lines,
// "%%MatrixMarket" banners and lines starting with a comment prefix are
// skipped; the first other line after a banner with exactly three tokens is
// the MatrixMarket size header ("rows cols nnz"); every other line must hold
// at least two tokens (separated by whitespace or commas) whose first two are
// Python int() literals; further tokens are ignored.  Errors carry the
// 1-based line number of the first offending line.
//
// Bytes the ASCII rules cannot decide like CPython does (non-ASCII bytes:
// Unicode whitespace and digits; a lone '\r' that universal newlines would
// treat as a line break; id literals beyond int64) set `fallback`, and the
// Python layer parses that input with its restatement of the reference loop.
#include <cub/cub.cuh>

#include "gd_common.cuh"
#include "gd_parse.cuh"

namespace gd {

namespace {

constexpr int kMaxPrefixes = 16;
constexpr int kMaxPrefixLen = 64;

struct Prefixes {
  int count;
  int len[kMaxPrefixes];
  char bytes[kMaxPrefixes][kMaxPrefixLen];
};

// Python str.isspace() on ASCII: \t \n \v \f \r, \x1c-\x1f and space.
__host__ __device__ __forceinline__ bool is_ws(unsigned char c) {
  return c == ' ' || (c >= 9 && c <= 13) || (c >= 0x1c && c <= 0x1f);
}
__host__ __device__ __forceinline__ bool is_sep(unsigned char c) { return is_ws(c) || c == ','; }

// int(token) for an ASCII token: optional sign, decimal digits with single
// underscores between digits.  0: ok, 1: not an int literal, 2: beyond int64.
__host__ __device__ __forceinline__ int parse_int(const unsigned char* t, int64_t len,
                                                  int64_t* out) {
  int64_t i = 0;
  bool neg = false;
  if (i < len && (t[i] == '+' || t[i] == '-')) {
    neg = t[i] == '-';
    i++;
  }
  if (i >= len || t[i] < '0' || t[i] > '9') return 1;
  unsigned long long v = 0;
  bool over = false;
  const unsigned long long lim = neg ? (1ull << 63) : (1ull << 63) - 1ull;
  bool prev_us = false;
  for (; i < len; i++) {
    const unsigned char c = t[i];
    if (c == '_') {
      if (prev_us) return 1;
      prev_us = true;
      continue;
    }
    if (c < '0' || c > '9') return 1;
    prev_us = false;
    const unsigned d = c - '0';
    if (!over) {
      if (v > (lim - d) / 10ull) over = true;
      else v = v * 10ull + d;
    }
  }
  if (prev_us) return 1;  // trailing underscore
  if (over) return 2;
  *out = neg ? (int64_t)(0ull - v) : (int64_t)v;
  return 0;
}

__host__ __device__ __forceinline__ bool starts_with(const unsigned char* s, int64_t len,
                                                     const char* p, int plen) {
  if (plen > len) return false;
  for (int k = 0; k < plen; k++)
    if (s[k] != (unsigned char)p[k]) return false;
  return true;
}

// Input the ASCII rules cannot decide, and the number of '\n' bytes.
__global__ void k_scan_bytes(const unsigned char* __restrict__ buf, int64_t len, int cr_newline,
                             unsigned long long* __restrict__ nnl, int* __restrict__ fallback) {
  unsigned cnt = 0;
  bool odd = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len;
       i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned char c = buf[i];
    cnt += c == '\n';
    odd |= c >= 0x80;
    if (c == '\r' && cr_newline && (i + 1 == len || buf[i + 1] != '\n')) odd = true;
  }
  for (int off = 16; off; off >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(nnl, (unsigned long long)cnt);
  if (odd) atomicOr(fallback, 1);
}

struct IsNewline {
  const unsigned char* buf;
  __device__ __forceinline__ bool operator()(int64_t i) const { return buf[i] == '\n'; }
};

enum LineKind : unsigned char { kSkip = 0, kData = 1 };
// error kinds (reported as (line << 2) | kind, minimum over lines)
enum { kErrTokens = 1, kErrNonInt = 2 };

__global__ void k_parse_lines(const unsigned char* __restrict__ buf, int64_t len,
                              const int64_t* __restrict__ nlpos, int64_t nlines,
                              int64_t header_line, Prefixes P, unsigned char* __restrict__ kind,
                              int64_t* __restrict__ uv, unsigned long long* __restrict__ err,
                              int* __restrict__ fallback, long long* __restrict__ minmax) {
  for (int64_t li = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; li < nlines;
       li += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = li == 0 ? 0 : nlpos[li - 1] + 1;
    int64_t b = nlpos[li];  // '\n' of the line (len for an unterminated last line)
    kind[li] = kSkip;
    while (a < b && is_ws(buf[a])) a++;
    while (b > a && is_ws(buf[b - 1])) b--;
    if (a == b || li == header_line) continue;
    const unsigned char* s = buf + a;
    const int64_t n = b - a;
    if (starts_with(s, n, "%%MatrixMarket", 14)) continue;
    bool comment = false;
    for (int p = 0; p < P.count && !comment; p++) comment = starts_with(s, n, P.bytes[p], P.len[p]);
    if (comment) continue;
    // first two tokens
    int64_t t0 = -1, e0 = -1, t1 = -1, e1 = -1, i = 0;
    while (i < n && is_sep(s[i])) i++;
    if (i < n) {
      t0 = i;
      while (i < n && !is_sep(s[i])) i++;
      e0 = i;
      while (i < n && is_sep(s[i])) i++;
      if (i < n) {
        t1 = i;
        while (i < n && !is_sep(s[i])) i++;
        e1 = i;
      }
    }
    if (t1 < 0) {
      atomicMin(err, ((unsigned long long)li << 2) | kErrTokens);
      continue;
    }
    int64_t u = 0, v = 0;
    const int ru = parse_int(s + t0, e0 - t0, &u);
    const int rv = parse_int(s + t1, e1 - t1, &v);
    if (ru == 1 || rv == 1) {
      atomicMin(err, ((unsigned long long)li << 2) | kErrNonInt);
      continue;
    }
    if (ru == 2 || rv == 2) {  // a Python int beyond int64: decided on the host
      atomicOr(fallback, 2);
      continue;
    }
    kind[li] = kData;
    uv[2 * li] = u;
    uv[2 * li + 1] = v;
    atomicMin(&minmax[0], (long long)(u < v ? u : v));
    atomicMax(&minmax[1], (long long)(u > v ? u : v));
  }
}

__global__ void k_compact_pairs(const unsigned char* __restrict__ kind,
                                const int64_t* __restrict__ pos, const int64_t* __restrict__ uv,
                                int64_t nlines, int64_t shift, int64_t* __restrict__ out) {
  for (int64_t li = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; li < nlines;
       li += (int64_t)gridDim.x * blockDim.x) {
    if (kind[li] != kData) continue;
    const int64_t p = pos[li];
    out[2 * p] = uv[2 * li] - shift;
    out[2 * p + 1] = uv[2 * li + 1] - shift;
  }
}

__global__ void k_kind_to_i64(const unsigned char* __restrict__ kind, int64_t n,
                              int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = kind[i] == kData;
}

int grid_for(int64_t work) {
  const int64_t b = (work + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)num_sms() * 16));
}

// Host pre-scan up to the first line that is not empty, a banner or a
// comment (graph.py:245-266): MatrixMarket size header or the first data line.
struct Prescan {
  int64_t header_line = -1;  // 0-based index of the size header line
  int64_t mm_rows = -1;
  int64_t err_kind = 0, err_line = 0, err_off = 0, err_len = 0;
  bool any = false;          // a data-relevant line exists
  bool fallback = false;
};

Prescan prescan(const unsigned char* buf, int64_t len, const Prefixes& P) {
  Prescan r;
  bool is_mm = false;
  int64_t pos = 0, li = 0;
  while (pos < len) {
    int64_t e = pos;
    while (e < len && buf[e] != '\n') e++;
    int64_t a = pos, b = e;
    while (a < b && is_ws(buf[a])) a++;
    while (b > a && is_ws(buf[b - 1])) b--;
    const unsigned char* s = buf + a;
    const int64_t n = b - a;
    if (n > 0) {
      bool skip = false;
      if (starts_with(s, n, "%%MatrixMarket", 14)) {
        is_mm = true;
        skip = true;
      } else {
        for (int p = 0; p < P.count && !skip; p++) skip = starts_with(s, n, P.bytes[p], P.len[p]);
      }
      if (!skip) {
        r.any = true;
        if (is_mm) {
          int64_t tok[4][2];
          int nt = 0, i = 0;
          while (i < n) {
            while (i < n && is_sep(s[i])) i++;
            if (i >= n) break;
            const int64_t t = i;
            while (i < n && !is_sep(s[i])) i++;
            if (nt < 4) { tok[nt][0] = t; tok[nt][1] = i; }
            nt++;
          }
          if (nt == 3) {
            int64_t rows = 0, cols = 0;
            const int a0 = parse_int(s + tok[0][0], tok[0][1] - tok[0][0], &rows);
            const int a1 = parse_int(s + tok[1][0], tok[1][1] - tok[1][0], &cols);
            if (a0 == 2 || a1 == 2) {
              r.fallback = true;
            } else if (a0 || a1) {
              r.err_kind = 3;  // malformed MatrixMarket size header
              r.err_line = li + 1;
              r.err_off = a;
              r.err_len = n;
            } else {
              r.header_line = li;
              r.mm_rows = rows > cols ? rows : cols;
            }
          }
        }
        return r;
      }
    }
    pos = e + 1;
    li++;
  }
  return r;
}

}  // namespace

void parse_edge_list(const char* text, int64_t len, const char* const* prefixes, int nprefixes,
                     int cr_newline, int mm_shift, ParseOut& out, cudaStream_t s) {
  Prefixes P{};
  if (nprefixes < 0 || nprefixes > kMaxPrefixes)
    throw Error(GD_EINVAL, "at most 16 comment prefixes");
  P.count = nprefixes;
  for (int p = 0; p < nprefixes; p++) {
    const size_t l = strlen(prefixes[p]);
    if (l >= (size_t)kMaxPrefixLen) throw Error(GD_EINVAL, "comment prefix longer than 63 bytes");
    P.len[p] = (int)l;
    memcpy(P.bytes[p], prefixes[p], l);
  }
  const unsigned char* hb = (const unsigned char*)text;
  for (int64_t k = 0; k < 12; k++) out.info[k] = 0;
  out.info[1] = -1;
  const Prescan pre = prescan(hb, len, P);
  if (pre.fallback) {
    out.info[6] = 1;
    return;
  }
  if (pre.err_kind) {
    out.info[2] = pre.err_kind;
    out.info[3] = pre.err_line;
    out.info[4] = pre.err_off;
    out.info[5] = pre.err_len;
    return;
  }
  if (!pre.any) {
    out.info[2] = 4;  // no data lines
    return;
  }
  out.info[1] = pre.mm_rows;
  // bytes to the device; '\n' positions
  DBuf<unsigned char> dbuf;
  dbuf.alloc(len, s);
  GD_CUDA(cudaMemcpyAsync(dbuf.p, text, len, cudaMemcpyHostToDevice, s));
  DBuf<int> dflag;
  DBuf<unsigned long long> dnnl;
  dflag.alloc(1, s);
  dflag.zero();
  dnnl.alloc(1, s);
  dnnl.zero();
  if (len) {
    k_scan_bytes<<<grid_for(len), 256, 0, s>>>(dbuf.p, len, cr_newline, dnnl.p, dflag.p);
    GD_LAUNCH_CHECK("parse_scan_bytes");
  }
  int64_t nnl = 0;
  int hflag0 = 0;
  GD_CUDA(cudaMemcpyAsync(&nnl, dnnl.p, 8, cudaMemcpyDeviceToHost, s));
  GD_CUDA(cudaMemcpyAsync(&hflag0, dflag.p, 4, cudaMemcpyDeviceToHost, s));
  GD_CUDA(cudaStreamSynchronize(s));
  if (hflag0) {
    out.info[6] = hflag0;
    return;
  }
  // '\n' positions (exact size; one more slot for an unterminated last line)
  DBuf<int64_t> nlpos, nsel;
  nlpos.alloc(nnl + 1, s);
  nsel.alloc(1, s);
  if (nnl) {
    cub::CountingInputIterator<int64_t> it(0);
    IsNewline pred{dbuf.p};
    size_t tb = 0;
    GD_CUDA(cub::DeviceSelect::If(nullptr, tb, it, nlpos.p, nsel.p, len, pred, s));
    DBuf<char> tmp;
    tmp.alloc(tb, s);
    GD_CUDA(cub::DeviceSelect::If(tmp.p, tb, it, nlpos.p, nsel.p, len, pred, s));
  }
  // lines: one per '\n', plus a last unterminated one
  const bool tail = len > 0 && hb[len - 1] != '\n';
  const int64_t nlines = nnl + (tail ? 1 : 0);
  if (tail) GD_CUDA(cudaMemcpyAsync(nlpos.p + nnl, &len, 8, cudaMemcpyHostToDevice, s));
  DBuf<unsigned char> kind;
  DBuf<int64_t> uv, pos;
  DBuf<unsigned long long> derr;
  DBuf<long long> mm;
  kind.alloc(nlines, s);
  uv.alloc(2 * nlines, s);
  pos.alloc(nlines + 1, s);
  derr.alloc(1, s);
  mm.alloc(2, s);
  const unsigned long long none = ~0ull;
  const long long mm_init[2] = {INT64_MAX, INT64_MIN};
  GD_CUDA(cudaMemcpyAsync(derr.p, &none, 8, cudaMemcpyHostToDevice, s));
  GD_CUDA(cudaMemcpyAsync(mm.p, mm_init, 16, cudaMemcpyHostToDevice, s));
  if (nlines) {
    k_parse_lines<<<grid_for(nlines), 256, 0, s>>>(dbuf.p, len, nlpos.p, nlines, pre.header_line,
                                                  P, kind.p, uv.p, derr.p, dflag.p, mm.p);
    GD_LAUNCH_CHECK("parse_lines");
  }
  unsigned long long herr = none;
  int hflag = 0;
  long long hmm[2];
  GD_CUDA(cudaMemcpyAsync(&herr, derr.p, 8, cudaMemcpyDeviceToHost, s));
  GD_CUDA(cudaMemcpyAsync(&hflag, dflag.p, 4, cudaMemcpyDeviceToHost, s));
  GD_CUDA(cudaMemcpyAsync(hmm, mm.p, 16, cudaMemcpyDeviceToHost, s));
  GD_CUDA(cudaStreamSynchronize(s));
  if (hflag) {
    out.info[6] = hflag;
    return;
  }
  if (herr != none) {
    const int64_t li = (int64_t)(herr >> 2);
    int64_t a = 0, b = 0;
    if (li > 0) {
      GD_CUDA(cudaMemcpy(&a, nlpos.p + li - 1, 8, cudaMemcpyDeviceToHost));
      a += 1;
    }
    GD_CUDA(cudaMemcpy(&b, nlpos.p + li, 8, cudaMemcpyDeviceToHost));
    out.info[2] = (int64_t)(herr & 3);
    out.info[3] = li + 1;
    out.info[4] = a;
    out.info[5] = b - a;
    return;
  }
  // compact the data lines into pairs (MatrixMarket: shifted to 0-based)
  DBuf<int64_t> flag64;
  flag64.alloc(nlines + 1, s);
  if (nlines) {
    k_kind_to_i64<<<grid_for(nlines), 256, 0, s>>>(kind.p, nlines, flag64.p);
    GD_LAUNCH_CHECK("parse_kind");
  }
  GD_CUDA(cudaMemsetAsync(flag64.p + nlines, 0, 8, s));
  {
    size_t tb = 0;
    GD_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, flag64.p, pos.p, nlines + 1, s));
    DBuf<char> tmp;
    tmp.alloc(tb, s);
    GD_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, flag64.p, pos.p, nlines + 1, s));
  }
  int64_t k = 0;
  GD_CUDA(cudaMemcpyAsync(&k, pos.p + nlines, 8, cudaMemcpyDeviceToHost, s));
  GD_CUDA(cudaStreamSynchronize(s));
  const int64_t shift = (pre.mm_rows >= 0 && mm_shift) ? 1 : 0;
  out.pairs.alloc(2 * k, s);
  if (k) {
    k_compact_pairs<<<grid_for(nlines), 256, 0, s>>>(kind.p, pos.p, uv.p, nlines, shift,
                                                     out.pairs.p);
    GD_LAUNCH_CHECK("parse_compact");
  }
  GD_CUDA(cudaStreamSynchronize(s));
  out.info[0] = k;
  out.info[7] = k ? hmm[0] : 0;  // min / max id (before the MatrixMarket shift)
  out.info[8] = k ? hmm[1] : 0;
  out.info[9] = shift;
  out.info[10] = nlines;
}

}  // namespace gd
