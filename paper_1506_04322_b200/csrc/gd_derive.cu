// Per-edge derived outputs on the B200: the reference's
// _derive_micro (census.py:574-596) fused over all edges, and micro_csv
// (census.py:603-623) formatted on the device.
//
// From one raw row (t, su, sv, cl, cy, uu1, vv1, ts1, ti1, si1):
//   i3 = n-2-t-su-sv   ss1 = uu1+vv1   out = m+1-(t+su+1)-(t+sv+1)
//   ii1 = out-(cl+ts1+ti1)-(ss1+cy+si1)
//   tt0 = C(t,2)-cl  susv0 = su*sv-cy  ts0 = t(su+sv)-ts1
//   ss0 = C(su,2)+C(sv,2)-ss1  ti0 = t*i3-ti1  si0 = (su+sv)*i3-si1
//   ii0 = C(i3,2)-ii1
// A negative tt0, susv0, ts0, ss0, ti0, ti1, si0, si1, ii0 or ii1 is a
// ConsistencyError; the first (edge, name) in the reference's order is
// reported.  The CSV is written in two passes (row lengths, exclusive scan,
// row text) into one device buffer that starts with the header line.
#include <cub/cub.cuh>

#include "gd_common.cuh"
#include "gd_derive.cuh"

namespace gd {

namespace {

constexpr int kRoles = 15;  // tt1 tt0 susv1 susv0 ts1 ts0 ss1 ss0 ti1 ti0 si1 si0 ii1 ii0 indep3
constexpr int kCsvCols = 19;

struct Derived {
  int64_t t, su, sv, cl, cy, tt0, susv0, ts1, ts0, ss1, ss0, ti1, ti0, si1, si0, ii1, ii0, i3;
};

__device__ __forceinline__ int64_t c2(int64_t x) { return x * (x - 1) / 2; }

__device__ __forceinline__ Derived derive_row(const long long* __restrict__ r, int64_t n,
                                              int64_t m) {
  Derived d;
  d.t = r[0];
  d.su = r[1];
  d.sv = r[2];
  d.cl = r[3];
  d.cy = r[4];
  const int64_t uu1 = r[5], vv1 = r[6];
  d.ts1 = r[7];
  d.ti1 = r[8];
  d.si1 = r[9];
  d.i3 = n - 2 - d.t - d.su - d.sv;
  d.ss1 = uu1 + vv1;
  const int64_t outside = m + 1 - (d.t + d.su + 1) - (d.t + d.sv + 1);
  d.ii1 = outside - (d.cl + d.ts1 + d.ti1) - (d.ss1 + d.cy + d.si1);
  d.tt0 = c2(d.t) - d.cl;
  d.susv0 = d.su * d.sv - d.cy;
  d.ts0 = d.t * (d.su + d.sv) - d.ts1;
  d.ss0 = c2(d.su) + c2(d.sv) - d.ss1;
  d.ti0 = d.t * d.i3 - d.ti1;
  d.si0 = (d.su + d.sv) * d.i3 - d.si1;
  d.ii0 = c2(d.i3) - d.ii1;
  return d;
}

// first negative field in the reference's check order (census.py:592-595)
__device__ __forceinline__ int first_negative(const Derived& d) {
  const int64_t v[10] = {d.tt0, d.susv0, d.ts0, d.ss0, d.ti0, d.ti1, d.si0, d.si1, d.ii0, d.ii1};
#pragma unroll
  for (int k = 0; k < 10; k++)
    if (v[k] < 0) return k;
  return -1;
}

__device__ __forceinline__ int dec_len(int64_t v) {
  unsigned long long u = v < 0 ? 0ull - (unsigned long long)v : (unsigned long long)v;
  int l = v < 0 ? 1 : 0;
  do {
    l++;
    u /= 10ull;
  } while (u);
  return l;
}

__device__ __forceinline__ char* put_dec(char* p, int64_t v) {
  unsigned long long u = v < 0 ? 0ull - (unsigned long long)v : (unsigned long long)v;
  if (v < 0) *p++ = '-';
  char tmp[20];
  int k = 0;
  do {
    tmp[k++] = (char)('0' + (int)(u % 10ull));
    u /= 10ull;
  } while (u);
  while (k) *p++ = tmp[--k];
  return p;
}

__device__ __forceinline__ void csv_fields(const Derived& d, int64_t src, int64_t dst,
                                           int64_t* f) {
  f[0] = src;     f[1] = dst;     f[2] = d.t;     f[3] = d.su;    f[4] = d.sv;
  f[5] = d.cl;    f[6] = d.cy;    f[7] = d.tt0;   f[8] = d.susv0; f[9] = d.ts1;
  f[10] = d.ss1;  f[11] = d.ss0;  f[12] = d.ti1;  f[13] = d.ti0;  f[14] = d.si1;
  f[15] = d.si0;  f[16] = d.ii1;  f[17] = d.ii0;  f[18] = d.i3;
}

struct DeriveIn {
  const long long* table;  // [m][10]
  const int32_t* eu;       // canonical edges (dense ids)
  const int32_t* ev;
  const int64_t* orig;     // [n] original ids
  int64_t n, m;
};

__global__ void k_roles(DeriveIn in, long long* __restrict__ roles,
                        unsigned long long* __restrict__ bad) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < in.m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const Derived d = derive_row(in.table + 10 * e, in.n, in.m);
    const int nb = first_negative(d);
    if (nb >= 0) atomicMin(bad, ((unsigned long long)e << 4) | (unsigned)nb);
    long long* o = roles + kRoles * e;
    o[0] = d.cl;   o[1] = d.tt0;  o[2] = d.cy;   o[3] = d.susv0; o[4] = d.ts1;
    o[5] = d.ts0;  o[6] = d.ss1;  o[7] = d.ss0;  o[8] = d.ti1;   o[9] = d.ti0;
    o[10] = d.si1; o[11] = d.si0; o[12] = d.ii1; o[13] = d.ii0;  o[14] = d.i3;
  }
}

__global__ void k_csv_len(DeriveIn in, int64_t* __restrict__ len,
                          unsigned long long* __restrict__ bad) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < in.m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const Derived d = derive_row(in.table + 10 * e, in.n, in.m);
    const int nb = first_negative(d);
    if (nb >= 0) atomicMin(bad, ((unsigned long long)e << 4) | (unsigned)nb);
    int64_t f[kCsvCols];
    csv_fields(d, in.orig[in.eu[e]], in.orig[in.ev[e]], f);
    int64_t l = kCsvCols;  // 18 commas + '\n'
#pragma unroll
    for (int k = 0; k < kCsvCols; k++) l += dec_len(f[k]);
    len[e] = l;
  }
}

__global__ void k_csv_write(DeriveIn in, const int64_t* __restrict__ off, int64_t base,
                            char* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < in.m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const Derived d = derive_row(in.table + 10 * e, in.n, in.m);
    int64_t f[kCsvCols];
    csv_fields(d, in.orig[in.eu[e]], in.orig[in.ev[e]], f);
    char* p = out + base + off[e];
#pragma unroll
    for (int k = 0; k < kCsvCols; k++) {
      p = put_dec(p, f[k]);
      *p++ = k + 1 < kCsvCols ? ',' : '\n';
    }
  }
}

int grid_for(int64_t work) {
  const int64_t b = (work + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)num_sms() * 16));
}

const char* kCsvHeader =
    "src,dst,tri,star_u,star_v,clique4,cycle4,chordal_chord,cycle_mid_path,"
    "chordal_cycle_edge,tailed_tail,star3,tailed_detached,tri_isolated,path_end,"
    "star_isolated,pair_edge,lone_edge,indep3\n";

// table and orig ids on the device (copied when the caller passed host memory)
struct Inputs {
  DBuf<long long> table;
  DBuf<int64_t> orig;
  DeriveIn in;
};

void stage(const DevGraph& g, const long long* table, bool table_dev, const int64_t* orig_host,
           Inputs& I, cudaStream_t s) {
  if (g.G != 1) throw Error(GD_EINVAL, "derived outputs need a single graph (not a batch)");
  I.in.n = g.n;
  I.in.m = g.m;
  I.in.eu = g.eu.p;
  I.in.ev = g.ev.p;
  if (table_dev) {
    I.in.table = table;
  } else {
    I.table.alloc((size_t)g.m * 10, s);
    if (g.m)
      GD_CUDA(cudaMemcpyAsync(I.table.p, table, (size_t)g.m * 80, cudaMemcpyHostToDevice, s));
    I.in.table = I.table.p;
  }
  I.orig.alloc(g.n, s);
  if (g.n)
    GD_CUDA(cudaMemcpyAsync(I.orig.p, orig_host, (size_t)g.n * 8, cudaMemcpyHostToDevice, s));
  I.in.orig = I.orig.p;
}

}  // namespace

int64_t micro_roles(const DevGraph& g, const long long* table, bool table_dev,
                    const int64_t* orig_host, long long* roles_host, cudaStream_t s) {
  Inputs I;
  stage(g, table, table_dev, orig_host, I, s);
  DBuf<long long> roles;
  DBuf<unsigned long long> bad;
  roles.alloc((size_t)g.m * kRoles, s);
  bad.alloc(1, s);
  GD_CUDA(cudaMemsetAsync(bad.p, 0xff, 8, s));
  if (g.m) {
    k_roles<<<grid_for(g.m), 256, 0, s>>>(I.in, roles.p, bad.p);
    GD_LAUNCH_CHECK("micro_roles");
    GD_CUDA(cudaMemcpyAsync(roles_host, roles.p, (size_t)g.m * kRoles * 8,
                            cudaMemcpyDeviceToHost, s));
  }
  unsigned long long hb = ~0ull;
  GD_CUDA(cudaMemcpyAsync(&hb, bad.p, 8, cudaMemcpyDeviceToHost, s));
  GD_CUDA(cudaStreamSynchronize(s));
  return hb == ~0ull ? -1 : (int64_t)hb;
}

int64_t micro_csv(const DevGraph& g, const long long* table, bool table_dev,
                  const int64_t* orig_host, CsvText& out, cudaStream_t s) {
  Inputs I;
  stage(g, table, table_dev, orig_host, I, s);
  const int64_t m = g.m;
  const int64_t hlen = (int64_t)strlen(kCsvHeader);
  DBuf<int64_t> len, off;
  DBuf<unsigned long long> bad;
  len.alloc(m + 1, s);
  off.alloc(m + 1, s);
  bad.alloc(1, s);
  GD_CUDA(cudaMemsetAsync(bad.p, 0xff, 8, s));
  GD_CUDA(cudaMemsetAsync(len.p + m, 0, 8, s));
  if (m) {
    k_csv_len<<<grid_for(m), 256, 0, s>>>(I.in, len.p, bad.p);
    GD_LAUNCH_CHECK("micro_csv_len");
  }
  {
    size_t tb = 0;
    GD_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, len.p, off.p, m + 1, s));
    DBuf<char> tmp;
    tmp.alloc(tb, s);
    GD_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, len.p, off.p, m + 1, s));
  }
  int64_t body = 0;
  unsigned long long hb = ~0ull;
  GD_CUDA(cudaMemcpyAsync(&body, off.p + m, 8, cudaMemcpyDeviceToHost, s));
  GD_CUDA(cudaMemcpyAsync(&hb, bad.p, 8, cudaMemcpyDeviceToHost, s));
  GD_CUDA(cudaStreamSynchronize(s));
  if (hb != ~0ull) return (int64_t)hb;
  out.bytes = hlen + body;
  out.text.alloc(out.bytes, s);
  GD_CUDA(cudaMemcpyAsync(out.text.p, kCsvHeader, hlen, cudaMemcpyHostToDevice, s));
  if (m) {
    k_csv_write<<<grid_for(m), 256, 0, s>>>(I.in, off.p, hlen, out.text.p);
    GD_LAUNCH_CHECK("micro_csv_write");
  }
  GD_CUDA(cudaStreamSynchronize(s));
  return -1;
}

}  // namespace gd
