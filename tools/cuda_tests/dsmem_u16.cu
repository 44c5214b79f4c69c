// DSMEM u16 counters (2 per word) with remote atomics + remote u16 reads.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void __launch_bounds__(512, 1) k(unsigned* out, int per, int mode) {
  extern __shared__ __align__(16) unsigned slab[];
  __shared__ int s_frame;
  cg::cluster_group cl = cg::this_cluster();
  const int words = per >> 1;
  for (int i = threadIdx.x; i < words; i += blockDim.x) slab[i] = 0;
  if (threadIdx.x == 0 && cl.block_rank() == 0) s_frame = 7;
  cl.sync();
  const int f = *cl.map_shared_rank(&s_frame, 0);
  const int cs = cl.num_blocks();
  for (int x = threadIdx.x; x < per * cs; x += blockDim.x) {
    const int owner = x / per, off = x - owner * per;
    unsigned* w = cl.map_shared_rank(slab, owner) + (off >> 1);
    atomicAdd(w, 1u << ((off & 1) << 4));
  }
  cl.sync();
  unsigned s = 0;
  for (int x = threadIdx.x; x < per * cs; x += blockDim.x) {
    const int owner = x / per, off = x - owner * per;
    const unsigned short* c = (const unsigned short*)cl.map_shared_rank(slab, owner);
    s += mode ? c[off] : 1u;
  }
  atomicAdd(out, s + (f == 7 ? 0 : 1000000));
  cl.sync();
}

int main() {
  unsigned* d;
  cudaMalloc(&d, 4);
  for (int mode = 0; mode < 2; mode++)
  for (int cs : {1, 2, 16}) {
    cudaMemset(d, 0, 4);
    int per = cs == 1 ? 98304 : (cs == 2 ? 50000 : 65536);
    size_t sm = per * 2;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (cs > 8) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = cs; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = sm; cfg.attrs = a; cfg.numAttrs = 1;
    cfg.gridDim = dim3(cs);
    int ncl = 0;
    cudaOccupancyMaxActiveClusters(&ncl, (void*)k, &cfg);
    cfg.gridDim = dim3(cs * 2);
    cudaError_t e1 = cudaLaunchKernelEx(&cfg, k, d, per, mode);
    cudaError_t e2 = cudaDeviceSynchronize();
    unsigned h = 0;
    cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
    printf("mode=%d cs=%d maxclusters=%d launch=%s sync=%s sum=%u expect=%u\n", mode, cs, ncl,
           cudaGetErrorString(e1), cudaGetErrorString(e2), h, (unsigned)(per * cs * 2 * (mode ? cs : 1)));
    if (e2 != cudaSuccess) return 1;
  }
}
