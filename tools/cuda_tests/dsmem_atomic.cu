// Minimal check of distributed-shared-memory atomics on B200 (cluster of 2 and 16).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k(unsigned* out, int per) {
  extern __shared__ unsigned slab[];
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < per; i += blockDim.x) slab[i] = 0;
  cl.sync();
  const int cs = cl.num_blocks();
  for (int i = threadIdx.x; i < per * cs; i += blockDim.x) {
    const int owner = i / per, off = i - owner * per;
    unsigned* w = cl.map_shared_rank(slab, owner) + off;
    atomicAdd(w, 1u);
  }
  cl.sync();
  unsigned s = 0;
  for (int i = threadIdx.x; i < per; i += blockDim.x) s += slab[i];
  atomicAdd(out, s);
  cl.sync();
}

int main() {
  unsigned* d;
  cudaMalloc(&d, 4);
  for (int cs : {2, 8, 16}) {
    cudaMemset(d, 0, 4);
    int per = 16384;
    size_t sm = per * 4;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (cs > 8) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = cs; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = sm; cfg.attrs = a; cfg.numAttrs = 1;
    cfg.gridDim = dim3(cs);
    int ncl = 0;
    cudaError_t e0 = cudaOccupancyMaxActiveClusters(&ncl, (void*)k, &cfg);
    cfg.gridDim = dim3(cs * 4);
    cudaError_t e1 = cudaLaunchKernelEx(&cfg, k, d, per);
    cudaError_t e2 = cudaDeviceSynchronize();
    unsigned h = 0;
    cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
    printf("cs=%d maxclusters=%d (%s) launch=%s sync=%s sum=%u expect=%u\n", cs, ncl,
           cudaGetErrorString(e0), cudaGetErrorString(e1), cudaGetErrorString(e2), h,
           (unsigned)(per * cs * cs * 4));
  }
}
