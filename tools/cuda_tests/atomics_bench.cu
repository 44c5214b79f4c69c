// Throughput of the scattered counter operations the wedge sweeps are made of
// (B200): shared-memory atomics / loads vs global RED / loads on L2-resident
// and DRAM-resident counter arrays.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ unsigned hash32(unsigned x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16;
  return x;
}

// mode 0: smem u16 atomic add (32-bit atomicAdd with shift)  1: smem u16 load
template <int MODE>
__global__ void __launch_bounds__(1024, 1) k_smem(int iters, int words, unsigned* out) {
  extern __shared__ unsigned tab[];
  for (int i = threadIdx.x; i < words; i += blockDim.x) tab[i] = 0;
  __syncthreads();
  unsigned x = blockIdx.x * 1024 + threadIdx.x, acc = 0;
  const unsigned mask = words * 2 - 1;
  for (int i = 0; i < iters; i++) {
    x = hash32(x + i);
    const unsigned c = x & mask;
    if (MODE == 0) atomicAdd(&tab[c >> 1], 1u << ((c & 1) << 4));
    else acc += ((const unsigned short*)tab)[c];
  }
  __syncthreads();
  if (threadIdx.x == 0) atomicAdd(out, tab[0] + acc);
}

// mode 0: global red.add u32   1: global u16 load   (array of `words` u32)
template <int MODE>
__global__ void __launch_bounds__(512, 4) k_gmem(int iters, unsigned* tab, unsigned mask, unsigned* out) {
  unsigned x = blockIdx.x * 512 + threadIdx.x, acc = 0;
  for (int i = 0; i < iters; i++) {
    x = hash32(x + i);
    const unsigned c = x & mask;
    if (MODE == 0)
      asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(tab + (c >> 1)), "r"(1u << ((c & 1) << 4)) : "memory");
    else acc += ((const unsigned short*)tab)[c];
  }
  if (acc == 0x12345) atomicAdd(out, acc);
}

int main() {
  unsigned* out;
  cudaMalloc(&out, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096;
  for (int words : {4096, 49152}) {
    const size_t sm = words * 4;
    cudaFuncSetAttribute(k_smem<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaFuncSetAttribute(k_smem<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    for (int mode = 0; mode < 2; mode++) {
      for (int rep = 0; rep < 2; rep++) {
        cudaEventRecord(a);
        if (mode == 0) k_smem<0><<<sms, 1024, sm>>>(iters, words, out);
        else k_smem<1><<<sms, 1024, sm>>>(iters, words, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
      }
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double ops = (double)sms * 1024 * iters;
      printf("smem %s words=%d: %.3f ms  %.1f Gop/s  %.3f op/clk/SM @1.965GHz\n",
             mode ? "u16 load " : "u16 atomic", words, ms, ops / ms / 1e6,
             ops / (ms * 1e-3) / 1.965e9 / sms);
    }
  }
  for (size_t bytes : {(size_t)8 << 20, (size_t)48 << 20, (size_t)96 << 20, (size_t)640 << 20}) {
    unsigned* tab;
    cudaMalloc(&tab, bytes);
    cudaMemset(tab, 0, bytes);
    const unsigned mask = (unsigned)(bytes / 2 - 1);
    for (int mode = 0; mode < 2; mode++) {
      for (int rep = 0; rep < 2; rep++) {
        cudaEventRecord(a);
        if (mode == 0) k_gmem<0><<<sms * 4, 512>>>(iters, tab, mask, out);
        else k_gmem<1><<<sms * 4, 512>>>(iters, tab, mask, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
      }
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double ops = (double)sms * 4 * 512 * iters;
      printf("gmem %s %4zu MB: %.3f ms  %.1f Gop/s  %.3f op/clk/SM\n", mode ? "u16 load " : "u16 red  ",
             bytes >> 20, ms, ops / ms / 1e6, ops / (ms * 1e-3) / 1.965e9 / sms);
    }
    cudaFree(tab);
  }
  printf("err=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
