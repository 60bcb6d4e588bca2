// HBM streaming rate with S tiles in flight per SM: per-row 1 KB bulk copies vs one 32 KB copy
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
template <int S>
__global__ void k(const double* X, long long tiles_total, int mode) {
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) unsigned long long bar[S];
  if (threadIdx.x == 0) { for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(&bar[s]))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  long long mine = (tiles_total - blockIdx.x + gridDim.x - 1) / gridDim.x;
  auto issue = [&](long long i) {
    int st = i % S; long long tile = blockIdx.x + i * gridDim.x;
    const double* src = X + tile * 32 * 128;
    double* dst = sm + st * 32 * 132;
    if (threadIdx.x == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sa(&bar[st])), "r"(32 * 1024) : "memory");
    __syncwarp();
    if (mode == 0) asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(sa(dst + threadIdx.x * 132)), "l"(src + threadIdx.x * 128), "r"(1024), "r"(sa(&bar[st])) : "memory");
    else if (threadIdx.x == 0) asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(sa(dst)), "l"(src), "r"(32 * 1024), "r"(sa(&bar[st])) : "memory");
  };
  if (threadIdx.x < 32) {
    for (long long i = 0; i < mine; ++i) {
      if (i >= S) { // wait for the consumer... here: wait for previous fill of this stage to land (no consumer)
        int st = i % S; unsigned par = ((i / S) - 1) & 1;
        asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" :: "r"(sa(&bar[st])), "r"(par) : "memory");
      }
      issue(i);
    }
    for (long long i = (mine > S ? mine - S : 0); i < mine; ++i) {
      int st = i % S; unsigned par = (i / S) & 1;
      asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" :: "r"(sa(&bar[st])), "r"(par) : "memory");
    }
  }
}
int main() {
  long long N = 800000; double* X; cudaMalloc(&X, N * 128 * 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  long long tiles = N / 32;
  auto run = [&](auto kern, int S, int mode) {
    size_t smem = S * 32 * 132 * 8;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<sms, 32, smem>>>(X, tiles, mode);
    cudaEventRecord(e0); kern<<<sms, 32, smem>>>(X, tiles, mode); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("stages %d %-18s: %.0f GB/s\n", S, mode ? "one 32KB copy" : "32 x 1KB row copies", N * 1024.0 / (ms * 1e6));
  };
  run(k<2>, 2, 0); run(k<2>, 2, 1); run(k<4>, 4, 0); run(k<4>, 4, 1); run(k<6>, 6, 0); run(k<6>, 6, 1);
}
