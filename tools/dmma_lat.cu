#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc) {
  double c[2] = {0, 0}, a = threadIdx.x * 1e-3, b = 1.0;
  long long t0 = clock64();
  for (int i = 0; i < 256; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
  long long t1 = clock64();
  out[threadIdx.x] = c[0] + c[1];
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / 256;
}
// bulk copy throughput: one CTA per SM copies `n` rows of `bytes` via per-row cp.async.bulk vs one big copy
__global__ void bulk(const double* X, int rows, int rowbytes, int reps, int mode, long long* cyc) {
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) unsigned long long bar;
  unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(b)); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    const double* src = X + ((size_t)(blockIdx.x * reps + r) * rows * rowbytes / 8) % ((size_t)1 << 27);
    if (threadIdx.x < 32) {
      if (threadIdx.x == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(rows * rowbytes) : "memory");
      __syncwarp();
      if (mode == 0) {
        for (int i = threadIdx.x; i < rows; i += 32)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"((unsigned)__cvta_generic_to_shared(sm + i * (rowbytes / 8 + 4))), "l"(src + (size_t)i * rowbytes / 8), "r"(rowbytes), "r"(b) : "memory");
      } else if (threadIdx.x == 0) {
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"((unsigned)__cvta_generic_to_shared(sm)), "l"(src), "r"(rows * rowbytes), "r"(b) : "memory");
      }
    }
    asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" :: "r"(b), "r"(r & 1) : "memory");
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[1 + mode] = (t1 - t0) / reps;
}
int main() {
  double* out; long long* cyc; double* X; cudaMalloc(&out, 4096); cudaMalloc(&cyc, 64); cudaMalloc(&X, (size_t)1 << 30);
  k<<<1, 32>>>(out, cyc); k<<<1, 32>>>(out, cyc);
  cudaFuncSetAttribute(bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int mode = 0; mode < 2; ++mode) {
    bulk<<<148, 256, 200 * 1024>>>(X, 32, 1024, 64, mode, cyc);
    cudaEventRecord(e0); bulk<<<148, 256, 200 * 1024>>>(X, 32, 1024, 256, mode, cyc); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("mode %s: %.1f GB/s aggregate (1 tile in flight per SM)\n", mode ? "one 32KB copy" : "32 x 1KB row copies", 148.0 * 256 * 32 * 1024 / (ms * 1e6));
  }
  long long c[3]; cudaMemcpy(c, cyc, 24, cudaMemcpyDeviceToHost);
  printf("DMMA dependent latency %lld cycles; per-tile cycles rows %lld one %lld\n", c[0], c[1], c[2]);
}
