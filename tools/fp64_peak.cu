// Measure FP64 peak on the device: DFMA (CUDA cores) vs DMMA (mma.sync m8n8k4 f64).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x[16];
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0; for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}
__global__ void dmma_loop(double* out, int iters) {
  double c[8][2]; double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-6;
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 1 << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    for (int tpb : {256, 512, 1024}) {
      int blocks = sms * (2048 / tpb); int iters = 20000;
      cudaEventRecord(e0); dfma_loop<<<blocks, tpb>>>(out, iters, 1.0000001, 1e-9); cudaEventRecord(e1);
      cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 16 * iters * (double)blocks * tpb;
      if (rep) printf("DFMA tpb=%4d: %.2f TFLOP/s\n", tpb, fl / ms / 1e9);
      iters = 4000;
      cudaEventRecord(e0); dmma_loop<<<blocks, tpb>>>(out, iters); cudaEventRecord(e1);
      cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      fl = 2.0 * 256 * 8 * iters * (double)blocks * (tpb / 32);
      if (rep) printf("DMMA tpb=%4d: %.2f TFLOP/s\n", tpb, fl / ms / 1e9);
    }
  }
  return 0;
}
