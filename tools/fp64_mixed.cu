// Do DFMA (FP64 CUDA-core pipe) and DMMA (FP64 tensor path) share hardware?
// Even warps run DMMA chains, odd warps DFMA chains, in one kernel; compare the
// combined rate with each alone.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
__device__ void dfma_part(double *out, int iters) {
  double x[16];
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], 1.0000001, 1e-9);
  }
  double s = 0; for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}
__device__ void dmma_part(double *out, int iters) {
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
// mode 0: all DFMA, 1: all DMMA, 2: half/half by warp parity
__global__ void mixed(double *out, int mode, int it_fma, int it_mma) {
  const int w = threadIdx.x >> 5;
  const bool mma = mode == 1 || (mode == 2 && (w & 1));
  if (mma) dmma_part(out, it_mma); else dfma_part(out, it_fma);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *out; cudaMalloc(&out, 1 << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int tpb = 512, blocks = sms * 4;
  // per-warp work: DFMA 2*16*32*it_fma flops; DMMA 2*256*8*it_mma flops
  const int it_fma = 20000, it_mma = 2500;  // DFMA warp: 20.5 MF, DMMA warp: 10.2 MF
  for (int rep = 0; rep < 2; ++rep)
    for (int mode = 0; mode < 3; ++mode) {
      cudaEventRecord(e0);
      mixed<<<blocks, tpb>>>(out, mode, it_fma, it_mma);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double warps = (double)blocks * tpb / 32;
      const double ffma = 2.0 * 16 * 32 * it_fma, fmma = 2.0 * 256 * 8 * it_mma;
      double fl = mode == 0 ? warps * ffma : mode == 1 ? warps * fmma : warps / 2 * (ffma + fmma);
      if (rep) printf("mode %d (%s): %.3f ms, %.2f TFLOP/s\n", mode,
                      mode == 0 ? "DFMA" : mode == 1 ? "DMMA" : "half/half", ms, fl / ms / 1e9);
    }
  return 0;
}
