// throughput of the group sweep (RB=16, 2 groups/warp) at realistic occupancy
#include <cstdio>
#include <cuda_runtime.h>
#define FULL_MASK 0xffffffffu
__device__ __forceinline__ double rcp_nr(double d) {
    double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    double e = fma(-d, r, 1.0); r = fma(r, e, r); e = fma(-d, r, 1.0); return fma(r, e, r);
}
template <int RB, int MODE>
__device__ __forceinline__ void sweep(double (&a)[RB], double* buf, int r) {
#pragma unroll
  for (int k = 0; k < RB; ++k) {
    double col[RB];
    if (MODE == 0) {
      buf[r] = a[k]; __syncwarp();
      const double2* b2 = reinterpret_cast<const double2*>(buf);
#pragma unroll
      for (int z = 0; z < RB/2; ++z) { double2 t = b2[z]; col[2*z] = t.x; col[2*z+1] = t.y; }
      __syncwarp();
    } else {
#pragma unroll
      for (int z = 0; z < RB; ++z) col[z] = __shfl_sync(FULL_MASK, a[k], z, RB);
    }
    const double d = col[k];
    const double id = rcp_nr(d);
    const bool piv = (r == k);
    const double f = a[k] * id;
    const double alpha = piv ? id : 1.0, beta = piv ? 0.0 : f;
#pragma unroll
    for (int z = 0; z < RB; ++z) { if (z == k) continue; a[z] = fma(-beta, col[z], a[z] * alpha); }
    a[k] = piv ? -id : f;
  }
}
template <int MODE>
__global__ void __launch_bounds__(128) kern(double* out, int iters) {
  constexpr int RB = 16;
  __shared__ __align__(16) double bufs[8][RB];
  const int lane = threadIdx.x & 31, r = lane % RB, gid = (threadIdx.x >> 5) * 2 + lane / RB;
  double a[RB];
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int z = 0; z < RB; ++z) a[z] = (z == r ? 20.0 : 0.0) + 1.0 / (1.0 + r + z + it);
    sweep<RB, MODE>(a, bufs[gid], r);
    double s = 0; 
#pragma unroll
    for (int z = 0; z < RB; ++z) s += a[z];
    if (s == 123.456) out[threadIdx.x] = s;
  }
}
int main() {
  double* out; cudaMalloc(&out, 1 << 20);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int mode = 0; mode < 2; ++mode) for (int cps : {1, 2, 4, 8, 16}) {
    int iters = 200, blocks = sms * cps;
    for (int w = 0; w < 2; ++w) {
      cudaEventRecord(e0);
      if (mode == 0) kern<0><<<blocks, 128>>>(out, iters); else kern<1><<<blocks, 128>>>(out, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
    }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double sweeps = (double)blocks * 8 * iters;  // 8 groups per CTA
    double cyc_per_sweep_per_sm = ms * 1e-3 * 1.965e9 * sms / sweeps;
    printf("mode %s ctas/SM %2d: %.1f ns per sweep (GPU-wide), %.0f SM-cycles per sweep, warp-step latency %.0f cyc\n",
           mode ? "shfl" : "smem", cps, ms * 1e6 / sweeps, cyc_per_sweep_per_sm,
           ms * 1e-3 * 1.965e9 / (iters * 16.0) / ((blocks + sms * 16 - 1) / (sms * 16) > 1 ? 1 : 1));
  }
}
