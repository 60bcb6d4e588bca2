// latency probes: dependent DFMA chain, rcp.approx.f64 chain, STS->LDS round trip, dependent LDG
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, const double* g, int n) {
  __shared__ double s[64];
  double x = out[threadIdx.x] + 1.0, y = 1.0;
  long long t0 = clock64();
  for (int i = 0; i < 256; ++i) x = fma(x, 1.0000001, 1e-9);
  long long t1 = clock64();
  for (int i = 0; i < 256; ++i) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r + 1.0; }
  long long t2 = clock64();
  for (int i = 0; i < 256; ++i) { s[threadIdx.x] = x; __syncwarp(); x = s[(threadIdx.x + 1) & 31] + 1e-9; __syncwarp(); }
  long long t3 = clock64();
  int idx = threadIdx.x;
  for (int i = 0; i < 64; ++i) { idx = (int)g[idx]; }
  long long t4 = clock64();
  for (int i = 0; i < 256; ++i) y = y / (x + i);
  long long t5 = clock64();
  out[threadIdx.x] = x + idx + y;
  if (threadIdx.x == 0) { cyc[0] = (t1-t0)/256; cyc[1] = (t2-t1)/256; cyc[2] = (t3-t2)/256; cyc[3] = (t4-t3)/64; cyc[4]=(t5-t4)/256; }
}
int main() {
  double *out, *g; long long *cyc; int n = 1 << 24;
  cudaMalloc(&out, 4096); cudaMalloc(&cyc, 64); cudaMalloc(&g, n * 8);
  double* h = new double[n]; for (int i = 0; i < n; ++i) h[i] = (double)((i * 2654435761u + 12345u) % n);
  cudaMemcpy(g, h, n * 8, cudaMemcpyHostToDevice); cudaMemset(out, 0, 4096);
  k<<<1, 32>>>(out, cyc, g, n); cudaDeviceSynchronize();
  k<<<1, 32>>>(out, cyc, g, n); cudaDeviceSynchronize();
  long long c[5]; cudaMemcpy(c, cyc, 40, cudaMemcpyDeviceToHost);
  printf("DFMA dep latency %lld cyc, rcp.approx.f64 %lld cyc (+DADD), STS-sync-LDS-sync %lld cyc, dependent LDG (DRAM) %lld cyc, IEEE div %lld cyc\n", c[0], c[1], c[2], c[3], c[4]);
}
