#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_lat(double* out, int iters, long long* cyc) {
  double x = threadIdx.x * 1e-3, a = 1.0000001, b = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
template <int NT>
__global__ void bar_loop(double* out, int iters, long long* cyc) {
  __shared__ double s[2][NT];
  double x = threadIdx.x * 1e-3;
  int par = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    s[par][threadIdx.x] = x;
    __syncthreads();
    const double l = s[par][(threadIdx.x + NT - 1) % NT], r = s[par][(threadIdx.x + 1) % NT];
    x = fma(0.25, l + r, 0.5 * x);
    par ^= 1;
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 8192); cudaMallocManaged(&cyc, 8);
  const int it = 10000;
  dfma_lat<<<1, 32>>>(out, it, cyc); cudaDeviceSynchronize();
  dfma_lat<<<1, 32>>>(out, it, cyc); cudaDeviceSynchronize();
  printf("DFMA dependent latency: %.2f cycles\n", (double)cyc[0] / it);
  bar_loop<32><<<1, 32>>>(out, it, cyc); cudaDeviceSynchronize();
  printf("exchange loop 1 warp: %.1f cycles/iter\n", (double)cyc[0] / it);
  bar_loop<160><<<1, 160>>>(out, it, cyc); cudaDeviceSynchronize();
  printf("exchange loop 5 warps: %.1f cycles/iter\n", (double)cyc[0] / it);
  bar_loop<512><<<1, 512>>>(out, it, cyc); cudaDeviceSynchronize();
  printf("exchange loop 16 warps: %.1f cycles/iter\n", (double)cyc[0] / it);
  bar_loop<1024><<<1, 1024>>>(out, it, cyc); cudaDeviceSynchronize();
  printf("exchange loop 32 warps: %.1f cycles/iter\n", (double)cyc[0] / it);
  return 0;
}
