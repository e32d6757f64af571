#include <cstdio>
#include <cuda_runtime.h>
struct Coef { double c[128]; };
template <int MODE>
__global__ void loop(double* out, const double* __restrict__ gco, Coef pc, int iters, long long* cyc) {
  constexpr int NT = 160;
  __shared__ double s[2][NT];
  __shared__ double sc[128];
  if (threadIdx.x < 128) sc[threadIdx.x] = gco[threadIdx.x];
  __syncthreads();
  double x[4] = {threadIdx.x * 1e-3, 1.0, 2.0, 3.0}, acc = 0.0, up[4] = {0, 0, 0, 0};
  int par = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    s[par][threadIdx.x] = x[0];
    __syncthreads();
    const double l = s[par][(threadIdx.x + NT - 1) % NT], r = s[par][(threadIdx.x + 1) % NT];
    double bj = 1.0;
    if (MODE == 1) bj = __ldg(gco + (i & 127));
    if (MODE == 2) bj = pc.c[i & 127];
    if (MODE == 3) bj = sc[i & 127];
    double un[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double wl = k == 0 ? l : x[k - 1], wr = k == 3 ? r : x[k + 1];
      double v = fma(0.3, x[k], 0.1 * up[k]);
      v = fma(0.2, wr, v);
      un[k] = fma(0.2, wl, v);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) { up[k] = x[k]; x[k] = un[k]; acc += bj * un[k]; }
    par ^= 1;
  }
  long long t1 = clock64();
  out[threadIdx.x] = x[0] + acc;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* out; double* gco; long long* cyc;
  cudaMalloc(&out, 8192); cudaMalloc(&gco, 128 * 8); cudaMemset(gco, 0, 128 * 8); cudaMallocManaged(&cyc, 8);
  Coef pc{}; for (int i = 0; i < 128; ++i) pc.c[i] = 1e-3 * i;
  const int it = 20000;
  const char* names[] = {"no coef", "__ldg coef", "param coef (LDC)", "smem coef"};
  for (int rep = 0; rep < 2; ++rep) {
    loop<0><<<1, 160>>>(out, gco, pc, it, cyc); cudaDeviceSynchronize(); if (rep) printf("%s: %.1f\n", names[0], (double)cyc[0] / it);
    loop<1><<<1, 160>>>(out, gco, pc, it, cyc); cudaDeviceSynchronize(); if (rep) printf("%s: %.1f\n", names[1], (double)cyc[0] / it);
    loop<2><<<1, 160>>>(out, gco, pc, it, cyc); cudaDeviceSynchronize(); if (rep) printf("%s: %.1f\n", names[2], (double)cyc[0] / it);
    loop<3><<<1, 160>>>(out, gco, pc, it, cyc); cudaDeviceSynchronize(); if (rep) printf("%s: %.1f\n", names[3], (double)cyc[0] / it);
  }
  return 0;
}
