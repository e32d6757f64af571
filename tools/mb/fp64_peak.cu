// fp64 FMA throughput on one B200: the denominator of the "fp64 pipe" fraction the bench reports.
//
// Every thread runs CH independent DFMA chains (enough to cover the DFMA latency), the grid is
// a multiple of the SM count with full occupancy, and the clock is left to the driver (no lock):
// the result is the DFMA rate the part sustains at its own clock, measured with CUDA events
// (best launch and the average over ~2 s of back-to-back launches, so the power cap settles
// as in a long step).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb/fp64_peak tools/mb/fp64_peak.cu
//   tools/mb/fp64_peak            -> one JSON line
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void __launch_bounds__(256) dfma_tput(double* out, int iters, long long* cyc) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = 1e-3 * (threadIdx.x + c);
  const double a = 0.999999999, b = 1e-12;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
  }
  const long long t1 = clock64();
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  int dev = 0, sms = 0, clk_khz = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  constexpr int CH = 8;
  const int threads = 256, blocks = sms * 8;  // 2048 threads per SM
  const int iters = 20000;
  double* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(double) * threads * blocks);
  cudaMallocManaged(&cyc, sizeof(long long));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) dfma_tput<CH><<<blocks, threads>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  float best_ms = 1e30f, total_ms = 0.f;
  int reps = 0;
  while (total_ms < 2000.f) {
    cudaEventRecord(e0);
    dfma_tput<CH><<<blocks, threads>>>(out, iters, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    total_ms += ms;
    ++reps;
    if (ms < best_ms) best_ms = ms;
  }
  const double dfma = (double)threads * blocks * iters * CH;
  const double best = dfma / (best_ms * 1e-3), avg = dfma * reps / (total_ms * 1e-3);
  cudaError_t err = cudaGetLastError();
  printf("{\"kernel\": \"dfma_tput<%d>\", \"sms\": %d, \"dfma_per_s_best\": %.4e, \"dfma_per_s_avg\": %.4e, "
         "\"fp64_tflops_best\": %.3f, \"fp64_tflops_avg\": %.3f, \"reps\": %d, \"error\": \"%s\"}\n",
         CH, sms, best, avg, 2e-12 * best, 2e-12 * avg, reps, cudaGetErrorString(err));
  return err == cudaSuccess ? 0 : 1;
}
