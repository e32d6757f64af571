// common.cuh — device helpers and plain types shared by every translation unit.
//
// Only __device__ __forceinline__ functions, templates and PODs live here, so any .cu
// may include it; each kernel family lives in its own header, included by exactly one
// translation unit (see internal.h for the layout).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace px {

// 5-point stencil (cc, ce, cw, cn, cs); 1D uses the first three (problems.py:106-152).
struct Stencil5 {
  double cc, ce, cw, cn, cs;
};

// periodic wrap for halo coordinates (tiles may be wider than the grid)
__device__ __forceinline__ int wrapi(int v, int n) {
  v %= n;
  return v < 0 ? v + n : v;
}

// (M u) at flat index i of a periodic nx×ny field (global memory, L1/L2 cached).
template <int DIM>
__device__ __forceinline__ double stencil_at(const double* __restrict__ u, const Stencil5& s,
                                             int x, int y, int nx, int ny) {
  const size_t row = (size_t)y * nx;
  const int xe = (x + 1 == nx) ? 0 : x + 1;
  const int xw = (x == 0) ? nx - 1 : x - 1;
  double r = s.cc * u[row + x];
  r += s.ce * __ldg(u + row + xe);
  r += s.cw * __ldg(u + row + xw);
  if (DIM == 2) {
    const int yn = (y + 1 == ny) ? 0 : y + 1;
    const int ys = (y == 0) ? ny - 1 : y - 1;
    r += s.cn * __ldg(u + (size_t)yn * nx + x);
    r += s.cs * __ldg(u + (size_t)ys * nx + x);
  }
  return r;
}

// --- cp.async (LDGSTS) ------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// --- 1D bulk copies (TMA engine, cp.async.bulk) completing on an mbarrier -------------
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, unsigned bytes, unsigned long long* bar) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem);
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(d),
               "l"(gmem), "r"(bytes), "r"(b)
               : "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// block-wide sum of NT threads (fixed order; result valid in thread 0); red: NT/32 doubles
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x < 32) {
    r = (threadIdx.x < NT / 32) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) r += __shfl_down_sync(0xffffffffu, r, o);
  }
  __syncthreads();
  return r;  // valid in thread 0
}

// compile-time constants for unrolled lambdas
template <int V> struct IC { static constexpr int value = V; };
template <bool V> struct BC { static constexpr bool value = V; };

// --- Krylov scratch (krylov.cuh) ------------------------------------------------------
constexpr int KRYLOV_MAX_M = 40;

struct KrylovWork {
  int m = 0, B = 0, nblk = 0;
  size_t n = 0;
  double* V = nullptr;        // (m+1) × B × n
  double* w = nullptr;        // 2 × B × n (ping-pong: step j's w feeds V_{j+1} at step j+1)
  double* H = nullptr;        // B × (m+1) × m   (row i, col j at i*m + j)
  double* hcol = nullptr;     // B × (MAX_M+1)  current column pass values
  double* part = nullptr;     // B × (MAX_M+1) × nblk partial dots
  double* beta = nullptr;     // B
  double* coef = nullptr;     // B × 2 × m  (exp column, φ column), β-scaled
  // delayed reorthogonalization (one reduction and two basis passes per step)
  double* u = nullptr;        // 2 × B × n  the candidate vector (ping-pong)
  double* kc = nullptr;       // B × KC_STRIDE  per-step coefficients (g, a/β, 1/β, κ)
  int* cnt = nullptr;         // B  ticket counters of the fused per-step finalisation
};
constexpr int KC_STRIDE = 2 * (KRYLOV_MAX_M + 1) + 4;

}  // namespace px
