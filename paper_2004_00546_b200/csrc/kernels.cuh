// kernels.cuh — sm_100a fp64 kernels of the Paraexp direct-adjoint path.
//
// Replaces the reference's per-stage Python/scipy arithmetic:
//   rk45_integrate stage loop (timestepping.py:162-201) + csr_matvec (linalg.py:70-74)
//     -> rk4.cuh (row-marching fused RK4 steps over all batch × slice lanes);
//   _LejaInterpolant.step Newton loop (timestepping.py:343-356)
//     -> k_cheb_first / k_cheb_term: stencil fused with the Chebyshev three-term
//        recurrence and the exp and φ₁ accumulators;
//   superposition / cost / gradient quadrature (paraexp.py:202-218,
//   optimization.py:84-112) -> elementwise, reduction and projection kernels with
//   fixed-order (deterministic) reductions.
// No tensor cores: nothing here is a dense contraction; fp64 CUDA-core math.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace px {

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

// ---------------------------------------------------------------------------
// Chebyshev exponential action: stencil fused with the three-term recurrence
// ---------------------------------------------------------------------------

struct ChebFirstArgs {
  const double* u0; long long u0_bstride;     // U_0 (batch-strided)
  double* u1;                                 // U_1 = (M U_0 − c0 U_0)/d  (B × n)
  double* acc;                                // b0 U_0 + b1 U_1 (+ addend)
  const double* addend; long long add_bstride;  // may be nullptr
  double* pacc;                               // += p0 U_0 + p1 U_1 (may be nullptr)
  Stencil5 st;
  double c0, d, b0, b1, p0, p1;
  int nx, ny;
};

template <int DIM>
__global__ void __launch_bounds__(256) k_cheb_first(ChebFirstArgs a) {
  const size_t n = (size_t)a.nx * a.ny;
  const int b = blockIdx.y;
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int y = (int)(i / a.nx), x = (int)(i - (size_t)y * a.nx);
  const double* u0 = a.u0 + b * a.u0_bstride;
  const double u = u0[i];
  const double v1 = (stencil_at<DIM>(u0, a.st, x, y, a.nx, a.ny) - a.c0 * u) / a.d;
  const size_t o = (size_t)b * n + i;
  a.u1[o] = v1;
  double r = a.b0 * u + a.b1 * v1;
  if (a.addend) r += a.addend[b * a.add_bstride + i];
  a.acc[o] = r;
  if (a.pacc) a.pacc[o] += a.p0 * u + a.p1 * v1;
}

struct ChebTermArgs {
  const double* ucur; long long ucur_bstride;
  const double* uprev; long long uprev_bstride;
  double* unext;      // B × n
  double* acc;        // B × n
  double* pacc;       // may be nullptr
  Stencil5 st;
  double c0, two_over_d, sigma, bk, pk;
  int nx, ny;
};

template <int DIM>
__global__ void __launch_bounds__(256) k_cheb_term(ChebTermArgs a) {
  const size_t n = (size_t)a.nx * a.ny;
  const int b = blockIdx.y;
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int y = (int)(i / a.nx), x = (int)(i - (size_t)y * a.nx);
  const double* uc = a.ucur + b * a.ucur_bstride;
  const double* up = a.uprev + b * a.uprev_bstride;
  const double u = uc[i];
  const double un = a.two_over_d * (stencil_at<DIM>(uc, a.st, x, y, a.nx, a.ny) - a.c0 * u) +
                    a.sigma * up[i];
  const size_t o = (size_t)b * n + i;
  a.unext[o] = un;
  a.acc[o] += a.bk * un;
  if (a.pacc) a.pacc[o] += a.pk * un;
}

// ---------------------------------------------------------------------------
// Elementwise helpers (batch in blockIdx.y)
// ---------------------------------------------------------------------------

// out[b] = alpha·x[b] + beta·y[b]  (x, y batch-strided; y may be nullptr)
__global__ void k_axpby(double* out, long long out_bstride, const double* x, long long x_bstride,
                        double alpha, const double* y, long long y_bstride, double beta, size_t n) {
  const int b = blockIdx.y;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    double r = alpha * x[b * x_bstride + i];
    if (y) r += beta * y[b * y_bstride + i];
    out[b * out_bstride + i] = r;
  }
}

// out[b] = M x[b] (+ f[b]) with f = Σ_k c[b,k] tx[ix_k][i] ty[iy_k][j] when ctrl != nullptr
template <int DIM>
__global__ void k_apply_plus_control(double* out, const double* src, long long src_bstride, Stencil5 st,
                                     const double* ctrl, const double* tx, const double* ty,
                                     const int* ix, const int* iy, int K, int nx, int ny) {
  const size_t n = (size_t)nx * ny;
  const int b = blockIdx.y;
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int y = (int)(i / nx), x = (int)(i - (size_t)y * nx);
  double r = stencil_at<DIM>(src + b * src_bstride, st, x, y, nx, ny);
  if (ctrl) {
    const double* c = ctrl + (size_t)b * K;
    double f = 0.0;
    for (int k = 0; k < K; ++k) f += c[k] * (tx[(size_t)ix[k] * nx + x] * ty[(size_t)iy[k] * ny + y]);
    r += f;
  }
  out[(size_t)b * n + i] = r;
}

// out[b][i] = Σ_{p<lanes_per_b} lanes[b*lanes_per_b + p][i]  (fixed order)
__global__ void k_lane_sum(double* out, const double* lanes, int lanes_per_b, size_t n) {
  const int b = blockIdx.y;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const double* src = lanes + (size_t)b * lanes_per_b * n + i;
    double r = 0.0;
    for (int p = 0; p < lanes_per_b; ++p) r += src[(size_t)p * n];
    out[(size_t)b * n + i] = r;
  }
}

// ---------------------------------------------------------------------------
// Deterministic reductions
// ---------------------------------------------------------------------------

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

// partial[b][blk] = Σ_{i in blk's grid-stride set} x[b][i]²
__global__ void __launch_bounds__(256) k_sumsq_partial(double* partial, const double* x, size_t n) {
  __shared__ double red[8];
  const int b = blockIdx.y;
  double v = 0.0;
  for (size_t i = (size_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (size_t)gridDim.x * 256) {
    const double t = x[(size_t)b * n + i];
    v += t * t;
  }
  v = block_sum<256>(v, red);
  if (threadIdx.x == 0) partial[(size_t)b * gridDim.x + blockIdx.x] = v;
}

// out[b] = scale · Σ_j partial[b][j]; flag set if non-finite
__global__ void __launch_bounds__(256) k_finalize_sum(double* out, const double* partial, int m,
                                                      double scale, int* nonfinite) {
  __shared__ double red[8];
  const int b = blockIdx.x;
  double v = 0.0;
  for (int j = threadIdx.x; j < m; j += 256) v += partial[(size_t)b * m + j];
  v = block_sum<256>(v, red);
  if (threadIdx.x == 0) {
    const double r = scale * v;
    out[b] = r;
    if (nonfinite && !isfinite(r)) atomicExch(nonfinite, 1);
  }
}

// R[b][a][j] = Σ_i tx[a][i] F[b][j][i] for all x-table rows a (grid: (ny, B))
template <int MAXR>
__global__ void __launch_bounds__(256) k_project_rows(double* R, const double* F, long long F_bstride,
                                                      const double* tx, int rows_x, int nx, int ny) {
  __shared__ double red[8];
  const int j = blockIdx.x, b = blockIdx.y;
  const double* row = F + b * F_bstride + (size_t)j * nx;
  double acc[MAXR];
#pragma unroll
  for (int a = 0; a < MAXR; ++a) acc[a] = 0.0;
  for (int i = threadIdx.x; i < nx; i += 256) {
    const double v = row[i];
#pragma unroll
    for (int a = 0; a < MAXR; ++a)
      if (a < rows_x) acc[a] += tx[(size_t)a * nx + i] * v;
  }
  for (int a = 0; a < rows_x; ++a) {
    const double s = block_sum<256>(acc[a], red);
    if (threadIdx.x == 0) R[((size_t)b * rows_x + a) * ny + j] = s;
  }
}

// grad[b][k] = beta·grad[b][k] + alpha·Σ_j ty[iy_k][j] R[b][ix_k][j]  (grid: (K, B))
__global__ void __launch_bounds__(256) k_project_cols(double* grad, const double* R, const double* ty,
                                                      const int* ix, const int* iy, int rows_x, int K,
                                                      int ny, double alpha, double beta) {
  __shared__ double red[8];
  const int k = blockIdx.x, b = blockIdx.y;
  const double* r = R + ((size_t)b * rows_x + ix[k]) * ny;
  const double* t = ty + (size_t)iy[k] * ny;
  double v = 0.0;
  for (int j = threadIdx.x; j < ny; j += 256) v += t[j] * r[j];
  v = block_sum<256>(v, red);
  if (threadIdx.x == 0) {
    const size_t o = (size_t)b * K + k;
    grad[o] = (beta == 0.0 ? 0.0 : beta * grad[o]) + alpha * v;
  }
}

// ---------------------------------------------------------------------------
// Closed-form adjoint ∫ for circulant (periodic, constant-coefficient) operators:
//   Σ_{k<n} h·S(hM)·y_k = M⁻¹(y_n − n·b)   (from y_{k+1} − y_k = hM·S(hM)·y_k + b, y_0 = 0)
// on the non-constant Fourier modes; the constant mode (M·1 = 0) has y_k = k·b̄, hence
// h·b̄·n(n−1)/2. One FFT solve per gradient replaces a per-step, per-lane accumulator.
// ---------------------------------------------------------------------------

// f[b][i] = (Σ_p lanes[b·Pl + p][i] − nscale·b[b][i], 0)
__global__ void k_zsrc_cplx(double2* f, const double* lanes, int lanes_per_b, const double* bsrc, double nscale,
                            size_t n) {
  const int b = blockIdx.y;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const double* src = lanes + (size_t)b * lanes_per_b * n + i;
    double r = 0.0;
    for (int p = 0; p < lanes_per_b; ++p) r += src[(size_t)p * n];
    f[(size_t)b * n + i] = make_double2(r - nscale * bsrc[(size_t)b * n + i], 0.0);
  }
}

// f̂(kx, ky) /= n·λ(kx, ky), λ = cc + ce·e^{iθx} + cw·e^{−iθx} + cn·e^{iθy} + cs·e^{−iθy}
// (the stencil's eigenvalues; θ = 2πk/N, cuFFT's forward sign); the constant mode -> 0
__global__ void k_circ_solve(double2* f, Stencil5 st, int nx, int ny, int B) {
  const size_t n = (size_t)nx * ny;
  const double inv_n = 1.0 / (double)n;
  const double two_pi = 6.283185307179586476925286766559;
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n * B;
       idx += (size_t)gridDim.x * blockDim.x) {
    const size_t i = idx % n;
    const int kx = (int)(i % nx), ky = (int)(i / nx);
    if (kx == 0 && ky == 0) {
      f[idx] = make_double2(0.0, 0.0);
      continue;
    }
    double sx, cx, sy, cy;
    sincos(two_pi * kx / nx, &sx, &cx);
    sincos(two_pi * ky / ny, &sy, &cy);
    const double lr = st.cc + (st.ce + st.cw) * cx + (st.cn + st.cs) * cy;
    const double li = (st.ce - st.cw) * sx + (st.cn - st.cs) * sy;
    const double den = (lr * lr + li * li) * (double)n;
    const double2 v = f[idx];
    // v / λ = v·conj(λ) / |λ|², and the inverse transform's 1/n
    f[idx] = make_double2((v.x * lr + v.y * li) / den, (v.y * lr - v.x * li) / den);
    (void)inv_n;
  }
}

// G[b][i] = Re f[b][i] + cscale·c[b][i] + kconst·bsum[b]
__global__ void k_z_finish(double* G, const double2* f, const double* c, double cscale, const double* bsum,
                           double kconst, size_t n) {
  const int b = blockIdx.y;
  const double kb = kconst * bsum[b];
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    G[(size_t)b * n + i] = f[(size_t)b * n + i].x + cscale * c[(size_t)b * n + i] + kb;
}

// partial[b][blk] = Σ_{i in blk's grid-stride set} x[b][i]
__global__ void __launch_bounds__(256) k_sum_partial(double* partial, const double* x, size_t n) {
  __shared__ double red[8];
  const int b = blockIdx.y;
  double v = 0.0;
  for (size_t i = (size_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (size_t)gridDim.x * 256) v += x[(size_t)b * n + i];
  v = block_sum<256>(v, red);
  if (threadIdx.x == 0) partial[(size_t)b * gridDim.x + blockIdx.x] = v;
}

}  // namespace px
