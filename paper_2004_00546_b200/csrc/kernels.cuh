// kernels.cuh — sm_100a fp64 kernels of the Paraexp direct-adjoint path.
//
// Replaces the reference's per-stage Python/scipy arithmetic:
//   rk45_integrate stage loop (timestepping.py:162-201) + csr_matvec (linalg.py:70-74)
//     -> rk4.cuh (row-marching fused RK4 steps over all batch × slice lanes);
//   superposition / cost / gradient quadrature (paraexp.py:202-218,
//   optimization.py:84-112) -> elementwise, reduction and projection kernels with
//   fixed-order (deterministic) reductions.
// No tensor cores: nothing here is a dense contraction; fp64 CUDA-core math.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace px {

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
  if (ctrl && K < 0) {  // field control (PX_FLAG_FIELD_CONTROL): f is given point by point
    r += ctrl[(size_t)b * n + i];
  } else if (ctrl) {
    const double* c = ctrl + (size_t)b * K;
    double f = 0.0;
    for (int k = 0; k < K; ++k) f += c[k] * (tx[(size_t)ix[k] * nx + x] * ty[(size_t)iy[k] * ny + y]);
    r += f;
  }
  out[(size_t)b * n + i] = r;
}

// ---------------------------------------------------------------------------
// Deterministic reductions
// ---------------------------------------------------------------------------


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
