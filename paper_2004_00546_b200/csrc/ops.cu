// ops.cu — elementwise, projection and reduction launches (kernels.cuh): superposition
// sums, the control source, the objective, the gradient projection and the closed-form
// adjoint ∫ (paraexp.py:202-218, optimization.py:84-117).
#include <algorithm>

#include "internal.h"
#include "kernels.cuh"

namespace pxi {

int axpby(Handle* h, double* out, long long obs, const double* x, long long xbs, double alpha, const double* y,
          long long ybs, double beta, cudaStream_t s) {
  px::k_axpby<<<grid_stride(h->n, h->B), 256, 0, s>>>(out, obs, x, xbs, alpha, y, ybs, beta, h->n);
  PX_CHECK_LAUNCH(h);
  return PX_OK;
}

// grad[b][k] = alpha·⟨φ_k, F[b]⟩ + beta·grad[b][k] (separable basis: rows then columns)
int project(Handle* h, double* grad, const double* F, long long Fbs, double alpha, double beta, cudaStream_t s) {
  if (h->d.flags & PX_FLAG_FIELD_CONTROL)  // field control: the gradient is the field itself
    return axpby(h, grad, (long long)h->n, F, Fbs, alpha, grad, (long long)h->n, beta, s);
  const int rx = h->rows_x;
  const dim3 g(h->d.ny, h->B);
  if (rx <= 8) px::k_project_rows<8><<<g, 256, 0, s>>>(h->R, F, Fbs, h->tx, rx, h->d.nx, h->d.ny);
  else if (rx <= 16) px::k_project_rows<16><<<g, 256, 0, s>>>(h->R, F, Fbs, h->tx, rx, h->d.nx, h->d.ny);
  else if (rx <= 32) px::k_project_rows<32><<<g, 256, 0, s>>>(h->R, F, Fbs, h->tx, rx, h->d.nx, h->d.ny);
  else px::k_project_rows<64><<<g, 256, 0, s>>>(h->R, F, Fbs, h->tx, rx, h->d.nx, h->d.ny);
  PX_CHECK_LAUNCH(h);
  px::k_project_cols<<<dim3(h->K, h->B), 256, 0, s>>>(grad, h->R, h->ty, h->ix, h->iy, rx, h->K, h->d.ny, alpha,
                                                      beta);
  PX_CHECK_LAUNCH(h);
  return PX_OK;
}

// out[b] = M·x[b] (+ f[b] = Σ_k c[b,k] φ_k when with_control)
int apply_plus_control(Handle* h, double* out, const double* x, long long xbs, const px::Stencil5& st,
                       bool with_control, cudaStream_t s) {
  const dim3 grid = grid1(h->n, h->B);
  const double* c = with_control ? h->ctrl : nullptr;
  const int K = (h->d.flags & PX_FLAG_FIELD_CONTROL) ? -1 : h->K;
  if (h->dim == 2)
    px::k_apply_plus_control<2><<<grid, 256, 0, s>>>(out, x, xbs, st, c, h->tx, h->ty, h->ix, h->iy, K, h->d.nx,
                                                     h->d.ny);
  else
    px::k_apply_plus_control<1><<<grid, 256, 0, s>>>(out, x, xbs, st, c, h->tx, h->ty, h->ix, h->iy, K, h->d.nx,
                                                     h->d.ny);
  PX_CHECK_LAUNCH(h);
  return PX_OK;
}

// J[b] = ½‖QT[b]‖² (fixed-order two-level reduction); raises the non-finite flag
int finalize_sum(Handle* h, double* out, const double* partial, int m, double scale, cudaStream_t s) {
  px::k_finalize_sum<<<h->B, 256, 0, s>>>(out, partial, m, scale, h->nonfinite);
  PX_CHECK_LAUNCH(h);
  return PX_OK;
}

int objective(Handle* h, cudaStream_t s) {
  px::k_sumsq_partial<<<dim3(h->red_blocks, h->B), 256, 0, s>>>(h->partial, h->QT, h->n);
  PX_CHECK_LAUNCH(h);
  px::k_finalize_sum<<<h->B, 256, 0, s>>>(h->J, h->partial, h->red_blocks, 0.5, h->nonfinite);
  PX_CHECK_LAUNCH(h);
  return PX_OK;
}

// G partial <- Σ_p z_p without per-lane accumulators (circulant 2D operator):
// Σ_p z_p = (Aᵀ)⁻¹₀(Σ_p w_n,p − Pl·n·b) + Pl·n·c + Pl·h·b̄·n(n−1)/2, the pseudo-inverse on the
// non-constant Fourier modes by one batched Z2Z FFT solve (kernels.cuh, k_circ_solve).
int z_closed_form(Handle* h, const double* wend, cudaStream_t s) {
  const double hs = (h->d.T / h->d.P) / h->d.nsteps;
  const double ns = (double)h->d.nsteps;
  const dim3 gs = grid_stride(h->n, h->B);
  px::k_zsrc_cplx<<<gs, 256, 0, s>>>(h->fbuf, wend, h->Pl, h->bsrc, (double)h->Pl * ns, h->n);
  PX_CHECK_LAUNCH(h);
  px::k_sum_partial<<<dim3(h->red_blocks, h->B), 256, 0, s>>>(h->partial, h->bsrc, h->n);
  PX_CHECK_LAUNCH(h);
  px::k_finalize_sum<<<h->B, 256, 0, s>>>(h->bsum, h->partial, h->red_blocks, 1.0, nullptr);
  PX_CHECK_LAUNCH(h);
  if (cufftSetStream(h->fft, s) != CUFFT_SUCCESS ||
      cufftExecZ2Z(h->fft, reinterpret_cast<cufftDoubleComplex*>(h->fbuf),
                   reinterpret_cast<cufftDoubleComplex*>(h->fbuf), CUFFT_FORWARD) != CUFFT_SUCCESS)
    return fail(h, PX_ERR_CUDA, "cufft forward failed");
  px::k_circ_solve<<<(unsigned)std::min<size_t>((h->n * h->B + 255) / 256, 148 * 16), 256, 0, s>>>(
      h->fbuf, h->AT, h->d.nx, h->d.ny, h->B);
  PX_CHECK_LAUNCH(h);
  if (cufftExecZ2Z(h->fft, reinterpret_cast<cufftDoubleComplex*>(h->fbuf),
                   reinterpret_cast<cufftDoubleComplex*>(h->fbuf), CUFFT_INVERSE) != CUFFT_SUCCESS)
    return fail(h, PX_ERR_CUDA, "cufft inverse failed");
  const double kconst = (double)h->Pl * hs * ns * (ns - 1.0) / 2.0 / (double)h->n;
  px::k_z_finish<<<gs, 256, 0, s>>>(h->G, h->fbuf, h->cz, (double)h->Pl * ns, h->bsum, kconst, h->n);
  PX_CHECK_LAUNCH(h);
  return PX_OK;
}

}  // namespace pxi
