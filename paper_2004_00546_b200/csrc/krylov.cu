// krylov.cu — batched Arnoldi (CGS2) exponential actions (krylov.cuh), BASELINE config 4.
#include "internal.h"
#include "krylov.cuh"

namespace pxi {

int krylov_alloc(px::KrylovWork& kw, int m, size_t n, int B, std::string* err) {
  return px::krylov_alloc(kw, m, n, B, err);
}

void krylov_free(px::KrylovWork& kw) { px::krylov_free(kw); }

// result <- exp(span·M)·src (+ addend);  pacc += span·φ₁(span·M)·src  (if pacc)
int krylov_action(Handle* h, const Plan& pl, const px::Stencil5& st, const double* src, long long src_bs,
                  const double* addend, long long add_bs, double* pacc, double** result, cudaStream_t s) {
  PX_TRY(px::krylov_action(h->kw, pl.span / pl.substeps, pl.substeps, h->d.krylov_m, st, src, src_bs, addend,
                           add_bs, pacc, h->ACC, h->B, h->d.nx, h->d.ny, h->dim, result, s, &h->stats,
                           h->var.krylov_ortho));
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(h, PX_ERR_CUDA, std::string("krylov launch: ") + cudaGetErrorString(e));
  return PX_OK;
}

}  // namespace pxi
