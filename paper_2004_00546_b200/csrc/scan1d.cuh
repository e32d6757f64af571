// scan1d.cuh — the whole summed-chain carry of a 1D linear sweep on chip.
//
// For 1D fields (n ≤ 4096: configs 1 and 2) one exp-action term touches only a
// few tens of KB, so per-term kernels are launch-bound. Here ONE CTA per batch
// member runs the complete recursion of SURVEY.md App. B,
//   direct : D ← v_{p0};  D ← exp(ΔA)D + v_p (p = p0+1 … p1−1);  [D ← exp(τ_long A)D]
//   adjoint: C ← w_{p1−1}; C ← exp(ΔAᵀ)C + w_p, G += Δφ₁(ΔAᵀ)C (p = p1−2 … p0); [long span]
// with the carry, the three Chebyshev basis vectors and the accumulators in
// registers (each thread owns a contiguous run of PPT points) and only the two
// run-edge values exchanged per term through shared memory (double buffered,
// one barrier per term). The plan coefficients are read from device memory
// (uniform across the CTA, broadcast through L1).
#pragma once
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace px {

struct Scan1DPlan {
  const double* be;  // degree+1 (device)
  const double* bp;  // degree+1 (device), may be null
  int degree, substeps, sigma;
  double c0, d;
};

struct Scan1DArgs {
  const double* lanes;  // L × n lane end states (member b: lanes b*Pl .. b*Pl+Pl−1)
  double* out;          // B × n result carry
  double* pacc;         // B × n running ∫ accumulator (adjoint), may be null
  Stencil5 st;
  Scan1DPlan slice, lng;
  int use_long;
  int adjoint;          // 0: forward order, 1: backward order with φ accumulation
  int n, Pl;
};

template <int PPT>
__global__ void __launch_bounds__(512) k_scan1d(Scan1DArgs a) {
  __shared__ double eL[2][512];
  __shared__ double eR[2][512];
  const int n = a.n;
  const int b = blockIdx.x;
  const int t = threadIdx.x;
  const int start = t * PPT;
  const int cnt = max(0, min(PPT, n - start));
  const int last = (n + PPT - 1) / PPT - 1;
  const int tl = (t == 0) ? last : t - 1;
  const int tr = (t >= last) ? 0 : t + 1;
  const Stencil5 st = a.st;
  const bool phi = a.adjoint && a.pacc != nullptr;
  const double* lanes = a.lanes + (size_t)b * a.Pl * n;
  double C[PPT], G[PPT];
  const int q0 = a.adjoint ? a.Pl - 1 : 0;
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    C[k] = (k < cnt) ? lanes[(size_t)q0 * n + start + k] : 0.0;
    G[k] = (phi && k < cnt) ? a.pacc[(size_t)b * n + start + k] : 0.0;
  }
  int par = 0;
  // (M u − c0 u) over the run, with the neighbours' edge values
  auto shifted = [&](const double* u, double c0, double* out) {
    if (t <= last) {
      eL[par][t] = u[0];
      eR[par][t] = u[cnt > 0 ? cnt - 1 : 0];
    }
    __syncthreads();
    const double left = eR[par][tl], right = eL[par][tr];
    par ^= 1;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      const double wl = (k == 0) ? left : u[k - 1];
      const double wr = (k + 1 == PPT || k + 1 >= cnt) ? right : u[k + 1];
      double v = st.cc * u[k];
      v += st.ce * wr;
      v += st.cw * wl;
      out[k] = v - c0 * u[k];
    }
  };
  auto action = [&](const Scan1DPlan& pl) {
    for (int sub = 0; sub < pl.substeps; ++sub) {
      double up[PPT], uc[PPT], un[PPT], acc[PPT], pc[PPT];
      const double b0 = __ldg(pl.be), b1 = __ldg(pl.be + 1);
      const double p0 = phi ? __ldg(pl.bp) : 0.0, p1 = phi ? __ldg(pl.bp + 1) : 0.0;
      shifted(C, pl.c0, un);
#pragma unroll
      for (int k = 0; k < PPT; ++k) {
        up[k] = C[k];
        uc[k] = un[k] / pl.d;
        acc[k] = b0 * up[k] + b1 * uc[k];
        pc[k] = p0 * up[k] + p1 * uc[k];
      }
      const double tod = 2.0 / pl.d, sg = (double)pl.sigma;
      for (int j = 2; j <= pl.degree; ++j) {
        shifted(uc, pl.c0, un);
        const double bj = __ldg(pl.be + j), pj = phi ? __ldg(pl.bp + j) : 0.0;
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
          const double v = tod * un[k] + sg * up[k];
          up[k] = uc[k];
          uc[k] = v;
          acc[k] += bj * v;
          pc[k] += pj * v;
        }
      }
#pragma unroll
      for (int k = 0; k < PPT; ++k) {
        C[k] = acc[k];
        G[k] += pc[k];
      }
    }
  };
  for (int s = 1; s < a.Pl; ++s) {
    const int q = a.adjoint ? a.Pl - 1 - s : s;
    action(a.slice);
#pragma unroll
    for (int k = 0; k < PPT; ++k)
      if (k < cnt) C[k] += lanes[(size_t)q * n + start + k];
  }
  if (a.use_long) action(a.lng);
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    if (k < cnt) {
      a.out[(size_t)b * n + start + k] = C[k];
      if (phi) a.pacc[(size_t)b * n + start + k] = G[k];
    }
  }
}

}  // namespace px
