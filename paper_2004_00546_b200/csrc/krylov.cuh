// krylov.cuh — batched Arnoldi exponential action (BASELINE config 4: m = 30).
//
// No reference equivalent (Krylov is out of the reference's scope, SPEC.md:13,204;
// the paper describes it). Per substep of width τ:
//   β = ‖y‖, V_0 = y/β; for j < m: w = M V_j, CGS2 against V_0..V_j (the
//   stencil application is fused with the first pass's dot products),
//   h_{j+1,j} = ‖w‖, V_{j+1} = w/h_{j+1,j};
//   E = exp([[τH_m, τe_1], [0, 0]]) (one CTA, Taylor-18 scaling and squaring);
//   y <- β·V_m·E[:m, 0],  φ-accumulator += β·V_m·E[:m, m]  (= τφ₁(τM)y).
// Reductions are two-level and fixed-order (deterministic). The basis for
// config 4 (31 × 2 MB) stays resident in the 126 MB L2.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "../../include/paraexp.h"
#include "common.cuh"

namespace px {

constexpr double KRYLOV_BREAKDOWN = 1e-13;
constexpr int KR_EXPM_MATS = 12;  // N×N matrices in k_kr_expm's shared memory (A … A⁶, 3 blocks, E, T)
#ifndef PX_KR_PPT
#define PX_KR_PPT 4
#endif
constexpr int KR_PPT = PX_KR_PPT;     // points per thread in the Arnoldi passes
constexpr int KR_BLK = 256 * KR_PPT;  // points per block


inline int krylov_alloc(KrylovWork& kw, int m, size_t n, int B, std::string* err) {
  kw.m = m;
  kw.n = n;
  kw.B = B;
  kw.nblk = (int)((n + KR_BLK - 1) / KR_BLK);
  auto al = [&](double** p, size_t cnt) -> bool {
    cudaError_t e = cudaMalloc(p, cnt * sizeof(double));
    if (e != cudaSuccess) {
      if (err) *err = std::string("krylov cudaMalloc: ") + cudaGetErrorString(e);
      return false;
    }
    return true;
  };
  if (!al(&kw.V, (size_t)(m + 1) * B * n) || !al(&kw.w, 2 * (size_t)B * n) ||
      !al(&kw.H, (size_t)B * (m + 1) * m) || !al(&kw.hcol, (size_t)B * (KRYLOV_MAX_M + 1)) ||
      !al(&kw.part, (size_t)B * (2 * (KRYLOV_MAX_M + 1) + 1) * std::max<size_t>((size_t)kw.nblk, 148 * 4)) || !al(&kw.beta, B) ||
      !al(&kw.coef, (size_t)B * 2 * m) || !al(&kw.u, 2 * (size_t)B * n) || !al(&kw.kc, (size_t)B * KC_STRIDE))
    return PX_ERR_NOMEM;
  if (cudaMalloc(&kw.cnt, sizeof(int) * B) != cudaSuccess || cudaMemset(kw.cnt, 0, sizeof(int) * B) != cudaSuccess) {
    if (err) *err = "krylov cudaMalloc: ticket counters";
    return PX_ERR_NOMEM;
  }

  return PX_OK;
}

inline void krylov_free(KrylovWork& kw) {
  cudaFree(kw.V); cudaFree(kw.w); cudaFree(kw.H); cudaFree(kw.hcol);
  cudaFree(kw.part); cudaFree(kw.beta); cudaFree(kw.coef); cudaFree(kw.u); cudaFree(kw.kc); cudaFree(kw.cnt);
  kw = KrylovWork{};
}

// partial[b][0][blk] = Σ y², one point per thread
__global__ void __launch_bounds__(256) k_kr_sumsq(double* part, int nblk, const double* y, long long ybs,
                                                  size_t n) {
  __shared__ double red[8];
  const int b = blockIdx.y;
  double v = 0.0;
#pragma unroll
  for (int k = 0; k < KR_PPT; ++k) {
    const size_t i = (size_t)blockIdx.x * KR_BLK + threadIdx.x + 256 * k;
    if (i < n) {
      const double t = y[b * ybs + i];
      v += t * t;
    }
  }
  v = block_sum<256>(v, red);
  if (threadIdx.x == 0) part[(size_t)b * nblk + blockIdx.x] = v;
}

// out[b] = sqrt(Σ part[b][:])
__global__ void __launch_bounds__(256) k_kr_beta(double* beta, const double* part, int nblk) {
  __shared__ double red[8];
  const int b = blockIdx.x;
  double v = 0.0;
  for (int j = threadIdx.x; j < nblk; j += 256) v += part[(size_t)b * nblk + j];
  v = block_sum<256>(v, red);
  if (threadIdx.x == 0) beta[b] = sqrt(v);
}

// V0[b] = y[b] / beta[b] (0 if beta == 0)
__global__ void k_kr_v0(double* V0, const double* y, long long ybs, const double* beta, size_t n) {
  const int b = blockIdx.y;
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double bt = beta[b];
  V0[(size_t)b * n + i] = bt > 0.0 ? y[b * ybs + i] / bt : 0.0;
}


// Block-reduce the per-thread values v[q], q ≤ j, with one barrier; thread q
// writes the block sum of column q to out[q * stride] (fixed order).
__device__ __forceinline__ void block_multi_sum(double (*red)[KRYLOV_MAX_M + 1], int nq,
                                                const double* v, double* out, size_t stride) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int q = 0; q < nq; ++q) {
    double x = v[q];
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if (l == 0) red[w][q] = x;
  }
  __syncthreads();
  if (threadIdx.x < nq) {
    double s = 0.0;
    for (int k = 0; k < 8; ++k) s += red[k][threadIdx.x];
    out[(size_t)threadIdx.x * stride] = s;
  }
}

// part[b][q][blk] = Σ_{i in block} V_q[i]·ws[i] for q ≤ j: one warp per column q
// (q = warp, warp+8, …), each lane streaming the block's chunk of V_q with 8 loads
// in flight; fixed order (deterministic).
__device__ __forceinline__ void warp_column_dots(const double* __restrict__ V, int B, int b, size_t n, int j,
                                                 const double* ws, double* part, int nblk) {
  const int wid = threadIdx.x >> 5, ln = threadIdx.x & 31;
  const size_t i0 = (size_t)blockIdx.x * KR_BLK;
  const int cnt = (int)min((size_t)KR_BLK, n - i0);
  for (int q = wid; q <= j; q += 8) {
    const double* __restrict__ Vq = V + ((size_t)q * B + b) * n + i0;
    double acc = 0.0;
#pragma unroll 8
    for (int t = ln; t < KR_BLK; t += 32)
      if (t < cnt) acc += Vq[t] * ws[t];
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if (ln == 0) part[((size_t)b * (KRYLOV_MAX_M + 1) + q) * nblk + blockIdx.x] = acc;
  }
}

// Arnoldi step j, first pass: V_j = w_prev·inv (materialised, fused scale of the
// previous step; j = 0 reads V_0 directly), w = M V_j, part[b][q][blk] = Σ V_q·w.
template <int DIM>
__global__ void __launch_bounds__(256) k_kr_spmv_dots(double* w, double* V, const double* w_prev,
                                                      const double* hcol, int j, Stencil5 st, double* part,
                                                      int nblk, int B, int nx, int ny) {
  const size_t n = (size_t)nx * ny;
  const int b = blockIdx.y;
  double* Vj = V + ((size_t)j * B + b) * n;
  const double* src = Vj;
  double inv = 1.0;
  if (j > 0) {
    src = w_prev + (size_t)b * n;
    inv = hcol[(size_t)b * (KRYLOV_MAX_M + 1)];
  }
  __shared__ double ws[KR_BLK];
#pragma unroll
  for (int k = 0; k < KR_PPT; ++k) {
    const size_t i = (size_t)blockIdx.x * KR_BLK + threadIdx.x + 256 * k;
    double wv = 0.0;
    if (i < n) {
      const int y = (int)(i / nx), x = (int)(i - (size_t)y * nx);
      wv = inv * stencil_at<DIM>(src, st, x, y, nx, ny);
      w[(size_t)b * n + i] = wv;
      if (j > 0) Vj[i] = src[i] * inv;
    }
    ws[threadIdx.x + 256 * k] = wv;
  }
  __syncthreads();  // V_j (global) and w (smem) of this block complete
  warp_column_dots(V, B, b, n, j, ws, part, nblk);
}

// w -= Σ_{q≤j} hcol[b][q] V_q; then part = dots (mode 0) or ‖w‖² (mode 1)
__global__ void __launch_bounds__(256) k_kr_update(double* __restrict__ w, const double* __restrict__ V, int j,
                                                   const double* __restrict__ hcol,
                                                   double* part, int nblk, int B, size_t n, int mode) {
  __shared__ double red[8][KRYLOV_MAX_M + 1];
  __shared__ double hs[KRYLOV_MAX_M + 1];
  const int b = blockIdx.y;
  if (threadIdx.x <= j) hs[threadIdx.x] = hcol[(size_t)b * (KRYLOV_MAX_M + 1) + threadIdx.x];
  __syncthreads();
  __shared__ double ws[KR_BLK];
  double wv[KR_PPT];
#pragma unroll
  for (int k = 0; k < KR_PPT; ++k) {
    const size_t i = (size_t)blockIdx.x * KR_BLK + threadIdx.x + 256 * k;
    wv[k] = i < n ? w[(size_t)b * n + i] : 0.0;
  }
#pragma unroll 4
  for (int q = 0; q <= j; ++q) {  // KR_PPT independent loads per column (× 4 columns in flight)
    const double hq = hs[q];
    const double* __restrict__ Vq = V + ((size_t)q * B + b) * n;
#pragma unroll
    for (int k = 0; k < KR_PPT; ++k) {
      const size_t i = (size_t)blockIdx.x * KR_BLK + threadIdx.x + 256 * k;
      if (i < n) wv[k] -= hq * Vq[i];
    }
  }
#pragma unroll
  for (int k = 0; k < KR_PPT; ++k) {
    const size_t i = (size_t)blockIdx.x * KR_BLK + threadIdx.x + 256 * k;
    if (i < n) w[(size_t)b * n + i] = wv[k];
    ws[threadIdx.x + 256 * k] = wv[k];
  }
  if (mode == 0) {
    __syncthreads();
    warp_column_dots(V, B, b, n, j, ws, part, nblk);
  } else {
    double vq[1];
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < KR_PPT; ++k) acc += wv[k] * wv[k];
    vq[0] = acc;
    block_multi_sum(red, 1, vq, part + ((size_t)b * (KRYLOV_MAX_M + 1)) * nblk + blockIdx.x, nblk);
  }
}

// hcol[b][q] = Σ_blk part[b][q][blk]; H[b][q][j] (+)= hcol  (grid: (j+1, B))
__global__ void __launch_bounds__(256) k_kr_finalize_dots(double* hcol, double* H, const double* part, int nblk,
                                                          int m, int j, int accumulate) {
  __shared__ double red[8];
  const int q = blockIdx.x, b = blockIdx.y;
  double v = 0.0;
  const double* p = part + ((size_t)b * (KRYLOV_MAX_M + 1) + q) * nblk;
  for (int t = threadIdx.x; t < nblk; t += 256) v += p[t];
  v = block_sum<256>(v, red);
  if (threadIdx.x == 0) {
    hcol[(size_t)b * (KRYLOV_MAX_M + 1) + q] = v;
    double* hq = H + ((size_t)b * (m + 1) + q) * m + j;
    *hq = accumulate ? *hq + v : v;
  }
}

// H[b][j+1][j] = ‖w‖ (0 on breakdown); hcol[b][0] = 1/‖w‖ (0 on breakdown)
__global__ void __launch_bounds__(256) k_kr_finalize_norm(double* hcol, double* H, const double* part, int nblk,
                                                          int m, int j) {
  __shared__ double red[8];
  const int b = blockIdx.x;
  double v = 0.0;
  const double* p = part + ((size_t)b * (KRYLOV_MAX_M + 1)) * nblk;
  for (int t = threadIdx.x; t < nblk; t += 256) v += p[t];
  v = block_sum<256>(v, red);
  if (threadIdx.x == 0) {
    const double nrm = sqrt(v);
    double mx = 1.0;
    for (int q = 0; q <= j; ++q) mx = fmax(mx, fabs(H[((size_t)b * (m + 1) + q) * m + j]));
    mx = fmax(mx, nrm);
    const bool brk = nrm <= KRYLOV_BREAKDOWN * mx;
    H[((size_t)b * (m + 1) + j + 1) * m + j] = brk ? 0.0 : nrm;
    hcol[(size_t)b * (KRYLOV_MAX_M + 1)] = brk ? 0.0 : 1.0 / nrm;
  }
}

// V_{j+1}[b] = w[b] · hcol[b][0]
__global__ void k_kr_scale(double* Vn, const double* w, const double* hcol, int B, size_t n) {
  const int b = blockIdx.y;
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  Vn[(size_t)b * n + i] = w[(size_t)b * n + i] * hcol[(size_t)b * (KRYLOV_MAX_M + 1)];
}

// One CTA per member: E = exp([[τH_m, τe_1],[0,0]]) by scaling and squaring + Taylor-18;
// coef[b] = (β·E[:m,0], β·E[:m,m]).  Truncation at the first zero subdiagonal is implicit:
// columns beyond a breakdown are zero and do not reach the first column.
__device__ void expm_aug_block(double* coef, const double* Hb, double bt, int m, double tau, double* sm) {
  const int N = m + 1;
  double* Aa = sm;            // N×N scaled matrix
  double* E = Aa + N * N;     // accumulator
  double* T = E + N * N;      // scratch
  __shared__ int s_sq;
  // meff: first zero subdiagonal
  for (int idx = threadIdx.x; idx < N * N; idx += blockDim.x) {
    const int r = idx / N, c = idx - r * N;
    double v = 0.0;
    if (c < m && r < m) v = tau * Hb[r * m + c];
    if (c == m && r == 0) v = tau;
    Aa[idx] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // truncate at breakdown: zero rows/cols beyond meff
    int meff = m;
    for (int j = 0; j < m - 1; ++j)
      if (Hb[(j + 1) * m + j] == 0.0) { meff = j + 1; break; }
    if (meff < m) {
      // move the τe_1 column to position meff and clear the rest
      for (int r = 0; r < N; ++r)
        for (int c = 0; c < N; ++c)
          if (r >= meff || c >= meff) Aa[r * N + c] = 0.0;
      Aa[0 * N + meff] = tau;
    }
    s_sq = meff;  // stash meff temporarily
  }
  __syncthreads();
  const int meff = s_sq;
  const int Ne = meff + 1;
  // compact to Ne×Ne in T then back to Aa
  for (int idx = threadIdx.x; idx < Ne * Ne; idx += blockDim.x) {
    const int r = idx / Ne, c = idx - r * Ne;
    T[idx] = Aa[r * N + c];
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < Ne * Ne; idx += blockDim.x) Aa[idx] = T[idx];
  __syncthreads();
  if (threadIdx.x == 0) {
    double nrm = 0.0;
    for (int c = 0; c < Ne; ++c) {
      double s = 0.0;
      for (int r = 0; r < Ne; ++r) s += fabs(Aa[r * Ne + c]);
      nrm = fmax(nrm, s);
    }
    s_sq = nrm <= 0.5 ? 0 : (int)ceil(log2(nrm / 0.5));
  }
  __syncthreads();
  const int sq = s_sq;
  const double scale = ldexp(1.0, -sq);
  const int NN = Ne * Ne;
  for (int idx = threadIdx.x; idx < NN; idx += blockDim.x) Aa[idx] *= scale;
  __syncthreads();
  // Taylor degree 18 by Paterson–Stockmeyer: p(A) = B0 + A⁶(B1 + A⁶(B2 + A⁶/18!)),
  // B_i = Σ_{l<6} A^l/(6i+l)!  — 7 matrix products instead of 18 (same polynomial)
  double* P[7];  // P[l] = A^l, l = 1 … 6
  P[1] = Aa;
  for (int l = 2; l <= 6; ++l) P[l] = sm + (size_t)(l + 1) * N * N;  // slots 3 … 8 (E, T: slots 1, 2)
  auto mul = [&](double* C, const double* X, const double* Y) {
    for (int idx = threadIdx.x; idx < NN; idx += blockDim.x) {
      const int r = idx / Ne, c = idx - r * Ne;
      double acc = 0.0;
      for (int q = 0; q < Ne; ++q) acc = fma(X[r * Ne + q], Y[q * Ne + c], acc);
      C[idx] = acc;
    }
    __syncthreads();
  };
  mul(P[2], P[1], P[1]);
  mul(P[3], P[2], P[1]);
  mul(P[4], P[2], P[2]);
  mul(P[5], P[4], P[1]);
  mul(P[6], P[3], P[3]);
  double* Bs[3] = {sm + 9 * (size_t)N * N, sm + 10 * (size_t)N * N, sm + 11 * (size_t)N * N};
  {
    double inv_fact[19];
    inv_fact[0] = 1.0;
    for (int k = 1; k <= 18; ++k) inv_fact[k] = inv_fact[k - 1] / k;
    for (int idx = threadIdx.x; idx < NN; idx += blockDim.x) {
      const double id = (idx / Ne == idx % Ne) ? 1.0 : 0.0;
      for (int i = 0; i < 3; ++i) {
        double v = inv_fact[6 * i] * id;
        for (int l = 1; l < 6; ++l) v = fma(inv_fact[6 * i + l], P[l][idx], v);
        Bs[i][idx] = v;
      }
      // X = B2 + A⁶/18!
      Bs[2][idx] = fma(inv_fact[18], P[6][idx], Bs[2][idx]);
    }
    __syncthreads();
  }
  mul(T, P[6], Bs[2]);  // A⁶·X
  for (int idx = threadIdx.x; idx < NN; idx += blockDim.x) Bs[1][idx] += T[idx];  // Y = B1 + A⁶X
  __syncthreads();
  mul(T, P[6], Bs[1]);  // A⁶·Y
  for (int idx = threadIdx.x; idx < NN; idx += blockDim.x) E[idx] = Bs[0][idx] + T[idx];
  __syncthreads();
  for (int it = 0; it < sq; ++it) {
    for (int idx = threadIdx.x; idx < Ne * Ne; idx += blockDim.x) {
      const int r = idx / Ne, c = idx - r * Ne;
      double s = 0.0;
      for (int q = 0; q < Ne; ++q) s += E[r * Ne + q] * E[q * Ne + c];
      T[idx] = s;
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < Ne * Ne; idx += blockDim.x) E[idx] = T[idx];
    __syncthreads();
  }
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    coef[i] = i < meff ? bt * E[i * Ne + 0] : 0.0;
    coef[m + i] = i < meff ? bt * E[i * Ne + meff] : 0.0;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) k_kr_expm(double* coef, const double* H, const double* beta, int m,
                                                 double tau) {
  extern __shared__ double sm[];
  const int b = blockIdx.x;
  expm_aug_block(coef + (size_t)b * 2 * m, H + (size_t)b * (m + 1) * m, beta[b], m, tau, sm);
}

// out[b] = Σ_i coef_e[b][i] V_i (+ addend);  pacc[b] += Σ_i coef_p[b][i] V_i
__global__ void k_kr_combine(double* out, const double* V, const double* coef, int m, int B, size_t n,
                             const double* addend, long long add_bs, double* pacc) {
  const int b = blockIdx.y;
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* ce = coef + (size_t)b * 2 * m;
  const double* cp = ce + m;
  double e = 0.0, p = 0.0;
  for (int q = 0; q < m; ++q) {
    const double v = V[((size_t)q * B + b) * n + i];
    e += ce[q] * v;
    p += cp[q] * v;
  }
  if (addend) e += addend[b * add_bs + i];
  out[(size_t)b * n + i] = e;
  if (pacc) pacc[(size_t)b * n + i] += p;
}

// ---------------------------------------------------------------------------
// Delayed reorthogonalization (DCGS2): one reduction and two basis passes per step.
//
// At step j the candidate u_j is orthogonal to Q_j = [v_0 … v_{j−1}] after ONE projection and
// not normalised. One pass computes w = M·u_j and, in the same read of Q_j, a = Q_jᵀu_j,
// b = Q_jᵀw, γ = ‖u_j‖², δ = u_jᵀw. Then (one CTA per member, k_kr_dfinal): the second
// projection of u_j is a, β = √(γ − ‖a‖²), v_j = (u_j − Q_j a)/β, H[:, j−1] = c_{j−1} + a,
// H[j, j−1] = β; the first projection of M·v_j = (w − Q_j H a − v_j β a_{j−1})/β follows from the
// Arnoldi relation without touching Q again: c_Q = (b − H a)/β, c_v = ((δ − aᵀb)/β − β a_{j−1})/β.
// The second pass (k_kr_dupdate) writes v_j = u_j/β − Q_j(a/β) and
// u_{j+1} = w/β − κ·u_j − Q_j g, κ = (a_{j−1} + c_v)/β, g = H a/β + c_Q − κ a — the basis is read
// twice per step instead of four times (CGS2), at the same orthogonality (equal to CGS2's H and V
// to rounding; tests/test_gpu_parity.py compares both with the oracle).
// ---------------------------------------------------------------------------

// One CTA per member: reduce the partials (one warp per slot, fixed order), then the step's small
// algebra in parallel over the rows (j ≤ 40). j = 0: β is ‖src‖ (kw.beta). final: only the last
// column's delayed correction H[:, m−1] += a and its subdiagonal.
__device__ __forceinline__ void kr_dfinal_body(int b, double* H, double* kc, double* beta0, const double* part,
                                               int nblk, int m, int j, int final_step) {
  const int t = threadIdx.x, wid = t >> 5, ln = t & 31;
  __shared__ double r[2 * (KRYLOV_MAX_M + 1) + 2];
  __shared__ double sh[4];  // β, 1/β, κ, a_{j−1}+c_v … (see below)
  const int nslot = 2 * j + 2;
  const double* pb = part + (size_t)b * (2 * (KRYLOV_MAX_M + 1) + 1) * nblk;
  // four threads per slot, each over a quarter of the block partials (independent loads in
  // flight), combined in a fixed order
  for (int base = 0; base < nslot; base += 64) {
    const int sl = base + (t >> 2), sub = t & 3;
    double s = 0.0;
    if (sl < nslot && (!final_step || sl < j || sl == 2 * j)) {
      const double* src = pb + (size_t)sl * nblk;
#pragma unroll 16
      for (int k = sub; k < nblk; k += 4) s += src[k];
    }
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    if (sub == 0 && sl < nslot) r[sl] = s;
  }
  (void)wid;
  (void)ln;
  __syncthreads();
  double* Hb = H + (size_t)b * (m + 1) * m;
  double* kb = kc + (size_t)b * KC_STRIDE;
  const double* a = r;
  const double* bq = r + j;
  // H's leading j×j block in shared memory (one parallel load; every later access is on chip)
  __shared__ double Hs[KRYLOV_MAX_M * KRYLOV_MAX_M];
  for (int idx = t; idx < j * j; idx += blockDim.x) {
    const int q = idx / j, c = idx - q * j;
    Hs[idx] = Hb[(size_t)q * m + c];
  }
  __syncthreads();
  // the previous column gets its delayed second projection (rows in parallel)
  if (j > 0 && t < j) {
    const double v = Hs[t * j + (j - 1)] + a[t];
    Hs[t * j + (j - 1)] = v;
    Hb[(size_t)t * m + (j - 1)] = v;
  }
  __syncthreads();
  if (t == 0) {
    double aa = 0.0, ab = 0.0, mx = 1.0;
    for (int q = 0; q < j; ++q) {
      aa = fma(a[q], a[q], aa);
      ab = fma(a[q], bq[q], ab);
      mx = fmax(mx, fabs(Hs[q * j + (j - 1)]));
    }
    const double gam = r[2 * j], dlt = r[2 * j + 1];
    double beta = sqrt(fmax(gam - aa, 0.0));
    if (j > 0) {
      if (beta <= KRYLOV_BREAKDOWN * fmax(mx, beta)) beta = 0.0;  // happy breakdown
      Hb[(size_t)j * m + (j - 1)] = beta;
    } else {
      beta0[b] = beta;
    }
    const double ib = beta > 0.0 ? 1.0 / beta : 0.0;
    const double am1 = j > 0 ? a[j - 1] : 0.0;
    const double cv = ib * (ib * (dlt - ab) - beta * am1);
    sh[0] = beta;
    sh[1] = ib;
    sh[2] = ib * (am1 + cv);  // κ
    sh[3] = cv;
  }
  __syncthreads();
  if (final_step) return;
  const double beta = sh[0], ib = sh[1], kap = sh[2];
  if (t < j) {  // row t: (H a)_t over the corrected columns 0 … j−1
    double ha = 0.0;
    for (int c = 0; c < j; ++c) ha = fma(Hs[t * j + c], a[c], ha);
    const double cq = ib * (bq[t] - ha);
    kb[t] = ib * ha + cq - kap * a[t];             // g
    kb[(KRYLOV_MAX_M + 1) + t] = ib * a[t];        // a/β
    Hb[(size_t)t * m + j] = beta > 0.0 ? cq : 0.0;  // column j: first projection (corrected next step)
  }
  if (t == 0) {
    Hb[(size_t)j * m + j] = beta > 0.0 ? sh[3] : 0.0;
    kb[2 * (KRYLOV_MAX_M + 1) + 0] = ib;
    kb[2 * (KRYLOV_MAX_M + 1) + 1] = beta > 0.0 ? kap : 0.0;
  }
}

__global__ void __launch_bounds__(256) k_kr_dfinal(double* H, double* kc, double* beta0, const double* part, int nblk,
                                                   int m, int j, int final_step) {
  kr_dfinal_body(blockIdx.x, H, kc, beta0, part, nblk, m, j, final_step);
}

// w = M·u (u from `u`, batch stride ubs); part slots: [0, j) Q_qᵀu, [j, 2j) Q_qᵀw, 2j γ, 2j+1 δ.
// spmv = false: no w (the final reorthogonalization of u_m): slots [0, j) and 2j only.
// fin != null: the last CTA of each member (atomic ticket after a fence, threadFenceReduction
// pattern) runs the step's finalisation (kr_dfinal_body) — no separate launch.
struct KrFin {
  double *H, *kc, *beta0;
  int* cnt;
  int m, final_step;
};

template <int DIM>
__global__ void __launch_bounds__(256) k_kr_ddots(double* w, const double* u, long long ubs, const double* V, int j,
                                                  Stencil5 st, double* part, int nblk, int B, int nx, int ny,
                                                  int spmv, KrFin fin) {
  const size_t n = (size_t)nx * ny;
  const int b = blockIdx.y;
  const double* ub = u + b * ubs;
  __shared__ double us[KR_BLK], wsh[KR_BLK];
  __shared__ double red[8][2];
  double gam = 0.0, dlt = 0.0;
#pragma unroll
  for (int k = 0; k < KR_PPT; ++k) {
    const size_t i = (size_t)blockIdx.x * KR_BLK + threadIdx.x + 256 * k;
    double uv = 0.0, wv = 0.0;
    if (i < n) {
      uv = ub[i];
      if (spmv) {
        const int y = (int)(i / nx), x = (int)(i - (size_t)y * nx);
        wv = stencil_at<DIM>(ub, st, x, y, nx, ny);
        w[(size_t)b * n + i] = wv;
      }
    }
    us[threadIdx.x + 256 * k] = uv;
    wsh[threadIdx.x + 256 * k] = wv;
    gam = fma(uv, uv, gam);
    dlt = fma(uv, wv, dlt);
  }
  // γ, δ: block sums in fixed order
  for (int o = 16; o > 0; o >>= 1) {
    gam += __shfl_down_sync(0xffffffffu, gam, o);
    dlt += __shfl_down_sync(0xffffffffu, dlt, o);
  }
  const int wid = threadIdx.x >> 5, ln = threadIdx.x & 31;
  if (ln == 0) {
    red[wid][0] = gam;
    red[wid][1] = dlt;
  }
  __syncthreads();
  double* pb = part + (size_t)b * (2 * (KRYLOV_MAX_M + 1) + 1) * nblk;
  if (threadIdx.x < 2 && (spmv || threadIdx.x == 0)) {
    double s2 = 0.0;
    for (int k = 0; k < 8; ++k) s2 += red[k][threadIdx.x];
    pb[(size_t)(2 * j + threadIdx.x) * nblk + blockIdx.x] = s2;
  }
  // Q_qᵀu and Q_qᵀw: one warp per column, the column chunk read once
  const size_t i0 = (size_t)blockIdx.x * KR_BLK;
  const int cnt = (int)min((size_t)KR_BLK, n - i0);
  for (int q = wid; q < j; q += 8) {
    const double* __restrict__ Vq = V + ((size_t)q * B + b) * n + i0;
    double au = 0.0, aw = 0.0;
#pragma unroll 8
    for (int t = ln; t < KR_BLK; t += 32)
      if (t < cnt) {
        const double v = Vq[t];
        au = fma(v, us[t], au);
        aw = fma(v, wsh[t], aw);
      }
    for (int o = 16; o > 0; o >>= 1) {
      au += __shfl_down_sync(0xffffffffu, au, o);
      aw += __shfl_down_sync(0xffffffffu, aw, o);
    }
    if (ln == 0) {
      pb[(size_t)q * nblk + blockIdx.x] = au;
      if (spmv) pb[(size_t)(j + q) * nblk + blockIdx.x] = aw;
    }
  }
  if (fin.cnt) {
    __shared__ int last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = (atomicAdd(fin.cnt + b, 1) == (int)gridDim.x - 1);
    __syncthreads();
    if (last) {
      __threadfence();
      kr_dfinal_body(b, fin.H, fin.kc, fin.beta0, part, nblk, fin.m, j, fin.final_step);
      if (threadIdx.x == 0) fin.cnt[b] = 0;
    }
  }
}

// v_j = u·(1/β) − Σ_q (a_q/β)·Q_q;  u_next = w·(1/β) − κ·u − Σ_q g_q·Q_q  (Q read once)
__global__ void __launch_bounds__(256) k_kr_dupdate(double* Vj, double* unext, const double* u, long long ubs,
                                                    const double* w, const double* V, const double* kc, int j, int B,
                                                    size_t n) {
  const int b = blockIdx.y;
  __shared__ double gs[KRYLOV_MAX_M + 1], as_[KRYLOV_MAX_M + 1];
  __shared__ double sc[2];
  const double* kb = kc + (size_t)b * KC_STRIDE;
  if (threadIdx.x < j) {
    gs[threadIdx.x] = kb[threadIdx.x];
    as_[threadIdx.x] = kb[(KRYLOV_MAX_M + 1) + threadIdx.x];
  }
  if (threadIdx.x < 2) sc[threadIdx.x] = kb[2 * (KRYLOV_MAX_M + 1) + threadIdx.x];
  __syncthreads();
  const double ib = sc[0], kap = sc[1];
  double vv[KR_PPT], uu[KR_PPT];
#pragma unroll
  for (int k = 0; k < KR_PPT; ++k) {
    const size_t i = (size_t)blockIdx.x * KR_BLK + threadIdx.x + 256 * k;
    const double ui = i < n ? u[b * ubs + i] : 0.0;
    const double wi = i < n ? w[(size_t)b * n + i] : 0.0;
    vv[k] = ib * ui;
    uu[k] = fma(-kap, ui, ib * wi);
  }
#pragma unroll 4
  for (int q = 0; q < j; ++q) {
    const double gq = gs[q], aq = as_[q];
    const double* __restrict__ Vq = V + ((size_t)q * B + b) * n;
#pragma unroll
    for (int k = 0; k < KR_PPT; ++k) {
      const size_t i = (size_t)blockIdx.x * KR_BLK + threadIdx.x + 256 * k;
      if (i < n) {
        const double v = Vq[i];
        vv[k] = fma(-aq, v, vv[k]);
        uu[k] = fma(-gq, v, uu[k]);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < KR_PPT; ++k) {
    const size_t i = (size_t)blockIdx.x * KR_BLK + threadIdx.x + 256 * k;
    if (i < n) {
      Vj[(size_t)b * n + i] = vv[k];
      unext[(size_t)b * n + i] = uu[k];
    }
  }
}

inline int krylov_action(KrylovWork& kw, double tau, int substeps, int m, const Stencil5& st,
                         const double* src, long long src_bs, const double* addend, long long add_bs,
                         double* pacc, double* const* ACC, int B, int nx, int ny, int dim,
                         double** result, cudaStream_t s, px_stats* stats, int ortho = 1) {
  const size_t n = kw.n;
  const dim3 g(kw.nblk, B);
  const long long nb = (long long)n;
  uint64_t launches = 0;
  for (int sub = 0; sub < substeps; ++sub) {
    double* out = (src == ACC[0]) ? ACC[1] : ACC[0];
    if (ortho == 1) {  // delayed reorthogonalization: 3 launches and two basis passes per step
      cudaMemsetAsync(kw.H, 0, sizeof(double) * B * (m + 1) * m, s);
      const double* u = src;
      long long ubs = src_bs;
      const KrFin fin{kw.H, kw.kc, kw.beta, kw.cnt, m, 0};
      for (int j = 0; j < m; ++j) {
        if (dim == 2)
          k_kr_ddots<2><<<g, 256, 0, s>>>(kw.w, u, ubs, kw.V, j, st, kw.part, kw.nblk, B, nx, ny, 1, fin);
        else
          k_kr_ddots<1><<<g, 256, 0, s>>>(kw.w, u, ubs, kw.V, j, st, kw.part, kw.nblk, B, nx, ny, 1, fin);
        double* un = kw.u + (size_t)(j & 1) * B * n;
        k_kr_dupdate<<<g, 256, 0, s>>>(kw.V + (size_t)j * B * n, un, u, ubs, kw.w, kw.V, kw.kc, j, B, n);
        u = un;
        ubs = nb;
        launches += 2;
      }
      // the delayed second projection of the last candidate completes H's last column
      const KrFin fin_last{kw.H, kw.kc, kw.beta, kw.cnt, m, 1};
      if (dim == 2)
        k_kr_ddots<2><<<g, 256, 0, s>>>(kw.w, u, ubs, kw.V, m, st, kw.part, kw.nblk, B, nx, ny, 0, fin_last);
      else
        k_kr_ddots<1><<<g, 256, 0, s>>>(kw.w, u, ubs, kw.V, m, st, kw.part, kw.nblk, B, nx, ny, 0, fin_last);
      const int N = m + 1;
      const size_t smem = KR_EXPM_MATS * (size_t)N * N * sizeof(double);
      cudaFuncSetAttribute(k_kr_expm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k_kr_expm<<<B, 256, smem, s>>>(kw.coef, kw.H, kw.beta, m, tau);
      k_kr_combine<<<dim3((unsigned)((n + 255) / 256), B), 256, 0, s>>>(
          out, kw.V, kw.coef, m, B, n, sub == substeps - 1 ? addend : nullptr, add_bs, pacc);
      launches += 3;
      src = out;
      src_bs = nb;
      continue;
    }
    k_kr_sumsq<<<g, 256, 0, s>>>(kw.part, kw.nblk, src, src_bs, n);
    k_kr_beta<<<B, 256, 0, s>>>(kw.beta, kw.part, kw.nblk);
    k_kr_v0<<<dim3((unsigned)((n + 255) / 256), B), 256, 0, s>>>(kw.V, src, src_bs, kw.beta, n);
    launches += 3;
    cudaMemsetAsync(kw.H, 0, sizeof(double) * B * (m + 1) * m, s);
    for (int j = 0; j < m; ++j) {
      double* wj = kw.w + (size_t)(j & 1) * B * n;
      const double* wprev = kw.w + (size_t)((j + 1) & 1) * B * n;
      if (dim == 2)
        k_kr_spmv_dots<2><<<g, 256, 0, s>>>(wj, kw.V, wprev, kw.hcol, j, st, kw.part, kw.nblk, B, nx, ny);
      else
        k_kr_spmv_dots<1><<<g, 256, 0, s>>>(wj, kw.V, wprev, kw.hcol, j, st, kw.part, kw.nblk, B, nx, ny);
      k_kr_finalize_dots<<<dim3(j + 1, B), 256, 0, s>>>(kw.hcol, kw.H, kw.part, kw.nblk, m, j, 0);
      k_kr_update<<<g, 256, 0, s>>>(wj, kw.V, j, kw.hcol, kw.part, kw.nblk, B, n, 0);
      k_kr_finalize_dots<<<dim3(j + 1, B), 256, 0, s>>>(kw.hcol, kw.H, kw.part, kw.nblk, m, j, 1);
      k_kr_update<<<g, 256, 0, s>>>(wj, kw.V, j, kw.hcol, kw.part, kw.nblk, B, n, 1);
      k_kr_finalize_norm<<<B, 256, 0, s>>>(kw.hcol, kw.H, kw.part, kw.nblk, m, j);
      launches += 6;
    }
    const int N = m + 1;
    const size_t smem = KR_EXPM_MATS * (size_t)N * N * sizeof(double);
    cudaFuncSetAttribute(k_kr_expm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_kr_expm<<<B, 256, smem, s>>>(kw.coef, kw.H, kw.beta, m, tau);
    k_kr_combine<<<dim3((unsigned)((n + 255) / 256), B), 256, 0, s>>>(
        out, kw.V, kw.coef, m, B, n, sub == substeps - 1 ? addend : nullptr, add_bs, pacc);
    launches += 2;
    src = out;
    src_bs = nb;
  }
  if (stats) {
    stats->kernel_launches += launches;
    stats->arnoldi_steps += (uint64_t)substeps * m * B;
    stats->exp_terms += (uint64_t)substeps * m * B;
    // Arnoldi step j (SURVEY §8(d)'s CGS unit, kept as the model for both forms): SpMV in/out
    // 16n + read V_0..V_j for the dots and again for the update, twice (CGS2) ≈ 16n + 32n(j+1);
    // the delayed form moves ≈ 16n + 16n·j + 40n of it
    double bytes = 0.0;
    for (int j = 0; j < m; ++j) bytes += 16.0 * n + 32.0 * n * (j + 1);
    bytes += 8.0 * n * (m + 2);  // combine (+ pacc)
    bytes *= (double)substeps * B;
    stats->exp_bytes += bytes;
    stats->algorithmic_bytes += bytes;
  }
  *result = const_cast<double*>(src);
  return PX_OK;
}

}  // namespace px

