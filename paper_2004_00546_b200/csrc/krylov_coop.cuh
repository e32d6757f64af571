// krylov_coop.cuh — cooperative persistent Arnoldi exponential action.
//
// Same arithmetic as the multi-kernel path in krylov.cuh (CGS2, happy-breakdown
// rule, augmented Taylor-18 exponential, β-scaled combination) but ONE launch per
// substep: every block owns a contiguous range of points and the phases are
// separated by grid-wide barriers (3 per Arnoldi step), removing ~6 dependent
// launches per step. All blocks reduce the per-block partials in the same fixed
// order, so every block holds bit-identical h, ‖w‖ and breakdown decisions.
// Partial-sum rows: [0, MAX_M] first CGS pass, [MAX_M+1, 2·MAX_M+1] second pass,
// 2·(MAX_M+1) norms — distinct rows so no block overwrites partials another block
// may still be reading.
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "krylov.cuh"

namespace px {

constexpr int KC_ROWS = 2 * (KRYLOV_MAX_M + 1) + 1;

struct KrCoopArgs {
  const double* src; long long src_bs;   // y (batch-strided)
  double* out;                           // B × n result
  const double* addend; long long add_bs;
  double* pacc;                          // may be null
  double* V;                             // (m+1) × B × n
  double* w;                             // 2 × B × n
  double* H;                             // B × (m+1) × m
  double* part;                          // B × KC_ROWS × nblk
  double* coef;                          // B × 2 × m
  Stencil5 st;
  double tau;
  int m, B, nx, ny;
};

// out[q] = Σ_{t<cnt} p[q·stride + t] for q < nq: one warp per column (fixed order:
// lane-strided partial sums, then a shuffle tree), one block barrier at the end.
__device__ __forceinline__ void multi_fixed_sum(const double* p, int nq, int cnt, size_t stride, double* out) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int q = w; q < nq; q += 8) {
    const double* col = p + (size_t)q * stride;
    double v = 0.0;
    for (int t = l; t < cnt; t += 32) v += col[t];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (l == 0) out[q] = v;
  }
  __syncthreads();
}

template <int DIM>
__global__ void __launch_bounds__(256) k_kr_coop(KrCoopArgs a) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double kc_sm[];  // expm scratch (block 0)
  __shared__ double red[8][KRYLOV_MAX_M + 1];
  __shared__ double red1[8];
  __shared__ double h1[KRYLOV_MAX_M + 1], h2[KRYLOV_MAX_M + 1];
  __shared__ double sc[2];
  const int nx = a.nx, ny = a.ny, m = a.m, B = a.B;
  const size_t n = (size_t)nx * ny;
  const int nblk = gridDim.x;
  const size_t per = (n + nblk - 1) / nblk;
  const size_t i0 = min(n, (size_t)blockIdx.x * per);
  const size_t i1 = min(n, i0 + per);
  const int NR = KRYLOV_MAX_M + 1;
  for (int b = 0; b < B; ++b) {
    const double* y = a.src + b * a.src_bs;
    double* P1 = a.part + (size_t)b * KC_ROWS * nblk;
    double* P2 = P1 + (size_t)NR * nblk;
    double* PN = P1 + (size_t)2 * NR * nblk;
    double* Hb = a.H + (size_t)b * (m + 1) * m;
    // β = ‖y‖
    double v = 0.0;
    for (size_t i = i0 + threadIdx.x; i < i1; i += 256) v += y[i] * y[i];
    v = block_sum<256>(v, red1);
    if (threadIdx.x == 0) PN[blockIdx.x] = v;
    grid.sync();
    multi_fixed_sum(PN, 1, nblk, nblk, sc);
    const double beta = sqrt(sc[0]);
    double inv = beta > 0.0 ? 1.0 / beta : 0.0;
    if (blockIdx.x == 0)
      for (int t = threadIdx.x; t < (m + 1) * m; t += 256) Hb[t] = 0.0;
    const double* srcj = y;  // V_j = srcj · inv
    for (int j = 0; j < m; ++j) {
      double* Vj = a.V + ((size_t)j * B + b) * n;
      double* wj = a.w + ((size_t)(j & 1) * B + b) * n;
      double dq[KRYLOV_MAX_M + 1];
      // (a) materialise V_j, w = M V_j, first-pass dots
      for (int q = 0; q <= j; ++q) dq[q] = 0.0;
      for (size_t i = i0 + threadIdx.x; i < i1; i += 256) {
        const int yy = (int)(i / nx), xx = (int)(i - (size_t)yy * nx);
        const double vj = srcj[i] * inv;
        Vj[i] = vj;
        const double wv = inv * stencil_at<DIM>(srcj, a.st, xx, yy, nx, ny);
        wj[i] = wv;
        for (int q = 0; q < j; ++q) dq[q] += a.V[((size_t)q * B + b) * n + i] * wv;
        dq[j] += vj * wv;
      }
      block_multi_sum(red, j + 1, dq, P1 + blockIdx.x, nblk);
      grid.sync();
      // (b) h1 = Σ partials; w -= V h1; second-pass dots
      multi_fixed_sum(P1, j + 1, nblk, nblk, h1);
      for (int q = 0; q <= j; ++q) dq[q] = 0.0;
      for (size_t i = i0 + threadIdx.x; i < i1; i += 256) {
        double x = wj[i];
        for (int q = 0; q <= j; ++q) x -= h1[q] * a.V[((size_t)q * B + b) * n + i];
        wj[i] = x;
        for (int q = 0; q <= j; ++q) dq[q] += a.V[((size_t)q * B + b) * n + i] * x;
      }
      block_multi_sum(red, j + 1, dq, P2 + blockIdx.x, nblk);
      grid.sync();
      // (c) h2; w -= V h2; ‖w‖² partials
      multi_fixed_sum(P2, j + 1, nblk, nblk, h2);
      double nn = 0.0;
      for (size_t i = i0 + threadIdx.x; i < i1; i += 256) {
        double x = wj[i];
        for (int q = 0; q <= j; ++q) x -= h2[q] * a.V[((size_t)q * B + b) * n + i];
        wj[i] = x;
        nn += x * x;
      }
      nn = block_sum<256>(nn, red1);
      if (threadIdx.x == 0) PN[blockIdx.x] = nn;
      grid.sync();
      // (d) column j of H, h_{j+1,j}, breakdown (identical in every block)
      {
        __shared__ double tot_s;
        multi_fixed_sum(PN, 1, nblk, nblk, &tot_s);
        if (threadIdx.x == 0) {
          const double nrm = sqrt(tot_s);
          double mx = fmax(1.0, nrm);
          for (int q = 0; q <= j; ++q) mx = fmax(mx, fabs(h1[q] + h2[q]));
          const bool brk = nrm <= KRYLOV_BREAKDOWN * mx;
          sc[0] = brk ? 0.0 : 1.0 / nrm;
          sc[1] = brk ? 0.0 : nrm;
        }
        __syncthreads();
      }
      if (blockIdx.x == 0) {
        if (threadIdx.x <= j) Hb[(size_t)threadIdx.x * m + j] = h1[threadIdx.x] + h2[threadIdx.x];
        if (threadIdx.x == 0) Hb[(size_t)(j + 1) * m + j] = sc[1];
      }
      inv = sc[0];
      srcj = wj;
      __syncthreads();
    }
    // exponential of the augmented Hessenberg matrix (block 0), then combine
    if (blockIdx.x == 0) {
      __syncthreads();
      expm_aug_block(a.coef + (size_t)b * 2 * m, Hb, beta, m, a.tau, kc_sm);
    }
    grid.sync();
    const double* ce = a.coef + (size_t)b * 2 * m;
    const double* cp = ce + m;
    for (size_t i = i0 + threadIdx.x; i < i1; i += 256) {
      double e = 0.0, p = 0.0;
      for (int q = 0; q < m; ++q) {
        const double vq = a.V[((size_t)q * B + b) * n + i];
        e += ce[q] * vq;
        p += cp[q] * vq;
      }
      if (a.addend) e += a.addend[b * a.add_bs + i];
      a.out[(size_t)b * n + i] = e;
      if (a.pacc) a.pacc[(size_t)b * n + i] += p;
    }
    grid.sync();  // next member reuses the shared partial rows / basis
  }
}

inline size_t kr_coop_smem(int m) { return 3 * (size_t)(m + 1) * (m + 1) * sizeof(double); }

}  // namespace px

namespace px {

// Blocks of the cooperative grid (all co-resident): SMs × occupancy, capped by
// the point count (each block needs at least a few warps' worth of points).
inline int kr_coop_blocks(int dim, int m, size_t n) {
  static int cached[2] = {0, 0};
  int& c = cached[dim == 2 ? 1 : 0];
  if (c == 0) {
    int dev = 0, sms = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (dim == 2) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_kr_coop<2>, 256, kr_coop_smem(KRYLOV_MAX_M));
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_kr_coop<1>, 256, kr_coop_smem(KRYLOV_MAX_M));
    c = sms * std::max(1, std::min(occ, 2));
  }
  return (int)std::max<size_t>(1, std::min<size_t>((size_t)c, (n + 255) / 256));
}

inline int krylov_action_coop(KrylovWork& kw, double tau, int substeps, int m, const Stencil5& st,
                              const double* src, long long src_bs, const double* addend, long long add_bs,
                              double* pacc, double* const* ACC, int B, int nx, int ny, int dim,
                              double** result, cudaStream_t s, px_stats* stats) {
  const size_t n = kw.n;
  const int nblk = kr_coop_blocks(dim, m, n);
  const size_t smem = kr_coop_smem(m);
  for (int sub = 0; sub < substeps; ++sub) {
    double* out = (src == ACC[0]) ? ACC[1] : ACC[0];
    KrCoopArgs a{};
    a.src = src; a.src_bs = src_bs;
    a.out = out;
    a.addend = (sub == substeps - 1) ? addend : nullptr;
    a.add_bs = add_bs;
    a.pacc = pacc;
    a.V = kw.V; a.w = kw.w; a.H = kw.H; a.part = kw.part; a.coef = kw.coef;
    a.st = st; a.tau = tau; a.m = m; a.B = B; a.nx = nx; a.ny = ny;
    void* args[] = {&a};
    cudaError_t e;
    if (dim == 2) e = cudaLaunchCooperativeKernel((const void*)k_kr_coop<2>, dim3(nblk), dim3(256), args, smem, s);
    else e = cudaLaunchCooperativeKernel((const void*)k_kr_coop<1>, dim3(nblk), dim3(256), args, smem, s);
    if (e != cudaSuccess) return PX_ERR_CUDA;
    src = out;
    src_bs = (long long)n;
  }
  if (stats) {
    stats->kernel_launches += substeps;
    stats->arnoldi_steps += (uint64_t)substeps * m * B;
    stats->exp_terms += (uint64_t)substeps * m * B;
    double bytes = 0.0;
    for (int j = 0; j < m; ++j) bytes += 16.0 * n + 32.0 * n * (j + 1);
    bytes += 8.0 * n * (m + 2);
    bytes *= (double)substeps * B;
    stats->exp_bytes += bytes;
    stats->algorithmic_bytes += bytes;
  }
  *result = const_cast<double*>(src);
  return PX_OK;
}

}  // namespace px
