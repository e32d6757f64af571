// burgers.cuh — BASELINE config 3: 1D viscous Burgers, serial direct sweep with
// the trajectory kept in HBM, Paraexp adjoint with piecewise-frozen linearisation.
//
// Reference pieces restated here (Option A of SURVEY.md §8(c)):
//   serial direct sweep        hybrid.py:185-191, serial.py:17-25 (rk45 -> fixed RK4)
//   Burgers rhs (V ≡ 0)        problems.py:177-185
//   Jᵀ(u)·y matrix-free        problems.py:316-343
//   linear interpolation of the stored trajectory at RK stages   timestepping.py:64-75
//   trapezoid-averaged frozen operator J(ū_p)ᵀ                   problems.py:346-366,
//                                                                systems.py:76-97
//   absorbed final condition, reflected time                    paraexp.py:256-295,329-353
// The states are small (n ≤ 8192): every sweep runs with the state in shared
// memory — the direct sweep is ONE persistent CTA per batch member stepping
// P·nsteps times, the adjoint slice solves are one CTA per (member, slice), and
// the homogeneous carry over all slices is one persistent CTA per member.
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "../../include/paraexp.h"
#include "common.cuh"

namespace px {

constexpr int BURGERS_MAX_N = 8192;
constexpr int BURGERS_NT = 1024;

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

struct BurgersDirectArgs {
  const double *u0, *ctrl, *tx;
  const int* ix;
  int K;
  double *traj, *ubar, *UT, *bpart, *bounds;
  int bounds_blocks;
  double D, hx, h;
  int nx, B, P, nsteps;
};

struct BurgersAdjointArgs {
  const double *traj, *ubar, *QT;
  double *W0, *W1, *Z, *G, *QDAG0;
  double* Wk[3];
  double* ACC[2];
  double D, hx, h;
  int nx, B, P, nsteps, p_begin, p_end;
  int substeps, degree, sigma;
  double center, scale;
  const double *be, *bp;
  // 1: the reference's solve_hybrid adjoint (hybrid.py:212-237) for a terminal objective:
  // no adjoint source, so the inhomogeneous solves (zero terminal data) vanish and q† is
  // q†_T propagated over [T, 0] through the frozen J(ū_p)ᵀ; 0: absorbed final condition
  int terminal_span;
};

// rhs(u)_i = −u_i·(u_{i+1} − u_{i−1})/(2h) + D·(u_{i+1} − 2u_i + u_{i−1})/h² + f_i
__device__ __forceinline__ double burgers_rhs_at(const double* s, int i, int n, double inv2h, double Dih2,
                                                 double f) {
  const int ip = (i + 1 == n) ? 0 : i + 1, im = (i == 0) ? n - 1 : i - 1;
  const double u = s[i], up = s[ip], um = s[im];
  const double dx = (up - um) * inv2h;
  const double lap = (up - 2.0 * u + um) * Dih2;
  return -u * dx + lap + f;
}

// One CTA per member; whole serial sweep (S = P·nsteps steps) with u in smem.
// Every node is written to traj[s][b][:] (the HBM-resident direct trajectory).
template <int PPT>
__global__ void __launch_bounds__(BURGERS_NT) k_burgers_direct(BurgersDirectArgs a) {
  extern __shared__ double sm[];
  const int n = a.nx;
  // stage inputs: s0 = u, s1 = u + (h/2)k1, s2 = u + (h/2)k2, s3 = u + h·k3 (aliases s1, whose
  // last readers, stage 2, finished before the barrier after stage 2); the new state goes back
  // into s0 (last read in stage 1): one barrier per stage, none for a separate state copy
  double* s0 = sm;
  double* s1 = sm + n;
  double* s2 = sm + 2 * n;
  double* s3 = s1;
  const int b = blockIdx.x;
  const double inv2h = 1.0 / (2.0 * a.hx);
  const double Dih2 = a.D / (a.hx * a.hx);
  const double h = a.h, hh = 0.5 * a.h, h6 = a.h / 6.0;
  double f[PPT], u[PPT], acc[PPT];
  const double* c = a.ctrl + (size_t)b * a.K;
#pragma unroll
  for (int t = 0; t < PPT; ++t) {
    const int i = threadIdx.x + t * BURGERS_NT;
    f[t] = 0.0;
    u[t] = 0.0;
    if (i < n) {
      double fv = 0.0;
      for (int k = 0; k < a.K; ++k) fv += c[k] * a.tx[(size_t)a.ix[k] * n + i];
      f[t] = fv;
      u[t] = a.u0[i];
      s0[i] = u[t];
      a.traj[(size_t)b * n + i] = u[t];
    }
  }
  __syncthreads();
  const size_t S = (size_t)a.P * a.nsteps;
  const size_t node_stride = (size_t)a.B * n;
  for (size_t st = 0; st < S; ++st) {
#pragma unroll
    for (int t = 0; t < PPT; ++t) {
      const int i = threadIdx.x + t * BURGERS_NT;
      if (i < n) {
        const double k = burgers_rhs_at(s0, i, n, inv2h, Dih2, f[t]);
        acc[t] = k;
        s1[i] = u[t] + hh * k;
      }
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < PPT; ++t) {
      const int i = threadIdx.x + t * BURGERS_NT;
      if (i < n) {
        const double k = burgers_rhs_at(s1, i, n, inv2h, Dih2, f[t]);
        acc[t] += 2.0 * k;
        s2[i] = u[t] + hh * k;
      }
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < PPT; ++t) {
      const int i = threadIdx.x + t * BURGERS_NT;
      if (i < n) {
        const double k = burgers_rhs_at(s2, i, n, inv2h, Dih2, f[t]);
        acc[t] += 2.0 * k;
        s3[i] = u[t] + h * k;
      }
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < PPT; ++t) {
      const int i = threadIdx.x + t * BURGERS_NT;
      if (i < n) {
        const double k = burgers_rhs_at(s3, i, n, inv2h, Dih2, f[t]);
        u[t] = u[t] + h6 * (acc[t] + k);
        s0[i] = u[t];
        a.traj[(st + 1) * node_stride + (size_t)b * n + i] = u[t];
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int t = 0; t < PPT; ++t) {
    const int i = threadIdx.x + t * BURGERS_NT;
    if (i < n) a.UT[(size_t)b * n + i] = u[t];
  }
}

// Same sweep with each thread owning a contiguous run of PPT points (n = PPT·blockDim):
// neighbours inside the run come from registers, only the run edges go through shared
// memory (one vector store + two scalar loads per stage), and the right-hand side is
// rearranged to 5 flops per point: rhs = D/h²·(u₊ + u₋) + f − u·(2D/h² + (u₊ − u₋)/(2h)).
template <int PPT>
__global__ void __launch_bounds__(BURGERS_NT) k_burgers_direct_run(BurgersDirectArgs a) {
  extern __shared__ double sm[];
  const int n = a.nx;
  const int T = n / PPT;  // threads with points (blockDim ≥ T)
  double* sA = sm;        // [2][n]: stage inputs, double buffered
  const int b = blockIdx.x;
  const int t = threadIdx.x;
  const bool act = t < T;
  const int i0 = t * PPT;
  const int il = (i0 == 0) ? n - 1 : i0 - 1;            // left neighbour of the run
  const int ir = (i0 + PPT >= n) ? 0 : i0 + PPT;        // right neighbour of the run
  const double inv2h = 1.0 / (2.0 * a.hx);
  const double Dih2 = a.D / (a.hx * a.hx), twoD = 2.0 * Dih2;
  const double h = a.h, hh = 0.5 * a.h, h6 = a.h / 6.0;
  double f[PPT], u[PPT], acc[PPT], x[PPT];
  const double* c = a.ctrl + (size_t)b * a.K;
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    f[k] = 0.0;
    u[k] = 0.0;
    if (act) {
      const int i = i0 + k;
      double fv = 0.0;
      for (int q = 0; q < a.K; ++q) fv += c[q] * a.tx[(size_t)a.ix[q] * n + i];
      f[k] = fv;
      u[k] = a.u0[i];
      a.traj[(size_t)b * n + i] = u[k];
    }
  }
  const size_t S = (size_t)a.P * a.nsteps;
  const size_t node_stride = (size_t)a.B * n;
  int par = 0;
  // rhs of the stage input x (run in registers, edges from the other threads via smem)
  auto rhs = [&](double* k_out) {
    double* sx = sA + par * n;
    if (act) {
#pragma unroll
      for (int k = 0; k < PPT; ++k) sx[i0 + k] = x[k];
    }
    __syncthreads();
    const double xl = act ? sx[il] : 0.0, xr = act ? sx[ir] : 0.0;
    par ^= 1;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      const double um = (k == 0) ? xl : x[k - 1];
      const double up = (k + 1 == PPT) ? xr : x[k + 1];
      const double A = up + um, B = up - um;
      const double t1 = fma(Dih2, A, f[k]);
      const double t2 = fma(inv2h, B, twoD);
      k_out[k] = fma(-x[k], t2, t1);
    }
  };
  double kk[PPT];
  for (size_t st = 0; st < S; ++st) {
#pragma unroll
    for (int k = 0; k < PPT; ++k) x[k] = u[k];
    rhs(kk);
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      acc[k] = kk[k];
      x[k] = fma(hh, kk[k], u[k]);
    }
    rhs(kk);
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      acc[k] = fma(2.0, kk[k], acc[k]);
      x[k] = fma(hh, kk[k], u[k]);
    }
    rhs(kk);
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      acc[k] = fma(2.0, kk[k], acc[k]);
      x[k] = fma(h, kk[k], u[k]);
    }
    rhs(kk);
#pragma unroll
    for (int k = 0; k < PPT; ++k) u[k] = fma(h6, acc[k] + kk[k], u[k]);
    if (act) {
      double* node = a.traj + (st + 1) * node_stride + (size_t)b * n + i0;
#pragma unroll
      for (int k = 0; k < PPT; ++k) node[k] = u[k];
    }
  }
  if (act) {
#pragma unroll
    for (int k = 0; k < PPT; ++k) a.UT[(size_t)b * n + i0 + k] = u[k];
  }
}

// ū_p[b][i] = Σ_j w_j traj[p·ns + j][b][i], trapezoid weights (½,1,…,1,½)/ns
__global__ void k_slice_means(double* ubar, const double* traj, int P, int nsteps, int B, int n) {
  const size_t total = (size_t)P * B * n;
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (size_t)gridDim.x * blockDim.x) {
    const int p = (int)(idx / ((size_t)B * n));
    const size_t rem = idx - (size_t)p * B * n;  // b*n + i
    const double* src = traj + (size_t)p * nsteps * B * n + rem;
    const double w = 1.0 / nsteps;
    double s = (0.5 * w) * src[0];
    for (int j = 1; j < nsteps; ++j) s += w * src[(size_t)j * B * n];
    s += (0.5 * w) * src[(size_t)nsteps * B * n];
    ubar[idx] = s;
  }
}

// min / max that propagate NaN (fmin/fmax drop it): a non-finite trajectory must reach the
// host as a non-finite bound, not as a silently smaller box
__device__ __forceinline__ double nan_min(double a, double b) { return (a < b || a != a) ? a : b; }
__device__ __forceinline__ double nan_max(double a, double b) { return (a > b || a != a) ? a : b; }

// Field-of-values box of B̄ = J(ū)ᵀ, union over slices and members (see
// problems.burgers_frozen_region): (min re_lo, max re_hi, max im) partials.
__global__ void __launch_bounds__(256) k_frozen_bounds(double* bpart, const double* ubar, size_t total, int n,
                                                       double hx, double D) {
  __shared__ double r0[8], r1[8], r2[8];
  double lo = 1e300, hi = -1e300, im = 0.0;
  const double inv2h = 1.0 / (2.0 * hx), inv4h = 1.0 / (4.0 * hx), dh2 = 2.0 * D / (hx * hx);
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (size_t)gridDim.x * blockDim.x) {
    const size_t row = idx / n;
    const int i = (int)(idx - row * n);
    const double* u = ubar + row * n;
    const double uc = u[i], up = u[i + 1 == n ? 0 : i + 1], um = u[i == 0 ? n - 1 : i - 1];
    const double dxu = (up - um) * inv2h;
    const double diag = -dxu - dh2;
    const double rad = (fabs(up - uc) + fabs(uc - um)) * inv4h + dh2;
    lo = nan_min(lo, diag - rad);
    hi = nan_max(hi, diag + rad);
    im = nan_max(im, (fabs(up + uc) + fabs(uc + um)) * inv4h);
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = nan_min(lo, __shfl_down_sync(0xffffffffu, lo, o));
    hi = nan_max(hi, __shfl_down_sync(0xffffffffu, hi, o));
    im = nan_max(im, __shfl_down_sync(0xffffffffu, im, o));
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { r0[w] = lo; r1[w] = hi; r2[w] = im; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < 8; ++k) { lo = nan_min(lo, r0[k]); hi = nan_max(hi, r1[k]); im = nan_max(im, r2[k]); }
    bpart[3 * blockIdx.x + 0] = lo;
    bpart[3 * blockIdx.x + 1] = hi;
    bpart[3 * blockIdx.x + 2] = im;
  }
}

// one CTA of 256 threads: min / max are order-independent, so the result is exact and
// deterministic whatever the reduction tree
__global__ void __launch_bounds__(256) k_frozen_bounds_final(double* bounds, const double* bpart, int m) {
  __shared__ double r0[8], r1[8], r2[8];
  double lo = 1e300, hi = -1e300, im = 0.0;
  for (int k = threadIdx.x; k < m; k += blockDim.x) {
    lo = nan_min(lo, bpart[3 * k]);
    hi = nan_max(hi, bpart[3 * k + 1]);
    im = nan_max(im, bpart[3 * k + 2]);
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = nan_min(lo, __shfl_down_sync(0xffffffffu, lo, o));
    hi = nan_max(hi, __shfl_down_sync(0xffffffffu, hi, o));
    im = nan_max(im, __shfl_down_sync(0xffffffffu, im, o));
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    r0[w] = lo;
    r1[w] = hi;
    r2[w] = im;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) {
      lo = nan_min(lo, r0[k]);
      hi = nan_max(hi, r1[k]);
      im = nan_max(im, r2[k]);
    }
    bounds[0] = lo;
    bounds[1] = hi;
    bounds[2] = im;
  }
}

// (Jᵀ(u) y)_i = (u_{i+1}y_{i+1} − u_{i−1}y_{i−1})/(2h) − (u_{i+1} − u_{i−1})/(2h)·y_i
//              + D(y_{i+1} − 2y_i + y_{i−1})/h²
__device__ __forceinline__ double jt_at(const double* su, const double* sy, int i, int n, double inv2h,
                                        double Dih2) {
  const int ip = (i + 1 == n) ? 0 : i + 1, im = (i == 0) ? n - 1 : i - 1;
  const double up = su[ip], um = su[im];
  const double yp = sy[ip], ym = sy[im], yc = sy[i];
  const double dxuy = (up * yp - um * ym) * inv2h;
  const double dxu = (up - um) * inv2h;
  const double lap = (yp - 2.0 * yc + ym) * Dih2;
  return dxuy - dxu * yc + lap;
}

// One CTA per lane (member b, slice p): reflected-time RK4 of
// w' = Jᵀ(u(t))(w + q†_T), w(0) = 0, z = ∫w; u at stage times by linear
// interpolation of the stored nodes (half steps: 0.5·u_j + 0.5·u_{j−1}).
template <int PPT>
__global__ void __launch_bounds__(BURGERS_NT) k_burgers_adjoint_rk4(BurgersAdjointArgs a) {
  extern __shared__ double sm[];
  const int n = a.nx;
  double* s_ua = sm;
  double* s_ub = sm + n;
  double* s_um = sm + 2 * n;
  double* s_y = sm + 3 * n;
  const int Pl = a.p_end - a.p_begin;
  const int lane = blockIdx.x;
  const int b = lane / Pl;
  const int p = a.p_begin + (lane - b * Pl);
  const double inv2h = 1.0 / (2.0 * a.hx);
  const double Dih2 = a.D / (a.hx * a.hx);
  const double h = a.h, hh = 0.5 * a.h, h6 = a.h / 6.0;
  const size_t node_stride = (size_t)a.B * n;
  const double* qT = a.QT + (size_t)b * n;
  double q[PPT], w[PPT], z[PPT], acc[PPT], zacc[PPT];
  const int top = (p + 1) * a.nsteps;
#pragma unroll
  for (int t = 0; t < PPT; ++t) {
    const int i = threadIdx.x + t * BURGERS_NT;
    w[t] = 0.0;
    z[t] = 0.0;
    q[t] = 0.0;
    if (i < n) {
      q[t] = qT[i];
      s_ua[i] = a.traj[(size_t)top * node_stride + (size_t)b * n + i];
    }
  }
  double* ua = s_ua;
  double* ub = s_ub;
  for (int st = 0; st < a.nsteps; ++st) {
    const double* nodeb = a.traj + (size_t)(top - st - 1) * node_stride + (size_t)b * n;
#pragma unroll
    for (int t = 0; t < PPT; ++t) {
      const int i = threadIdx.x + t * BURGERS_NT;
      if (i < n) {
        const double vb = nodeb[i];
        ub[i] = vb;
        s_um[i] = 0.5 * ua[i] + 0.5 * vb;
        s_y[i] = w[t] + q[t];
      }
    }
    __syncthreads();
    double Y[PPT];
#pragma unroll
    for (int t = 0; t < PPT; ++t) {
      const int i = threadIdx.x + t * BURGERS_NT;
      if (i < n) {
        const double k = jt_at(ua, s_y, i, n, inv2h, Dih2);
        acc[t] = k;
        Y[t] = w[t] + hh * k;
        zacc[t] = w[t] + 2.0 * Y[t];
      }
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < PPT; ++t) {
      const int i = threadIdx.x + t * BURGERS_NT;
      if (i < n) s_y[i] = Y[t] + q[t];
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < PPT; ++t) {
      const int i = threadIdx.x + t * BURGERS_NT;
      if (i < n) {
        const double k = jt_at(s_um, s_y, i, n, inv2h, Dih2);
        acc[t] += 2.0 * k;
        Y[t] = w[t] + hh * k;
        zacc[t] += 2.0 * Y[t];
      }
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < PPT; ++t) {
      const int i = threadIdx.x + t * BURGERS_NT;
      if (i < n) s_y[i] = Y[t] + q[t];
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < PPT; ++t) {
      const int i = threadIdx.x + t * BURGERS_NT;
      if (i < n) {
        const double k = jt_at(s_um, s_y, i, n, inv2h, Dih2);
        acc[t] += 2.0 * k;
        Y[t] = w[t] + h * k;
        zacc[t] += Y[t];
      }
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < PPT; ++t) {
      const int i = threadIdx.x + t * BURGERS_NT;
      if (i < n) s_y[i] = Y[t] + q[t];
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < PPT; ++t) {
      const int i = threadIdx.x + t * BURGERS_NT;
      if (i < n) {
        const double k = jt_at(ub, s_y, i, n, inv2h, Dih2);
        z[t] = z[t] + h6 * zacc[t];
        w[t] = w[t] + h6 * (acc[t] + k);
      }
    }
    __syncthreads();
    double* tmp = ua;
    ua = ub;
    ub = tmp;
  }
#pragma unroll
  for (int t = 0; t < PPT; ++t) {
    const int i = threadIdx.x + t * BURGERS_NT;
    if (i < n) {
      a.W0[(size_t)lane * n + i] = w[t];
      a.Z[(size_t)lane * n + i] = z[t];
    }
  }
}

// One CTA per member: the homogeneous carry over all slices, frozen operators
// J(ū_p)ᵀ, Chebyshev substeps with exp and φ₁ accumulators, state in smem.
//   C <- w_{p1−1};  for p = p1−2 … p0: C <- exp(ΔB̄_p)C + w_p,  G += Δφ₁(ΔB̄_p)C
//   for p = p0−1 … 0: C <- exp(ΔB̄_p)C (carry through earlier ranks' slices)
template <int PPT>
__global__ void __launch_bounds__(BURGERS_NT) k_burgers_scan(BurgersAdjointArgs a, const double* coef) {
  extern __shared__ double sm[];
  const int n = a.nx;
  double* s_cur = sm;  // [2][n]: U_k, double buffered (one barrier per term)
  const int b = blockIdx.x;
  const int Pl = a.p_end - a.p_begin;
  const double inv2h = 1.0 / (2.0 * a.hx);
  const double Dih2 = a.D / (a.hx * a.hx);
  const double c0 = a.center, two_over = 2.0 / a.scale, sigma = (double)a.sigma;
  const double* __restrict__ be = coef;
  const double* __restrict__ bp = coef + a.degree + 1;
  const int degree = a.degree, substeps = a.substeps;
  double C[PPT], Gp[PPT], prev[PPT], cur[PPT], acc[PPT], pac[PPT];
  // per point, per slice: J(ū)ᵀy = kp·y₊ + km·y₋ + kc·y with kp = ū₊/(2h) + D/h²,
  // km = −ū₋/(2h) + D/h², kc = −(ū₊ − ū₋)/(2h) − 2D/h² (problems.py:316-343), folded with the
  // Chebyshev shift/scale: first term f·(y₊, y₋, y), later terms g·(y₊, y₋, y) + σ·U_{k−1}
  double gp[PPT], gm[PPT], gc[PPT];  // the first term uses f = g/2
  auto ipx = [&](int t) { const int i = threadIdx.x + t * BURGERS_NT; return (i + 1 >= n) ? 0 : i + 1; };
  auto imx = [&](int t) { const int i = threadIdx.x + t * BURGERS_NT; return (i == 0) ? n - 1 : i - 1; };
#pragma unroll
  for (int t = 0; t < PPT; ++t) {
    const int i = threadIdx.x + t * BURGERS_NT;
    C[t] = Gp[t] = 0.0;
    if (i < n) {
      C[t] = a.terminal_span ? a.QT[(size_t)b * n + i] : a.W0[((size_t)b * Pl + (Pl - 1)) * n + i];
      Gp[t] = a.terminal_span ? 0.0 : a.G[(size_t)b * n + i];
    }
  }
  int par = 0;
  for (int p = a.p_end - (a.terminal_span ? 1 : 2); p >= 0; --p) {
    const bool own = p >= a.p_begin;
    const double* ub = a.ubar + ((size_t)p * a.B + b) * n;
#pragma unroll
    for (int t = 0; t < PPT; ++t) {
      const int i = threadIdx.x + t * BURGERS_NT;
      const double up = (i < n) ? ub[ipx(t)] : 0.0, um = (i < n) ? ub[imx(t)] : 0.0;
      const double kp = up * inv2h + Dih2, km = Dih2 - um * inv2h, kc = -(up - um) * inv2h - 2.0 * Dih2;
      gp[t] = two_over * kp;
      gm[t] = two_over * km;
      gc[t] = two_over * (kc - c0);
    }
    for (int sub = 0; sub < substeps; ++sub) {
#pragma unroll
      for (int t = 0; t < PPT; ++t) {
        const int i = threadIdx.x + t * BURGERS_NT;
        if (i < n) s_cur[par * n + i] = C[t];
      }
      __syncthreads();
      {
        const double b0 = __ldg(be), b1 = __ldg(be + 1), p0 = __ldg(bp), p1 = __ldg(bp + 1);
        const double* sc = s_cur + par * n;
#pragma unroll
        for (int t = 0; t < PPT; ++t) {
          if (threadIdx.x + t * BURGERS_NT >= n) continue;  // inactive point (n % BURGERS_NT ≠ 0)
          const double u0 = C[t];
          double u1 = gc[t] * u0;
          u1 = fma(gp[t], sc[ipx(t)], u1);
          u1 = 0.5 * fma(gm[t], sc[imx(t)], u1);
          prev[t] = u0;
          cur[t] = u1;
          acc[t] = b0 * u0 + b1 * u1;
          pac[t] = p0 * u0 + p1 * u1;
        }
      }
      par ^= 1;
      for (int k = 2; k <= degree; ++k) {
#pragma unroll
        for (int t = 0; t < PPT; ++t) {
          const int i = threadIdx.x + t * BURGERS_NT;
          if (i < n) s_cur[par * n + i] = cur[t];
        }
        __syncthreads();
        const double bk = __ldg(be + k), pk = __ldg(bp + k);
        const double* sc = s_cur + par * n;
#pragma unroll
        for (int t = 0; t < PPT; ++t) {
          if (threadIdx.x + t * BURGERS_NT >= n) continue;
          double un = fma(gc[t], cur[t], sigma * prev[t]);
          un = fma(gp[t], sc[ipx(t)], un);
          un = fma(gm[t], sc[imx(t)], un);
          prev[t] = cur[t];
          cur[t] = un;
          acc[t] = fma(bk, un, acc[t]);
          pac[t] = fma(pk, un, pac[t]);
        }
        par ^= 1;
      }
#pragma unroll
      for (int t = 0; t < PPT; ++t) {
        C[t] = acc[t];
        Gp[t] += pac[t];
      }
    }
    if (own) {
#pragma unroll
      for (int t = 0; t < PPT; ++t) {
        const int i = threadIdx.x + t * BURGERS_NT;
        if (i < n && !a.terminal_span) C[t] += a.W0[((size_t)b * Pl + (p - a.p_begin)) * n + i];
      }
    }
  }
#pragma unroll
  for (int t = 0; t < PPT; ++t) {
    const int i = threadIdx.x + t * BURGERS_NT;
    if (i < n) {
      a.QDAG0[(size_t)b * n + i] = C[t];
      a.G[(size_t)b * n + i] = Gp[t];
    }
  }
}

// The frozen-operator carry with contiguous runs of PPT points per thread (n = PPT·T):
// run-interior neighbours from registers, only the two run edges through shared memory.
template <int PPT>
__global__ void __launch_bounds__(BURGERS_NT) k_burgers_scan_run(BurgersAdjointArgs a, const double* coef) {
  extern __shared__ double sm[];
  const int n = a.nx;
  const int T = n / PPT;
  double* sE = sm;  // [2][2][T]: (first, last) run values, double buffered
  const int b = blockIdx.x;
  const int t = threadIdx.x;
  const bool act = t < T;
  const int i0 = t * PPT;
  const int tl = (t == 0) ? T - 1 : t - 1, tr = (t + 1 >= T) ? 0 : t + 1;
  const int Pl = a.p_end - a.p_begin;
  const double inv2h = 1.0 / (2.0 * a.hx);
  const double Dih2 = a.D / (a.hx * a.hx);
  const double c0 = a.center, two_over = 2.0 / a.scale, sigma = (double)a.sigma;
  const double* __restrict__ be = coef;
  const double* __restrict__ bp = coef + a.degree + 1;
  const int degree = a.degree, substeps = a.substeps;
  double C[PPT], Gp[PPT], prev[PPT], cur[PPT], acc[PPT], pac[PPT], gp[PPT], gm[PPT], gc[PPT];
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    C[k] = !act ? 0.0 : a.terminal_span ? a.QT[(size_t)b * n + i0 + k] : a.W0[((size_t)b * Pl + (Pl - 1)) * n + i0 + k];
    Gp[k] = (act && !a.terminal_span) ? a.G[(size_t)b * n + i0 + k] : 0.0;
  }
  int par = 0;
  // (left, right) neighbours of the run of v
  auto edges = [&](const double* v, double& l, double& r) {
    if (act) {
      sE[(par * 2 + 0) * T + t] = v[0];
      sE[(par * 2 + 1) * T + t] = v[PPT - 1];
    }
    __syncthreads();
    l = act ? sE[(par * 2 + 1) * T + tl] : 0.0;
    r = act ? sE[(par * 2 + 0) * T + tr] : 0.0;
    par ^= 1;
  };
  for (int p = a.p_end - (a.terminal_span ? 1 : 2); p >= 0; --p) {
    const bool own = p >= a.p_begin;
    const double* ub = a.ubar + ((size_t)p * a.B + b) * n;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      const int i = i0 + k;
      const int ip = (i + 1 >= n) ? 0 : i + 1, im = (i == 0) ? n - 1 : i - 1;
      const double up = act ? ub[ip] : 0.0, um = act ? ub[im] : 0.0;
      const double kp = up * inv2h + Dih2, km = Dih2 - um * inv2h, kc = -(up - um) * inv2h - 2.0 * Dih2;
      gp[k] = two_over * kp;
      gm[k] = two_over * km;
      gc[k] = two_over * (kc - c0);
    }
    for (int sub = 0; sub < substeps; ++sub) {
      double l, r;
      edges(C, l, r);
      {
        const double b0 = __ldg(be), b1 = __ldg(be + 1), p0 = __ldg(bp), p1 = __ldg(bp + 1);
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
          const double yp = (k + 1 == PPT) ? r : C[k + 1];
          const double ym = (k == 0) ? l : C[k - 1];
          double u1 = gc[k] * C[k];
          u1 = fma(gp[k], yp, u1);
          u1 = 0.5 * fma(gm[k], ym, u1);
          prev[k] = C[k];
          cur[k] = u1;
          acc[k] = b0 * C[k] + b1 * u1;
          pac[k] = p0 * C[k] + p1 * u1;
        }
      }
      for (int j = 2; j <= degree; ++j) {
        edges(cur, l, r);
        const double bk = __ldg(be + j), pk = __ldg(bp + j);
        double un[PPT];
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
          const double yp = (k + 1 == PPT) ? r : cur[k + 1];
          const double ym = (k == 0) ? l : cur[k - 1];
          double v = fma(gc[k], cur[k], sigma * prev[k]);
          v = fma(gp[k], yp, v);
          un[k] = fma(gm[k], ym, v);
        }
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
          prev[k] = cur[k];
          cur[k] = un[k];
          acc[k] = fma(bk, un[k], acc[k]);
          pac[k] = fma(pk, un[k], pac[k]);
        }
      }
#pragma unroll
      for (int k = 0; k < PPT; ++k) {
        C[k] = acc[k];
        Gp[k] += pac[k];
      }
    }
    if (own && act && !a.terminal_span) {
#pragma unroll
      for (int k = 0; k < PPT; ++k) C[k] += a.W0[((size_t)b * Pl + (p - a.p_begin)) * n + i0 + k];
    }
  }
  if (act) {
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      a.QDAG0[(size_t)b * n + i0 + k] = C[k];
      a.G[(size_t)b * n + i0 + k] = Gp[k];
    }
  }
}

// The frozen-operator carry spread over the CS CTAs of a thread-block cluster (CS SMs
// instead of one): CTA r owns W = n/CS points plus a ghost zone of G points per side that it
// recomputes redundantly (with the ghost points' own J(ū_p)ᵀ coefficients), so the Chebyshev
// terms need CTA barriers only; the ghost zones are refreshed from the neighbouring CTAs'
// shared memory (DSMEM) after one cluster barrier every G terms and at every action start
// (the k_scan1d_cluster scheme with per-point, per-slice coefficients). Same arithmetic per
// point as k_burgers_scan_run.
template <int PPT, int CS, int G>
__global__ void __launch_bounds__(256) k_burgers_scan_cluster(BurgersAdjointArgs a, const double* coef) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  static_assert(G % PPT == 0, "ghost width must be whole runs");
  constexpr int GR = G / PPT;
  __shared__ double eL[2][256], eR[2][256];
  __shared__ double xbuf[2][2][2][G];  // [parity][side: 0 my left edge, 1 right][cur/prev][G]
  const int n = a.nx;
  const int W = n / CS;
  const int rank = (int)cluster.block_rank();
  const int b = blockIdx.x / CS;  // member
  const int t = threadIdx.x;
  const int NR = W / PPT + 2 * GR;
  const bool act = t < NR;
  const int g0 = rank * W - G + t * PPT;
  const bool owned = act && t >= GR && t < NR - GR;
  const int tl = (t == 0) ? 0 : t - 1, tr = (t + 1 >= NR) ? NR - 1 : t + 1;
  auto gidx = [&](int k) { int g = g0 + k; g %= n; return g < 0 ? g + n : g; };
  const int Pl = a.p_end - a.p_begin;
  const double inv2h = 1.0 / (2.0 * a.hx);
  const double Dih2 = a.D / (a.hx * a.hx);
  const double c0 = a.center, two_over = 2.0 / a.scale, sigma = (double)a.sigma;
  const double* __restrict__ be = coef;
  const double* __restrict__ bp = coef + a.degree + 1;
  const int degree = a.degree, substeps = a.substeps;
  double C[PPT], Gp[PPT], gp[PPT], gm[PPT], gc[PPT];
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    const int i = gidx(k);
    C[k] = !act ? 0.0 : a.terminal_span ? a.QT[(size_t)b * n + i] : a.W0[((size_t)b * Pl + (Pl - 1)) * n + i];
    Gp[k] = (owned && !a.terminal_span) ? a.G[(size_t)b * n + i] : 0.0;
  }
  int par = 0, xpar = 0;
  auto exchange = [&](const double* u, double& l, double& r) {
    if (act) {
      eL[par][t] = u[0];
      eR[par][t] = u[PPT - 1];
    }
    __syncthreads();
    l = eR[par][tl];
    r = eL[par][tr];
    par ^= 1;
  };
  auto refresh = [&](double* u, double* v) {
    if (act) {
      if (t >= GR && t < 2 * GR) {
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
          xbuf[xpar][0][0][(t - GR) * PPT + k] = u[k];
          if (v) xbuf[xpar][0][1][(t - GR) * PPT + k] = v[k];
        }
      }
      if (t >= NR - 2 * GR && t < NR - GR) {
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
          xbuf[xpar][1][0][(t - (NR - 2 * GR)) * PPT + k] = u[k];
          if (v) xbuf[xpar][1][1][(t - (NR - 2 * GR)) * PPT + k] = v[k];
        }
      }
    }
    cluster.sync();
    if (act && t < GR) {
      const double* src = cluster.map_shared_rank(&xbuf[xpar][1][0][0], (unsigned)((rank + CS - 1) % CS));
#pragma unroll
      for (int k = 0; k < PPT; ++k) {
        u[k] = src[t * PPT + k];
        if (v) v[k] = src[G + t * PPT + k];
      }
    }
    if (act && t >= NR - GR) {
      const double* src = cluster.map_shared_rank(&xbuf[xpar][0][0][0], (unsigned)((rank + 1) % CS));
#pragma unroll
      for (int k = 0; k < PPT; ++k) {
        u[k] = src[(t - (NR - GR)) * PPT + k];
        if (v) v[k] = src[G + (t - (NR - GR)) * PPT + k];
      }
    }
    xpar ^= 1;
  };
  for (int p = a.p_end - (a.terminal_span ? 1 : 2); p >= 0; --p) {
    const bool own = p >= a.p_begin;
    const double* ub = a.ubar + ((size_t)p * a.B + b) * n;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      const int i = gidx(k);
      const int ip = (i + 1 >= n) ? 0 : i + 1, im = (i == 0) ? n - 1 : i - 1;
      const double up = act ? ub[ip] : 0.0, um = act ? ub[im] : 0.0;
      const double kp = up * inv2h + Dih2, km = Dih2 - um * inv2h, kc = -(up - um) * inv2h - 2.0 * Dih2;
      gp[k] = two_over * kp;
      gm[k] = two_over * km;
      gc[k] = two_over * (kc - c0);
    }
    for (int sub = 0; sub < substeps; ++sub) {
      double prev[PPT], cur[PPT], acc[PPT], pac[PPT];
      refresh(C, nullptr);
      int valid = G;
      double l, r;
      exchange(C, l, r);
      {
        const double b0 = __ldg(be), b1 = __ldg(be + 1), p0 = __ldg(bp), p1 = __ldg(bp + 1);
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
          const double yp = (k + 1 == PPT) ? r : C[k + 1];
          const double ym = (k == 0) ? l : C[k - 1];
          double u1 = gc[k] * C[k];
          u1 = fma(gp[k], yp, u1);
          u1 = 0.5 * fma(gm[k], ym, u1);
          prev[k] = C[k];
          cur[k] = u1;
          acc[k] = b0 * C[k] + b1 * u1;
          pac[k] = p0 * C[k] + p1 * u1;
        }
      }
      --valid;
      for (int j = 2; j <= degree; ++j) {
        if (valid == 0) {
          refresh(cur, prev);
          valid = G;
        }
        exchange(cur, l, r);
        const double bk = __ldg(be + j), pk = __ldg(bp + j);
        double un[PPT];
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
          const double yp = (k + 1 == PPT) ? r : cur[k + 1];
          const double ym = (k == 0) ? l : cur[k - 1];
          double v = fma(gc[k], cur[k], sigma * prev[k]);
          v = fma(gp[k], yp, v);
          un[k] = fma(gm[k], ym, v);
        }
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
          prev[k] = cur[k];
          cur[k] = un[k];
          acc[k] = fma(bk, un[k], acc[k]);
          pac[k] = fma(pk, un[k], pac[k]);
        }
        --valid;
      }
#pragma unroll
      for (int k = 0; k < PPT; ++k) {
        C[k] = acc[k];
        Gp[k] += pac[k];
      }
    }
    if (own && act && !a.terminal_span) {
#pragma unroll
      for (int k = 0; k < PPT; ++k) C[k] += a.W0[((size_t)b * Pl + (p - a.p_begin)) * n + gidx(k)];
    }
  }
  if (owned) {
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      a.QDAG0[(size_t)b * n + gidx(k)] = C[k];
      a.G[(size_t)b * n + gidx(k)] = Gp[k];
    }
  }
  cluster.sync();  // no CTA leaves while a neighbour may still read its exchange buffers
}

// The serial direct sweep spread over the CS CTAs of a thread-block cluster: CTA r owns
// W = n/CS points plus G ghost points per side, recomputed redundantly (each RK4 stage
// consumes one ghost layer per side), so the 4·G/4 stages between refreshes need CTA
// barriers only; every G/4 steps the ghost zones of u are refreshed from the neighbouring
// CTAs' shared memory (DSMEM) after one cluster barrier. Nodes and u(T) are written for the
// owned points. Same arithmetic per point as k_burgers_direct_run.
template <int PPT, int CS, int G>
__global__ void __launch_bounds__(256) k_burgers_direct_cluster(BurgersDirectArgs a) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  static_assert(G % (4 * PPT) == 0, "ghost width: whole runs, whole steps");
  constexpr int GR = G / PPT;
  constexpr int STEPS_PER_REFRESH = G / 4;
  __shared__ double eL[2][256], eR[2][256];
  __shared__ double xbuf[2][2][G];  // [parity][side: 0 my left edge, 1 my right edge][G]
  const int n = a.nx;
  const int W = n / CS;
  const int rank = (int)cluster.block_rank();
  const int b = blockIdx.x / CS;
  const int t = threadIdx.x;
  const int NR = W / PPT + 2 * GR;
  const bool act = t < NR;
  const int g0 = rank * W - G + t * PPT;
  const bool owned = act && t >= GR && t < NR - GR;
  const int tl = (t == 0) ? 0 : t - 1, tr = (t + 1 >= NR) ? NR - 1 : t + 1;
  auto gidx = [&](int k) { int g = g0 + k; g %= n; return g < 0 ? g + n : g; };
  const double inv2h = 1.0 / (2.0 * a.hx);
  const double Dih2 = a.D / (a.hx * a.hx), twoD = 2.0 * Dih2;
  const double h = a.h, hh = 0.5 * a.h, h6 = a.h / 6.0;
  double f[PPT], u[PPT], acc[PPT], x[PPT], kk[PPT];
  const double* c = a.ctrl + (size_t)b * a.K;
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    f[k] = 0.0;
    u[k] = 0.0;
    if (act) {
      const int i = gidx(k);
      double fv = 0.0;
      for (int q = 0; q < a.K; ++q) fv += c[q] * a.tx[(size_t)a.ix[q] * n + i];
      f[k] = fv;
      u[k] = a.u0[i];
      if (owned) a.traj[(size_t)b * n + i] = u[k];
    }
  }
  const size_t S = (size_t)a.P * a.nsteps;
  const size_t node_stride = (size_t)a.B * n;
  int par = 0, xpar = 0;
  auto rhs = [&](double* k_out) {
    if (act) {
      eL[par][t] = x[0];
      eR[par][t] = x[PPT - 1];
    }
    __syncthreads();
    const double xl = eR[par][tl], xr = eL[par][tr];
    par ^= 1;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      const double um = (k == 0) ? xl : x[k - 1];
      const double up = (k + 1 == PPT) ? xr : x[k + 1];
      const double A = up + um, B = up - um;
      const double t1 = fma(Dih2, A, f[k]);
      const double t2 = fma(inv2h, B, twoD);
      k_out[k] = fma(-x[k], t2, t1);
    }
  };
  auto refresh = [&]() {
    if (act) {
      if (t >= GR && t < 2 * GR) {
#pragma unroll
        for (int k = 0; k < PPT; ++k) xbuf[xpar][0][(t - GR) * PPT + k] = u[k];
      }
      if (t >= NR - 2 * GR && t < NR - GR) {
#pragma unroll
        for (int k = 0; k < PPT; ++k) xbuf[xpar][1][(t - (NR - 2 * GR)) * PPT + k] = u[k];
      }
    }
    cluster.sync();
    if (act && t < GR) {
      const double* src = cluster.map_shared_rank(&xbuf[xpar][1][0], (unsigned)((rank + CS - 1) % CS));
#pragma unroll
      for (int k = 0; k < PPT; ++k) u[k] = src[t * PPT + k];
    }
    if (act && t >= NR - GR) {
      const double* src = cluster.map_shared_rank(&xbuf[xpar][0][0], (unsigned)((rank + 1) % CS));
#pragma unroll
      for (int k = 0; k < PPT; ++k) u[k] = src[(t - (NR - GR)) * PPT + k];
    }
    xpar ^= 1;
  };
  int valid = STEPS_PER_REFRESH;  // the ghost zones start exact (u0 read at global indices)
  for (size_t st = 0; st < S; ++st) {
    if (valid == 0) {
      refresh();
      valid = STEPS_PER_REFRESH;
    }
#pragma unroll
    for (int k = 0; k < PPT; ++k) x[k] = u[k];
    rhs(kk);
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      acc[k] = kk[k];
      x[k] = fma(hh, kk[k], u[k]);
    }
    rhs(kk);
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      acc[k] = fma(2.0, kk[k], acc[k]);
      x[k] = fma(hh, kk[k], u[k]);
    }
    rhs(kk);
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      acc[k] = fma(2.0, kk[k], acc[k]);
      x[k] = fma(h, kk[k], u[k]);
    }
    rhs(kk);
#pragma unroll
    for (int k = 0; k < PPT; ++k) u[k] = fma(h6, acc[k] + kk[k], u[k]);
    --valid;
    if (owned) {
      double* node = a.traj + (st + 1) * node_stride + (size_t)b * n;
#pragma unroll
      for (int k = 0; k < PPT; ++k) node[gidx(k)] = u[k];
    }
  }
  if (owned) {
#pragma unroll
    for (int k = 0; k < PPT; ++k) a.UT[(size_t)b * n + gidx(k)] = u[k];
  }
  cluster.sync();  // no CTA leaves while a neighbour may still read its exchange buffers
}

inline int burgers_direct(const BurgersDirectArgs& a, cudaStream_t s, px_stats* stats, bool use_cluster) {
  if (a.nx > BURGERS_MAX_N) return PX_ERR_ARG;
  const size_t smem = 3 * (size_t)a.nx * sizeof(double);
  const int ppt = (a.nx + BURGERS_NT - 1) / BURGERS_NT;
#define PX_BD(PP)                                                                              \
  do {                                                                                         \
    cudaFuncSetAttribute(k_burgers_direct<PP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    k_burgers_direct<PP><<<a.B, BURGERS_NT, smem, s>>>(a);                                     \
  } while (0)
#define PX_BR(PP)                                                                              \
  do {                                                                                         \
    const size_t sm2 = 2 * (size_t)a.nx * sizeof(double);                                     \
    cudaFuncSetAttribute(k_burgers_direct_run<PP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2); \
    k_burgers_direct_run<PP><<<a.B, ((a.nx / PP + 31) / 32) * 32, sm2, s>>>(a);                \
  } while (0)
  // contiguous runs when n is a multiple of the run length (the strided kernel otherwise)
  const int rp = ppt <= 1 ? 1 : (ppt <= 2 ? 2 : (ppt <= 4 ? 4 : 8));
  // cluster sweep (8 CTAs per member, 64-point ghost zones refreshed every 16 steps) for the
  // larger grids
  constexpr int kCS = 8, kPPT = 4, kG = 64;
  if (use_cluster && a.nx >= 2048 && a.nx % (kCS * kPPT) == 0 && a.nx / kCS >= kG &&
      a.nx / kCS / kPPT + 2 * (kG / kPPT) <= 256) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(a.B * kCS));
    cfg.blockDim = dim3((unsigned)(((a.nx / kCS / kPPT + 2 * (kG / kPPT) + 31) / 32) * 32));
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kCS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, k_burgers_direct_cluster<kPPT, kCS, kG>, a) != cudaSuccess) return PX_ERR_CUDA;
  } else if (a.nx % rp == 0) {
    if (rp == 1) PX_BR(1);
    else if (rp == 2) PX_BR(2);
    else if (rp == 4) PX_BR(4);
    else PX_BR(8);
  } else if (ppt <= 1) PX_BD(1);
  else if (ppt <= 2) PX_BD(2);
  else if (ppt <= 4) PX_BD(4);
  else PX_BD(8);
#undef PX_BD
#undef PX_BR
  const size_t total = (size_t)a.P * a.B * a.nx;
  k_slice_means<<<(unsigned)std::min<size_t>((total + 255) / 256, 4096), 256, 0, s>>>(a.ubar, a.traj, a.P,
                                                                                       a.nsteps, a.B, a.nx);
  k_frozen_bounds<<<a.bounds_blocks, 256, 0, s>>>(a.bpart, a.ubar, total, a.nx, a.hx, a.D);
  k_frozen_bounds_final<<<1, 256, 0, s>>>(a.bounds, a.bpart, a.bounds_blocks);
  if (cudaGetLastError() != cudaSuccess) return PX_ERR_CUDA;
  if (stats) {
    stats->kernel_launches += 4;
    const double S = (double)a.P * a.nsteps;
    stats->rk4_lane_steps += (uint64_t)(S * a.B);
    const double bytes = 24.0 * a.nx * S * a.B;  // read u_n, (f), write node u_{n+1}
    stats->rk4_bytes += bytes;
    stats->algorithmic_bytes += bytes;
  }
  return PX_OK;
}

inline int burgers_adjoint(const BurgersAdjointArgs& a, cudaStream_t s, px_stats* stats, const double** wend,
                           bool use_cluster) {
  if (a.nx > BURGERS_MAX_N) return PX_ERR_ARG;
  const int Pl = a.p_end - a.p_begin;
  const int ppt = (a.nx + BURGERS_NT - 1) / BURGERS_NT;
  const size_t smem_rk = 4 * (size_t)a.nx * sizeof(double);
#define PX_BA(PP)                                                                                  \
  do {                                                                                             \
    cudaFuncSetAttribute(k_burgers_adjoint_rk4<PP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_rk); \
    k_burgers_adjoint_rk4<PP><<<a.B * Pl, BURGERS_NT, smem_rk, s>>>(a);                            \
  } while (0)
  if (!a.terminal_span) {  // terminal span: the inhomogeneous solves are identically zero
    if (ppt <= 1) PX_BA(1);
    else if (ppt <= 2) PX_BA(2);
    else if (ppt <= 4) PX_BA(4);
    else PX_BA(8);
    k_lane_sum<<<dim3((unsigned)std::min<size_t>(((size_t)a.nx + 255) / 256, 64), a.B), 256, 0, s>>>(
        a.G, a.Z, Pl, (size_t)a.nx);
  }
#undef PX_BA
  // coefficients to device (scratch ACC[0] is free here: n ≥ 2·(degree+1) not guaranteed, use Wk[2])
  double* coef = a.Wk[2];
  const size_t ncoef = 2 * (size_t)(a.degree + 1);
  if ((size_t)a.B * a.nx < ncoef) return PX_ERR_ARG;
  if (a.be && a.bp) {  // no plan: one slice, no carry (the scan only finalises q†(0) and G)
    cudaMemcpyAsync(coef, a.be, sizeof(double) * (a.degree + 1), cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(coef + a.degree + 1, a.bp, sizeof(double) * (a.degree + 1), cudaMemcpyHostToDevice, s);
  }
  const size_t smem_sc = 2 * (size_t)a.nx * sizeof(double);
#define PX_BS(PP)                                                                               \
  do {                                                                                          \
    cudaFuncSetAttribute(k_burgers_scan<PP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_sc); \
    k_burgers_scan<PP><<<a.B, BURGERS_NT, smem_sc, s>>>(a, coef);                               \
  } while (0)
#define PX_BSR(PP)                                                                                   \
  do {                                                                                             \
    const size_t sm2 = 4 * (size_t)(a.nx / PP) * sizeof(double);                                   \
    cudaFuncSetAttribute(k_burgers_scan_run<PP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2); \
    k_burgers_scan_run<PP><<<a.B, ((a.nx / PP + 31) / 32) * 32, sm2, s>>>(a, coef);                \
  } while (0)
  // cluster scan (8 CTAs per member, 64-point DSMEM ghost zones) for the larger grids
  constexpr int kCS = 8, kPPT = 4, kG = 64;
  const int rps = ppt <= 1 ? 1 : (ppt <= 2 ? 2 : (ppt <= 4 ? 4 : 8));
  if (use_cluster && a.nx >= 2048 && a.nx % (kCS * kPPT) == 0 && a.nx / kCS >= kG &&
      a.nx / kCS / kPPT + 2 * (kG / kPPT) <= 256 && a.degree >= 1) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(a.B * kCS));
    cfg.blockDim = dim3((unsigned)(((a.nx / kCS / kPPT + 2 * (kG / kPPT) + 31) / 32) * 32));
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kCS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, k_burgers_scan_cluster<kPPT, kCS, kG>, a, (const double*)coef) != cudaSuccess)
      return PX_ERR_CUDA;
  } else if (a.nx % rps == 0) {
    if (rps == 1) PX_BSR(1);
    else if (rps == 2) PX_BSR(2);
    else if (rps == 4) PX_BSR(4);
    else PX_BSR(8);
  } else if (ppt <= 1) PX_BS(1);
  else if (ppt <= 2) PX_BS(2);
  else if (ppt <= 4) PX_BS(4);
  else PX_BS(8);
#undef PX_BS
#undef PX_BSR
  if (cudaGetLastError() != cudaSuccess) return PX_ERR_CUDA;
  *wend = a.W0;
  if (stats) {
    stats->kernel_launches += a.terminal_span ? 1 : 3;
    if (!a.terminal_span) stats->rk4_lane_steps += (uint64_t)a.B * Pl * a.nsteps;
    const double rb = a.terminal_span ? 0.0 : 40.0 * a.nx * (double)a.B * Pl * a.nsteps;  // y, q†_T, node, y', z
    stats->rk4_bytes += rb;
    const uint64_t acts = (uint64_t)(a.p_end - (a.terminal_span ? 0 : 1));
    const uint64_t terms = acts * a.substeps * a.degree * a.B;
    stats->exp_terms += terms;
    const double eb = 56.0 * a.nx * (double)terms;
    stats->exp_bytes += eb;
    stats->algorithmic_bytes += rb + eb;
  }
  return PX_OK;
}

}  // namespace px
