// hybrid.cuh — the reference's hybrid algorithm (hybrid.py:1-290) with its tracking objective
// (optimization.py:84-112, 172-189) on the GPU: 1D Burgers (V ≡ 0), forcing field × time law
// θ(t) = α + β sin ωt + γ cos ωt, variable (geometric) slices on the serial sweep's node grid.
//
//   k_hyb_direct  one CTA per member: the serial RK4 sweep, every node to HBM, the tracking
//                 cost (1/T)∫‖u − u_t‖² (trapezoid on the nodes) on the fly, and a progress
//                 flag per slice released the moment the slice's last node is stored;
//   k_hyb_lanes   one CTA per (member, slice): the slice's adjoint inhomogeneous solve from
//                 zero terminal data (hybrid.py:194-203) with exact Jᵀ(u(t)) and the source
//                 s = 2(u − u_t), plus its θ-weighted ∫ — started by the flag, so the slice
//                 solves run WHILE the serial sweep continues (the reference's overlap);
//   k_hyb_means   trapezoid slice means ū_p of variable slices (problems.py:346-366);
//   k_hyb_scan    one CTA per member: the slice ends propagated through the frozen J(ū_m)ᵀ of
//                 every earlier slice (propagate_span, hybrid.py:212-225, summed as one carry),
//                 per-slice Chebyshev plans, the θ-weighted φ-type series for ∫θ·q† dt.
// Every thread owns a contiguous run of PPT points; run edges are exchanged through double-
// buffered shared arrays (one CTA barrier per stage / term).
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "hybrid_args.h"

namespace px {

// θ at half-step k (t = k·h/2): the host tabulates the law once per handle
__device__ __forceinline__ double hyb_theta(const HybArgs& a, int k) { return __ldg(a.theta + k); }

// Exchange the run edges of y (PPT values per thread) and return the left / right neighbours
// of the run; `par` selects the buffer (double buffering: one barrier per call).
template <int PPT>
__device__ __forceinline__ void hyb_edges(const double* y, double (*eL)[HYB_NT], double (*eR)[HYB_NT], int& par,
                                          bool act, int t, int tl, int tr, double& l, double& r) {
  if (act) {
    eL[par][t] = y[0];
    eR[par][t] = y[PPT - 1];
  }
  __syncthreads();
  l = eR[par][tl];
  r = eL[par][tr];
  par ^= 1;
}

template <int PPT>
__global__ void __launch_bounds__(HYB_NT) k_hyb_direct(HybArgs a) {
  __shared__ double eL[2][HYB_NT], eR[2][HYB_NT];
  __shared__ double red[8];
  const int n = a.nx, b = blockIdx.x, t = threadIdx.x;
  const int NR = n / PPT;
  const bool act = t < NR;
  const int tl = (t == 0) ? NR - 1 : t - 1, tr = (t + 1 >= NR) ? 0 : t + 1;
  const int i0 = t * PPT;
  const double inv2h = 1.0 / (2.0 * a.hx), Dih2 = a.D / (a.hx * a.hx);
  const size_t ns = (size_t)a.B * n;
  const size_t tstride = (size_t)a.target_b * n;
  const double* tg = a.target + (a.target_b > 1 ? (size_t)b * n : 0);
  double u[PPT], f[PPT];
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    u[k] = act ? a.u0[(size_t)b * n + i0 + k] : 0.0;
    f[k] = act ? a.f[(size_t)b * n + i0 + k] : 0.0;
  }
  double jacc = 0.0;
  // the target row of the node a step is about to produce is loaded one step ahead, so its
  // latency overlaps the step's four stages instead of stalling the sweep at every node
  double tnext[PPT];
  auto load_target = [&](int s) {
#pragma unroll
    for (int k = 0; k < PPT; ++k) tnext[k] = (act && s <= a.S) ? __ldg(tg + (size_t)s * tstride + i0 + k) : 0.0;
  };
  auto node = [&](int s, double w) {
    if (!act) return;
    double e = 0.0;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      a.traj[(size_t)s * ns + (size_t)b * n + i0 + k] = u[k];
      const double d = u[k] - tnext[k];
      e = fma(d, d, e);
    }
    jacc = fma(w, e, jacc);
  };
  load_target(0);
  node(0, 0.5);
  load_target(1);
  int par = 0;
  // k = −y∘Dx y + D·L y + θ·f (problems.py:177-185, V ≡ 0)
  auto rhs = [&](const double* y, double th, double* k) {
    double l, r;
    hyb_edges<PPT>(y, eL, eR, par, act, t, tl, tr, l, r);
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      const double ym = (q == 0) ? l : y[q - 1];
      const double yp = (q + 1 == PPT) ? r : y[q + 1];
      k[q] = fma(th, f[q], fma(-y[q], (yp - ym) * inv2h, (yp - 2.0 * y[q] + ym) * Dih2));
    }
  };
  int p = 0;
  int next = a.offsets[1];
  for (int s = 0; s < a.S; ++s) {
    const double th1 = hyb_theta(a, 2 * s), th2 = hyb_theta(a, 2 * s + 1), th4 = hyb_theta(a, 2 * s + 2);
    double k[PPT], Y[PPT], acc[PPT];
    rhs(u, th1, k);
#pragma unroll
    for (int q = 0; q < PPT; ++q) { acc[q] = k[q]; Y[q] = fma(0.5 * a.h, k[q], u[q]); }
    rhs(Y, th2, k);
#pragma unroll
    for (int q = 0; q < PPT; ++q) { acc[q] = fma(2.0, k[q], acc[q]); Y[q] = fma(0.5 * a.h, k[q], u[q]); }
    rhs(Y, th2, k);
#pragma unroll
    for (int q = 0; q < PPT; ++q) { acc[q] = fma(2.0, k[q], acc[q]); Y[q] = fma(a.h, k[q], u[q]); }
    rhs(Y, th4, k);
#pragma unroll
    for (int q = 0; q < PPT; ++q) u[q] = fma(a.h / 6.0, acc[q] + k[q], u[q]);
    node(s + 1, s + 1 == a.S ? 0.5 : 1.0);
    load_target(s + 2);
    if (s + 1 == next) {
      // slice p's nodes are stored: publish (every writer fences, then one release flag)
      __threadfence();
      __syncthreads();
      if (t == 0) atomicExch(a.flags + (size_t)b * a.P + p, 1);
      ++p;
      next = (p < a.P) ? a.offsets[p + 1] : -1;
    }
  }
  const double tot = block_sum<HYB_NT>(jacc, red);
  if (t == 0) a.J[b] = (a.h / a.T) * tot;
}

// The serial sweep of k_hyb_direct spread over the CS CTAs of a thread-block cluster (the
// k_burgers_direct_cluster scheme): CTA r owns W = n/CS points plus G ghost points per side,
// recomputed redundantly (one ghost layer per RK4 stage), the ghost zones of u refreshed from
// the neighbouring CTAs' shared memory (DSMEM) after one cluster barrier every G/4 steps. A slice
// is published when every CTA of the cluster has stored its part of the slice's last node (each
// writer fences, one cluster barrier, one flag store); the tracking cost is reduced over the
// cluster through DSMEM in a fixed order.
template <int PPT, int CS, int G>
__global__ void __launch_bounds__(256) k_hyb_direct_cluster(HybArgs a) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  static_assert(G % (4 * PPT) == 0, "ghost width: whole runs, whole steps");
  constexpr int GR = G / PPT;
  constexpr int STEPS_PER_REFRESH = G / 4;
  __shared__ double eL[2][256], eR[2][256];
  __shared__ double xbuf[2][2][G];
  __shared__ double red[8];
  __shared__ double jpart;
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
  const double Dih2 = a.D / (a.hx * a.hx);
  const double h = a.h, hh = 0.5 * a.h, h6 = a.h / 6.0;
  const size_t ns = (size_t)a.B * n;
  const size_t tstride = (size_t)a.target_b * n;
  const double* tg = a.target + (a.target_b > 1 ? (size_t)b * n : 0);
  double f[PPT], u[PPT], acc[PPT], x[PPT], kk[PPT];
  double jacc = 0.0;
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    f[k] = act ? a.f[(size_t)b * n + gidx(k)] : 0.0;
    u[k] = act ? a.u0[(size_t)b * n + gidx(k)] : 0.0;
  }
  double tnext[PPT];  // the next node's target row, loaded a step ahead (see k_hyb_direct)
  auto load_target = [&](int s) {
#pragma unroll
    for (int k = 0; k < PPT; ++k) tnext[k] = (owned && s <= a.S) ? __ldg(tg + (size_t)s * tstride + gidx(k)) : 0.0;
  };
  auto node = [&](int s, double w) {
    if (!owned) return;
    double e = 0.0;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      const int i = gidx(k);
      a.traj[(size_t)s * ns + (size_t)b * n + i] = u[k];
      const double d = u[k] - tnext[k];
      e = fma(d, d, e);
    }
    jacc = fma(w, e, jacc);
  };
  load_target(0);
  node(0, 0.5);
  load_target(1);
  int par = 0, xpar = 0;
  auto rhs = [&](double th, double* k_out) {
    if (act) {
      eL[par][t] = x[0];
      eR[par][t] = x[PPT - 1];
    }
    __syncthreads();
    const double xl = eR[par][tl], xr = eL[par][tr];
    par ^= 1;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      const double ym = (k == 0) ? xl : x[k - 1];
      const double yp = (k + 1 == PPT) ? xr : x[k + 1];
      k_out[k] = fma(th, f[k], fma(-x[k], (yp - ym) * inv2h, (yp - 2.0 * x[k] + ym) * Dih2));
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
  int valid = STEPS_PER_REFRESH;
  int p = 0, next = a.offsets[1];
  double n1 = hyb_theta(a, 0), n2 = hyb_theta(a, 1), n4 = hyb_theta(a, 2);  // θ of the next step
  for (int st = 0; st < a.S; ++st) {
    if (valid == 0) {
      refresh();
      valid = STEPS_PER_REFRESH;
    }
    const double th1 = n1, th2 = n2, th4 = n4;
    if (st + 1 < a.S) {
      n1 = hyb_theta(a, 2 * st + 2);
      n2 = hyb_theta(a, 2 * st + 3);
      n4 = hyb_theta(a, 2 * st + 4);
    }
#pragma unroll
    for (int k = 0; k < PPT; ++k) x[k] = u[k];
    rhs(th1, kk);
#pragma unroll
    for (int k = 0; k < PPT; ++k) { acc[k] = kk[k]; x[k] = fma(hh, kk[k], u[k]); }
    rhs(th2, kk);
#pragma unroll
    for (int k = 0; k < PPT; ++k) { acc[k] = fma(2.0, kk[k], acc[k]); x[k] = fma(hh, kk[k], u[k]); }
    rhs(th2, kk);
#pragma unroll
    for (int k = 0; k < PPT; ++k) { acc[k] = fma(2.0, kk[k], acc[k]); x[k] = fma(h, kk[k], u[k]); }
    rhs(th4, kk);
#pragma unroll
    for (int k = 0; k < PPT; ++k) u[k] = fma(h6, acc[k] + kk[k], u[k]);
    --valid;
    node(st + 1, st + 1 == a.S ? 0.5 : 1.0);
    load_target(st + 2);
    if (st + 1 == next) {
      __threadfence();
      cluster.sync();
      if (rank == 0 && t == 0) atomicExch(a.flags + (size_t)b * a.P + p, 1);
      ++p;
      next = (p < a.P) ? a.offsets[p + 1] : -1;
    }
  }
  if (t < 8) red[t] = 0.0;  // the CTA may have fewer than 8 warps
  __syncthreads();
  const double tot = block_sum<256>(jacc, red);
  if (t == 0) jpart = tot;
  cluster.sync();
  if (rank == 0 && t == 0) {
    double s = 0.0;
    for (int r = 0; r < CS; ++r) s += *cluster.map_shared_rank(&jpart, (unsigned)r);
    a.J[b] = (a.h / a.T) * s;
  }
  cluster.sync();  // no CTA leaves while a neighbour may still read its exchange buffers
}

// The adjoint slice solve of lane (b, p) in reflected time, nodes o_{p+1} → o_p:
//   a' = Jᵀ(u(t))·a + 2(u(t) − u_t(t)), a = 0 at t = T_{p+1};  z' = θ(t)·a  (RK4 on (a, z))
// u and u_t at the half steps are the node means (linear interpolation, timestepping.py:64-75).
template <int PPT>
__global__ void __launch_bounds__(HYB_NT) k_hyb_lanes(HybArgs a) {
  extern __shared__ double hyb_sm[];  // two node rows: [2][n]
  __shared__ double eL[2][HYB_NT], eR[2][HYB_NT];
  const int n = a.nx, t = threadIdx.x;
  const int lane = blockIdx.x;
  const int b = lane / a.P, p = lane - b * a.P;
  const int NR = n / PPT;
  const bool act = t < NR;
  const int tl = (t == 0) ? NR - 1 : t - 1, tr = (t + 1 >= NR) ? 0 : t + 1;
  const int i0 = t * PPT;
  const double inv2h = 1.0 / (2.0 * a.hx), Dih2 = a.D / (a.hx * a.hx);
  const size_t ns = (size_t)a.B * n;
  const size_t tstride = (size_t)a.target_b * n;
  const double* tg = a.target + (a.target_b > 1 ? (size_t)b * n : 0);
  const int o0 = a.offsets[p], o1 = a.offsets[p + 1];
  if (a.wait) {
    if (t == 0) {
      volatile int* fl = a.flags + (size_t)b * a.P + p;
      while (*fl == 0) __nanosleep(200);
      __threadfence();
    }
    __syncthreads();
  }
  double* ua = hyb_sm;
  double* ub = hyb_sm + n;
  const double* nb = a.traj + (size_t)b * n;
  for (int j = t; j < n; j += HYB_NT) ua[j] = __ldcg(nb + (size_t)o1 * ns + j);
  double av[PPT], z[PPT], tga[PPT], tgb[PPT];
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    av[q] = 0.0;
    z[q] = 0.0;
    tga[q] = act ? tg[(size_t)o1 * tstride + i0 + q] : 0.0;
  }
  int par = 0;
  // out = Jᵀ(U)·y + src, U a node row (or the mean of the two rows when MEAN)
  auto jt = [&](auto meanc, const double* U, const double* y, const double* src, double* out) {
    constexpr bool MEAN = decltype(meanc)::value;
    double l, r;
    hyb_edges<PPT>(y, eL, eR, par, act, t, tl, tr, l, r);
    if (!act) return;
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      const int i = i0 + q;
      const int ip = (i + 1 == n) ? 0 : i + 1, im = (i == 0) ? n - 1 : i - 1;
      const double up = MEAN ? 0.5 * ua[ip] + 0.5 * ub[ip] : U[ip];
      const double um = MEAN ? 0.5 * ua[im] + 0.5 * ub[im] : U[im];
      const double ym = (q == 0) ? l : y[q - 1];
      const double yp = (q + 1 == PPT) ? r : y[q + 1];
      const double dxuy = (up * yp - um * ym) * inv2h;
      const double dxu = (up - um) * inv2h;
      out[q] = dxuy - dxu * y[q] + (yp - 2.0 * y[q] + ym) * Dih2 + src[q];
    }
  };
  const double h = a.h, hh = 0.5 * a.h, h6 = a.h / 6.0;
  // the next node row and its target values are fetched one step ahead (registers), so their
  // latency overlaps the current step's stages
  double rnext[PPT], tnext[PPT];
  auto prefetch = [&](int node) {
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      const int j = t + q * HYB_NT;
      rnext[q] = (j < n) ? __ldcg(nb + (size_t)node * ns + j) : 0.0;
      tnext[q] = act ? __ldg(tg + (size_t)node * tstride + i0 + q) : 0.0;
    }
  };
  prefetch(o1 - 1);
  for (int it = 0; it < o1 - o0; ++it) {
    const int top = o1 - it;
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      const int j = t + q * HYB_NT;
      if (j < n) ub[j] = rnext[q];
      tgb[q] = tnext[q];
    }
    if (top - 2 >= o0) prefetch(top - 2);
    __syncthreads();
    const double tha = hyb_theta(a, 2 * top), thm = hyb_theta(a, 2 * top - 1), thb = hyb_theta(a, 2 * top - 2);
    double sa[PPT], sm[PPT], sb[PPT];
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      const double va = act ? ua[i0 + q] : 0.0, vb = act ? ub[i0 + q] : 0.0;
      sa[q] = 2.0 * (va - tga[q]);
      sm[q] = 2.0 * ((0.5 * va + 0.5 * vb) - (0.5 * tga[q] + 0.5 * tgb[q]));
      sb[q] = 2.0 * (vb - tgb[q]);
    }
    double k[PPT], Y[PPT], acc[PPT], zacc[PPT];
    jt(BC<false>{}, ua, av, sa, k);
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      acc[q] = k[q];
      Y[q] = fma(hh, k[q], av[q]);
      zacc[q] = fma(2.0 * thm, Y[q], tha * av[q]);
    }
    jt(BC<true>{}, nullptr, Y, sm, k);
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      acc[q] = fma(2.0, k[q], acc[q]);
      Y[q] = fma(hh, k[q], av[q]);
      zacc[q] = fma(2.0 * thm, Y[q], zacc[q]);
    }
    jt(BC<true>{}, nullptr, Y, sm, k);
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      acc[q] = fma(2.0, k[q], acc[q]);
      Y[q] = fma(h, k[q], av[q]);
      zacc[q] = fma(thb, Y[q], zacc[q]);
    }
    jt(BC<false>{}, ub, Y, sb, k);
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      z[q] = fma(h6, zacc[q], z[q]);
      av[q] = fma(h6, acc[q] + k[q], av[q]);
      tga[q] = tgb[q];
    }
    double* tmp = ua;
    ua = ub;
    ub = tmp;
  }
  if (act) {
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      a.aend[(size_t)lane * n + i0 + q] = av[q];
      a.zl[(size_t)lane * n + i0 + q] = z[q];
    }
  }
}

// ū_p[b][i] = Σ_j w_j traj[o_p + j][b][i], trapezoid weights (½, 1, …, 1, ½)/(o_{p+1} − o_p)
__global__ void k_hyb_means(double* ubar, const double* traj, const int* offsets, int P, int B, int n) {
  const size_t total = (size_t)P * B * n;
  const size_t ns = (size_t)B * n;
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (size_t)gridDim.x * blockDim.x) {
    const int p = (int)(idx / ns);
    const size_t rem = idx - (size_t)p * ns;
    const int o0 = offsets[p], m = offsets[p + 1] - o0;
    const double* src = traj + (size_t)o0 * ns + rem;
    const double w = 1.0 / m;
    double s = (0.5 * w) * src[0];
    for (int j = 1; j < m; ++j) s += w * src[(size_t)j * ns];
    s += (0.5 * w) * src[(size_t)m * ns];
    ubar[idx] = s;
  }
}

// Frozen-operator carry of member b: C ← exp(Δ_p J(ū_p)ᵀ)·C + a_p for p = top … 0, with
// G += ∫θ(t)·e^{(T_{p+1}−t)J(ū_p)ᵀ}C dt from the law series of every substep.
template <int PPT>
__global__ void __launch_bounds__(HYB_NT) k_hyb_scan(HybScanArgs a) {
  __shared__ double eL[2][HYB_NT], eR[2][HYB_NT];
  const int n = a.nx, b = blockIdx.x, t = threadIdx.x;
  const int NR = n / PPT;
  const bool act = t < NR;
  const int tl = (t == 0) ? NR - 1 : t - 1, tr = (t + 1 >= NR) ? 0 : t + 1;
  const int i0 = t * PPT;
  const double inv2h = 1.0 / (2.0 * a.hx), Dih2 = a.D / (a.hx * a.hx);
  const int P = a.P;
  double C[PPT], Gh[PPT], Zs[PPT], gp[PPT], gm[PPT], gc[PPT];
  const bool has_qT = a.qT != nullptr;
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    const int i = i0 + q;
    C[q] = !act ? 0.0 : has_qT ? a.qT[(size_t)b * n + i] : a.aend[((size_t)b * P + P - 1) * n + i];
    Gh[q] = 0.0;
    Zs[q] = 0.0;
  }
  if (act) {
    for (int p = 0; p < P; ++p) {
#pragma unroll
      for (int q = 0; q < PPT; ++q) Zs[q] += a.zl[((size_t)b * P + p) * n + i0 + q];
    }
  }
  int par = 0;
  for (int p = has_qT ? P - 1 : P - 2; p >= 0; --p) {
    const HybSlicePlan pl = a.plans[p];
    const double two_over = 2.0 / pl.d, sigma = (double)pl.sigma;
    const double* ubp = a.ubar + ((size_t)p * a.B + b) * n;
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      const int i = i0 + q;
      const int ip = (i + 1 >= n) ? 0 : i + 1, im = (i == 0) ? n - 1 : i - 1;
      const double up = act ? ubp[ip] : 0.0, um = act ? ubp[im] : 0.0;
      // (J(ū)ᵀy)_i = kp·y_{i+1} + km·y_{i−1} + kc·y_i (problems.py:316-343, V ≡ 0)
      const double kp = up * inv2h + Dih2, km = Dih2 - um * inv2h, kc = -(up - um) * inv2h - 2.0 * Dih2;
      gp[q] = two_over * kp;
      gm[q] = two_over * km;
      gc[q] = two_over * (kc - pl.c0);
    }
    const double* be = a.coef + pl.exp_off;
    for (int sub = 0; sub < pl.substeps; ++sub) {
      const double* bl = a.coef + pl.law_off + (size_t)sub * (pl.degree + 1);
      double prev[PPT], cur[PPT], acc[PPT], lac[PPT], l, r;
      hyb_edges<PPT>(C, eL, eR, par, act, t, tl, tr, l, r);
      const double b0 = be[0], b1 = be[1], l0 = bl[0], l1 = bl[1];
#pragma unroll
      for (int q = 0; q < PPT; ++q) {
        const double yp = (q + 1 == PPT) ? r : C[q + 1];
        const double ym = (q == 0) ? l : C[q - 1];
        const double u1 = 0.5 * fma(gm[q], ym, fma(gp[q], yp, gc[q] * C[q]));
        prev[q] = C[q];
        cur[q] = u1;
        acc[q] = fma(b1, u1, b0 * C[q]);
        lac[q] = fma(l1, u1, l0 * C[q]);
      }
      for (int j = 2; j <= pl.degree; ++j) {
        hyb_edges<PPT>(cur, eL, eR, par, act, t, tl, tr, l, r);
        const double bk = be[j], lk = bl[j];
        double un[PPT];
#pragma unroll
        for (int q = 0; q < PPT; ++q) {
          const double yp = (q + 1 == PPT) ? r : cur[q + 1];
          const double ym = (q == 0) ? l : cur[q - 1];
          un[q] = fma(gm[q], ym, fma(gp[q], yp, fma(gc[q], cur[q], sigma * prev[q])));
        }
#pragma unroll
        for (int q = 0; q < PPT; ++q) {
          prev[q] = cur[q];
          cur[q] = un[q];
          acc[q] = fma(bk, un[q], acc[q]);
          lac[q] = fma(lk, un[q], lac[q]);
        }
      }
#pragma unroll
      for (int q = 0; q < PPT; ++q) {
        C[q] = acc[q];
        Gh[q] += lac[q];
      }
    }
    if (act) {
#pragma unroll
      for (int q = 0; q < PPT; ++q) C[q] += a.aend[((size_t)b * P + p) * n + i0 + q];
    }
  }
  if (act) {
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      a.qdag0[(size_t)b * n + i0 + q] = C[q];
      a.grad[(size_t)b * n + i0 + q] = (Zs[q] + Gh[q]) / a.T;
    }
  }
}

}  // namespace px
