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

#include <cooperative_groups.h>

#include "common.cuh"

namespace px {

struct Scan1DPlan {
  const double* be;  // degree+1 (device)
  const double* bp;  // degree+1 (device), may be null
  int degree, substeps, sigma;
  double c0, d;
  double f[3];  // (cc − c0, ce, cw)/d      : U_1 = f·(u, e, w)
  double g[3];  // (2/d)(cc − c0, ce, cw)   : U_{j+1} = g·(U_j, e, w) + σ U_{j−1}
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

template <int PPT, bool FULL>
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
  // publish the run's edge values of u and return the neighbours' (left, right)
  auto exchange = [&](double first, double lastv, double& left, double& right) {
    if (t <= last) {
      eL[par][t] = first;
      eR[par][t] = lastv;
    }
    __syncthreads();
    left = eR[par][tl];
    right = eL[par][tr];
    par ^= 1;
  };
  // Chebyshev terms with pre-scaled coefficients, every array indexed at compile time
  // (no pointers to register arrays, so nothing is demoted to local memory):
  //   U_1 = f·(u, e, w);  U_{j+1} = g·(U_j, e, w) + σ U_{j−1}
  // last valid element of a run: selects over compile-time indices (an indexed read would
  // demote the register array to local memory)
// FULL (n a multiple of PPT): every run has PPT points and the last index is static.
#define PX_RUN_LAST(arr, out)                                                                      \
  do {                                                                                             \
    if (FULL) {                                                                                    \
      out = arr[PPT - 1];                                                                          \
    } else {                                                                                       \
      out = arr[0];                                                                                \
      _Pragma("unroll") for (int kk = 1; kk < PPT; ++kk) out = (kk == cnt - 1) ? arr[kk] : out;    \
    }                                                                                              \
  } while (0)
  auto action = [&](const Scan1DPlan& pl) {
    const double f0 = pl.f[0], f1 = pl.f[1], f2 = pl.f[2];
    const double g0 = pl.g[0], g1 = pl.g[1], g2 = pl.g[2];
    const double sg = (double)pl.sigma;
    const double* __restrict__ be = pl.be;   // plan fields hoisted out of the term loop
    const double* __restrict__ bp = pl.bp;
    const int degree = pl.degree, substeps = pl.substeps;
    for (int sub = 0; sub < substeps; ++sub) {
      double up[PPT], uc[PPT], acc[PPT], pc[PPT];
      const double b0 = __ldg(be), b1 = __ldg(be + 1);
      const double p0 = phi ? __ldg(bp) : 0.0, p1 = phi ? __ldg(bp + 1) : 0.0;
      double left, right, lastv;
      PX_RUN_LAST(C, lastv);
      exchange(C[0], lastv, left, right);
#pragma unroll
      for (int k = 0; k < PPT; ++k) {
        const double wl = (k == 0) ? left : C[k - 1];
        const double wr = (k + 1 == PPT || (!FULL && k + 1 >= cnt)) ? right : C[k + 1];
        double v = f0 * C[k];
        v = fma(f1, wr, v);
        uc[k] = fma(f2, wl, v);
      }
#pragma unroll
      for (int k = 0; k < PPT; ++k) {
        up[k] = C[k];
        acc[k] = b0 * up[k] + b1 * uc[k];
        pc[k] = p0 * up[k] + p1 * uc[k];
      }
      for (int j = 2; j <= degree; ++j) {
        PX_RUN_LAST(uc, lastv);
        exchange(uc[0], lastv, left, right);
        const double bj = __ldg(be + j), pj = phi ? __ldg(bp + j) : 0.0;
        double un[PPT];
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
          const double wl = (k == 0) ? left : uc[k - 1];
          const double wr = (k + 1 == PPT || (!FULL && k + 1 >= cnt)) ? right : uc[k + 1];
          double v = fma(g0, uc[k], sg * up[k]);
          v = fma(g1, wr, v);
          un[k] = fma(g2, wl, v);
        }
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
          up[k] = uc[k];
          uc[k] = un[k];
          acc[k] += bj * un[k];
          if (phi) pc[k] += pj * un[k];
        }
      }
#pragma unroll
      for (int k = 0; k < PPT; ++k) {
        C[k] = acc[k];
        G[k] += pc[k];
      }
    }
  };
  // one call site of `action` (a second one would out-line it and demote the captured
  // register arrays C, G to local memory): Pl−1 slice carries, then the optional long span
  const int n_act = a.Pl - 1 + (a.use_long ? 1 : 0);
  for (int s = 1; s <= n_act; ++s) {
    const bool lng = s == a.Pl;
    action(lng ? a.lng : a.slice);
    if (!lng) {
      const int q = a.adjoint ? a.Pl - 1 - s : s;
#pragma unroll
      for (int k = 0; k < PPT; ++k)
        if (k < cnt) C[k] += lanes[(size_t)q * n + start + k];
    }
  }
#undef PX_RUN_LAST
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    if (k < cnt) {
      a.out[(size_t)b * n + start + k] = C[k];
      if (phi) a.pacc[(size_t)b * n + start + k] = G[k];
    }
  }
}

// ---------------------------------------------------------------------------
// Thread-block-cluster version: one member's carry recursion spread over the CS CTAs
// of a cluster (CS SMs instead of one). CTA r owns W = n/CS points and also computes a
// ghost zone of G points on each side (redundantly), so the Chebyshev terms run with
// CTA-local barriers only; every G terms (and at the start of every action) the ghost
// zones are refreshed from the neighbouring CTAs' shared memory (DSMEM) after one
// cluster barrier. Exchange buffers are double buffered, so one cluster barrier per
// refresh suffices. Same arithmetic per point as k_scan1d (pre-scaled terms).
// ---------------------------------------------------------------------------
template <int PPT, int CS, int G, int MB>
__global__ void __launch_bounds__(256) k_scan1d_cluster(Scan1DArgs a, int B) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  static_assert(G % PPT == 0, "ghost width must be whole runs");
  constexpr int GR = G / PPT;            // ghost runs per side
  // MB members per CTA: their recurrences are independent, so interleaving them hides the
  // per-term latency chain (edge store → barrier → neighbour load → 3 FMAs) MB-fold
  __shared__ double eL[2][MB][256];
  __shared__ double eR[2][MB][256];
  __shared__ double xbuf[2][2][2][MB][G];  // [parity][side 0 = my left edge, 1 = right][cur/prev][member][G]
  const int n = a.n;
  const int W = n / CS;                  // owned points
  const int rank = (int)cluster.block_rank();
  const int bb = (blockIdx.x / CS) * MB; // first member of this CTA
  const int t = threadIdx.x;
  const int NR = W / PPT + 2 * GR;       // runs in the local domain (threads with points)
  const bool act = t < NR;
  // local run t covers global points g0 + k, g0 = rank·W − G + t·PPT (mod n)
  const int g0 = rank * W - G + t * PPT;
  const bool owned = act && t >= GR && t < NR - GR;
  const int tl = (t == 0) ? 0 : t - 1, tr = (t + 1 >= NR) ? NR - 1 : t + 1;  // domain ends: clamped
  const bool phi = a.adjoint && a.pacc != nullptr;
  auto gidx = [&](int k) { int g = g0 + k; g %= n; return g < 0 ? g + n : g; };
  auto mact = [&](int m) { return bb + m < B; };
  double C[MB][PPT], G_[MB][PPT];
  const int q0 = a.adjoint ? a.Pl - 1 : 0;
#pragma unroll
  for (int m = 0; m < MB; ++m) {
    const double* lanes = a.lanes + (size_t)(bb + m) * a.Pl * n;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      C[m][k] = (act && mact(m)) ? lanes[(size_t)q0 * n + gidx(k)] : 0.0;
      G_[m][k] = (phi && owned && mact(m)) ? a.pacc[(size_t)(bb + m) * n + gidx(k)] : 0.0;
    }
  }
  int par = 0, xpar = 0;
  // run-edge exchange inside the CTA for all members: (left, right) neighbours
  auto exchange = [&](double (*u)[PPT], double* left, double* right) {
    if (act) {
#pragma unroll
      for (int m = 0; m < MB; ++m) {
        eL[par][m][t] = u[m][0];
        eR[par][m][t] = u[m][PPT - 1];
      }
    }
    __syncthreads();
#pragma unroll
    for (int m = 0; m < MB; ++m) {
      left[m] = eR[par][m][tl];
      right[m] = eL[par][m][tr];
    }
    par ^= 1;
  };
  // refresh the ghost runs of u (and v, when given) from the neighbouring CTAs
  auto refresh = [&](double (*u)[PPT], double (*v)[PPT]) {
    if (act) {
      if (t >= GR && t < 2 * GR) {
#pragma unroll
        for (int m = 0; m < MB; ++m)
#pragma unroll
          for (int k = 0; k < PPT; ++k) {
            xbuf[xpar][0][0][m][(t - GR) * PPT + k] = u[m][k];
            if (v) xbuf[xpar][0][1][m][(t - GR) * PPT + k] = v[m][k];
          }
      }
      if (t >= NR - 2 * GR && t < NR - GR) {
#pragma unroll
        for (int m = 0; m < MB; ++m)
#pragma unroll
          for (int k = 0; k < PPT; ++k) {
            xbuf[xpar][1][0][m][(t - (NR - 2 * GR)) * PPT + k] = u[m][k];
            if (v) xbuf[xpar][1][1][m][(t - (NR - 2 * GR)) * PPT + k] = v[m][k];
          }
      }
    }
    cluster.sync();
    // my left ghosts = left neighbour's right edge; my right ghosts = right neighbour's left edge
    if (act && t < GR) {
      const double* src = cluster.map_shared_rank(&xbuf[xpar][1][0][0][0], (unsigned)((rank + CS - 1) % CS));
#pragma unroll
      for (int m = 0; m < MB; ++m)
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
          u[m][k] = src[m * G + t * PPT + k];
          if (v) v[m][k] = src[MB * G + m * G + t * PPT + k];
        }
    }
    if (act && t >= NR - GR) {
      const double* src = cluster.map_shared_rank(&xbuf[xpar][0][0][0][0], (unsigned)((rank + 1) % CS));
#pragma unroll
      for (int m = 0; m < MB; ++m)
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
          u[m][k] = src[m * G + (t - (NR - GR)) * PPT + k];
          if (v) v[m][k] = src[MB * G + m * G + (t - (NR - GR)) * PPT + k];
        }
    }
    xpar ^= 1;
  };
  auto action = [&](const Scan1DPlan& pl) {
    const double f0 = pl.f[0], f1 = pl.f[1], f2 = pl.f[2];
    const double g0c = pl.g[0], g1 = pl.g[1], g2 = pl.g[2];
    const double sg = (double)pl.sigma;
    const double* __restrict__ be = pl.be;
    const double* __restrict__ bp = pl.bp;
    const int degree = pl.degree, substeps = pl.substeps;
    for (int sub = 0; sub < substeps; ++sub) {
      double up[MB][PPT], uc[MB][PPT], acc[MB][PPT], pc[MB][PPT];
      refresh(C, nullptr);
      int valid = G;  // ghost depth still exact
      const double b0 = __ldg(be), b1 = __ldg(be + 1);
      const double p0 = phi ? __ldg(bp) : 0.0, p1 = phi ? __ldg(bp + 1) : 0.0;
      double left[MB], right[MB];
      exchange(C, left, right);
#pragma unroll
      for (int m = 0; m < MB; ++m)
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
          const double wl = (k == 0) ? left[m] : C[m][k - 1];
          const double wr = (k + 1 == PPT) ? right[m] : C[m][k + 1];
          double v = f0 * C[m][k];
          v = fma(f1, wr, v);
          uc[m][k] = fma(f2, wl, v);
          up[m][k] = C[m][k];
          acc[m][k] = b0 * up[m][k] + b1 * uc[m][k];
          pc[m][k] = p0 * up[m][k] + p1 * uc[m][k];
        }
      --valid;
      for (int j = 2; j <= degree; ++j) {
        if (valid == 0) {
          refresh(uc, up);
          valid = G;
        }
        exchange(uc, left, right);
        const double bj = __ldg(be + j), pj = phi ? __ldg(bp + j) : 0.0;
#pragma unroll
        for (int m = 0; m < MB; ++m) {
          double un[PPT];
#pragma unroll
          for (int k = 0; k < PPT; ++k) {
            const double wl = (k == 0) ? left[m] : uc[m][k - 1];
            const double wr = (k + 1 == PPT) ? right[m] : uc[m][k + 1];
            double v = fma(g0c, uc[m][k], sg * up[m][k]);
            v = fma(g1, wr, v);
            un[k] = fma(g2, wl, v);
          }
#pragma unroll
          for (int k = 0; k < PPT; ++k) {
            up[m][k] = uc[m][k];
            uc[m][k] = un[k];
            acc[m][k] += bj * un[k];
            if (phi) pc[m][k] += pj * un[k];
          }
        }
        --valid;
      }
#pragma unroll
      for (int m = 0; m < MB; ++m)
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
          C[m][k] = acc[m][k];
          G_[m][k] += pc[m][k];
        }
    }
  };
  const int n_act = a.Pl - 1 + (a.use_long ? 1 : 0);
  for (int s = 1; s <= n_act; ++s) {
    const bool lng = s == a.Pl;
    action(lng ? a.lng : a.slice);
    if (!lng) {
      const int q = a.adjoint ? a.Pl - 1 - s : s;
      if (act) {
#pragma unroll
        for (int m = 0; m < MB; ++m) {
          if (!mact(m)) continue;
          const double* lanes = a.lanes + (size_t)(bb + m) * a.Pl * n;
#pragma unroll
          for (int k = 0; k < PPT; ++k) C[m][k] += lanes[(size_t)q * n + gidx(k)];
        }
      }
    }
  }
  if (owned) {
#pragma unroll
    for (int m = 0; m < MB; ++m) {
      if (!mact(m)) continue;
#pragma unroll
      for (int k = 0; k < PPT; ++k) {
        a.out[(size_t)(bb + m) * n + gidx(k)] = C[m][k];
        if (phi) a.pacc[(size_t)(bb + m) * n + gidx(k)] = G_[m][k];
      }
    }
  }
  cluster.sync();  // no CTA leaves while a neighbour may still read its exchange buffers
}

}  // namespace px
