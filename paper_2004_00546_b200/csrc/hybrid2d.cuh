// hybrid2d.cuh — kernels of the reference's 2D two-field Burgers testbed (instantiated in hybrid2d.cu):
// the two-field rhs (problems.py:177-186), J(q)ᵀ (problems.py:316-343), the forward Jacobian
// (problems.py:213-287), slice means and FOV box, tracking cost; per-stage-launch kernels for any
// grid (k_b2_*) and on-chip kernels for nx·ny ≤ 2048 (k_b2s_*: the serial sweep, the slice adjoint
// solves, the frozen-operator carry, Algorithm 2's sweep) — DESIGN.md §3.5.
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"
#include "hybrid_args.h"

namespace px {

struct B2Geom {
  int nx, ny;
  double i2hx, i2hy;  // 1/(2hx), 1/(2hy)
  double dx2, dy2;    // D/hx², D/hy²
};

__device__ __forceinline__ void b2_nbrs(int i, const B2Geom& g, int& e, int& w, int& n, int& s) {
  const int y = i / g.nx, x = i - y * g.nx;
  e = (x + 1 == g.nx) ? i + 1 - g.nx : i + 1;
  w = (x == 0) ? i + g.nx - 1 : i - 1;
  n = (y + 1 == g.ny) ? x : i + g.nx;
  s = (y == 0) ? i + (g.ny - 1) * g.nx : i - g.nx;
}

// ---- serial direct sweep: one RK4 stage ------------------------------------------------------
struct B2DirectArgs {
  const double* win; long long win_bs;      // stage input W (neighbours read)
  const double* base; long long base_bs;    // u_i
  const double* accin; long long accin_bs;  // running u_i + Σ weights·k
  double* wout;                             // next stage input u_i + cw·k (B × 2n; null at stage 4)
  double* accout; long long accout_bs;
  const double* f;                          // B × 2n forcing field
  double cw, ca, theta;
  B2Geom g;
};

__global__ void __launch_bounds__(256) k_b2_direct_stage(B2DirectArgs a) {
  const int n = a.g.nx * a.g.ny;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const size_t b = blockIdx.y;
  const double* U = a.win + b * a.win_bs;
  const double* V = U + n;
  int e, w, nn, s;
  b2_nbrs(i, a.g, e, w, nn, s);
  const double uc = U[i], ue = U[e], uw = U[w], un = U[nn], us = U[s];
  const double vc = V[i], ve = V[e], vw = V[w], vn = V[nn], vs = V[s];
  const double dUx = (ue - uw) * a.g.i2hx, dUy = (un - us) * a.g.i2hy;
  const double dVx = (ve - vw) * a.g.i2hx, dVy = (vn - vs) * a.g.i2hy;
  const double lU = a.g.dx2 * (ue - 2.0 * uc + uw) + a.g.dy2 * (un - 2.0 * uc + us);
  const double lV = a.g.dx2 * (ve - 2.0 * vc + vw) + a.g.dy2 * (vn - 2.0 * vc + vs);
  const double* f = a.f + b * 2 * n;
  const double ku = -uc * dUx - vc * dUy + lU + a.theta * f[i];
  const double kv = -uc * dVx - vc * dVy + lV + a.theta * f[n + i];
  const double* bs = a.base + b * a.base_bs;
  if (a.wout) {
    double* wo = a.wout + b * 2 * n;
    wo[i] = bs[i] + a.cw * ku;
    wo[n + i] = bs[n + i] + a.cw * kv;
  }
  const double* ai = a.accin + b * a.accin_bs;
  double* ao = a.accout + b * a.accout_bs;
  ao[i] = ai[i] + a.ca * ku;
  ao[n + i] = ai[n + i] + a.ca * kv;
}

// ---- tracking cost: per-member partial sums of w_j·‖traj_j − target_j‖² (fixed order) --------
__global__ void __launch_bounds__(256) k_b2_cost_partial(double* partial, const double* traj, const double* target,
                                                         int target_b, size_t n2, int S, int B) {
  __shared__ double red[8];
  const size_t b = blockIdx.y;
  const size_t total = (size_t)(S + 1) * n2;
  double acc = 0.0;
  for (size_t m = (size_t)blockIdx.x * blockDim.x + threadIdx.x; m < total; m += (size_t)gridDim.x * blockDim.x) {
    const size_t j = m / n2, i = m - j * n2;
    const double d = traj[(j * B + b) * n2 + i] - target[(target_b > 1 ? j * B + b : j) * n2 + i];
    acc += (j == 0 || j == (size_t)S ? 0.5 : 1.0) * d * d;
  }
  const double r = block_sum<256>(acc, red);
  if (threadIdx.x == 0) partial[b * gridDim.x + blockIdx.x] = r;
}

__global__ void k_b2_cost_final(double* J, const double* partial, int m, double scale, int B) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  double s = 0.0;
  for (int k = 0; k < m; ++k) s += partial[(size_t)b * m + k];
  J[b] = scale * s;
}

// ---- slice means (trapezoid on the slice's nodes, problems.py:346-366) -----------------------
__global__ void __launch_bounds__(256) k_b2_means(double* ubar, const double* traj, const int* offs, int B, size_t n2) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n2) return;
  const size_t b = blockIdx.y, p = blockIdx.z;
  const int lo = offs[p], hi = offs[p + 1];
  double acc = 0.5 * traj[((size_t)lo * B + b) * n2 + i];
  for (int j = lo + 1; j < hi; ++j) acc += traj[((size_t)j * B + b) * n2 + i];
  acc += 0.5 * traj[((size_t)hi * B + b) * n2 + i];
  ubar[(p * B + b) * n2 + i] = acc / (double)(hi - lo);
}

// ---- FOV box of the frozen operators J(q̄_p)ᵀ (problems.frozen_bounds_2d), per-block partials --
__global__ void __launch_bounds__(256) k_b2_bounds(double* part, const double* ubar, int rows, B2Geom g, double D) {
  __shared__ double red[3][8];
  const int n = g.nx * g.ny;
  double lo = INFINITY, hi = -INFINITY, im = 0.0;
  bool bad = false;
  const size_t total = (size_t)rows * n;
  const double dd = 2.0 * g.dx2 + 2.0 * g.dy2;
  for (size_t m = (size_t)blockIdx.x * blockDim.x + threadIdx.x; m < total; m += (size_t)gridDim.x * blockDim.x) {
    const size_t r = m / n;
    const int i = (int)(m - r * n);
    const double* U = ubar + r * 2 * n;
    const double* V = U + n;
    int e, w, nn, s;
    b2_nbrs(i, g, e, w, nn, s);
    const double uc = U[i], ue = U[e], uw = U[w], un = U[nn], us = U[s];
    const double vc = V[i], ve = V[e], vw = V[w], vn = V[nn], vs = V[s];
    const double dUx = (ue - uw) * g.i2hx, dUy = (un - us) * g.i2hy;
    const double dVx = (ve - vw) * g.i2hx, dVy = (vn - vs) * g.i2hy;
    const double rad = (fabs(ue - uc) + fabs(uc - uw)) * (0.5 * g.i2hx) + (fabs(vn - vc) + fabs(vc - vs)) * (0.5 * g.i2hy) +
                       dd + 0.5 * fabs(dVx + dUy);
    const double imv = (fabs(ue + uc) + fabs(uc + uw)) * (0.5 * g.i2hx) + (fabs(vn + vc) + fabs(vc + vs)) * (0.5 * g.i2hy) +
                       0.5 * fabs(dUy - dVx);
    const double da = -dUx - dd, db = -dVy - dd;
    if (!(isfinite(rad) && isfinite(imv) && isfinite(da) && isfinite(db))) bad = true;
    lo = fmin(lo, fmin(da, db) - rad);
    hi = fmax(hi, fmax(da, db) + rad);
    im = fmax(im, imv);
  }
  if (bad) lo = hi = im = NAN;  // fmin/fmax drop NaN: carry it explicitly
  // block reduction (NaN-propagating)
  auto comb = [](double x, double y, int op) {
    if (x != x || y != y) return (double)NAN;
    return op == 0 ? fmin(x, y) : fmax(x, y);
  };
  for (int o = 16; o > 0; o >>= 1) {
    lo = comb(lo, __shfl_down_sync(0xffffffffu, lo, o), 0);
    hi = comb(hi, __shfl_down_sync(0xffffffffu, hi, o), 1);
    im = comb(im, __shfl_down_sync(0xffffffffu, im, o), 1);
  }
  const int wp = threadIdx.x >> 5, ln = threadIdx.x & 31;
  if (ln == 0) { red[0][wp] = lo; red[1][wp] = hi; red[2][wp] = im; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < 8; ++k) {
      lo = comb(lo, red[0][k], 0);
      hi = comb(hi, red[1][k], 1);
      im = comb(im, red[2][k], 1);
    }
    part[3 * blockIdx.x + 0] = lo;
    part[3 * blockIdx.x + 1] = hi;
    part[3 * blockIdx.x + 2] = im;
  }
}

// J(q)ᵀ(a, b) at point i (problems.py:316-343): out_a = ∂x(Ua) + ∂y(Va) − (∂xU)a − (∂xV)b + D∇²a,
// out_b = ∂x(Ub) + ∂y(Vb) − (∂yU)a − (∂yV)b + D∇²b
struct B2Pt {
  double ue, uw, un, us, ve, vw, vn, vs;
};
__device__ __forceinline__ void b2_adj_apply(const B2Geom& g, const B2Pt& q, const double* A, const double* Bf, int i,
                                             int e, int w, int nn, int s, double& oa, double& ob) {
  const double ac = A[i], ae = A[e], aw = A[w], an = A[nn], as = A[s];
  const double bc = Bf[i], be = Bf[e], bw = Bf[w], bn = Bf[nn], bs = Bf[s];
  const double dUx = (q.ue - q.uw) * g.i2hx, dUy = (q.un - q.us) * g.i2hy;
  const double dVx = (q.ve - q.vw) * g.i2hx, dVy = (q.vn - q.vs) * g.i2hy;
  oa = (q.ue * ae - q.uw * aw) * g.i2hx + (q.vn * an - q.vs * as) * g.i2hy - dUx * ac - dVx * bc +
       g.dx2 * (ae - 2.0 * ac + aw) + g.dy2 * (an - 2.0 * ac + as);
  ob = (q.ue * be - q.uw * bw) * g.i2hx + (q.vn * bn - q.vs * bs) * g.i2hy - dUy * ac - dVy * bc +
       g.dx2 * (be - 2.0 * bc + bw) + g.dy2 * (bn - 2.0 * bc + bs);
}

// ---- slice adjoint solves (hybrid.py:194-203): one RK4 stage of every active lane ------------
struct B2AdjArgs {
  const double* yin;    // L × 2n stage input (neighbours read)
  double* a;            // L × 2n: a_i (base); stage 4 writes a_{i+1} here
  const double* accin;  // L × 2n (stage 1: a)
  double* accout;       // L × 2n (stage 4: a)
  double* yout;         // L × 2n next stage input (null at stage 4)
  double* z;            // L × 2n: ∫θ·a dt (RK4-consistent)
  const double* traj;   // (S+1) × B × 2n
  const double* target; // (S+1) × (B | 1) × 2n
  const int* offs;
  const double* theta;  // θ(k·h/2)
  double wa, wb;        // stage state = wa·node[top] + wb·node[top − 1]
  double cw, ca, cz;
  int tsel;             // θ at node top (0), top − ½ (1), top − 1 (2)
  int step, p0, pcount, P, B, target_b;
  B2Geom g;
};

__global__ void __launch_bounds__(256) k_b2_adj_stage(B2AdjArgs a) {
  const int n = a.g.nx * a.g.ny;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int b = blockIdx.y / a.pcount;
  const int p = a.p0 + blockIdx.y % a.pcount;
  const int np = a.offs[p + 1] - a.offs[p];
  if (a.step >= np) return;
  const int top = a.offs[p + 1] - a.step;
  const size_t n2 = 2 * (size_t)n;
  const size_t lane = (size_t)b * a.P + p;
  const double* qa = a.traj + ((size_t)top * a.B + b) * n2;
  const double* qb = a.traj + ((size_t)(top - 1) * a.B + b) * n2;
  const double* ta = a.target + ((size_t)top * a.target_b + (a.target_b > 1 ? b : 0)) * n2;
  const double* tb = a.target + ((size_t)(top - 1) * a.target_b + (a.target_b > 1 ? b : 0)) * n2;
  int e, w, nn, s;
  b2_nbrs(i, a.g, e, w, nn, s);
  auto st = [&](size_t k) { return a.wa * qa[k] + a.wb * qb[k]; };
  B2Pt q;
  q.ue = st(e); q.uw = st(w); q.un = st(nn); q.us = st(s);
  q.ve = st(n + e); q.vw = st(n + w); q.vn = st(n + nn); q.vs = st(n + s);
  const double su = 2.0 * (st(i) - (a.wa * ta[i] + a.wb * tb[i]));
  const double sv = 2.0 * (st(n + i) - (a.wa * ta[n + i] + a.wb * tb[n + i]));
  const double* Y = a.yin + lane * n2;
  double ka, kb;
  b2_adj_apply(a.g, q, Y, Y + n, i, e, w, nn, s, ka, kb);
  ka += su;
  kb += sv;
  const double th = a.theta[2 * top - a.tsel];
  double* z = a.z + lane * n2;
  z[i] += a.cz * th * Y[i];
  z[n + i] += a.cz * th * Y[n + i];
  const double* base = a.a + lane * n2;
  const double* ai = a.accin + lane * n2;
  const double ra = ai[i] + a.ca * ka, rb = ai[n + i] + a.ca * kb;
  if (a.yout) {
    double* yo = a.yout + lane * n2;
    yo[i] = base[i] + a.cw * ka;
    yo[n + i] = base[n + i] + a.cw * kb;
  }
  double* ao = a.accout + lane * n2;
  ao[i] = ra;
  ao[n + i] = rb;
}

// ---- frozen-operator carry: one Chebyshev term of exp(τ·J(q̄_p)ᵀ) with the law series ----------
struct B2ChebArgs {
  const double* x;     // B × 2n: U_k (neighbours read)
  const double* prev;  // B × 2n: U_{k−1} (unused on the first term)
  double* out;         // B × 2n: U_{k+1}
  double* acc;         // B × 2n: Σ be_k U_k
  double* G;           // B × 2n: += Σ bl_k U_k (the θ-weighted integral)
  const double* qbar;  // B × 2n: the slice mean q̄_p
  double alpha, c0, sg, be0, bek, bl0, blk;
  int first;
  B2Geom g;
};

__global__ void __launch_bounds__(256) k_b2_cheb_term(B2ChebArgs a) {
  const int n = a.g.nx * a.g.ny;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const size_t off = (size_t)blockIdx.y * 2 * n;
  const double* U = a.qbar + off;
  const double* V = U + n;
  int e, w, nn, s;
  b2_nbrs(i, a.g, e, w, nn, s);
  B2Pt q{U[e], U[w], U[nn], U[s], V[e], V[w], V[nn], V[s]};
  const double* X = a.x + off;
  double oa, ob;
  b2_adj_apply(a.g, q, X, X + n, i, e, w, nn, s, oa, ob);
  const double xa = X[i], xb = X[n + i];
  double ua = a.alpha * (oa - a.c0 * xa), ub = a.alpha * (ob - a.c0 * xb);
  double* acc = a.acc + off;
  double* G = a.G + off;
  if (a.first) {
    acc[i] = a.be0 * xa + a.bek * ua;
    acc[n + i] = a.be0 * xb + a.bek * ub;
    G[i] += a.bl0 * xa + a.blk * ua;
    G[n + i] += a.bl0 * xb + a.blk * ub;
  } else {
    const double* P = a.prev + off;
    ua += a.sg * P[i];
    ub += a.sg * P[n + i];
    acc[i] += a.bek * ua;
    acc[n + i] += a.bek * ub;
    G[i] += a.blk * ua;
    G[n + i] += a.blk * ub;
  }
  double* o = a.out + off;
  o[i] = ua;
  o[n + i] = ub;
}

// C[b] = (add ? C[b] : 0) + lanes[b·P + p]
__global__ void k_b2_take_lane(double* C, const double* lanes, int P, int p, int add, size_t n2) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n2) return;
  const size_t b = blockIdx.y;
  const double v = lanes[(b * P + p) * n2 + i];
  C[b * n2 + i] = add ? C[b * n2 + i] + v : v;
}

// grad[b] = (Σ_p zl[b·P + p] + G[b]) / T
__global__ void k_b2_grad(double* grad, const double* zl, const double* G, int P, double invT, size_t n2) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n2) return;
  const size_t b = blockIdx.y;
  double s = 0.0;
  for (int p = 0; p < P; ++p) s += zl[(b * P + p) * n2 + i];
  grad[b * n2 + i] = (s + G[b * n2 + i]) * invT;
}


// =============================================================================================
// On-chip variants for small grids (nx·ny ≤ B2S_MAX_N — the reference's 32×32 configs): the
// whole state of a member (or of a slice lane) stays in shared memory and registers, so the
// serial sweep is ONE kernel (one CTA per member, a CTA barrier per RK4 stage) instead of 4·S
// dependent launches, every slice's adjoint solve is one CTA of a second kernel that waits on a
// per-slice progress flag while the sweep is still running (as the 1D path, hybrid.cuh), and the
// frozen-operator carry is one kernel per gradient.
// =============================================================================================
constexpr int B2S_NT = 512;
constexpr int B2S_MAX_N = 2048;  // points per field: 4 state arrays of 2n doubles = 128 KB in the lane kernel

// the two-field rhs at point i from a shared-memory state W = (U | V)
__device__ __forceinline__ void b2s_rhs(const B2Geom& g, const double* W, int n, int i, int e, int w, int nn, int s,
                                        double& ku, double& kv) {
  const double* V = W + n;
  const double uc = W[i], ue = W[e], uw = W[w], un = W[nn], us = W[s];
  const double vc = V[i], ve = V[e], vw = V[w], vn = V[nn], vs = V[s];
  const double dUx = (ue - uw) * g.i2hx, dUy = (un - us) * g.i2hy;
  const double dVx = (ve - vw) * g.i2hx, dVy = (vn - vs) * g.i2hy;
  ku = -uc * dUx - vc * dUy + g.dx2 * (ue - 2.0 * uc + uw) + g.dy2 * (un - 2.0 * uc + us);
  kv = -uc * dVx - vc * dVy + g.dx2 * (ve - 2.0 * vc + vw) + g.dy2 * (vn - 2.0 * vc + vs);
}

struct B2sDirectArgs {
  const double* u0;     // B × 2n
  const double* f;      // B × 2n
  double* traj;         // (S+1) × B × 2n
  const double* theta;  // θ(k·h/2)
  int* flags;           // B × P progress flags
  const int* offs;      // P+1
  int P, B, S;
  double h;
  B2Geom g;
};

template <int PPT>
__global__ void __launch_bounds__(B2S_NT) k_b2s_direct(B2sDirectArgs a) {
  extern __shared__ double b2s_sm[];
  const int n = a.g.nx * a.g.ny, n2 = 2 * n;
  const int t = threadIdx.x;
  const size_t b = blockIdx.x;
  double* W0 = b2s_sm;
  double* W1 = b2s_sm + n2;
  double u[PPT][2], acc[PPT][2], fr[PPT][2];
  int ie[PPT], iw[PPT], in[PPT], is[PPT];
  const double* u0 = a.u0 + b * n2;
  const double* f = a.f + b * n2;
  double* tr = a.traj + b * n2;
  const size_t ns = (size_t)a.B * n2;
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    const int i = t + q * B2S_NT;
    if (i < n) {
      b2_nbrs(i, a.g, ie[q], iw[q], in[q], is[q]);
      u[q][0] = u0[i]; u[q][1] = u0[n + i];
      fr[q][0] = f[i]; fr[q][1] = f[n + i];
      W0[i] = u[q][0]; W0[n + i] = u[q][1];
      tr[i] = u[q][0]; tr[n + i] = u[q][1];
    }
  }
  __syncthreads();
  auto stage = [&](const double* Wi, double* Wo, double cw, double ca, double th, bool first) {
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      const int i = t + q * B2S_NT;
      if (i < n) {
        double ku, kv;
        b2s_rhs(a.g, Wi, n, i, ie[q], iw[q], in[q], is[q], ku, kv);
        ku += th * fr[q][0];
        kv += th * fr[q][1];
        acc[q][0] = (first ? u[q][0] : acc[q][0]) + ca * ku;
        acc[q][1] = (first ? u[q][1] : acc[q][1]) + ca * kv;
        Wo[i] = u[q][0] + cw * ku;
        Wo[n + i] = u[q][1] + cw * kv;
      }
    }
  };
  const double h = a.h;
  int p = 0, next = a.offs[1];
  for (int s = 0; s < a.S; ++s) {
    const double th1 = a.theta[2 * s], th2 = a.theta[2 * s + 1], th4 = a.theta[2 * s + 2];
    stage(W0, W1, 0.5 * h, h / 6.0, th1, true);
    __syncthreads();
    stage(W1, W0, 0.5 * h, h / 3.0, th2, false);
    __syncthreads();
    stage(W0, W1, h, h / 3.0, th2, false);
    __syncthreads();
    double* node = tr + (size_t)(s + 1) * ns;
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      const int i = t + q * B2S_NT;
      if (i < n) {
        double ku, kv;
        b2s_rhs(a.g, W1, n, i, ie[q], iw[q], in[q], is[q], ku, kv);
        u[q][0] = acc[q][0] + (h / 6.0) * (ku + th4 * fr[q][0]);
        u[q][1] = acc[q][1] + (h / 6.0) * (kv + th4 * fr[q][1]);
        W0[i] = u[q][0]; W0[n + i] = u[q][1];
        node[i] = u[q][0]; node[n + i] = u[q][1];
      }
    }
    if (s + 1 == next) {  // slice p's nodes are stored: every writer fences, then one flag
      __threadfence();
      __syncthreads();
      if (t == 0) atomicExch(a.flags + b * a.P + p, 1);
      ++p;
      next = (p < a.P) ? a.offs[p + 1] : -1;
    } else {
      __syncthreads();
    }
  }
}

struct B2sLaneArgs {
  const double* traj;    // (S+1) × B × 2n
  const double* target;  // (S+1) × tb × 2n
  const int* offs;
  const double* theta;
  int* flags;
  double* aend;          // (B·P) × 2n
  double* zl;            // (B·P) × 2n
  int P, B, target_b, wait;
  double h;
  B2Geom g;
};

// J(q)ᵀy at point i with the stage state q = wa·Qa + wb·Qb (MODE 0: Qa, 1: the node mean, 2: Qb)
template <int MODE>
__device__ __forceinline__ double b2s_state(const double* Qa, const double* Qb, int k) {
  if constexpr (MODE == 0) return Qa[k];
  else if constexpr (MODE == 2) return Qb[k];
  else return 0.5 * Qa[k] + 0.5 * Qb[k];
}

template <int PPT>
__global__ void __launch_bounds__(B2S_NT) k_b2s_lanes(B2sLaneArgs a) {
  extern __shared__ double b2s_sm[];
  const int n = a.g.nx * a.g.ny, n2 = 2 * n;
  const int t = threadIdx.x;
  const int lane = blockIdx.x, b = lane / a.P, p = lane % a.P;
  const int o0 = a.offs[p], o1 = a.offs[p + 1];
  if (a.wait) {
    if (t == 0) {
      volatile int* fl = a.flags + lane;
      while (*fl == 0) __nanosleep(200);
      __threadfence();
    }
    __syncthreads();
  }
  double* Y0 = b2s_sm;
  double* Y1 = Y0 + n2;
  double* Qa = Y1 + n2;
  double* Qb = Qa + n2;
  const size_t ns = (size_t)a.B * n2, ts = (size_t)a.target_b * n2;
  const double* nb = a.traj + (size_t)b * n2;
  const double* tg = a.target + (a.target_b > 1 ? (size_t)b * n2 : 0);
  double av[PPT][2], acc[PPT][2], z[PPT][2], ta[PPT][2], tb[PPT][2];
  int ie[PPT], iw[PPT], in[PPT], is[PPT];
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    const int i = t + q * B2S_NT;
    if (i < n) {
      b2_nbrs(i, a.g, ie[q], iw[q], in[q], is[q]);
      av[q][0] = av[q][1] = z[q][0] = z[q][1] = 0.0;
      Y0[i] = 0.0; Y0[n + i] = 0.0;
      Qa[i] = __ldcg(nb + (size_t)o1 * ns + i);
      Qa[n + i] = __ldcg(nb + (size_t)o1 * ns + n + i);
      ta[q][0] = tg[(size_t)o1 * ts + i];
      ta[q][1] = tg[(size_t)o1 * ts + n + i];
    }
  }
  const double h = a.h;
  auto stage = [&](auto mode, const double* Yi, double* Yo, double cw, double ca, double cz, double th, bool first,
                   bool last) {
    constexpr int MODE = decltype(mode)::value;
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      const int i = t + q * B2S_NT;
      if (i < n) {
        B2Pt s;
        s.ue = b2s_state<MODE>(Qa, Qb, ie[q]); s.uw = b2s_state<MODE>(Qa, Qb, iw[q]);
        s.un = b2s_state<MODE>(Qa, Qb, in[q]); s.us = b2s_state<MODE>(Qa, Qb, is[q]);
        s.ve = b2s_state<MODE>(Qa, Qb, n + ie[q]); s.vw = b2s_state<MODE>(Qa, Qb, n + iw[q]);
        s.vn = b2s_state<MODE>(Qa, Qb, n + in[q]); s.vs = b2s_state<MODE>(Qa, Qb, n + is[q]);
        double ka, kb;
        b2_adj_apply(a.g, s, Yi, Yi + n, i, ie[q], iw[q], in[q], is[q], ka, kb);
        double tu, tv;
        if constexpr (MODE == 0) { tu = ta[q][0]; tv = ta[q][1]; }
        else if constexpr (MODE == 2) { tu = tb[q][0]; tv = tb[q][1]; }
        else { tu = 0.5 * ta[q][0] + 0.5 * tb[q][0]; tv = 0.5 * ta[q][1] + 0.5 * tb[q][1]; }
        ka += 2.0 * (b2s_state<MODE>(Qa, Qb, i) - tu);
        kb += 2.0 * (b2s_state<MODE>(Qa, Qb, n + i) - tv);
        z[q][0] += cz * th * Yi[i];
        z[q][1] += cz * th * Yi[n + i];
        const double ra = (first ? av[q][0] : acc[q][0]) + ca * ka;
        const double rb = (first ? av[q][1] : acc[q][1]) + ca * kb;
        if (last) {
          av[q][0] = ra; av[q][1] = rb;
          Yo[i] = ra; Yo[n + i] = rb;
        } else {
          acc[q][0] = ra; acc[q][1] = rb;
          Yo[i] = av[q][0] + cw * ka;
          Yo[n + i] = av[q][1] + cw * kb;
        }
      }
    }
  };
  for (int top = o1; top > o0; --top) {
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      const int i = t + q * B2S_NT;
      if (i < n) {
        Qb[i] = __ldcg(nb + (size_t)(top - 1) * ns + i);
        Qb[n + i] = __ldcg(nb + (size_t)(top - 1) * ns + n + i);
        tb[q][0] = tg[(size_t)(top - 1) * ts + i];
        tb[q][1] = tg[(size_t)(top - 1) * ts + n + i];
      }
    }
    __syncthreads();
    const double th0 = a.theta[2 * top], th1 = a.theta[2 * top - 1], th2 = a.theta[2 * top - 2];
    stage(IC<0>{}, Y0, Y1, 0.5 * h, h / 6.0, h / 6.0, th0, true, false);
    __syncthreads();
    stage(IC<1>{}, Y1, Y0, 0.5 * h, h / 3.0, h / 3.0, th1, false, false);
    __syncthreads();
    stage(IC<1>{}, Y0, Y1, h, h / 3.0, h / 3.0, th1, false, false);
    __syncthreads();
    stage(IC<2>{}, Y1, Y0, 0.0, h / 6.0, h / 6.0, th2, false, true);
    __syncthreads();
    double* sw = Qa; Qa = Qb; Qb = sw;
#pragma unroll
    for (int q = 0; q < PPT; ++q) { ta[q][0] = tb[q][0]; ta[q][1] = tb[q][1]; }
  }
  double* ae = a.aend + (size_t)lane * n2;
  double* zo = a.zl + (size_t)lane * n2;
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    const int i = t + q * B2S_NT;
    if (i < n) {
      ae[i] = av[q][0]; ae[n + i] = av[q][1];
      zo[i] = z[q][0]; zo[n + i] = z[q][1];
    }
  }
}

struct B2sScanArgs {
  const double* ubar;         // P × B × 2n
  const double* aend;         // (B·P) × 2n
  const double* zl;           // (B·P) × 2n
  const double* qT;           // B × 2n or null
  const HybSlicePlan* plans;  // P
  const double* coef;         // pool: exp series per slice, law series per (slice, substep)
  double* qdag0;              // B × 2n
  double* grad;               // B × 2n
  int P, B;
  double invT;
  B2Geom g;
};

template <int PPT>
__global__ void __launch_bounds__(B2S_NT) k_b2s_scan(B2sScanArgs a) {
  extern __shared__ double b2s_sm[];
  const int n = a.g.nx * a.g.ny, n2 = 2 * n;
  const int t = threadIdx.x;
  const size_t b = blockIdx.x;
  double* X[3] = {b2s_sm, b2s_sm + n2, b2s_sm + 2 * n2};
  double* Qm = b2s_sm + 3 * n2;
  double acc[PPT][2], G[PPT][2];
  int ie[PPT], iw[PPT], in[PPT], is[PPT];
  const int top = a.qT ? a.P - 1 : a.P - 2;
  const double* c0src = a.qT ? a.qT + b * n2 : a.aend + (b * a.P + (a.P - 1)) * n2;
  int c = 0;
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    const int i = t + q * B2S_NT;
    if (i < n) {
      b2_nbrs(i, a.g, ie[q], iw[q], in[q], is[q]);
      G[q][0] = G[q][1] = 0.0;
      X[0][i] = c0src[i]; X[0][n + i] = c0src[n + i];
    }
  }
  for (int p = top; p >= 0; --p) {
    const double* qb = a.ubar + ((size_t)p * a.B + b) * n2;
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      const int i = t + q * B2S_NT;
      if (i < n) { Qm[i] = qb[i]; Qm[n + i] = qb[n + i]; }
    }
    __syncthreads();
    const HybSlicePlan pl = a.plans[p];
    const double* be = a.coef + pl.exp_off;
    const int K = pl.degree;
    for (int j = 0; j < pl.substeps; ++j) {
      const double* bl = a.coef + pl.law_off + (size_t)j * (K + 1);
      int prv = c, cur = (c + 1) % 3, nxt = (c + 2) % 3;
      // term 1
      {
        const double inv = 1.0 / pl.d;
        const double* Xc = X[c];
        double* Xo = X[cur];
#pragma unroll
        for (int q = 0; q < PPT; ++q) {
          const int i = t + q * B2S_NT;
          if (i < n) {
            B2Pt s{Qm[ie[q]], Qm[iw[q]], Qm[in[q]], Qm[is[q]], Qm[n + ie[q]], Qm[n + iw[q]], Qm[n + in[q]], Qm[n + is[q]]};
            double oa, ob;
            b2_adj_apply(a.g, s, Xc, Xc + n, i, ie[q], iw[q], in[q], is[q], oa, ob);
            const double xa = Xc[i], xb = Xc[n + i];
            const double ua = inv * (oa - pl.c0 * xa), ub = inv * (ob - pl.c0 * xb);
            acc[q][0] = be[0] * xa + be[1] * ua;
            acc[q][1] = be[0] * xb + be[1] * ub;
            G[q][0] += bl[0] * xa + bl[1] * ua;
            G[q][1] += bl[0] * xb + bl[1] * ub;
            Xo[i] = ua; Xo[n + i] = ub;
          }
        }
        __syncthreads();
      }
      const double two = 2.0 / pl.d, sg = (double)pl.sigma;
      for (int k = 2; k <= K; ++k) {
        const double* Xc = X[cur];
        const double* Xp = X[prv];
        double* Xo = X[nxt];
        const double bek = be[k], blk = bl[k];
#pragma unroll
        for (int q = 0; q < PPT; ++q) {
          const int i = t + q * B2S_NT;
          if (i < n) {
            B2Pt s{Qm[ie[q]], Qm[iw[q]], Qm[in[q]], Qm[is[q]], Qm[n + ie[q]], Qm[n + iw[q]], Qm[n + in[q]], Qm[n + is[q]]};
            double oa, ob;
            b2_adj_apply(a.g, s, Xc, Xc + n, i, ie[q], iw[q], in[q], is[q], oa, ob);
            const double ua = two * (oa - pl.c0 * Xc[i]) + sg * Xp[i];
            const double ub = two * (ob - pl.c0 * Xc[n + i]) + sg * Xp[n + i];
            acc[q][0] += bek * ua; acc[q][1] += bek * ub;
            G[q][0] += blk * ua; G[q][1] += blk * ub;
            Xo[i] = ua; Xo[n + i] = ub;   // Xo ≠ Xc, Xp: safe without a barrier before the write
          }
        }
        __syncthreads();
        const int tmp = prv; prv = cur; cur = nxt; nxt = tmp;
      }
      // the substep's result becomes the next input (nxt is free: its last readers passed the barrier)
      const bool slice_end = j + 1 == pl.substeps;
      const double* ae = a.aend + (b * a.P + p) * n2;
#pragma unroll
      for (int q = 0; q < PPT; ++q) {
        const int i = t + q * B2S_NT;
        if (i < n) {
          X[nxt][i] = acc[q][0] + (slice_end ? ae[i] : 0.0);       // + a_p(T_p) after slice p's action
          X[nxt][n + i] = acc[q][1] + (slice_end ? ae[n + i] : 0.0);
        }
      }
      c = nxt;
      __syncthreads();
    }
  }
  double* qo = a.qdag0 + b * n2;
  double* go = a.grad + b * n2;
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    const int i = t + q * B2S_NT;
    if (i < n) {
      qo[i] = X[c][i]; qo[n + i] = X[c][n + i];
      double su = 0.0, sv = 0.0;
      for (int p = 0; p < a.P; ++p) {
        su += a.zl[(b * a.P + p) * n2 + i];
        sv += a.zl[(b * a.P + p) * n2 + n + i];
      }
      go[i] = (su + G[q][0]) * a.invT;
      go[n + i] = (sv + G[q][1]) * a.invT;
    }
  }
}


// ---------------------------------------------------------------------------------------------
// Algorithm 2 on the two-field testbed (nonlinear.py:69-194), on chip (small grids): one sweep =
// k_b2s_nl_lanes (per slice the Jacobian-augmented linear problem from zero data, RK4 with the
// previous iterate linearly interpolated at the stages), k_b2s_nl_carry (the summed chain through
// exp(Δ(D∇² + J̄_p))), k_b2s_nl_hom (the homogeneous part on every node, step-width actions) and
// k_b2s_nl_err (per-slice relative change).
// ---------------------------------------------------------------------------------------------

// forward operator (D∇² + ∂N/∂q at q̄)·x at point i; q̄ and x in shared memory
__device__ __forceinline__ void b2s_jfull(const B2Geom& g, const double* Qm, const double* X, int n, int i, int e, int w,
                                          int nn, int s, double& oa, double& ob) {
  const double* Vm = Qm + n;
  const double* Xb = X + n;
  const double Ub = Qm[i], Vb = Vm[i];
  const double dUx = (Qm[e] - Qm[w]) * g.i2hx, dUy = (Qm[nn] - Qm[s]) * g.i2hy;
  const double dVx = (Vm[e] - Vm[w]) * g.i2hx, dVy = (Vm[nn] - Vm[s]) * g.i2hy;
  const double ac = X[i], ae = X[e], aw = X[w], an = X[nn], as = X[s];
  const double bc = Xb[i], be = Xb[e], bw = Xb[w], bn = Xb[nn], bs = Xb[s];
  oa = -Ub * (ae - aw) * g.i2hx - Vb * (an - as) * g.i2hy - dUx * ac - dUy * bc +
       g.dx2 * (ae - 2.0 * ac + aw) + g.dy2 * (an - 2.0 * ac + as);
  ob = -Ub * (be - bw) * g.i2hx - Vb * (bn - bs) * g.i2hy - dVx * ac - dVy * bc +
       g.dx2 * (be - 2.0 * bc + bw) + g.dy2 * (bn - 2.0 * bc + bs);
}

struct B2sNlArgs {
  const double* Q;      // (S+1) × B × 2n: the current iterate
  double* Qn;           // (S+1) × B × 2n: the next iterate
  const double* ubar;   // P × B × 2n slice means of Q
  const double* u0;     // B × 2n
  const double* f;      // B × 2n
  const double* theta;  // θ(k·h/2)
  double* yend;         // (B·P) × 2n
  double* Dc;           // (P+1) × B × 2n carried homogeneous parts at the slice starts
  double* err;          // B·P
  const double* coef;   // be_slice[0..Ks], be_step[0..Kh]
  int P, B, nsteps, S;
  int Ks, subs_s, sig_s, Kh, subs_h, sig_h;
  double c0_s, d_s, c0_h, d_h;
  double h;
  B2Geom g;
};

template <int PPT>
__global__ void __launch_bounds__(B2S_NT) k_b2s_nl_lanes(B2sNlArgs a) {
  extern __shared__ double b2s_sm[];
  const int n = a.g.nx * a.g.ny, n2 = 2 * n;
  const int t = threadIdx.x;
  const int lane = blockIdx.x, b = lane / a.P, p = lane % a.P;
  double* Y0 = b2s_sm;
  double* Y1 = Y0 + n2;
  double* Qm = Y1 + n2;
  double* Qa = Qm + n2;
  double* Qb = Qa + n2;
  const size_t ns = (size_t)a.B * n2;
  const double* Qg = a.Q + (size_t)b * n2;
  double* Qo = a.Qn + (size_t)b * n2;
  const double* u0 = a.u0 + (size_t)b * n2;
  const double* f = a.f + (size_t)b * n2;
  const double* qb = a.ubar + ((size_t)p * a.B + b) * n2;
  double y[PPT][2], acc[PPT][2], cst[PPT][2];
  int ie[PPT], iw[PPT], in[PPT], is[PPT];
  const int node0 = p * a.nsteps;
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    const int i = t + q * B2S_NT;
    if (i < n) {
      b2_nbrs(i, a.g, ie[q], iw[q], in[q], is[q]);
      Qm[i] = qb[i]; Qm[n + i] = qb[n + i];
      Qb[i] = u0[i]; Qb[n + i] = u0[n + i];   // u0 with neighbours, for the constant part of the source
      Qa[i] = Qg[(size_t)node0 * ns + i]; Qa[n + i] = Qg[(size_t)node0 * ns + n + i];
      Y0[i] = 0.0; Y0[n + i] = 0.0;
      y[q][0] = y[q][1] = 0.0;
    }
  }
  __syncthreads();
  // cst = D∇²u0 + J̄_adv·u0 (so that s(t) = cst + θ f + N(Q) − J̄_adv·Q): the full operator on u0
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    const int i = t + q * B2S_NT;
    if (i < n) b2s_jfull(a.g, Qm, Qb, n, i, ie[q], iw[q], in[q], is[q], cst[q][0], cst[q][1]);
  }
  __syncthreads();
  const double h = a.h;
  auto stage = [&](auto mode, const double* Yi, double* Yo, double cw, double ca, double th, bool first, bool last) {
    constexpr int MODE = decltype(mode)::value;
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      const int i = t + q * B2S_NT;
      if (i < n) {
        const int e = ie[q], w = iw[q], nn = in[q], s = is[q];
        // stage state qs (the previous iterate at the stage time) with neighbours
        const double uc = b2s_state<MODE>(Qa, Qb, i), ue = b2s_state<MODE>(Qa, Qb, e), uw = b2s_state<MODE>(Qa, Qb, w);
        const double un = b2s_state<MODE>(Qa, Qb, nn), us = b2s_state<MODE>(Qa, Qb, s);
        const double vc = b2s_state<MODE>(Qa, Qb, n + i), ve = b2s_state<MODE>(Qa, Qb, n + e);
        const double vw = b2s_state<MODE>(Qa, Qb, n + w), vn = b2s_state<MODE>(Qa, Qb, n + nn);
        const double vs = b2s_state<MODE>(Qa, Qb, n + s);
        // N(qs)
        const double Nu = -uc * (ue - uw) * a.g.i2hx - vc * (un - us) * a.g.i2hy;
        const double Nv = -uc * (ve - vw) * a.g.i2hx - vc * (vn - vs) * a.g.i2hy;
        // J̄_adv·qs
        const double* Vm = Qm + n;
        const double Ub = Qm[i], Vb = Vm[i];
        const double dUx = (Qm[e] - Qm[w]) * a.g.i2hx, dUy = (Qm[nn] - Qm[s]) * a.g.i2hy;
        const double dVx = (Vm[e] - Vm[w]) * a.g.i2hx, dVy = (Vm[nn] - Vm[s]) * a.g.i2hy;
        const double Ja = -Ub * (ue - uw) * a.g.i2hx - Vb * (un - us) * a.g.i2hy - dUx * uc - dUy * vc;
        const double Jb = -Ub * (ve - vw) * a.g.i2hx - Vb * (vn - vs) * a.g.i2hy - dVx * uc - dVy * vc;
        double ka, kb;
        b2s_jfull(a.g, Qm, Yi, n, i, e, w, nn, s, ka, kb);
        ka += cst[q][0] + th * f[i] + Nu - Ja;
        kb += cst[q][1] + th * f[n + i] + Nv - Jb;
        const double ra = (first ? y[q][0] : acc[q][0]) + ca * ka;
        const double rb = (first ? y[q][1] : acc[q][1]) + ca * kb;
        if (last) {
          y[q][0] = ra; y[q][1] = rb;
          Yo[i] = ra; Yo[n + i] = rb;
        } else {
          acc[q][0] = ra; acc[q][1] = rb;
          Yo[i] = y[q][0] + cw * ka;
          Yo[n + i] = y[q][1] + cw * kb;
        }
      }
    }
  };
  for (int k = 0; k < a.nsteps; ++k) {
    const int node = node0 + k;
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      const int i = t + q * B2S_NT;
      if (i < n) {
        Qb[i] = Qg[(size_t)(node + 1) * ns + i];
        Qb[n + i] = Qg[(size_t)(node + 1) * ns + n + i];
      }
    }
    __syncthreads();
    const double th0 = a.theta[2 * node], th1 = a.theta[2 * node + 1], th2 = a.theta[2 * node + 2];
    stage(IC<0>{}, Y0, Y1, 0.5 * h, h / 6.0, th0, true, false);
    __syncthreads();
    stage(IC<1>{}, Y1, Y0, 0.5 * h, h / 3.0, th1, false, false);
    __syncthreads();
    stage(IC<1>{}, Y0, Y1, h, h / 3.0, th1, false, false);
    __syncthreads();
    stage(IC<2>{}, Y1, Y0, 0.0, h / 6.0, th2, false, true);
    if (k + 1 < a.nsteps) {
#pragma unroll
      for (int q = 0; q < PPT; ++q) {
        const int i = t + q * B2S_NT;
        if (i < n) {
          Qo[(size_t)(node + 1) * ns + i] = u0[i] + y[q][0];
          Qo[(size_t)(node + 1) * ns + n + i] = u0[n + i] + y[q][1];
        }
      }
    }
    __syncthreads();
    double* sw = Qa; Qa = Qb; Qb = sw;
  }
  double* ye = a.yend + (size_t)lane * n2;
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    const int i = t + q * B2S_NT;
    if (i < n) { ye[i] = y[q][0]; ye[n + i] = y[q][1]; }
  }
}

// One planned action exp(span·(D∇² + J̄))·X[c] on chip: `subs` substeps of a degree-K Chebyshev
// series (coefficients be); X: three rotating vectors in shared memory; returns the buffer index
// of the result. Every thread holds the accumulator of its own points.
template <int PPT>
__device__ __forceinline__ int b2s_fwd_action(const B2Geom& g, double* const* X, const double* Qm, int n, int c,
                                              const double* be, int K, int subs, double c0, double d, int sigma,
                                              const int* ie, const int* iw, const int* in, const int* is) {
  const int t = threadIdx.x;
  double acc[PPT][2];
  for (int j = 0; j < subs; ++j) {
    int prv = c, cur = (c + 1) % 3, nxt = (c + 2) % 3;
    {
      const double inv = 1.0 / d;
      const double* Xc = X[c];
      double* Xo = X[cur];
#pragma unroll
      for (int q = 0; q < PPT; ++q) {
        const int i = t + q * B2S_NT;
        if (i < n) {
          double oa, ob;
          b2s_jfull(g, Qm, Xc, n, i, ie[q], iw[q], in[q], is[q], oa, ob);
          const double xa = Xc[i], xb = Xc[n + i];
          const double ua = inv * (oa - c0 * xa), ub = inv * (ob - c0 * xb);
          acc[q][0] = be[0] * xa + be[1] * ua;
          acc[q][1] = be[0] * xb + be[1] * ub;
          Xo[i] = ua; Xo[n + i] = ub;
        }
      }
      __syncthreads();
    }
    const double two = 2.0 / d, sg = (double)sigma;
    for (int k = 2; k <= K; ++k) {
      const double* Xc = X[cur];
      const double* Xp = X[prv];
      double* Xo = X[nxt];
      const double bek = be[k];
#pragma unroll
      for (int q = 0; q < PPT; ++q) {
        const int i = t + q * B2S_NT;
        if (i < n) {
          double oa, ob;
          b2s_jfull(g, Qm, Xc, n, i, ie[q], iw[q], in[q], is[q], oa, ob);
          const double ua = two * (oa - c0 * Xc[i]) + sg * Xp[i];
          const double ub = two * (ob - c0 * Xc[n + i]) + sg * Xp[n + i];
          acc[q][0] += bek * ua; acc[q][1] += bek * ub;
          Xo[i] = ua; Xo[n + i] = ub;
        }
      }
      __syncthreads();
      const int tmp = prv; prv = cur; cur = nxt; nxt = tmp;
    }
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      const int i = t + q * B2S_NT;
      if (i < n) { X[nxt][i] = acc[q][0]; X[nxt][n + i] = acc[q][1]; }
    }
    c = nxt;
    __syncthreads();
  }
  return c;
}

template <int PPT>
__global__ void __launch_bounds__(B2S_NT) k_b2s_nl_carry(B2sNlArgs a) {
  extern __shared__ double b2s_sm[];
  const int n = a.g.nx * a.g.ny, n2 = 2 * n;
  const int t = threadIdx.x;
  const size_t b = blockIdx.x;
  double* X[3] = {b2s_sm, b2s_sm + n2, b2s_sm + 2 * n2};
  double* Qm = b2s_sm + 3 * n2;
  int ie[PPT], iw[PPT], in[PPT], is[PPT];
  const size_t ns = (size_t)a.B * n2;
  int c = 0;
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    const int i = t + q * B2S_NT;
    if (i < n) {
      b2_nbrs(i, a.g, ie[q], iw[q], in[q], is[q]);
      a.Dc[b * n2 + i] = 0.0; a.Dc[b * n2 + n + i] = 0.0;   // D_0 = 0
    }
  }
  for (int p = 0; p < a.P; ++p) {
    const double* ye = a.yend + (b * a.P + p) * n2;
    if (p > 0) {
      const double* qb = a.ubar + ((size_t)p * a.B + b) * n2;
#pragma unroll
      for (int q = 0; q < PPT; ++q) {
        const int i = t + q * B2S_NT;
        if (i < n) { Qm[i] = qb[i]; Qm[n + i] = qb[n + i]; }
      }
      __syncthreads();
      c = b2s_fwd_action<PPT>(a.g, X, Qm, n, c, a.coef, a.Ks, a.subs_s, a.c0_s, a.d_s, a.sig_s, ie, iw, in, is);
    }
    double* Dn = a.Dc + (size_t)(p + 1) * ns + b * n2;
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      const int i = t + q * B2S_NT;
      if (i < n) {
        const double va = (p > 0 ? X[c][i] : 0.0) + ye[i], vb = (p > 0 ? X[c][n + i] : 0.0) + ye[n + i];
        X[c][i] = va; X[c][n + i] = vb;
        Dn[i] = va; Dn[n + i] = vb;
      }
    }
    __syncthreads();
  }
}

template <int PPT>
__global__ void __launch_bounds__(B2S_NT) k_b2s_nl_hom(B2sNlArgs a) {
  extern __shared__ double b2s_sm[];
  const int n = a.g.nx * a.g.ny, n2 = 2 * n;
  const int t = threadIdx.x;
  const int lane = blockIdx.x, b = lane / a.P, p = lane % a.P;
  double* X[3] = {b2s_sm, b2s_sm + n2, b2s_sm + 2 * n2};
  double* Qm = b2s_sm + 3 * n2;
  int ie[PPT], iw[PPT], in[PPT], is[PPT];
  const size_t ns = (size_t)a.B * n2;
  const double* u0 = a.u0 + (size_t)b * n2;
  const double* Dp = a.Dc + (size_t)p * ns + (size_t)b * n2;
  const double* qb = a.ubar + ((size_t)p * a.B + b) * n2;
  double* Qo = a.Qn + (size_t)b * n2;
  const int node0 = p * a.nsteps;
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    const int i = t + q * B2S_NT;
    if (i < n) {
      b2_nbrs(i, a.g, ie[q], iw[q], in[q], is[q]);
      Qm[i] = qb[i]; Qm[n + i] = qb[n + i];
      X[0][i] = Dp[i]; X[0][n + i] = Dp[n + i];
      Qo[(size_t)node0 * ns + i] = u0[i] + Dp[i];
      Qo[(size_t)node0 * ns + n + i] = u0[n + i] + Dp[n + i];
      if (p == a.P - 1) {   // the last node: u0 + D_P
        const double* DP = a.Dc + (size_t)a.P * ns + (size_t)b * n2;
        Qo[(size_t)a.S * ns + i] = u0[i] + DP[i];
        Qo[(size_t)a.S * ns + n + i] = u0[n + i] + DP[n + i];
      }
    }
  }
  __syncthreads();
  if (p == 0) return;   // D_0 = 0: nothing to propagate
  int c = 0;
  const double* be = a.coef + (a.Ks + 1);
  for (int k = 1; k < a.nsteps; ++k) {
    c = b2s_fwd_action<PPT>(a.g, X, Qm, n, c, be, a.Kh, a.subs_h, a.c0_h, a.d_h, a.sig_h, ie, iw, in, is);
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      const int i = t + q * B2S_NT;
      if (i < n) {
        Qo[(size_t)(node0 + k) * ns + i] += X[c][i];
        Qo[(size_t)(node0 + k) * ns + n + i] += X[c][n + i];
      }
    }
  }
}

// per (member, slice): ‖Qn − Q‖ / ‖Q‖ over the slice's nodes (both ends included), nonlinear.py:44-66
__global__ void __launch_bounds__(256) k_b2s_nl_err(B2sNlArgs a) {
  __shared__ double red[8];
  const int n2 = 2 * a.g.nx * a.g.ny;
  const int lane = blockIdx.x, b = lane / a.P, p = lane % a.P;
  const size_t ns = (size_t)a.B * n2;
  const size_t total = (size_t)(a.nsteps + 1) * n2;
  double num = 0.0, den = 0.0;
  for (size_t m = threadIdx.x; m < total; m += blockDim.x) {
    const size_t j = m / n2, i = m - j * n2;
    const size_t off = (size_t)(p * a.nsteps + j) * ns + (size_t)b * n2 + i;
    const double qo = a.Q[off], d = a.Qn[off] - qo;
    num += d * d;
    den += qo * qo;
  }
  const double rn = block_sum<256>(num, red);
  const double rd = block_sum<256>(den, red);
  if (threadIdx.x == 0) a.err[lane] = rd > 0.0 ? sqrt(rn) / sqrt(rd) : sqrt(rn);
}


// ---------------------------------------------------------------------------------------------
// Algorithm 2 with the fields in HBM (grids above B2S_MAX_N points): one launch per RK4 stage /
// Chebyshev term over (points, lanes), the same operation sequence as the on-chip kernels.
// ---------------------------------------------------------------------------------------------

// forward operator (D∇² + ∂N/∂q at q̄)·x at point i, q̄ and x in global memory
__device__ __forceinline__ void b2_jfull(const B2Geom& g, const double* Qm, const double* X, int n, int i, int e, int w,
                                         int nn, int s, double& oa, double& ob) {
  b2s_jfull(g, Qm, X, n, i, e, w, nn, s, oa, ob);  // plain pointer arithmetic: any address space
}

struct B2NlStageArgs {
  const double* yin;    // L × 2n stage input (neighbours read)
  double* y;            // L × 2n: y_k (base); stage 4 writes y_{k+1}
  const double* accin;  // L × 2n (stage 1: y)
  double* accout;       // L × 2n (stage 4: y)
  double* yout;         // L × 2n or null
  const double* cst;    // L × 2n: (D∇² + J̄_p)·u0
  const double* Q;      // (S+1) × B × 2n iterate
  double* Qn;           // next iterate (stage 4: node + 1 ← u0 + y_{k+1} when write_node)
  const double* ubar;   // P × B × 2n
  const double* u0;     // B × 2n
  const double* f;      // B × 2n
  const double* theta;
  double wa, wb, cw, ca;
  int tsel;             // θ at node (0), node + ½ (1), node + 1 (2)
  int k, nsteps, P, B, write_node;
  B2Geom g;
};

__global__ void __launch_bounds__(256) k_b2_nl_stage(B2NlStageArgs a) {
  const int n = a.g.nx * a.g.ny;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int lane = blockIdx.y, b = lane / a.P, p = lane % a.P;
  const size_t n2 = 2 * (size_t)n, ns = (size_t)a.B * n2;
  const int node = p * a.nsteps + a.k;
  const double* qa = a.Q + (size_t)node * ns + (size_t)b * n2;
  const double* qc = a.Q + (size_t)(node + 1) * ns + (size_t)b * n2;
  const double* Qm = a.ubar + ((size_t)p * a.B + b) * n2;
  int e, w, nn, s;
  b2_nbrs(i, a.g, e, w, nn, s);
  auto st = [&](size_t k) { return a.wa * qa[k] + a.wb * qc[k]; };
  const double uc = st(i), ue = st(e), uw = st(w), un = st(nn), us = st(s);
  const double vc = st(n + i), ve = st(n + e), vw = st(n + w), vn = st(n + nn), vs = st(n + s);
  const double Nu = -uc * (ue - uw) * a.g.i2hx - vc * (un - us) * a.g.i2hy;
  const double Nv = -uc * (ve - vw) * a.g.i2hx - vc * (vn - vs) * a.g.i2hy;
  const double* Vm = Qm + n;
  const double Ub = Qm[i], Vb = Vm[i];
  const double dUx = (Qm[e] - Qm[w]) * a.g.i2hx, dUy = (Qm[nn] - Qm[s]) * a.g.i2hy;
  const double dVx = (Vm[e] - Vm[w]) * a.g.i2hx, dVy = (Vm[nn] - Vm[s]) * a.g.i2hy;
  const double Ja = -Ub * (ue - uw) * a.g.i2hx - Vb * (un - us) * a.g.i2hy - dUx * uc - dUy * vc;
  const double Jb = -Ub * (ve - vw) * a.g.i2hx - Vb * (vn - vs) * a.g.i2hy - dVx * uc - dVy * vc;
  const double* Y = a.yin + (size_t)lane * n2;
  double ka, kb;
  b2_jfull(a.g, Qm, Y, n, i, e, w, nn, s, ka, kb);
  const double th = a.theta[2 * node + a.tsel];
  const double* cs = a.cst + (size_t)lane * n2;
  const double* f = a.f + (size_t)b * n2;
  ka += cs[i] + th * f[i] + Nu - Ja;
  kb += cs[n + i] + th * f[n + i] + Nv - Jb;
  const double* base = a.y + (size_t)lane * n2;
  const double* ai = a.accin + (size_t)lane * n2;
  const double ra = ai[i] + a.ca * ka, rb = ai[n + i] + a.ca * kb;
  if (a.yout) {
    double* yo = a.yout + (size_t)lane * n2;
    yo[i] = base[i] + a.cw * ka;
    yo[n + i] = base[n + i] + a.cw * kb;
  }
  double* ao = a.accout + (size_t)lane * n2;
  ao[i] = ra;
  ao[n + i] = rb;
  if (a.write_node) {
    const double* u0 = a.u0 + (size_t)b * n2;
    double* qo = a.Qn + (size_t)(node + 1) * ns + (size_t)b * n2;
    qo[i] = u0[i] + ra;
    qo[n + i] = u0[n + i] + rb;
  }
}

// cst[lane] = (D∇² + J̄_p)·u0, y[lane] = 0
__global__ void __launch_bounds__(256) k_b2_nl_prepare(double* cst, double* y, const double* ubar, const double* u0,
                                                       int P, int B, B2Geom g) {
  const int n = g.nx * g.ny;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int lane = blockIdx.y, b = lane / P, p = lane % P;
  const size_t n2 = 2 * (size_t)n;
  int e, w, nn, s;
  b2_nbrs(i, g, e, w, nn, s);
  double oa, ob;
  b2_jfull(g, ubar + ((size_t)p * B + b) * n2, u0 + (size_t)b * n2, n, i, e, w, nn, s, oa, ob);
  cst[(size_t)lane * n2 + i] = oa;
  cst[(size_t)lane * n2 + n + i] = ob;
  y[(size_t)lane * n2 + i] = 0.0;
  y[(size_t)lane * n2 + n + i] = 0.0;
}

// one Chebyshev term of exp(τ(D∇² + J̄))·x over `rows` vectors; row r uses q̄ of slice
// (pfix ≥ 0 ? pfix : r mod P) and member (pfix ≥ 0 ? r : r / P); rows with skip0 and slice 0 idle
struct B2FwdTermArgs {
  const double* x; const double* prev; double* out; double* acc;
  const double* ubar;
  double alpha, c0, sg, be0, bek;
  int first, P, B, pfix, skip0;
  B2Geom g;
};

__global__ void __launch_bounds__(256) k_b2_fwd_term(B2FwdTermArgs a) {
  const int n = a.g.nx * a.g.ny;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int r = blockIdx.y;
  const int p = a.pfix >= 0 ? a.pfix : r % a.P, b = a.pfix >= 0 ? r : r / a.P;
  if (a.skip0 && p == 0) return;
  const size_t n2 = 2 * (size_t)n, off = (size_t)r * n2;
  int e, w, nn, s;
  b2_nbrs(i, a.g, e, w, nn, s);
  const double* X = a.x + off;
  double oa, ob;
  b2_jfull(a.g, a.ubar + ((size_t)p * a.B + b) * n2, X, n, i, e, w, nn, s, oa, ob);
  const double xa = X[i], xb = X[n + i];
  double ua = a.alpha * (oa - a.c0 * xa), ub = a.alpha * (ob - a.c0 * xb);
  double* acc = a.acc + off;
  if (a.first) {
    acc[i] = a.be0 * xa + a.bek * ua;
    acc[n + i] = a.be0 * xb + a.bek * ub;
  } else {
    const double* P_ = a.prev + off;
    ua += a.sg * P_[i];
    ub += a.sg * P_[n + i];
    acc[i] += a.bek * ua;
    acc[n + i] += a.bek * ub;
  }
  double* o = a.out + off;
  o[i] = ua;
  o[n + i] = ub;
}

// D_{p+1}[b] = (p > 0 ? C[b] : 0) + yend[b·P + p]; C ← D_{p+1}
__global__ void k_b2_nl_carry_add(double* C, double* Dnext, const double* yend, int P, int p, size_t n2) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n2) return;
  const size_t b = blockIdx.y;
  const double v = (p > 0 ? C[b * n2 + i] : 0.0) + yend[(b * P + p) * n2 + i];
  C[b * n2 + i] = v;
  Dnext[b * n2 + i] = v;
}

// H[lane] = D_p[b]; Qn[p·ns][b] = u0 + D_p; lane P−1 also Qn[S][b] = u0 + D_P
__global__ void k_b2_nl_hom_init(double* H, double* Qn, const double* Dc, const double* u0, int P, int B, int nsteps,
                                 int S, size_t n2) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n2) return;
  const int lane = blockIdx.y, b = lane / P, p = lane % P;
  const size_t ns = (size_t)B * n2;
  const double d = Dc[(size_t)p * ns + (size_t)b * n2 + i], u = u0[(size_t)b * n2 + i];
  H[(size_t)lane * n2 + i] = d;
  Qn[(size_t)(p * nsteps) * ns + (size_t)b * n2 + i] = u + d;
  if (p == P - 1) Qn[(size_t)S * ns + (size_t)b * n2 + i] = u + Dc[(size_t)P * ns + (size_t)b * n2 + i];
}

// Qn[p·ns + k][b] += H[lane] (lanes of slice 0 idle: D_0 = 0)
__global__ void k_b2_nl_hom_add(double* Qn, const double* H, int P, int B, int nsteps, int k, size_t n2) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n2) return;
  const int lane = blockIdx.y, b = lane / P, p = lane % P;
  if (p == 0) return;
  Qn[(size_t)(p * nsteps + k) * (size_t)B * n2 + (size_t)b * n2 + i] += H[(size_t)lane * n2 + i];
}

}  // namespace px
