// burgers_iter.cuh — Algorithm 2 on the GPU: the iterative Jacobian-augmented
// Paraexp direct solve of the Burgers testbed (`nonlinear.py:69-194`), with the
// configs' numerics (fixed-step RK4, planned Chebyshev actions).
//
// One sweep, given the iterate Q (all RK4 nodes) and its trapezoid slice means ū_p:
//   1. k_nl_inhom   (one CTA per member × slice): y' = J(ū_p)y + s(t), y(T_p) = 0,
//      s = D·L u0 + f − Q∘Dx Q + ū_p∘Dx(Q − u0) + (Dx ū_p)∘(Q − u0)
//      (= A·q0 + f + N(Q) − J̄_p(Q − q0), `nonlinear.py:113-116`), Q linearly
//      interpolated at the RK4 stages; writes u0 + y at the slice's interior nodes;
//   2. k_nl_scan    (one CTA per member): D_{p+1} = exp(Δ·J(ū_p))·D_p + y_p(end);
//   3. k_nl_record  (one CTA per member × slice): node p·n_s + k gets
//      + exp(k·h·J(ū_p))·D_p (h-width actions), node p·n_s gets u0 + D_p;
//   4. k_nl_error   : per slice ‖Q_new − Q‖/‖Q‖ over its nodes (max-reduced on the host,
//      `nonlinear.py:48-66,137-143`).
// All fields live on chip per CTA (n ≤ 8192), as in burgers.cuh.
#pragma once
#include <cuda_runtime.h>

#include "burgers.cuh"
#include "common.cuh"

namespace px {

struct NlPlan {
  const double* be;  // device, degree+1
  int degree, substeps, sigma;
  double c0, d;
};

struct NlArgs {
  const double* Q;     // iterate, (S+1) × B × n
  double* Qn;          // next iterate
  const double* ubar;  // P × B × n (means of Q)
  const double* u0;    // n
  const double* ctrl;  // B × K
  const double* tx;
  const int* ix;
  int K;
  double* yend;        // B·P lanes × n
  double* Dc;          // (P+1) × B × n carries
  double* err;         // B × P
  NlPlan slice, step;
  double D, hx, h;
  int nx, B, P, nsteps;
};

// J(u)·y = D·L y − u∘Dx y − (Dx u)∘y at i
__device__ __forceinline__ double j_at(const double* su, const double* sy, int i, int n, double inv2h,
                                       double Dih2) {
  const int ip = (i + 1 == n) ? 0 : i + 1, im = (i == 0) ? n - 1 : i - 1;
  const double yc = sy[i], yp = sy[ip], ym = sy[im];
  const double dxy = (yp - ym) * inv2h;
  const double dxu = (su[ip] - su[im]) * inv2h;
  return (yp - 2.0 * yc + ym) * Dih2 - su[i] * dxy - dxu * yc;
}

template <int PPT>
__global__ void __launch_bounds__(BURGERS_NT) k_nl_inhom(NlArgs a) {
  extern __shared__ double sm[];
  const int n = a.nx;
  double* s_u = sm;        // ū_p
  double* s_y = sm + n;    // stage argument
  double* s_q = sm + 2 * n;  // iterate at the stage time
  const int lane = blockIdx.x;
  const int b = lane / a.P, p = lane - b * a.P;
  const double inv2h = 1.0 / (2.0 * a.hx), Dih2 = a.D / (a.hx * a.hx);
  const double h = a.h, hh = 0.5 * a.h, h6 = a.h / 6.0;
  const size_t ns = (size_t)a.B * n;  // node stride
  const double* ub = a.ubar + ((size_t)p * a.B + b) * n;
  const double* c = a.ctrl + (size_t)b * a.K;
  double u0v[PPT], c0v[PPT], y[PPT], acc[PPT], Y[PPT];
#pragma unroll
  for (int t = 0; t < PPT; ++t) {
    const int i = threadIdx.x + t * BURGERS_NT;
    y[t] = 0.0;
    u0v[t] = c0v[t] = 0.0;
    if (i < n) {
      s_u[i] = ub[i];
      s_y[i] = a.u0[i];
    }
  }
  __syncthreads();
#pragma unroll
  for (int t = 0; t < PPT; ++t) {
    const int i = threadIdx.x + t * BURGERS_NT;
    if (i < n) {
      double fv = 0.0;
      for (int k = 0; k < a.K; ++k) fv += c[k] * a.tx[(size_t)a.ix[k] * n + i];
      const int ip = (i + 1 == n) ? 0 : i + 1, im = (i == 0) ? n - 1 : i - 1;
      u0v[t] = s_y[i];
      c0v[t] = (s_y[ip] - 2.0 * s_y[i] + s_y[im]) * Dih2 + fv;  // D·L u0 + f
    }
  }
  __syncthreads();
  // s(q) at i, with q's neighbours in s_q
  // s(q) = c0 − q∘Dx q + ū∘Dx q + (Dx ū)∘(q − u0), with c0 = D·L u0 + f − ū∘Dx u0
  auto src = [&](int t, int i) -> double {
    const int ip = (i + 1 == n) ? 0 : i + 1, im = (i == 0) ? n - 1 : i - 1;
    const double q = s_q[i];
    const double dxq = (s_q[ip] - s_q[im]) * inv2h;
    const double dxu = (s_u[ip] - s_u[im]) * inv2h;
    return c0v[t] - q * dxq + s_u[i] * dxq + dxu * (q - u0v[t]);
  };
  // fold −ū∘Dx u0 into c0
#pragma unroll
  for (int t = 0; t < PPT; ++t) {
    const int i = threadIdx.x + t * BURGERS_NT;
    if (i < n) {
      const int ip = (i + 1 == n) ? 0 : i + 1, im = (i == 0) ? n - 1 : i - 1;
      c0v[t] -= s_u[i] * ((s_y[ip] - s_y[im]) * inv2h);
    }
  }
  __syncthreads();
  const size_t top = (size_t)p * a.nsteps;
  for (int k = 0; k < a.nsteps; ++k) {
    const double* qa = a.Q + (top + k) * ns + (size_t)b * n;
    const double* qb = a.Q + (top + k + 1) * ns + (size_t)b * n;
    // stage 1 (q at the node t_k)
#pragma unroll
    for (int t = 0; t < PPT; ++t) {
      const int i = threadIdx.x + t * BURGERS_NT;
      if (i < n) {
        s_y[i] = y[t];
        s_q[i] = qa[i];
      }
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < PPT; ++t) {
      const int i = threadIdx.x + t * BURGERS_NT;
      if (i < n) {
        const double kk = j_at(s_u, s_y, i, n, inv2h, Dih2) + src(t, i);
        acc[t] = kk;
        Y[t] = y[t] + hh * kk;
      }
    }
    __syncthreads();
    // stages 2, 3 (q at the midpoint: mean of the two nodes)
#pragma unroll
    for (int t = 0; t < PPT; ++t) {
      const int i = threadIdx.x + t * BURGERS_NT;
      if (i < n) {
        s_y[i] = Y[t];
        s_q[i] = 0.5 * qa[i] + 0.5 * qb[i];
      }
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < PPT; ++t) {
      const int i = threadIdx.x + t * BURGERS_NT;
      if (i < n) {
        const double kk = j_at(s_u, s_y, i, n, inv2h, Dih2) + src(t, i);
        acc[t] += 2.0 * kk;
        Y[t] = y[t] + hh * kk;
      }
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < PPT; ++t) {
      const int i = threadIdx.x + t * BURGERS_NT;
      if (i < n) s_y[i] = Y[t];
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < PPT; ++t) {
      const int i = threadIdx.x + t * BURGERS_NT;
      if (i < n) {
        const double kk = j_at(s_u, s_y, i, n, inv2h, Dih2) + src(t, i);
        acc[t] += 2.0 * kk;
        Y[t] = y[t] + h * kk;
      }
    }
    __syncthreads();
    // stage 4 (q at the node t_{k+1})
#pragma unroll
    for (int t = 0; t < PPT; ++t) {
      const int i = threadIdx.x + t * BURGERS_NT;
      if (i < n) {
        s_y[i] = Y[t];
        s_q[i] = qb[i];
      }
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < PPT; ++t) {
      const int i = threadIdx.x + t * BURGERS_NT;
      if (i < n) {
        const double kk = j_at(s_u, s_y, i, n, inv2h, Dih2) + src(t, i);
        y[t] = y[t] + h6 * (acc[t] + kk);
        if (k + 1 < a.nsteps) a.Qn[(top + k + 1) * ns + (size_t)b * n + i] = u0v[t] + y[t];
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int t = 0; t < PPT; ++t) {
    const int i = threadIdx.x + t * BURGERS_NT;
    if (i < n) a.yend[(size_t)lane * n + i] = y[t];
  }
}

// One planned Chebyshev action exp(τ_s·J(ū))^substeps applied to C (registers),
// ū in s_u, scratch s_c (n doubles); all threads of the CTA participate.
template <int PPT>
__device__ void nl_action(double* C, const NlPlan& pl, const double* s_u, double* s_c, int n, double inv2h,
                          double Dih2) {
  const double tod = 2.0 / pl.d, sg = (double)pl.sigma;
  for (int sub = 0; sub < pl.substeps; ++sub) {
    double up[PPT], uc[PPT], acc[PPT];
#pragma unroll
    for (int t = 0; t < PPT; ++t) {
      const int i = threadIdx.x + t * BURGERS_NT;
      if (i < n) s_c[i] = C[t];
    }
    __syncthreads();
    const double b0 = __ldg(pl.be), b1 = __ldg(pl.be + 1);
#pragma unroll
    for (int t = 0; t < PPT; ++t) {
      const int i = threadIdx.x + t * BURGERS_NT;
      up[t] = C[t];
      uc[t] = 0.0;
      if (i < n) uc[t] = (j_at(s_u, s_c, i, n, inv2h, Dih2) - pl.c0 * C[t]) / pl.d;
      acc[t] = b0 * up[t] + b1 * uc[t];
    }
    for (int k = 2; k <= pl.degree; ++k) {
      __syncthreads();
#pragma unroll
      for (int t = 0; t < PPT; ++t) {
        const int i = threadIdx.x + t * BURGERS_NT;
        if (i < n) s_c[i] = uc[t];
      }
      __syncthreads();
      const double bk = __ldg(pl.be + k);
#pragma unroll
      for (int t = 0; t < PPT; ++t) {
        const int i = threadIdx.x + t * BURGERS_NT;
        double un = 0.0;
        if (i < n) un = tod * (j_at(s_u, s_c, i, n, inv2h, Dih2) - pl.c0 * uc[t]) + sg * up[t];
        up[t] = uc[t];
        uc[t] = un;
        acc[t] += bk * un;
      }
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < PPT; ++t) C[t] = acc[t];
  }
}

template <int PPT>
__global__ void __launch_bounds__(BURGERS_NT) k_nl_scan(NlArgs a) {
  extern __shared__ double sm[];
  const int n = a.nx;
  double* s_u = sm;
  double* s_c = sm + n;
  const int b = blockIdx.x;
  const double inv2h = 1.0 / (2.0 * a.hx), Dih2 = a.D / (a.hx * a.hx);
  const size_t ns = (size_t)a.B * n;
  double C[PPT];
#pragma unroll
  for (int t = 0; t < PPT; ++t) {
    const int i = threadIdx.x + t * BURGERS_NT;
    C[t] = 0.0;
    if (i < n) a.Dc[(size_t)b * n + i] = 0.0;  // D_0
  }
  for (int p = 0; p < a.P; ++p) {
    if (p > 0) {
      const double* ub = a.ubar + ((size_t)p * a.B + b) * n;
#pragma unroll
      for (int t = 0; t < PPT; ++t) {
        const int i = threadIdx.x + t * BURGERS_NT;
        if (i < n) s_u[i] = ub[i];
      }
      nl_action<PPT>(C, a.slice, s_u, s_c, n, inv2h, Dih2);
    }
    const double* ye = a.yend + ((size_t)b * a.P + p) * n;
#pragma unroll
    for (int t = 0; t < PPT; ++t) {
      const int i = threadIdx.x + t * BURGERS_NT;
      if (i < n) {
        C[t] += ye[i];
        a.Dc[(size_t)(p + 1) * ns + (size_t)b * n + i] = C[t];
      }
    }
    __syncthreads();
  }
}

template <int PPT>
__global__ void __launch_bounds__(BURGERS_NT) k_nl_record(NlArgs a) {
  extern __shared__ double sm[];
  const int n = a.nx;
  double* s_u = sm;
  double* s_c = sm + n;
  const int lane = blockIdx.x;
  const int b = lane / a.P, p = lane - b * a.P;
  const double inv2h = 1.0 / (2.0 * a.hx), Dih2 = a.D / (a.hx * a.hx);
  const size_t ns = (size_t)a.B * n;
  const size_t top = (size_t)p * a.nsteps;
  const double* ub = a.ubar + ((size_t)p * a.B + b) * n;
  const double* Dp = a.Dc + (size_t)p * ns + (size_t)b * n;
  double H[PPT], u0v[PPT];
#pragma unroll
  for (int t = 0; t < PPT; ++t) {
    const int i = threadIdx.x + t * BURGERS_NT;
    H[t] = u0v[t] = 0.0;
    if (i < n) {
      s_u[i] = ub[i];
      H[t] = Dp[i];
      u0v[t] = a.u0[i];
      a.Qn[top * ns + (size_t)b * n + i] = u0v[t] + H[t];
      if (p == a.P - 1) a.Qn[(top + a.nsteps) * ns + (size_t)b * n + i] =
          u0v[t] + a.Dc[(size_t)a.P * ns + (size_t)b * n + i];
    }
  }
  __syncthreads();
  if (p == 0) return;  // D_0 = 0: no homogeneous part on the first slice
  for (int k = 1; k < a.nsteps; ++k) {
    nl_action<PPT>(H, a.step, s_u, s_c, n, inv2h, Dih2);
#pragma unroll
    for (int t = 0; t < PPT; ++t) {
      const int i = threadIdx.x + t * BURGERS_NT;
      if (i < n) a.Qn[(top + k) * ns + (size_t)b * n + i] += H[t];
    }
  }
}

// err[b·P + p] = ‖Qn − Q‖ / ‖Q‖ over the nodes p·ns … (p+1)·ns of member b
__global__ void __launch_bounds__(256) k_nl_error(NlArgs a) {
  __shared__ double r1[8], r2[8];
  const int lane = blockIdx.x;
  const int b = lane / a.P, p = lane - b * a.P;
  const int n = a.nx;
  const size_t ns = (size_t)a.B * n;
  double num = 0.0, den = 0.0;
  const int cnt = (a.nsteps + 1) * n;
  for (int idx = threadIdx.x; idx < cnt; idx += 256) {
    const int k = idx / n, i = idx - k * n;
    const size_t o = ((size_t)p * a.nsteps + k) * ns + (size_t)b * n + i;
    const double qn = a.Qn[o], q = a.Q[o];
    num += (qn - q) * (qn - q);
    den += q * q;
  }
  num = block_sum<256>(num, r1);
  den = block_sum<256>(den, r2);
  if (threadIdx.x == 0) {
    const double nn = sqrt(num), dd = sqrt(den);
    a.err[lane] = dd > 0.0 ? nn / dd : nn;
  }
}

// iterate ← u0 at every node
__global__ void k_nl_init(double* Q, const double* u0, size_t nodes, int B, int n) {
  const size_t total = nodes * B * (size_t)n;
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (size_t)gridDim.x * blockDim.x)
    Q[idx] = u0[idx % n];
}

}  // namespace px
