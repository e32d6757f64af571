// tracking.cuh — kernels of the linear testbed's tracking objective (the reference's linear loop,
// optimization.py:154-231 with algorithm "linear"): J = (1/T)∫‖u − u_t‖² dt, the adjoint source
// 2(u − u_t) and zero terminal data, ∂L/∂f = (1/T)∫θ(t)·q† dt.
//
//   recording sweep: every slice p marches u' = A u + θ(t)·f from its Paraexp edge state u(T_p)
//                    (all slices × batch as lanes, one launch per RK4 stage) and writes the nodes
//                    into the trajectory (S+1, B, n) — the solution inside slice p, by linearity the
//                    reference's lane plus the propagated incoming state (paraexp.py:202-218);
//   cost:            trapezoid of ‖u − u_t‖² over the nodes, per member (deterministic partials);
//   adjoint lanes:   a' = Aᵀa + 2(u − u_t) from a = 0 at T_{p+1} in reflected time, trajectory and
//                    target linearly interpolated at the half steps, with the θ-weighted
//                    RK4-consistent ∫ z += h/6[θa·a + 2θm(Y2 + Y3) + θb·Y4] (paraexp.py:298-326).
// The slice ends then go through the ordinary adjoint carries (sweeps.cu) with pacc = Σ z_p.
// Included by tracking.cu only.
#pragma once
#include "common.cuh"

namespace px {

struct TrackArgs {
  Stencil5 st;            // A (direct) or Aᵀ (adjoint)
  int nx, ny;
  size_t n;
  int P, ns;              // slices (lanes per member) and RK4 steps per slice
  int B;
  double h;               // RK4 step
  const double* theta;    // θ(j·h/2), j = 0 … 2S (S = P·ns)
  const double* f;        // B × n forcing field (direct)
  const double* y;        // lanes × n: the lane state at the step start (direct) / a (adjoint)
  const double* x;        // lanes × n: the stage argument (stages 1–3)
  double* xo;             // lanes × n: the next stage argument (stages 0–2)
  double* acc;            // lanes × n: k1 + 2k2 + 2k3
  double* ynew;           // lanes × n: the state after the step (stage 3; may alias y)
  double* traj;           // (S+1) × B × n: trajectory (written by the direct, read by the adjoint)
  const double* target;   // (S+1) × n or (S+1) × B × n
  int target_bs;          // 0 (shared target) or 1 (per member)
  double* z;              // lanes × n: θ-weighted ∫ (adjoint)
};

__device__ __forceinline__ void trk_lane(int lane, int P, int& b, int& p) {
  b = lane / P;
  p = lane - b * P;
}

// One stage of one step of every recording lane. Lane (b, p), step k of its slice: node j0 =
// p·ns + k; stage s evaluates k_{s+1} = A·x_s + θ(t_s)·f at t_s = j0·h + {0, h/2, h/2, h}.
template <int DIM>
__global__ void __launch_bounds__(256) k_trk_direct_stage(TrackArgs a, int stage, int k) {
  const int lane = blockIdx.y;
  int b, p;
  trk_lane(lane, a.P, b, p);
  const size_t base = (size_t)lane * a.n;
  const int j0 = p * a.ns + k;
  const int tj = stage == 0 ? 2 * j0 : (stage == 3 ? 2 * j0 + 2 : 2 * j0 + 1);
  const double th = a.theta[tj];
  const double* xin = (stage == 0 ? a.y : a.x) + base;
  const double* fb = a.f + (size_t)b * a.n;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += (size_t)gridDim.x * blockDim.x) {
    const int xx = (int)(i % a.nx), yy = (int)(i / a.nx);
    const double kv = stencil_at<DIM>(xin, a.st, xx, yy, a.nx, a.ny) + th * fb[i];
    const double yv = a.y[base + i];
    if (stage == 0) {
      a.acc[base + i] = kv;
      a.xo[base + i] = yv + (0.5 * a.h) * kv;
    } else if (stage < 3) {
      a.acc[base + i] += 2.0 * kv;
      a.xo[base + i] = yv + (stage == 1 ? 0.5 * a.h : a.h) * kv;
    } else {
      const double yn = yv + (a.h / 6.0) * (a.acc[base + i] + kv);
      a.ynew[base + i] = yn;
      a.traj[((size_t)(j0 + 1) * a.B + b) * a.n + i] = yn;
    }
  }
}

// One stage of one reflected-time step of every adjoint lane. Lane (b, p), step i of its slice
// from the top node top = (p+1)·ns − i: sources 2(u − u_t) at top, at the half step (the mean
// of the two nodes) and at top − 1; the ∫ gathers θa·a (stage 0) and the stage arguments.
template <int DIM>
__global__ void __launch_bounds__(256) k_trk_adjoint_stage(TrackArgs a, int stage, int step) {
  const int lane = blockIdx.y;
  int b, p;
  trk_lane(lane, a.P, b, p);
  const size_t base = (size_t)lane * a.n;
  const int top = (p + 1) * a.ns - step;
  const double h6 = a.h / 6.0;
  const double tha = a.theta[2 * top], thm = a.theta[2 * top - 1], thb = a.theta[2 * top - 2];
  const double* xin = (stage == 0 ? a.y : a.x) + base;
  const double* ua = a.traj + ((size_t)top * a.B + b) * a.n;
  const double* ub = ua - (size_t)a.B * a.n;
  const size_t tstride = a.target_bs ? (size_t)a.B * a.n : a.n;
  const double* ta = a.target + (size_t)top * tstride + (a.target_bs ? (size_t)b * a.n : 0);
  const double* tb = ta - tstride;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += (size_t)gridDim.x * blockDim.x) {
    const int xx = (int)(i % a.nx), yy = (int)(i / a.nx);
    double src;
    if (stage == 0) src = 2.0 * (ua[i] - ta[i]);
    else if (stage == 3) src = 2.0 * (ub[i] - tb[i]);
    else src = 2.0 * ((0.5 * ua[i] + 0.5 * ub[i]) - (0.5 * ta[i] + 0.5 * tb[i]));
    const double kv = stencil_at<DIM>(xin, a.st, xx, yy, a.nx, a.ny) + src;
    const double yv = a.y[base + i];
    if (stage == 0) {
      const double x2 = yv + (0.5 * a.h) * kv;
      a.acc[base + i] = kv;
      a.xo[base + i] = x2;
      const double z0 = step == 0 ? 0.0 : a.z[base + i];
      a.z[base + i] = z0 + h6 * (tha * yv + 2.0 * thm * x2);
    } else if (stage < 3) {
      const double xn = yv + (stage == 1 ? 0.5 * a.h : a.h) * kv;
      a.acc[base + i] += 2.0 * kv;
      a.xo[base + i] = xn;
      a.z[base + i] += h6 * (stage == 1 ? 2.0 * thm : thb) * xn;
    } else {
      a.ynew[base + i] = yv + h6 * (a.acc[base + i] + kv);
    }
  }
}

// Per-member partial sums of w_j·‖traj_j − target_j‖² over blocks of the flattened (node, point)
// range (trapezoid weights w = ½ at both ends, 1 inside); fixed order for determinism.
__global__ void __launch_bounds__(256) k_trk_cost_partial(double* partial, const double* traj, const double* target,
                                                          int target_bs, size_t n, int S, int B) {
  __shared__ double red[8];
  const int b = blockIdx.y;
  const size_t total = (size_t)(S + 1) * n;
  double acc = 0.0;
  for (size_t m = (size_t)blockIdx.x * blockDim.x + threadIdx.x; m < total; m += (size_t)gridDim.x * blockDim.x) {
    const size_t j = m / n, i = m - j * n;
    const double u = traj[(j * B + b) * n + i];
    const double t = target[(target_bs ? j * B + b : j) * n + i];
    const double d = u - t;
    acc += (j == 0 || j == (size_t)S ? 0.5 : 1.0) * d * d;
  }
  const double r = block_sum<256>(acc, red);
  if (threadIdx.x == 0) partial[(size_t)b * gridDim.x + blockIdx.x] = r;
}

// Lane state initialisation: lane (b, p) ← u(T_p) of member b (boundary states (B, P+1, n)),
// trajectory node 0 ← u0 for every member.
__global__ void k_trk_init(double* y, const double* ubnd, double* traj, const double* u0, size_t n, int P, int B) {
  const int lane = blockIdx.y;
  int b, p;
  trk_lane(lane, P, b, p);
  const double* src = ubnd + ((size_t)b * (P + 1) + p) * n;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    y[(size_t)lane * n + i] = src[i];
    if (p == 0) traj[(size_t)b * n + i] = u0[i];
  }
}

}  // namespace px
