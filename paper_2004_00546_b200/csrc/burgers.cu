// burgers.cu — config 3 (Burgers): the serial direct sweep keeping the trajectory in HBM
// (hybrid.py:185-191), the Paraexp adjoint with exact Jᵀ(u(t)) in the slices and frozen
// J(ū_p)ᵀ carries (paraexp.py:329-353, systems.py:64-97), and Algorithm 2's iterative
// direct (nonlinear.py:69-194) — burgers.cuh, burgers_iter.cuh.
#include <algorithm>
#include <cmath>

#include "internal.h"
#include "burgers.cuh"
#include "burgers_iter.cuh"
#include "hybrid.cuh"

namespace pxi {

int burgers_direct(Handle* h, cudaStream_t s) {
  px::BurgersDirectArgs a{};
  a.u0 = h->u0; a.ctrl = h->ctrl; a.tx = h->tx; a.ix = h->ix; a.K = h->K;
  a.traj = h->traj; a.ubar = h->ubar; a.UT = h->UT;
  a.bpart = h->bpart; a.bounds = h->bounds; a.bounds_blocks = h->bounds_blocks;
  a.D = h->d.D; a.hx = h->d.hx; a.h = (h->d.T / h->d.P) / h->d.nsteps;
  a.nx = h->d.nx; a.B = h->B; a.P = h->d.P; a.nsteps = h->d.nsteps;
  const int rc = px::burgers_direct(a, s, &h->stats, h->var.burgers_cluster != 0);
  if (rc != PX_OK)
    return fail(h, rc, "Burgers direct sweep failed: " + std::string(cudaGetErrorString(cudaGetLastError())));
  return PX_OK;
}

int burgers_adjoint(Handle* h, cudaStream_t s) {
  const Plan& pl = h->plans[PX_PLAN_FROZEN];
  const bool span = h->adjoint_mode == PX_ADJOINT_FROZEN_SPAN;
  if (span && (h->d.p_begin != 0 || h->d.p_end != h->d.P))
    return fail(h, PX_ERR_ARG, "the frozen-span adjoint runs on one rank (it is one sequential chain)");
  // one slice and no earlier ranks (the serial loop): no homogeneous carry, no plan needed
  const bool no_carry = h->Pl == 1 && h->d.p_begin == 0 && !span;
  if ((!pl.set || pl.krylov) && !no_carry) return fail(h, PX_ERR_STATE, "frozen-operator plan not set");
  const bool use_plan = pl.set && !pl.krylov;
  px::BurgersAdjointArgs a{};
  a.traj = h->traj; a.ubar = h->ubar; a.QT = h->QT;
  a.W0 = h->Y0; a.W1 = h->Y1; a.Z = h->Z;
  a.G = h->G; a.QDAG0 = h->QDAG0;
  a.Wk[0] = h->Wk[0]; a.Wk[1] = h->Wk[1]; a.Wk[2] = h->Wk[2];
  a.ACC[0] = h->ACC[0]; a.ACC[1] = h->ACC[1];
  a.D = h->d.D; a.hx = h->d.hx; a.h = (h->d.T / h->d.P) / h->d.nsteps;
  a.nx = h->d.nx; a.B = h->B; a.P = h->d.P; a.nsteps = h->d.nsteps;
  a.p_begin = h->d.p_begin; a.p_end = h->d.p_end;
  a.terminal_span = span ? 1 : 0;
  if (use_plan) {
    a.substeps = pl.substeps; a.degree = pl.degree; a.center = pl.center; a.scale = pl.scale;
    a.sigma = pl.sigma; a.be = pl.be.data(); a.bp = pl.bp.data();
  } else {
    a.substeps = 0; a.degree = 0; a.center = 0.0; a.scale = 1.0; a.sigma = 1;
    a.be = a.bp = nullptr;
  }
  const int rc = px::burgers_adjoint(a, s, &h->stats, &h->wend, h->var.burgers_cluster != 0);
  if (rc != PX_OK) return fail(h, rc, "Burgers adjoint sweep failed");
  return PX_OK;
}

int nl_init(Handle* h, cudaStream_t s) {
  const size_t nodes = (size_t)h->d.P * h->d.nsteps + 1;
  px::k_nl_init<<<1024, 256, 0, s>>>(h->traj, h->u0, nodes, h->B, (int)h->n);
  PX_CHECK_LAUNCH(h);
  return PX_OK;
}

// slice means ū_p of the stored trajectory and the frozen-operator FOV union (3 doubles)
int nl_means_bounds(Handle* h, cudaStream_t s) {
  const size_t total = (size_t)h->d.P * h->B * h->n;
  px::k_slice_means<<<(unsigned)std::min<size_t>((total + 255) / 256, 4096), 256, 0, s>>>(
      h->ubar, h->traj, h->d.P, h->d.nsteps, h->B, (int)h->n);
  PX_CHECK_LAUNCH(h);
  px::k_frozen_bounds<<<h->bounds_blocks, 256, 0, s>>>(h->bpart, h->ubar, total, (int)h->n, h->d.hx, h->d.D);
  PX_CHECK_LAUNCH(h);
  px::k_frozen_bounds_final<<<1, 256, 0, s>>>(h->bounds, h->bpart, h->bounds_blocks);
  PX_CHECK_LAUNCH(h);
  return PX_OK;
}

px::NlPlan nl_plan(const Plan& pl) {
  px::NlPlan p{};
  p.be = pl.dcoef;
  p.degree = pl.degree;
  p.substeps = pl.substeps;
  p.sigma = pl.sigma;
  p.c0 = pl.center;
  p.d = pl.scale;
  return p;
}

// One Jacobian-augmented sweep of Algorithm 2; *err_max = max over slices of the relative
// L2 change (NaN when any slice's change is NaN: `nonlinear.py:137-146` stops on it).
int nl_sweep(Handle* h, double* err_max, cudaStream_t s) {
  const Plan& ps = h->plans[PX_PLAN_NL_SLICE];
  const Plan& pt = h->plans[PX_PLAN_NL_STEP];
  if (!ps.set || !pt.set || ps.krylov || pt.krylov) return fail(h, PX_ERR_STATE, "iterative-direct plans not set");
  px::NlArgs a{};
  a.Q = h->traj; a.Qn = h->traj_b; a.ubar = h->ubar; a.u0 = h->u0; a.ctrl = h->ctrl;
  a.tx = h->tx; a.ix = h->ix; a.K = h->K;
  a.yend = h->Y0; a.Dc = h->Dc; a.err = h->nl_err;
  a.slice = nl_plan(ps); a.step = nl_plan(pt);
  a.D = h->d.D; a.hx = h->d.hx; a.h = (h->d.T / h->d.P) / h->d.nsteps;
  a.nx = h->d.nx; a.B = h->B; a.P = h->d.P; a.nsteps = h->d.nsteps;
  const int ppt = (a.nx + px::BURGERS_NT - 1) / px::BURGERS_NT;
  const unsigned lanes = (unsigned)(h->B * h->d.P);
  const size_t sm3 = 3 * (size_t)a.nx * sizeof(double), sm2 = 2 * (size_t)a.nx * sizeof(double);
#define PX_NL(PP)                                                                 \
  do {                                                                            \
    PX_TRY(smem_attr(h, (const void*)px::k_nl_inhom<PP>, sm3));                   \
    px::k_nl_inhom<PP><<<lanes, px::BURGERS_NT, sm3, s>>>(a);                     \
    PX_CHECK_LAUNCH(h);                                                           \
    PX_TRY(smem_attr(h, (const void*)px::k_nl_scan<PP>, sm2));                    \
    px::k_nl_scan<PP><<<h->B, px::BURGERS_NT, sm2, s>>>(a);                       \
    PX_CHECK_LAUNCH(h);                                                           \
    PX_TRY(smem_attr(h, (const void*)px::k_nl_record<PP>, sm2));                  \
    px::k_nl_record<PP><<<lanes, px::BURGERS_NT, sm2, s>>>(a);                    \
    PX_CHECK_LAUNCH(h);                                                           \
  } while (0)
  if (ppt <= 1) PX_NL(1);
  else if (ppt <= 2) PX_NL(2);
  else if (ppt <= 4) PX_NL(4);
  else PX_NL(8);
#undef PX_NL
  px::k_nl_error<<<lanes, 256, 0, s>>>(a);
  PX_CHECK_LAUNCH(h);
  h->nl_err_host.resize(lanes);
  PX_CUDA(h, cudaMemcpyAsync(h->nl_err_host.data(), h->nl_err, sizeof(double) * lanes, cudaMemcpyDeviceToHost, s));
  PX_CUDA(h, cudaStreamSynchronize(s));
  double mx = 0.0;
  for (double e : h->nl_err_host) {
    if (!(e == e)) {  // std::max would drop a NaN
      mx = NAN;
      break;
    }
    mx = std::max(mx, e);
  }
  *err_max = mx;
  std::swap(h->traj, h->traj_b);
  // stats: one inhomogeneous RK4 sweep + the carry and the node recordings
  const double n = (double)h->n;
  h->stats.rk4_lane_steps += (uint64_t)lanes * h->d.nsteps;
  h->stats.rk4_bytes += 32.0 * n * lanes * h->d.nsteps;
  const uint64_t terms = (uint64_t)h->B * ((h->d.P - 1) * ps.substeps * ps.degree +
                                            (uint64_t)(h->d.P - 1) * (h->d.nsteps - 1) * pt.substeps * pt.degree);
  h->stats.exp_terms += terms;
  h->stats.exp_bytes += 40.0 * n * terms;
  h->stats.algorithmic_bytes += 32.0 * n * lanes * h->d.nsteps + 40.0 * n * terms;
  if (!std::isfinite(mx)) return fail(h, PX_ERR_NONFINITE, "non-finite iterate in the nonlinear sweep");
  return PX_OK;
}

}  // namespace pxi

// ---- the reference's hybrid with its tracking objective (hybrid.cuh; hybrid.cu drives it) ----
namespace pxi {

namespace {
template <int PPT>
cudaError_t hyb_direct_t(const px::HybArgs& a, cudaStream_t s) {
  px::k_hyb_direct<PPT><<<a.B, px::HYB_NT, 0, s>>>(a);
  return cudaGetLastError();
}
template <int PPT>
cudaError_t hyb_lanes_t(const px::HybArgs& a, size_t smem, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute((const void*)px::k_hyb_lanes<PPT>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  px::k_hyb_lanes<PPT><<<a.B * a.P, px::HYB_NT, smem, s>>>(a);
  return cudaGetLastError();
}
template <int PPT>
cudaError_t hyb_scan_t(const px::HybScanArgs& a, cudaStream_t s) {
  px::k_hyb_scan<PPT><<<a.B, px::HYB_NT, 0, s>>>(a);
  return cudaGetLastError();
}
}  // namespace

#define PX_HYB_DISPATCH(PPT_VAR, CALL)   \
  switch (PPT_VAR) {                     \
    case 1: return CALL(1);              \
    case 2: return CALL(2);              \
    case 4: return CALL(4);              \
    case 8: return CALL(8);              \
    case 16: return CALL(16);            \
    case 32: return CALL(32);            \
    default: return cudaErrorInvalidValue; \
  }

cudaError_t hyb_launch_direct(const px::HybArgs& a, int ppt, cudaStream_t s) {
  // the cluster sweep (8 CTAs per member, 64-point ghost zones refreshed every 16 steps) for the
  // larger grids, as the config-3 direct sweep
  constexpr int kCS = 8, kPPT = 4, kG = 64;
  if (a.nx >= 2048 && a.nx % (kCS * kPPT) == 0 && a.nx / kCS >= kG && a.nx / kCS / kPPT + 2 * (kG / kPPT) <= 256) {
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
    return cudaLaunchKernelEx(&cfg, px::k_hyb_direct_cluster<kPPT, kCS, kG>, a);
  }
#define PX_C(P) hyb_direct_t<P>(a, s)
  PX_HYB_DISPATCH(ppt, PX_C)
#undef PX_C
}

int hyb_direct_ctas(int nx, int B) {
  constexpr int kCS = 8, kPPT = 4, kG = 64;
  const bool cl = nx >= 2048 && nx % (kCS * kPPT) == 0 && nx / kCS >= kG && nx / kCS / kPPT + 2 * (kG / kPPT) <= 256;
  return cl ? B * kCS : B;
}

cudaError_t hyb_launch_lanes(const px::HybArgs& a, int ppt, size_t smem, cudaStream_t s) {
#define PX_C(P) hyb_lanes_t<P>(a, smem, s)
  PX_HYB_DISPATCH(ppt, PX_C)
#undef PX_C
}

cudaError_t hyb_launch_scan(const px::HybScanArgs& a, int ppt, cudaStream_t s) {
#define PX_C(P) hyb_scan_t<P>(a, s)
  PX_HYB_DISPATCH(ppt, PX_C)
#undef PX_C
}

cudaError_t hyb_lanes_occupancy(int ppt, size_t smem, int* per_sm) {
#define PX_C(P)                                                                                    \
  (cudaFuncSetAttribute((const void*)px::k_hyb_lanes<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                        (int)smem),                                                                \
   cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, px::k_hyb_lanes<P>, px::HYB_NT, smem))
  PX_HYB_DISPATCH(ppt, PX_C)
#undef PX_C
}
#undef PX_HYB_DISPATCH

cudaError_t hyb_launch_means_bounds(double* ubar, const double* traj, const int* offsets, int P, int B, int n,
                                    double* bpart, int bblocks, double* bounds, double hx, double D,
                                    cudaStream_t s) {
  const size_t total = (size_t)P * B * n;
  px::k_hyb_means<<<(unsigned)std::min<size_t>((total + 255) / 256, 4096), 256, 0, s>>>(ubar, traj, offsets, P,
                                                                                         B, n);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  px::k_frozen_bounds<<<bblocks, 256, 0, s>>>(bpart, ubar, total, n, hx, D);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  px::k_frozen_bounds_final<<<1, 256, 0, s>>>(bounds, bpart, bblocks);
  return cudaGetLastError();
}

}  // namespace pxi
