// tracking.cu — the linear testbed with the reference's own objective (its linear loop,
// optimization.py:84-112,154-231): the recording sweep and the tracking cost after the Paraexp
// direct, the adjoint lanes with the source 2(u − u_t); kernels in tracking.cuh. The carries of
// the adjoint are the ordinary ones (sweeps.cu).
#include <algorithm>
#include <cmath>

#include "internal.h"
#include "tracking.cuh"

namespace pxi {

namespace {

double step_h(const Handle* h) { return h->d.T / ((double)h->d.P * h->d.nsteps); }

dim3 lane_grid(const Handle* h) {
  const size_t bx = std::min<size_t>((h->n + 255) / 256, 1024);
  return dim3((unsigned)std::max<size_t>(bx, 1), (unsigned)h->L);
}

px::TrackArgs base_args(const Handle* h, bool adjoint) {
  px::TrackArgs a{};
  a.st = adjoint ? h->AT : h->A;
  a.nx = h->d.nx;
  a.ny = h->dim == 2 ? h->d.ny : 1;
  a.n = h->n;
  a.P = h->Pl;
  a.ns = h->d.nsteps;
  a.B = h->B;
  a.h = step_h(h);
  a.theta = h->trk_theta;
  a.f = h->fctl;
  a.y = h->trk_y;
  a.acc = h->trk_acc;
  a.ynew = h->trk_y;
  a.traj = h->traj;
  a.target = h->trk_target;
  a.target_bs = h->trk_per_member;
  a.z = h->trk_z;
  return a;
}

template <bool ADJ>
int launch_stage(Handle* h, const px::TrackArgs& a, int stage, int step, cudaStream_t s) {
  const dim3 g = lane_grid(h);
  if (ADJ) {
    if (h->dim == 2) px::k_trk_adjoint_stage<2><<<g, 256, 0, s>>>(a, stage, step);
    else px::k_trk_adjoint_stage<1><<<g, 256, 0, s>>>(a, stage, step);
  } else {
    if (h->dim == 2) px::k_trk_direct_stage<2><<<g, 256, 0, s>>>(a, stage, step);
    else px::k_trk_direct_stage<1><<<g, 256, 0, s>>>(a, stage, step);
  }
  PX_CHECK_LAUNCH(h);
  return PX_OK;
}

// the four stage launches of one RK4 step (x ping-pong: X0 → X1 → X0)
template <bool ADJ>
int rk4_step(Handle* h, px::TrackArgs a, int step, cudaStream_t s) {
  for (int stage = 0; stage < 4; ++stage) {
    a.x = stage == 2 ? h->trk_x[1] : h->trk_x[0];
    a.xo = stage == 1 ? h->trk_x[1] : h->trk_x[0];
    PX_TRY(launch_stage<ADJ>(h, a, stage, step, s));
  }
  h->stats.rk4_lane_steps += (uint64_t)h->L;
  return PX_OK;
}

}  // namespace

int tracking_theta(Handle* h) {
  const int S = h->d.P * h->d.nsteps;
  const double hh = 0.5 * step_h(h);
  std::vector<double> th(2 * (size_t)S + 1);
  for (size_t j = 0; j < th.size(); ++j) {
    const double t = j * hh;
    th[j] = h->law[0] + h->law[1] * std::sin(h->law[3] * t) + h->law[2] * std::cos(h->law[3] * t);
  }
  PX_CUDA(h, cudaMemcpy(h->trk_theta, th.data(), sizeof(double) * th.size(), cudaMemcpyHostToDevice));
  return PX_OK;
}

int tracking_set(Handle* h, const double* target, int per_member, int mem, cudaStream_t s) {
  if (!target) {
    h->tracking = false;
    h->graph_valid = false;
    return PX_OK;
  }
  const size_t S = (size_t)h->d.P * h->d.nsteps;
  const size_t Bn = (size_t)h->B * h->n;
  const size_t L = (size_t)h->L;
  if (!h->trk_theta) {
    PX_TRY(dalloc_t(h, &h->trk_theta, 2 * S + 1));
    PX_TRY(dalloc_t(h, &h->trk_target, (S + 1) * Bn));
    if (!h->traj) PX_TRY(dalloc_t(h, &h->traj, (S + 1) * Bn));
    if (!h->UBND) PX_TRY(dalloc_t(h, &h->UBND, Bn * (size_t)(h->d.P + 1)));
    if (!h->fctl) PX_TRY(dalloc_t(h, &h->fctl, Bn));
    PX_TRY(dalloc_t(h, &h->trk_y, L * h->n));
    PX_TRY(dalloc_t(h, &h->trk_acc, L * h->n));
    PX_TRY(dalloc_t(h, &h->trk_z, L * h->n));
    for (auto& p : h->trk_x) PX_TRY(dalloc_t(h, &p, L * h->n));
  }
  const size_t cnt = (S + 1) * (per_member ? Bn : h->n);
  const cudaMemcpyKind kind = mem == PX_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  PX_CUDA(h, cudaMemcpyAsync(h->trk_target, target, sizeof(double) * cnt, kind, s));
  h->trk_per_member = per_member ? 1 : 0;
  PX_TRY(tracking_theta(h));
  h->tracking = true;
  h->graph_valid = false;
  return PX_OK;
}

// After the Paraexp direct (boundary states in UBND): the recording sweep of every slice from its
// edge state into the trajectory, then J = (1/T)·trapezoid of ‖u − u_t‖² on the nodes.
int track_direct(Handle* h, cudaStream_t s) {
  int tm = tbegin(h, PX_PHASE_RK4_DIRECT, s);
  if (!h->has_law)  // the forcing field f (with a law the direct built it already)
    PX_TRY(apply_plus_control(h, h->fctl, h->u0, 0, px::Stencil5{0.0, 0.0, 0.0, 0.0, 0.0}, true, s));
  px::k_trk_init<<<lane_grid(h), 256, 0, s>>>(h->trk_y, h->UBND, h->traj, h->u0, h->n, h->Pl, h->B);
  PX_CHECK_LAUNCH(h);
  const px::TrackArgs a = base_args(h, false);
  for (int k = 0; k < h->d.nsteps; ++k) PX_TRY(rk4_step<false>(h, a, k, s));
  tend(h, tm, s);
  tm = tbegin(h, PX_PHASE_OTHER, s);
  const int S = h->d.P * h->d.nsteps;
  px::k_trk_cost_partial<<<dim3(h->red_blocks, h->B), 256, 0, s>>>(h->partial, h->traj, h->trk_target,
                                                                    h->trk_per_member, h->n, S, h->B);
  PX_CHECK_LAUNCH(h);
  PX_TRY(finalize_sum(h, h->J, h->partial, h->red_blocks, step_h(h) / h->d.T, s));
  tend(h, tm, s);
  return PX_OK;
}

// The adjoint lanes from zero data with the tracking source; the lane ends go to *wend and
// G ← Σ_p z_p (the θ-weighted lane integrals).
int track_adjoint_lanes(Handle* h, const double** wend, cudaStream_t s) {
  const int tm = tbegin(h, PX_PHASE_RK4_ADJOINT, s);
  PX_CUDA(h, cudaMemsetAsync(h->trk_y, 0, sizeof(double) * (size_t)h->L * h->n, s));
  const px::TrackArgs a = base_args(h, true);
  for (int i = 0; i < h->d.nsteps; ++i) PX_TRY(rk4_step<true>(h, a, i, s));
  tend(h, tm, s);
  *wend = h->trk_y;
  return lane_sum_plus(h, h->G, h->trk_z, nullptr, 0.0, true, s);
}

}  // namespace pxi
