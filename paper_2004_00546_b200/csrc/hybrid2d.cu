// hybrid2d.cu — the reference's hybrid loop on its own 2D two-field Burgers testbed
// (px_hybrid_* with desc.ny > 1): problems.py:177-186 (rhs), :316-343 (J(q)ᵀ), :346-366 (slice
// means), hybrid.py:185-237 (serial direct sweep, per-slice adjoint solves, frozen spans),
// optimization.py:84-112 (tracking cost, adjoint source, ∂L/∂f).
//
// State q = (U, V), 2n doubles per member, x fastest, the U block first (problems.py:170-174).
// This unit is the host side (handle, launches, streams, plans); the kernels are hybrid2d.cuh.
// Two kernel families per handle: on chip for nx·ny ≤ 2048 (the serial sweep, every slice's
// adjoint solve and the frozen carry are one kernel each; slices released by progress flags), and
// one launch per RK4 stage / Chebyshev term with the fields in HBM above that, where the overlap
// pipeline is stream-level: when the serial sweep has stored the last node of slice p an event
// releases that slice's adjoint solve on a side stream while the sweep goes on.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "hybrid2d.h"
#include "hybrid2d.cuh"

namespace pxi {

namespace {

int cuda_fail2(Hybrid2D* hy, cudaError_t e, const char* what) {
  return fail(&hy->base, e == cudaErrorMemoryAllocation ? PX_ERR_NOMEM : PX_ERR_CUDA,
              std::string(what) + ": " + cudaGetErrorString(e));
}

#define H2_CUDA(hy, call)                                      \
  do {                                                         \
    cudaError_t _e = (call);                                   \
    if (_e != cudaSuccess) return cuda_fail2((hy), _e, #call); \
  } while (0)

#define H2_LAUNCHED(hy)                                                                       \
  do {                                                                                        \
    cudaError_t _e = cudaGetLastError();                                                      \
    if (_e != cudaSuccess) return cuda_fail2((hy), _e, "kernel launch");                      \
    (hy)->base.stats.kernel_launches++;                                                       \
  } while (0)

px::B2Geom geom(const Hybrid2D* hy) {
  px::B2Geom g;
  g.nx = hy->nx; g.ny = hy->ny;
  g.i2hx = 1.0 / (2.0 * hy->hx); g.i2hy = 1.0 / (2.0 * hy->hy);
  g.dx2 = hy->D / (hy->hx * hy->hx); g.dy2 = hy->D / (hy->hy * hy->hy);
  return g;
}

int copy_in2(Hybrid2D* hy, double* dst, const double* src, size_t count, int mem, cudaStream_t s) {
  H2_CUDA(hy, cudaMemcpyAsync(dst, src, count * sizeof(double),
                              mem == PX_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
  return PX_OK;
}

// the four RK4 stages of local step `step` of slices [p0, p0 + pcount) (all members)
int adjoint_step(Hybrid2D* hy, int step, int p0, int pcount, cudaStream_t s) {
  const int n = hy->nx * hy->ny;
  px::B2AdjArgs a{};
  a.a = hy->la; a.z = hy->lz; a.traj = hy->traj; a.target = hy->target; a.offs = hy->d_offs; a.theta = hy->theta;
  a.step = step; a.p0 = p0; a.pcount = pcount; a.P = hy->P; a.B = hy->B; a.target_b = hy->target_b;
  a.g = geom(hy);
  const double h = hy->h;
  const dim3 grid((unsigned)((n + 255) / 256), (unsigned)(hy->B * pcount));
  // stage 1 at node top
  a.yin = hy->la; a.accin = hy->la; a.accout = hy->lacc; a.yout = hy->ly[0];
  a.wa = 1.0; a.wb = 0.0; a.tsel = 0; a.cw = 0.5 * h; a.ca = h / 6.0; a.cz = h / 6.0;
  px::k_b2_adj_stage<<<grid, 256, 0, s>>>(a);
  H2_LAUNCHED(hy);
  // stages 2 and 3 at the half step (trajectory and target linearly interpolated, timestepping.py:64-75)
  a.yin = hy->ly[0]; a.accin = hy->lacc; a.yout = hy->ly[1];
  a.wa = 0.5; a.wb = 0.5; a.tsel = 1; a.ca = h / 3.0; a.cz = h / 3.0;
  px::k_b2_adj_stage<<<grid, 256, 0, s>>>(a);
  H2_LAUNCHED(hy);
  a.yin = hy->ly[1]; a.yout = hy->ly[0]; a.cw = h;
  px::k_b2_adj_stage<<<grid, 256, 0, s>>>(a);
  H2_LAUNCHED(hy);
  // stage 4 at node top − 1
  a.yin = hy->ly[0]; a.accout = hy->la; a.yout = nullptr;
  a.wa = 0.0; a.wb = 1.0; a.tsel = 2; a.ca = h / 6.0; a.cz = h / 6.0;
  px::k_b2_adj_stage<<<grid, 256, 0, s>>>(a);
  H2_LAUNCHED(hy);
  return PX_OK;
}


template <typename F>
cudaError_t b2s_dispatch(int ppt, F&& f) {
  switch (ppt) {
    case 1: return f(px::IC<1>{});
    case 2: return f(px::IC<2>{});
    default: return f(px::IC<4>{});
  }
}

cudaError_t b2s_launch_direct(const px::B2sDirectArgs& a, int ppt, size_t smem, cudaStream_t s) {
  return b2s_dispatch(ppt, [&](auto pc) {
    constexpr int PPT = decltype(pc)::value;
    cudaError_t e = cudaFuncSetAttribute(px::k_b2s_direct<PPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    px::k_b2s_direct<PPT><<<a.B, px::B2S_NT, smem, s>>>(a);
    return cudaGetLastError();
  });
}

cudaError_t b2s_launch_lanes(const px::B2sLaneArgs& a, int ppt, size_t smem, cudaStream_t s) {
  return b2s_dispatch(ppt, [&](auto pc) {
    constexpr int PPT = decltype(pc)::value;
    cudaError_t e = cudaFuncSetAttribute(px::k_b2s_lanes<PPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    px::k_b2s_lanes<PPT><<<a.B * a.P, px::B2S_NT, smem, s>>>(a);
    return cudaGetLastError();
  });
}

cudaError_t b2s_launch_scan(const px::B2sScanArgs& a, int ppt, size_t smem, cudaStream_t s) {
  return b2s_dispatch(ppt, [&](auto pc) {
    constexpr int PPT = decltype(pc)::value;
    cudaError_t e = cudaFuncSetAttribute(px::k_b2s_scan<PPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    px::k_b2s_scan<PPT><<<a.B, px::B2S_NT, smem, s>>>(a);
    return cudaGetLastError();
  });
}

// the on-chip sweep: one kernel for the serial direct (one CTA per member), one for every slice's
// adjoint solve (one CTA per lane), overlapped through the progress flags when all CTAs fit
int direct_small(Hybrid2D* hy, int overlap, cudaStream_t s) {
  const size_t n2 = 2 * (size_t)hy->nx * hy->ny;
  int sms = 0;
  H2_CUDA(hy, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, hy->base.device));
  const bool ov = overlap && hy->P > 1 && (long long)hy->B * hy->P + hy->B <= sms;
  px::B2sDirectArgs d{};
  d.u0 = hy->u0; d.f = hy->f; d.traj = hy->traj; d.theta = hy->theta; d.flags = hy->flags; d.offs = hy->d_offs;
  d.P = hy->P; d.B = hy->B; d.S = hy->S; d.h = hy->h; d.g = geom(hy);
  px::B2sLaneArgs l{};
  l.traj = hy->traj; l.target = hy->target; l.offs = hy->d_offs; l.theta = hy->theta; l.flags = hy->flags;
  l.aend = hy->la; l.zl = hy->lz; l.P = hy->P; l.B = hy->B; l.target_b = hy->target_b; l.wait = ov ? 1 : 0;
  l.h = hy->h; l.g = geom(hy);
  H2_CUDA(hy, cudaMemsetAsync(hy->flags, 0, sizeof(int) * hy->B * hy->P, s));
  H2_CUDA(hy, cudaEventRecord(hy->ev[0], s));
  if (ov) {
    cudaStream_t sd = hy->side[0];
    H2_CUDA(hy, cudaStreamWaitEvent(sd, hy->ev[0], 0));
    H2_CUDA(hy, b2s_launch_direct(d, hy->ppt, 2 * n2 * sizeof(double), s));
    H2_CUDA(hy, cudaEventRecord(hy->ev[1], s));
    H2_CUDA(hy, cudaEventRecord(hy->ev[2], sd));
    H2_CUDA(hy, b2s_launch_lanes(l, hy->ppt, 4 * n2 * sizeof(double), sd));
    H2_CUDA(hy, cudaEventRecord(hy->ev[3], sd));
    H2_CUDA(hy, cudaStreamWaitEvent(s, hy->ev[3], 0));
  } else {
    H2_CUDA(hy, b2s_launch_direct(d, hy->ppt, 2 * n2 * sizeof(double), s));
    H2_CUDA(hy, cudaEventRecord(hy->ev[1], s));
    H2_CUDA(hy, cudaEventRecord(hy->ev[2], s));
    H2_CUDA(hy, b2s_launch_lanes(l, hy->ppt, 4 * n2 * sizeof(double), s));
    H2_CUDA(hy, cudaEventRecord(hy->ev[3], s));
  }
  hy->base.stats.kernel_launches += 2;
  hy->overlapped = ov ? 1 : 0;
  return PX_OK;
}

int adjoint_small(Hybrid2D* hy, cudaStream_t s) {
  const size_t n2 = 2 * (size_t)hy->nx * hy->ny;
  if (hy->plans_dirty) {
    std::vector<double> pool;
    std::vector<px::HybSlicePlan> table(hy->P);
    for (int q = 0; q < hy->P; ++q) {
      const Hybrid2D::SlicePlan& sp = hy->plans[q];
      px::HybSlicePlan& t = table[q];
      t.substeps = sp.set ? sp.substeps : 0;
      t.degree = sp.degree; t.sigma = sp.sigma; t.c0 = sp.c0; t.d = sp.set ? sp.d : 1.0;
      t.exp_off = (int)pool.size();
      pool.insert(pool.end(), sp.be.begin(), sp.be.end());
      t.law_off = (int)pool.size();
      pool.insert(pool.end(), sp.law.begin(), sp.law.end());
    }
    if (pool.empty()) pool.push_back(0.0);
    if (pool.size() > hy->coef_cap) {
      if (hy->d_coef) cudaFree(hy->d_coef);
      hy->d_coef = nullptr;
      H2_CUDA(hy, cudaMalloc(&hy->d_coef, pool.size() * sizeof(double)));
      hy->coef_cap = pool.size();
    }
    H2_CUDA(hy, cudaMemcpy(hy->d_coef, pool.data(), pool.size() * sizeof(double), cudaMemcpyHostToDevice));
    H2_CUDA(hy, cudaMemcpy(hy->d_plans, table.data(), sizeof(px::HybSlicePlan) * hy->P, cudaMemcpyHostToDevice));
    hy->plans_dirty = false;
  }
  px::B2sScanArgs a{};
  a.ubar = hy->ubar; a.aend = hy->la; a.zl = hy->lz; a.qT = hy->has_qT ? hy->qT : nullptr;
  a.plans = hy->d_plans; a.coef = hy->d_coef; a.qdag0 = hy->qdag0; a.grad = hy->grad;
  a.P = hy->P; a.B = hy->B; a.invT = 1.0 / hy->T; a.g = geom(hy);
  H2_CUDA(hy, b2s_launch_scan(a, hy->ppt, 4 * n2 * sizeof(double), s));
  hy->base.stats.kernel_launches += 1;
  return PX_OK;
}

}  // namespace

int h2_create(const px_hybrid_desc* d, void** out) {
  if (d->nx < 3 || d->ny < 3) return fail(nullptr, PX_ERR_ARG, "hybrid 2D: nx, ny must be ≥ 3");
  if ((long long)d->nx * d->ny > (1LL << 28)) return fail(nullptr, PX_ERR_ARG, "hybrid 2D: grid too large");
  if (!(d->hy > 0)) return fail(nullptr, PX_ERR_ARG, "hybrid 2D: hy must be positive");
  const int P = d->nslices;
  auto* hy = new Hybrid2D();
  Handle* hb = &hy->base;
  cudaGetDevice(&hb->device);
  hy->nx = d->nx; hy->ny = d->ny; hy->B = d->batch; hy->P = P; hy->S = d->offsets[P];
  hy->D = d->D; hy->hx = d->hx; hy->hy = d->hy; hy->T = d->T; hy->h = d->T / hy->S;
  for (int k = 0; k < 4; ++k) hy->law[k] = d->law[k];
  hy->target_b = d->target_batched ? hy->B : 1;
  hy->offs.assign(d->offsets, d->offsets + P + 1);
  hy->plans.resize(P);
  hy->max_np = 0;
  for (int p = 0; p < P; ++p) hy->max_np = std::max(hy->max_np, hy->offs[p + 1] - hy->offs[p]);
  const size_t n2 = 2 * (size_t)hy->nx * hy->ny, B = hy->B, S = hy->S, L = B * P;
  const char* onchip = std::getenv("PX_HYB2D_ONCHIP");
  hy->small = n2 / 2 <= (size_t)px::B2S_MAX_N && !(onchip && onchip[0] == '0');
  hy->ppt = n2 / 2 <= (size_t)px::B2S_NT ? 1 : (n2 / 2 <= 2 * (size_t)px::B2S_NT ? 2 : 4);
  hy->cost_blocks = (int)std::min<size_t>(148 * 4, ((S + 1) * n2 + 255) / 256);
  hy->bounds_blocks = (int)std::min<size_t>(148 * 2, ((size_t)P * B * (n2 / 2) + 255) / 256);
  int rc = PX_OK;
  auto al = [&](double** p, size_t cnt) { if (rc == PX_OK) rc = dalloc_t(hb, p, cnt); };
  al(&hy->u0, B * n2); al(&hy->f, B * n2); al(&hy->target, (S + 1) * hy->target_b * n2); al(&hy->qT, B * n2);
  al(&hy->traj, (S + 1) * B * n2); al(&hy->J, B); al(&hy->ubar, (size_t)P * B * n2);
  al(&hy->qdag0, B * n2); al(&hy->grad, B * n2); al(&hy->G, B * n2);
  al(&hy->w[0], B * n2); al(&hy->w[1], B * n2); al(&hy->w[2], B * n2); al(&hy->w[3], B * n2);
  al(&hy->la, L * n2); al(&hy->lz, L * n2); al(&hy->lacc, L * n2); al(&hy->ly[0], L * n2); al(&hy->ly[1], L * n2);
  al(&hy->cpart, B * (size_t)hy->cost_blocks); al(&hy->bpart, 3 * (size_t)hy->bounds_blocks);
  if (rc == PX_OK) rc = dalloc_t(hb, &hy->d_offs, (size_t)P + 1);
  if (rc == PX_OK) rc = dalloc_t(hb, &hy->flags, B * P);
  if (rc == PX_OK) rc = dalloc_t(hb, &hy->d_plans, (size_t)P);
  if (rc == PX_OK && cudaMemcpy(hy->d_offs, d->offsets, sizeof(int) * (P + 1), cudaMemcpyHostToDevice) != cudaSuccess)
    rc = fail(hb, PX_ERR_CUDA, "hybrid 2D: offsets upload");
  if (rc == PX_OK) rc = dalloc_t(hb, &hy->theta, 2 * S + 1);
  if (rc == PX_OK) {
    hy->theta_host.resize(2 * S + 1);
    for (size_t k = 0; k <= 2 * S; ++k) {
      const double t = (double)k * (0.5 * hy->h);
      hy->theta_host[k] = hy->law[0] + hy->law[1] * std::sin(hy->law[3] * t) + hy->law[2] * std::cos(hy->law[3] * t);
    }
    if (cudaMemcpy(hy->theta, hy->theta_host.data(), sizeof(double) * hy->theta_host.size(), cudaMemcpyHostToDevice) !=
        cudaSuccess)
      rc = fail(hb, PX_ERR_CUDA, "hybrid 2D: law table upload");
  }
  for (int k = 0; k < Hybrid2D::NSIDE && rc == PX_OK; ++k)
    if (cudaStreamCreateWithFlags(&hy->side[k], cudaStreamNonBlocking) != cudaSuccess)
      rc = fail(hb, PX_ERR_CUDA, "hybrid 2D: stream creation");
  hy->ev_slice.assign(P, nullptr);
  for (int p = 0; p < P && rc == PX_OK; ++p)
    if (cudaEventCreateWithFlags(&hy->ev_slice[p], cudaEventDisableTiming) != cudaSuccess)
      rc = fail(hb, PX_ERR_CUDA, "hybrid 2D: event creation");
  for (int k = 0; k < Hybrid2D::NSIDE && rc == PX_OK; ++k)
    if (cudaEventCreateWithFlags(&hy->ev_join[k], cudaEventDisableTiming) != cudaSuccess)
      rc = fail(hb, PX_ERR_CUDA, "hybrid 2D: event creation");
  for (int k = 0; k < 4 && rc == PX_OK; ++k)
    if (cudaEventCreate(&hy->ev[k]) != cudaSuccess) rc = fail(hb, PX_ERR_CUDA, "hybrid 2D: event creation");
  if (rc != PX_OK) {
    h2_destroy(hy);
    return rc;
  }
  *out = hy;
  return PX_OK;
}

void h2_destroy(Hybrid2D* hy) {
  cudaSetDevice(hy->base.device);
  for (auto st : hy->side)
    if (st) cudaStreamSynchronize(st);
  for (void* a : hy->base.allocs) cudaFree(a);
  if (hy->d_coef) cudaFree(hy->d_coef);
  for (auto st : hy->side)
    if (st) cudaStreamDestroy(st);
  for (auto e : hy->ev_slice)
    if (e) cudaEventDestroy(e);
  for (auto e : hy->ev_join)
    if (e) cudaEventDestroy(e);
  for (auto e : hy->ev)
    if (e) cudaEventDestroy(e);
  delete hy;
}

int h2_set_inputs(Hybrid2D* hy, const double* u0, const double* f, const double* target, const double* qdag_T, int mem,
                  cudaStream_t s) {
  cudaSetDevice(hy->base.device);
  const size_t n2 = 2 * (size_t)hy->nx * hy->ny, B = hy->B;
  PX_TRY(copy_in2(hy, hy->u0, u0, B * n2, mem, s));
  PX_TRY(copy_in2(hy, hy->f, f, B * n2, mem, s));
  PX_TRY(copy_in2(hy, hy->target, target, (size_t)(hy->S + 1) * hy->target_b * n2, mem, s));
  hy->has_qT = qdag_T != nullptr;
  if (qdag_T) PX_TRY(copy_in2(hy, hy->qT, qdag_T, B * n2, mem, s));
  hy->inputs = true;
  hy->direct_done = hy->adjoint_done = hy->means_done = false;
  return PX_OK;
}

int h2_direct(Hybrid2D* hy, int overlap, cudaStream_t s) {
  if (!hy->inputs) return fail(&hy->base, PX_ERR_STATE, "hybrid: inputs not set");
  cudaSetDevice(hy->base.device);
  const int n = hy->nx * hy->ny;
  const size_t n2 = 2 * (size_t)n, B = hy->B, L = B * hy->P;
  const double h = hy->h;
  if (hy->small) {
    PX_TRY(direct_small(hy, overlap, s));
    px::k_b2_cost_partial<<<dim3((unsigned)hy->cost_blocks, (unsigned)B), 256, 0, s>>>(hy->cpart, hy->traj, hy->target,
                                                                                     hy->target_b, n2, hy->S, hy->B);
    H2_LAUNCHED(hy);
    px::k_b2_cost_final<<<(hy->B + 63) / 64, 64, 0, s>>>(hy->J, hy->cpart, hy->cost_blocks, h / hy->T, hy->B);
    H2_LAUNCHED(hy);
    hy->base.stats.rk4_lane_steps += (uint64_t)hy->B * hy->S * 2;
    hy->direct_done = true;
    hy->adjoint_done = hy->means_done = false;
    return PX_OK;
  }
  const bool ov = overlap && hy->P > 1;
  H2_CUDA(hy, cudaMemsetAsync(hy->la, 0, L * n2 * sizeof(double), s));
  H2_CUDA(hy, cudaMemsetAsync(hy->lz, 0, L * n2 * sizeof(double), s));
  H2_CUDA(hy, cudaMemcpyAsync(hy->traj, hy->u0, B * n2 * sizeof(double), cudaMemcpyDeviceToDevice, s));
  H2_CUDA(hy, cudaEventRecord(hy->ev[0], s));
  if (ov) {  // the side streams start after the lane buffers are cleared
    for (int k = 0; k < Hybrid2D::NSIDE; ++k) H2_CUDA(hy, cudaStreamWaitEvent(hy->side[k], hy->ev[0], 0));
  }
  px::B2DirectArgs a{};
  a.f = hy->f;
  a.g = geom(hy);
  const dim3 grid((unsigned)((n + 255) / 256), (unsigned)B);
  const long long bs = (long long)n2;
  bool slices_marked = false;
  int p = 0;
  for (int i = 0; i < hy->S; ++i) {
    const double* ui = hy->traj + (size_t)i * B * n2;
    double* un = hy->traj + (size_t)(i + 1) * B * n2;
    a.base = ui; a.base_bs = bs;
    a.win = ui; a.win_bs = bs; a.accin = ui; a.accin_bs = bs; a.wout = hy->w[0]; a.accout = hy->w[2]; a.accout_bs = bs;
    a.cw = 0.5 * h; a.ca = h / 6.0; a.theta = hy->theta_host[2 * i];
    px::k_b2_direct_stage<<<grid, 256, 0, s>>>(a);
    H2_LAUNCHED(hy);
    a.win = hy->w[0]; a.accin = hy->w[2]; a.wout = hy->w[1]; a.ca = h / 3.0; a.theta = hy->theta_host[2 * i + 1];
    px::k_b2_direct_stage<<<grid, 256, 0, s>>>(a);
    H2_LAUNCHED(hy);
    a.win = hy->w[1]; a.wout = hy->w[0]; a.cw = h;
    px::k_b2_direct_stage<<<grid, 256, 0, s>>>(a);
    H2_LAUNCHED(hy);
    a.win = hy->w[0]; a.wout = nullptr; a.accout = un; a.ca = h / 6.0; a.theta = hy->theta_host[2 * i + 2];
    px::k_b2_direct_stage<<<grid, 256, 0, s>>>(a);
    H2_LAUNCHED(hy);
    if (ov && i + 1 == hy->offs[p + 1]) {  // slice p is stored: release its adjoint solve on a side stream
      cudaStream_t sd = hy->side[p % Hybrid2D::NSIDE];
      H2_CUDA(hy, cudaEventRecord(hy->ev_slice[p], s));
      H2_CUDA(hy, cudaStreamWaitEvent(sd, hy->ev_slice[p], 0));
      if (!slices_marked) {
        H2_CUDA(hy, cudaEventRecord(hy->ev[2], sd));
        slices_marked = true;
      }
      const int np = hy->offs[p + 1] - hy->offs[p];
      for (int k = 0; k < np; ++k) PX_TRY(adjoint_step(hy, k, p, 1, sd));
      ++p;
    }
  }
  H2_CUDA(hy, cudaEventRecord(hy->ev[1], s));
  if (ov) {
    // join: the last slice's stream carries the end-of-slices mark after every other side stream
    cudaStream_t last = hy->side[(hy->P - 1) % Hybrid2D::NSIDE];
    for (int k = 0; k < Hybrid2D::NSIDE; ++k) {
      if (hy->side[k] == last) continue;
      H2_CUDA(hy, cudaEventRecord(hy->ev_join[k], hy->side[k]));
      H2_CUDA(hy, cudaStreamWaitEvent(last, hy->ev_join[k], 0));
    }
    H2_CUDA(hy, cudaEventRecord(hy->ev[3], last));
    H2_CUDA(hy, cudaStreamWaitEvent(s, hy->ev[3], 0));
  } else {
    H2_CUDA(hy, cudaEventRecord(hy->ev[2], s));
    for (int k = 0; k < hy->max_np; ++k) PX_TRY(adjoint_step(hy, k, 0, hy->P, s));
    H2_CUDA(hy, cudaEventRecord(hy->ev[3], s));
  }
  // tracking cost
  px::k_b2_cost_partial<<<dim3((unsigned)hy->cost_blocks, (unsigned)B), 256, 0, s>>>(hy->cpart, hy->traj, hy->target,
                                                                                   hy->target_b, n2, hy->S, hy->B);
  H2_LAUNCHED(hy);
  px::k_b2_cost_final<<<(hy->B + 63) / 64, 64, 0, s>>>(hy->J, hy->cpart, hy->cost_blocks, h / hy->T, hy->B);
  H2_LAUNCHED(hy);
  hy->base.stats.rk4_lane_steps += (uint64_t)hy->B * hy->S * 2;
  hy->overlapped = ov ? 1 : 0;
  hy->direct_done = true;
  hy->adjoint_done = hy->means_done = false;
  return PX_OK;
}

int h2_bounds(Hybrid2D* hy, double* out3, cudaStream_t s) {
  if (!hy->direct_done) return fail(&hy->base, PX_ERR_STATE, "hybrid: run px_hybrid_direct first");
  cudaSetDevice(hy->base.device);
  const int n = hy->nx * hy->ny;
  const size_t n2 = 2 * (size_t)n;
  px::k_b2_means<<<dim3((unsigned)((n2 + 255) / 256), (unsigned)hy->B, (unsigned)hy->P), 256, 0, s>>>(
      hy->ubar, hy->traj, hy->d_offs, hy->B, n2);
  H2_LAUNCHED(hy);
  px::k_b2_bounds<<<hy->bounds_blocks, 256, 0, s>>>(hy->bpart, hy->ubar, hy->P * hy->B, geom(hy), hy->D);
  H2_LAUNCHED(hy);
  std::vector<double> part(3 * (size_t)hy->bounds_blocks);
  H2_CUDA(hy, cudaMemcpyAsync(part.data(), hy->bpart, part.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
  H2_CUDA(hy, cudaStreamSynchronize(s));
  double lo = INFINITY, hi = -INFINITY, im = 0.0;
  bool bad = false;
  for (int k = 0; k < hy->bounds_blocks; ++k) {
    const double a = part[3 * k], b = part[3 * k + 1], c = part[3 * k + 2];
    if (a != a || b != b || c != c) bad = true;
    lo = std::min(lo, a); hi = std::max(hi, b); im = std::max(im, c);
  }
  if (bad || !std::isfinite(lo) || !std::isfinite(hi) || !std::isfinite(im))
    return fail(&hy->base, PX_ERR_NONFINITE, "hybrid: non-finite direct trajectory");
  out3[0] = lo; out3[1] = hi; out3[2] = im;
  hy->means_done = true;
  return PX_OK;
}

int h2_set_slice_plan(Hybrid2D* hy, int sl, const px_cheb_plan* plan, const double* gc, const double* gs) {
  if (sl < 0 || sl >= hy->P) return fail(&hy->base, PX_ERR_ARG, "hybrid plan: slice out of range");
  if (plan->substeps < 1 || plan->degree < 1 || !(plan->scale > 0) || (plan->sigma != 1 && plan->sigma != -1))
    return fail(&hy->base, PX_ERR_ARG, "hybrid plan: bad substeps/degree/scale/sigma");
  if (hy->law[3] != 0.0 && (!gc || !gs))
    return fail(&hy->base, PX_ERR_ARG, "hybrid plan: a sine/cosine time law needs the coef_gc / coef_gs series");
  const double span = (hy->offs[sl + 1] - hy->offs[sl]) * hy->h;
  if (std::fabs(plan->span - span) > 1e-12 * std::max(1.0, span))
    return fail(&hy->base, PX_ERR_ARG, "hybrid plan: span does not match the slice width");
  Hybrid2D::SlicePlan& sp = hy->plans[sl];
  const int K = plan->degree;
  sp.set = true;
  hy->plans_dirty = true;
  sp.substeps = plan->substeps; sp.degree = K; sp.sigma = plan->sigma;
  sp.c0 = plan->center; sp.d = plan->scale; sp.span = plan->span;
  sp.be.assign(plan->coef_exp, plan->coef_exp + K + 1);
  sp.law.assign((size_t)sp.substeps * (K + 1), 0.0);
  const double tau = plan->span / plan->substeps;
  const double t_top = hy->offs[sl + 1] * hy->h;
  const double la = hy->law[0], lb = hy->law[1], lc = hy->law[2], lw = hy->law[3];
  for (int j = 0; j < sp.substeps; ++j) {
    double* out = sp.law.data() + (size_t)j * (K + 1);
    const double tt = t_top - j * tau;
    if (lw == 0.0) {
      for (int k = 0; k <= K; ++k) out[k] = (la + lc) * plan->coef_phi[k];
    } else {
      const double A = lb * std::sin(lw * tt) + lc * std::cos(lw * tt);
      const double Bc = -lb * std::cos(lw * tt) + lc * std::sin(lw * tt);
      for (int k = 0; k <= K; ++k) out[k] = la * plan->coef_phi[k] + A * gc[k] + Bc * gs[k];
    }
  }
  return PX_OK;
}

int h2_adjoint(Hybrid2D* hy, cudaStream_t s) {
  if (!hy->direct_done) return fail(&hy->base, PX_ERR_STATE, "hybrid: run px_hybrid_direct first");
  if (!hy->means_done) return fail(&hy->base, PX_ERR_STATE, "hybrid: run px_hybrid_bounds first (slice means)");
  cudaSetDevice(hy->base.device);
  const int top = hy->has_qT ? hy->P - 1 : hy->P - 2;
  for (int q = 0; q <= top; ++q)
    if (!hy->plans[q].set) return fail(&hy->base, PX_ERR_STATE, "hybrid: slice plan " + std::to_string(q) + " not set");
  if (hy->small) {
    PX_TRY(adjoint_small(hy, s));
    uint64_t tm = 0;
    for (int q = 0; q <= top; ++q) tm += (uint64_t)hy->plans[q].substeps * hy->plans[q].degree;
    hy->base.stats.exp_terms += tm * hy->B;
    hy->adjoint_done = true;
    return PX_OK;
  }
  const int n = hy->nx * hy->ny;
  const size_t n2 = 2 * (size_t)n, B = hy->B;
  const dim3 gridn((unsigned)((n + 255) / 256), (unsigned)B);
  const dim3 grid2((unsigned)((n2 + 255) / 256), (unsigned)B);
  H2_CUDA(hy, cudaMemsetAsync(hy->G, 0, B * n2 * sizeof(double), s));
  // the carry C lives in w[c]; the other three buffers hold the recurrence and the accumulator
  int c = 0;
  if (hy->has_qT) {
    H2_CUDA(hy, cudaMemcpyAsync(hy->w[c], hy->qT, B * n2 * sizeof(double), cudaMemcpyDeviceToDevice, s));
  } else {
    px::k_b2_take_lane<<<grid2, 256, 0, s>>>(hy->w[c], hy->la, hy->P, hy->P - 1, 0, n2);
    H2_LAUNCHED(hy);
  }
  px::B2ChebArgs a{};
  a.G = hy->G;
  a.g = geom(hy);
  uint64_t terms = 0;
  for (int p = top; p >= 0; --p) {
    const Hybrid2D::SlicePlan& sp = hy->plans[p];
    const int K = sp.degree;
    a.qbar = hy->ubar + (size_t)p * B * n2;
    a.c0 = sp.c0;
    for (int j = 0; j < sp.substeps; ++j) {
      const double* bl = sp.law.data() + (size_t)j * (K + 1);
      int f1 = (c + 1) & 3, f2 = (c + 2) & 3, f3 = (c + 3) & 3;
      // term 1: U_1 = (M − c0)U_0/d, acc = be0 U_0 + be1 U_1
      a.x = hy->w[c]; a.prev = nullptr; a.out = hy->w[f1]; a.acc = hy->w[f2];
      a.alpha = 1.0 / sp.d; a.sg = 0.0; a.first = 1;
      a.be0 = sp.be[0]; a.bek = sp.be[1]; a.bl0 = bl[0]; a.blk = bl[1];
      px::k_b2_cheb_term<<<gridn, 256, 0, s>>>(a);
      H2_LAUNCHED(hy);
      int prev = c, cur = f1, nxt = f3;
      a.alpha = 2.0 / sp.d; a.sg = (double)sp.sigma; a.first = 0;
      for (int k = 2; k <= K; ++k) {
        a.x = hy->w[cur]; a.prev = hy->w[prev]; a.out = hy->w[nxt];
        a.bek = sp.be[k]; a.blk = bl[k];
        px::k_b2_cheb_term<<<gridn, 256, 0, s>>>(a);
        H2_LAUNCHED(hy);
        const int t = prev;
        prev = cur; cur = nxt; nxt = t;
      }
      c = f2;  // the substep's result
      terms += (uint64_t)K;
    }
    px::k_b2_take_lane<<<grid2, 256, 0, s>>>(hy->w[c], hy->la, hy->P, p, 1, n2);  // + a_p(T_p)
    H2_LAUNCHED(hy);
  }
  H2_CUDA(hy, cudaMemcpyAsync(hy->qdag0, hy->w[c], B * n2 * sizeof(double), cudaMemcpyDeviceToDevice, s));
  px::k_b2_grad<<<grid2, 256, 0, s>>>(hy->grad, hy->lz, hy->G, hy->P, 1.0 / hy->T, n2);
  H2_LAUNCHED(hy);
  hy->base.stats.exp_terms += terms * hy->B;
  hy->adjoint_done = true;
  return PX_OK;
}

// One planned forward action on `rows` vectors held in four rotating buffers buf[0..3] (each
// rows × 2n); the input is buf[*c], the result's index is returned in *c.
int fwd_action_launches(Hybrid2D* hy, double* const* buf, int* c, int rows, int pfix, int skip0,
                        const Hybrid2D::NlPlan& pl, const std::vector<double>& be, cudaStream_t s) {
  const int n = hy->nx * hy->ny;
  const dim3 grid((unsigned)((n + 255) / 256), (unsigned)rows);
  px::B2FwdTermArgs a{};
  a.ubar = hy->ubar; a.c0 = pl.c0; a.P = hy->P; a.B = hy->B; a.pfix = pfix; a.skip0 = skip0; a.g = geom(hy);
  for (int j = 0; j < pl.subs; ++j) {
    const int f1 = (*c + 1) & 3, f2 = (*c + 2) & 3, f3 = (*c + 3) & 3;
    a.x = buf[*c]; a.prev = nullptr; a.out = buf[f1]; a.acc = buf[f2];
    a.alpha = 1.0 / pl.d; a.sg = 0.0; a.first = 1; a.be0 = be[0]; a.bek = be[1];
    px::k_b2_fwd_term<<<grid, 256, 0, s>>>(a);
    H2_LAUNCHED(hy);
    int prev = *c, cur = f1, nxt = f3;
    a.alpha = 2.0 / pl.d; a.sg = (double)pl.sigma; a.first = 0;
    for (int k = 2; k <= pl.K; ++k) {
      a.x = buf[cur]; a.prev = buf[prev]; a.out = buf[nxt]; a.bek = be[k];
      px::k_b2_fwd_term<<<grid, 256, 0, s>>>(a);
      H2_LAUNCHED(hy);
      const int t = prev;
      prev = cur; cur = nxt; nxt = t;
    }
    *c = f2;
  }
  return PX_OK;
}

// Algorithm 2's sweep with one launch per stage / term (any grid size)
int nl_sweep_launches(Hybrid2D* hy, cudaStream_t s) {
  const int n = hy->nx * hy->ny;
  const size_t n2 = 2 * (size_t)n, B = hy->B;
  const int P = hy->P, L = hy->B * P, ns = hy->offs[1];
  const double h = hy->h;
  const dim3 gl((unsigned)((n + 255) / 256), (unsigned)L), gl2((unsigned)((n2 + 255) / 256), (unsigned)L);
  const dim3 gb2((unsigned)((n2 + 255) / 256), (unsigned)B);
  // slice lanes: y = la, cst = lz, acc = lacc, stage inputs ly[0/1]
  px::k_b2_nl_prepare<<<gl, 256, 0, s>>>(hy->lz, hy->la, hy->ubar, hy->u0, P, hy->B, geom(hy));
  H2_LAUNCHED(hy);
  px::B2NlStageArgs a{};
  a.y = hy->la; a.cst = hy->lz; a.Q = hy->traj; a.Qn = hy->Qn; a.ubar = hy->ubar; a.u0 = hy->u0; a.f = hy->f;
  a.theta = hy->theta; a.nsteps = ns; a.P = P; a.B = hy->B; a.g = geom(hy);
  for (int k = 0; k < ns; ++k) {
    a.k = k; a.write_node = 0;
    a.yin = hy->la; a.accin = hy->la; a.accout = hy->lacc; a.yout = hy->ly[0];
    a.wa = 1.0; a.wb = 0.0; a.tsel = 0; a.cw = 0.5 * h; a.ca = h / 6.0;
    px::k_b2_nl_stage<<<gl, 256, 0, s>>>(a);
    H2_LAUNCHED(hy);
    a.yin = hy->ly[0]; a.accin = hy->lacc; a.yout = hy->ly[1];
    a.wa = 0.5; a.wb = 0.5; a.tsel = 1; a.ca = h / 3.0;
    px::k_b2_nl_stage<<<gl, 256, 0, s>>>(a);
    H2_LAUNCHED(hy);
    a.yin = hy->ly[1]; a.yout = hy->ly[0]; a.cw = h;
    px::k_b2_nl_stage<<<gl, 256, 0, s>>>(a);
    H2_LAUNCHED(hy);
    a.yin = hy->ly[0]; a.accout = hy->la; a.yout = nullptr;
    a.wa = 0.0; a.wb = 1.0; a.tsel = 2; a.ca = h / 6.0; a.write_node = (k + 1 < ns) ? 1 : 0;
    px::k_b2_nl_stage<<<gl, 256, 0, s>>>(a);
    H2_LAUNCHED(hy);
  }
  // summed-chain carry (member vectors in w[0..3]); yend = la
  int c = 0;
  H2_CUDA(hy, cudaMemsetAsync(hy->Dc, 0, B * n2 * sizeof(double), s));
  for (int p = 0; p < P; ++p) {
    if (p > 0) PX_TRY(fwd_action_launches(hy, hy->w, &c, hy->B, p, 0, hy->nl_s, hy->nl_be_s, s));
    px::k_b2_nl_carry_add<<<gb2, 256, 0, s>>>(hy->w[c], hy->Dc + (size_t)(p + 1) * B * n2, hy->la, P, p, n2);
    H2_LAUNCHED(hy);
  }
  // homogeneous parts on every node: lane vectors rotate through ly[0], ly[1], lacc, lz
  double* hb[4] = {hy->ly[0], hy->ly[1], hy->lacc, hy->lz};
  int hc = 0;
  px::k_b2_nl_hom_init<<<gl2, 256, 0, s>>>(hb[0], hy->Qn, hy->Dc, hy->u0, P, hy->B, ns, hy->S, n2);
  H2_LAUNCHED(hy);
  if (P > 1) {
    for (int k = 1; k < ns; ++k) {
      PX_TRY(fwd_action_launches(hy, hb, &hc, L, -1, 1, hy->nl_h, hy->nl_be_h, s));
      px::k_b2_nl_hom_add<<<gl2, 256, 0, s>>>(hy->Qn, hb[hc], P, hy->B, ns, k, n2);
      H2_LAUNCHED(hy);
    }
  }
  return PX_OK;
}

// ---- Algorithm 2 (iterative nonlinear direct) on the two-field testbed --------------------------
int h2_nl_init(Hybrid2D* hy, cudaStream_t s) {
  if (!hy->inputs) return fail(&hy->base, PX_ERR_STATE, "hybrid: inputs not set");
  const int ns = hy->offs[1];
  for (int p = 0; p <= hy->P; ++p)
    if (hy->offs[p] != p * ns) return fail(&hy->base, PX_ERR_ARG, "Algorithm 2 needs equal slices (nonlinear.py: equidistant)");
  cudaSetDevice(hy->base.device);
  const size_t n2 = 2 * (size_t)hy->nx * hy->ny, B = hy->B, S = hy->S, P = hy->P;
  if (!hy->Qn) {
    int rc = dalloc_t(&hy->base, &hy->Qn, (S + 1) * B * n2);
    if (rc == PX_OK) rc = dalloc_t(&hy->base, &hy->Dc, (P + 1) * B * n2);
    if (rc == PX_OK) rc = dalloc_t(&hy->base, &hy->nl_err, B * P);
    if (rc == PX_OK) rc = dalloc_t(&hy->base, &hy->nl_coef, 2 * (size_t)(PX_MAX_CHEB_DEGREE + 1));
    if (rc != PX_OK) return rc;
  }
  // constant-in-time initial guess (nonlinear.py:98-100)
  for (size_t j = 0; j <= S; ++j)
    H2_CUDA(hy, cudaMemcpyAsync(hy->traj + j * B * n2, hy->u0, B * n2 * sizeof(double), cudaMemcpyDeviceToDevice, s));
  hy->nl_active = true;
  hy->nl_plans = false;
  hy->direct_done = true;   // the iterate is a trajectory: px_hybrid_bounds gives its slice means and FOV box
  hy->adjoint_done = hy->means_done = false;
  return PX_OK;
}

int h2_nl_set_plans(Hybrid2D* hy, const px_cheb_plan* ps, const px_cheb_plan* ph) {
  if (!hy->nl_active) return fail(&hy->base, PX_ERR_STATE, "hybrid: run px_hybrid_nl_init first");
  const px_cheb_plan* pl[2] = {ps, ph};
  const double spans[2] = {hy->offs[1] * hy->h, hy->h};
  for (int k = 0; k < 2; ++k) {
    if (pl[k]->substeps < 1 || pl[k]->degree < 1 || pl[k]->degree > PX_MAX_CHEB_DEGREE || !(pl[k]->scale > 0) ||
        (pl[k]->sigma != 1 && pl[k]->sigma != -1) || !pl[k]->coef_exp)
      return fail(&hy->base, PX_ERR_ARG, "hybrid nl plan: bad substeps/degree/scale/sigma");
    if (std::fabs(pl[k]->span - spans[k]) > 1e-12 * std::max(1.0, spans[k]))
      return fail(&hy->base, PX_ERR_ARG, "hybrid nl plan: span does not match the slice / step width");
  }
  cudaSetDevice(hy->base.device);
  std::vector<double> pool(ps->coef_exp, ps->coef_exp + ps->degree + 1);
  pool.insert(pool.end(), ph->coef_exp, ph->coef_exp + ph->degree + 1);
  H2_CUDA(hy, cudaMemcpy(hy->nl_coef, pool.data(), pool.size() * sizeof(double), cudaMemcpyHostToDevice));
  hy->nl_be_s.assign(ps->coef_exp, ps->coef_exp + ps->degree + 1);
  hy->nl_be_h.assign(ph->coef_exp, ph->coef_exp + ph->degree + 1);
  hy->nl_s = {ps->degree, ps->substeps, ps->sigma, ps->center, ps->scale};
  hy->nl_h = {ph->degree, ph->substeps, ph->sigma, ph->center, ph->scale};
  hy->nl_plans = true;
  return PX_OK;
}

int h2_nl_sweep(Hybrid2D* hy, double* err_out, cudaStream_t s) {
  if (!hy->nl_active || !hy->nl_plans) return fail(&hy->base, PX_ERR_STATE, "hybrid: nl_init / nl_set_plans first");
  if (!hy->means_done) return fail(&hy->base, PX_ERR_STATE, "hybrid: run px_hybrid_bounds on the iterate first");
  cudaSetDevice(hy->base.device);
  const size_t n2 = 2 * (size_t)hy->nx * hy->ny;
  px::B2sNlArgs a{};
  a.Q = hy->traj; a.Qn = hy->Qn; a.ubar = hy->ubar; a.u0 = hy->u0; a.f = hy->f; a.theta = hy->theta;
  a.yend = hy->lacc; a.Dc = hy->Dc; a.err = hy->nl_err; a.coef = hy->nl_coef;
  a.P = hy->P; a.B = hy->B; a.nsteps = hy->offs[1]; a.S = hy->S;
  a.Ks = hy->nl_s.K; a.subs_s = hy->nl_s.subs; a.sig_s = hy->nl_s.sigma; a.c0_s = hy->nl_s.c0; a.d_s = hy->nl_s.d;
  a.Kh = hy->nl_h.K; a.subs_h = hy->nl_h.subs; a.sig_h = hy->nl_h.sigma; a.c0_h = hy->nl_h.c0; a.d_h = hy->nl_h.d;
  a.h = hy->h; a.g = geom(hy);
  const int lanes = hy->B * hy->P;
  if (!hy->small) {
    PX_TRY(nl_sweep_launches(hy, s));
  } else
  H2_CUDA(hy, b2s_dispatch(hy->ppt, [&](auto pc) {
    constexpr int PPT = decltype(pc)::value;
    const size_t sm5 = 5 * n2 * sizeof(double), sm4 = 4 * n2 * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(px::k_b2s_nl_lanes<PPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm5);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(px::k_b2s_nl_carry<PPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm4);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(px::k_b2s_nl_hom<PPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm4);
    if (e != cudaSuccess) return e;
    px::k_b2s_nl_lanes<PPT><<<lanes, px::B2S_NT, sm5, s>>>(a);
    px::k_b2s_nl_carry<PPT><<<hy->B, px::B2S_NT, sm4, s>>>(a);
    px::k_b2s_nl_hom<PPT><<<lanes, px::B2S_NT, sm4, s>>>(a);
    return cudaGetLastError();
  }));
  px::k_b2s_nl_err<<<lanes, 256, 0, s>>>(a);
  H2_LAUNCHED(hy);
  hy->base.stats.kernel_launches += 3;
  std::vector<double> e(lanes);
  H2_CUDA(hy, cudaMemcpyAsync(e.data(), hy->nl_err, lanes * sizeof(double), cudaMemcpyDeviceToHost, s));
  H2_CUDA(hy, cudaStreamSynchronize(s));
  double mx = 0.0;
  for (double v : e) {
    if (v != v) mx = NAN;
    else if (mx == mx) mx = std::max(mx, v);
  }
  std::swap(hy->traj, hy->Qn);
  hy->means_done = false;
  hy->base.stats.rk4_lane_steps += (uint64_t)hy->B * hy->S;
  if (!std::isfinite(mx)) return fail(&hy->base, PX_ERR_NONFINITE, "hybrid: non-finite iterate in the nonlinear sweep");
  *err_out = mx;
  return PX_OK;
}

// the converged iterate is the direct trajectory: tracking cost and every slice's adjoint solve
int h2_nl_finish(Hybrid2D* hy, cudaStream_t s) {
  if (!hy->nl_active) return fail(&hy->base, PX_ERR_STATE, "hybrid: run px_hybrid_nl_init first");
  cudaSetDevice(hy->base.device);
  const size_t n2 = 2 * (size_t)hy->nx * hy->ny;
  px::B2sLaneArgs l{};
  l.traj = hy->traj; l.target = hy->target; l.offs = hy->d_offs; l.theta = hy->theta; l.flags = hy->flags;
  l.aend = hy->la; l.zl = hy->lz; l.P = hy->P; l.B = hy->B; l.target_b = hy->target_b; l.wait = 0;
  l.h = hy->h; l.g = geom(hy);
  H2_CUDA(hy, cudaEventRecord(hy->ev[0], s));
  H2_CUDA(hy, cudaEventRecord(hy->ev[1], s));
  H2_CUDA(hy, cudaEventRecord(hy->ev[2], s));
  if (hy->small) {
    H2_CUDA(hy, b2s_launch_lanes(l, hy->ppt, 4 * n2 * sizeof(double), s));
  } else {
    const size_t L = (size_t)hy->B * hy->P;
    H2_CUDA(hy, cudaMemsetAsync(hy->la, 0, L * n2 * sizeof(double), s));
    H2_CUDA(hy, cudaMemsetAsync(hy->lz, 0, L * n2 * sizeof(double), s));
    for (int k = 0; k < hy->max_np; ++k) PX_TRY(adjoint_step(hy, k, 0, hy->P, s));
  }
  H2_CUDA(hy, cudaEventRecord(hy->ev[3], s));
  px::k_b2_cost_partial<<<dim3((unsigned)hy->cost_blocks, (unsigned)hy->B), 256, 0, s>>>(
      hy->cpart, hy->traj, hy->target, hy->target_b, n2, hy->S, hy->B);
  H2_LAUNCHED(hy);
  px::k_b2_cost_final<<<(hy->B + 63) / 64, 64, 0, s>>>(hy->J, hy->cpart, hy->cost_blocks, hy->h / hy->T, hy->B);
  H2_LAUNCHED(hy);
  hy->base.stats.kernel_launches += 1;
  hy->overlapped = 0;
  hy->nl_active = false;
  hy->direct_done = true;
  hy->adjoint_done = hy->means_done = false;
  return PX_OK;
}

int h2_get(Hybrid2D* hy, int field, double* dst, size_t count, int mem, cudaStream_t s) {
  cudaSetDevice(hy->base.device);
  const size_t n2 = 2 * (size_t)hy->nx * hy->ny, B = hy->B, P = hy->P, S = hy->S;
  const double* src = nullptr;
  size_t have = 0;
  switch (field) {
    case PX_HFIELD_J: src = hy->J; have = B; break;
    case PX_HFIELD_GRAD: src = hy->grad; have = B * n2; break;
    case PX_HFIELD_UT: src = hy->traj + S * B * n2; have = B * n2; break;
    case PX_HFIELD_QDAG0: src = hy->qdag0; have = B * n2; break;
    case PX_HFIELD_TRAJ: src = hy->traj; have = (S + 1) * B * n2; break;
    case PX_HFIELD_AEND: src = hy->la; have = B * P * n2; break;
    case PX_HFIELD_ZL: src = hy->lz; have = B * P * n2; break;
    case PX_HFIELD_UBAR: src = hy->ubar; have = P * B * n2; break;
    default: return fail(&hy->base, PX_ERR_ARG, "hybrid: unknown field");
  }
  const bool needs_adj = field == PX_HFIELD_GRAD || field == PX_HFIELD_QDAG0;
  if ((needs_adj && !hy->adjoint_done) || (!needs_adj && !hy->direct_done) || (field == PX_HFIELD_UBAR && !hy->means_done))
    return fail(&hy->base, PX_ERR_STATE, "hybrid: field not computed yet");
  if (count != have) return fail(&hy->base, PX_ERR_ARG, "hybrid: count mismatch (" + std::to_string(have) + ")");
  H2_CUDA(hy, cudaMemcpyAsync(dst, src, count * sizeof(double),
                              mem == PX_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
  if (mem != PX_MEM_DEVICE) H2_CUDA(hy, cudaStreamSynchronize(s));
  return PX_OK;
}

int h2_get_timing(Hybrid2D* hy, double* ms) {
  if (!hy->direct_done) return fail(&hy->base, PX_ERR_STATE, "hybrid: no direct sweep timed");
  cudaSetDevice(hy->base.device);
  H2_CUDA(hy, cudaEventSynchronize(hy->ev[3]));
  H2_CUDA(hy, cudaEventSynchronize(hy->ev[1]));
  float a = 0, b = 0, c = 0, e = 0;
  H2_CUDA(hy, cudaEventElapsedTime(&a, hy->ev[0], hy->ev[1]));
  H2_CUDA(hy, cudaEventElapsedTime(&b, hy->ev[2], hy->ev[3]));
  H2_CUDA(hy, cudaEventElapsedTime(&c, hy->ev[0], hy->ev[3]));
  H2_CUDA(hy, cudaEventElapsedTime(&e, hy->ev[1], hy->ev[3]));
  ms[0] = a;
  ms[1] = b;
  ms[2] = std::max(a, c);
  ms[3] = std::max(0.0f, e);
  ms[4] = hy->overlapped;
  return PX_OK;
}

}  // namespace pxi
