// hybrid.cu — C ABI of the reference's hybrid algorithm with its tracking objective
// (px_hybrid_*, include/paraexp.h): hybrid.py:1-290 and optimization.py:84-112,172-189 on one
// GPU. The kernels are hybrid.cuh (instantiated in burgers.cu).
//
// One gradient: px_hybrid_direct (serial sweep + J; every slice's adjoint solve, overlapped with
// the sweep through per-slice progress flags when all CTAs can be co-resident) →
// px_hybrid_bounds (slice means, FOV box to the host, which plans the frozen actions) →
// px_hybrid_set_slice_plan × P → px_hybrid_adjoint (frozen-operator carry, ∂L/∂f).
#include <algorithm>
#include <cmath>
#include <vector>

#include "hybrid2d.h"
#include "internal.h"

namespace pxi {

struct Hybrid : HybridHead {  // dim = 1 (hybrid2d.h: the common head)
  int nx = 0, B = 1, P = 1, S = 1, ppt = 1, target_b = 1;
  double D = 0.0, hx = 0.0, T = 1.0, h = 1.0;
  double law[4] = {1.0, 0.0, 0.0, 0.0};
  std::vector<int> offs;
  int* d_offs = nullptr;
  int* flags = nullptr;
  double* theta = nullptr;  // θ(k·h/2), k = 0 … 2S
  double *u0 = nullptr, *f = nullptr, *target = nullptr, *qT = nullptr;
  double *traj = nullptr, *J = nullptr, *aend = nullptr, *zl = nullptr, *ubar = nullptr;
  double *qdag0 = nullptr, *grad = nullptr, *bpart = nullptr, *bounds = nullptr;
  int bounds_blocks = 0;
  bool has_qT = false, inputs = false, direct_done = false, adjoint_done = false;
  size_t lane_smem = 0;
  // per-slice plans: host records, device table and coefficient pool
  struct SlicePlan {
    bool set = false;
    int substeps = 0, degree = 0, sigma = -1;
    double c0 = 0.0, d = 1.0, span = 0.0;
    std::vector<double> be, law;  // exp series; law series per substep (substeps × (degree+1))
  };
  std::vector<SlicePlan> plans;
  px::HybSlicePlan* d_plans = nullptr;
  double* d_coef = nullptr;
  size_t coef_cap = 0;
  bool plans_dirty = true;
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev[4] = {nullptr, nullptr, nullptr, nullptr};
  int overlapped = 0;
};

namespace {

Hybrid* H(void* p) { return static_cast<Hybrid*>(p); }
// the 2D two-field handle (desc.ny > 1, hybrid2d.cu), or null for the 1D one
Hybrid2D* H2(void* p) {
  return p && static_cast<HybridHead*>(p)->dim == 2 ? static_cast<Hybrid2D*>(static_cast<HybridHead*>(p)) : nullptr;
}

int cuda_fail(Hybrid* hy, cudaError_t e, const char* what) {
  return fail(&hy->base, e == cudaErrorMemoryAllocation ? PX_ERR_NOMEM : PX_ERR_CUDA,
              std::string(what) + ": " + cudaGetErrorString(e));
}

#define HY_CUDA(hy, call)                                 \
  do {                                                    \
    cudaError_t _e = (call);                              \
    if (_e != cudaSuccess) return cuda_fail((hy), _e, #call); \
  } while (0)

int copy_in(Hybrid* hy, double* dst, const double* src, size_t count, int mem, cudaStream_t s) {
  HY_CUDA(hy, cudaMemcpyAsync(dst, src, count * sizeof(double),
                              mem == PX_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
  return PX_OK;
}

// the law series of one substep: ∫₀^τ θ(t_top − s)·e^{sM} ds = α·τφ₁ + A·Gc + B·Gs
void law_coef(const double* law, double t_top, const std::vector<double>& bp, const double* gc, const double* gs,
              int K, double* out) {
  const double a = law[0], b = law[1], c = law[2], w = law[3];
  if (w == 0.0) {
    for (int k = 0; k <= K; ++k) out[k] = (a + c) * bp[k];
    return;
  }
  const double A = b * std::sin(w * t_top) + c * std::cos(w * t_top);
  const double Bc = -b * std::cos(w * t_top) + c * std::sin(w * t_top);
  for (int k = 0; k <= K; ++k) out[k] = a * bp[k] + A * gc[k] + Bc * gs[k];
}

}  // namespace
}  // namespace pxi

using pxi::Hybrid;

extern "C" {

int px_hybrid_create(const px_hybrid_desc* d, void** out) {
  using namespace pxi;
  if (!d || !out) return fail(nullptr, PX_ERR_ARG, "px_hybrid_create: null argument");
  *out = nullptr;
  if (d->nx < 3 || (d->ny <= 1 && d->nx > 8192)) return fail(nullptr, PX_ERR_ARG, "hybrid: nx must be in [3, 8192]");
  if (d->batch < 1 || d->nslices < 1 || !d->offsets) return fail(nullptr, PX_ERR_ARG, "hybrid: batch/nslices/offsets");
  if (!(d->T > 0) || !(d->D > 0) || !(d->hx > 0)) return fail(nullptr, PX_ERR_ARG, "hybrid: T, D, hx must be positive");
  if (!(d->law[3] >= 0.0)) return fail(nullptr, PX_ERR_ARG, "hybrid: law ω must be non-negative");
  const int P = d->nslices;
  if (d->offsets[0] != 0) return fail(nullptr, PX_ERR_ARG, "hybrid: offsets must start at 0");
  for (int p = 0; p < P; ++p)
    if (d->offsets[p + 1] <= d->offsets[p]) return fail(nullptr, PX_ERR_ARG, "hybrid: offsets must increase");
  if (d->ny > 1) return h2_create(d, out);  // the reference's 2D two-field testbed (hybrid2d.cu)
  // runs of PPT points per thread, PPT a power of two dividing n, n/PPT ≤ HYB_NT
  int ppt = 0;
  for (int c = 1; c <= 32; c *= 2)
    if (d->nx % c == 0 && d->nx / c <= px::HYB_NT) { ppt = c; break; }
  if (!ppt) return fail(nullptr, PX_ERR_ARG, "hybrid: nx must be a multiple of a power of two ≤ 32 with nx/PPT ≤ 256");
  auto* hy = new Hybrid();
  Handle* hb = &hy->base;
  cudaGetDevice(&hb->device);
  hy->nx = d->nx; hy->B = d->batch; hy->P = P; hy->S = d->offsets[P]; hy->ppt = ppt;
  hy->D = d->D; hy->hx = d->hx; hy->T = d->T; hy->h = d->T / hy->S;
  for (int k = 0; k < 4; ++k) hy->law[k] = d->law[k];
  hy->target_b = d->target_batched ? hy->B : 1;
  hy->offs.assign(d->offsets, d->offsets + P + 1);
  hy->plans.resize(P);
  const size_t n = hy->nx, B = hy->B, S = hy->S;
  hy->lane_smem = 2 * n * sizeof(double);
  hy->bounds_blocks = 148 * 2;
  int rc = PX_OK;
  auto al = [&](double** p, size_t cnt) { if (rc == PX_OK) rc = dalloc_t(hb, p, cnt); };
  al(&hy->u0, B * n); al(&hy->f, B * n); al(&hy->target, (S + 1) * hy->target_b * n); al(&hy->qT, B * n);
  al(&hy->traj, (S + 1) * B * n); al(&hy->J, B); al(&hy->aend, B * P * n); al(&hy->zl, B * P * n);
  al(&hy->ubar, (size_t)P * B * n); al(&hy->qdag0, B * n); al(&hy->grad, B * n);
  al(&hy->bpart, 3 * (size_t)hy->bounds_blocks); al(&hy->bounds, 3);
  if (rc == PX_OK) rc = dalloc_t(hb, &hy->d_offs, (size_t)P + 1);
  if (rc == PX_OK) rc = dalloc_t(hb, &hy->flags, B * P);
  if (rc == PX_OK) rc = dalloc_t(hb, &hy->d_plans, (size_t)P);
  if (rc == PX_OK && cudaMemcpy(hy->d_offs, d->offsets, sizeof(int) * (P + 1), cudaMemcpyHostToDevice) != cudaSuccess)
    rc = fail(hb, PX_ERR_CUDA, "hybrid: offsets upload");
  if (rc == PX_OK) rc = dalloc_t(hb, &hy->theta, 2 * S + 1);
  if (rc == PX_OK) {
    std::vector<double> th(2 * S + 1);
    for (size_t k = 0; k <= 2 * S; ++k) {
      const double t = (double)k * (0.5 * hy->h);
      th[k] = hy->law[0] + hy->law[1] * std::sin(hy->law[3] * t) + hy->law[2] * std::cos(hy->law[3] * t);
    }
    if (cudaMemcpy(hy->theta, th.data(), sizeof(double) * th.size(), cudaMemcpyHostToDevice) != cudaSuccess)
      rc = fail(hb, PX_ERR_CUDA, "hybrid: law table upload");
  }
  if (rc == PX_OK && (cudaStreamCreateWithFlags(&hy->side, cudaStreamNonBlocking) != cudaSuccess ||
                      cudaEventCreateWithFlags(&hy->ev_fork, cudaEventDisableTiming) != cudaSuccess))
    rc = fail(hb, PX_ERR_CUDA, "hybrid: stream/event creation");
  for (int k = 0; k < 4 && rc == PX_OK; ++k)
    if (cudaEventCreate(&hy->ev[k]) != cudaSuccess) rc = fail(hb, PX_ERR_CUDA, "hybrid: event creation");
  if (rc != PX_OK) {
    px_hybrid_destroy(hy);
    return rc;
  }
  *out = hy;
  return PX_OK;
}

void px_hybrid_destroy(void* p) {
  if (!p) return;
  if (pxi::Hybrid2D* h2 = pxi::H2(p)) return pxi::h2_destroy(h2);
  Hybrid* hy = pxi::H(p);
  cudaSetDevice(hy->base.device);
  if (hy->side) cudaStreamSynchronize(hy->side);
  for (void* a : hy->base.allocs) cudaFree(a);
  if (hy->d_coef) cudaFree(hy->d_coef);
  if (hy->side) cudaStreamDestroy(hy->side);
  if (hy->ev_fork) cudaEventDestroy(hy->ev_fork);
  for (auto e : hy->ev)
    if (e) cudaEventDestroy(e);
  delete hy;
}

const char* px_hybrid_last_error(const void* p) {
  return p ? static_cast<const pxi::HybridHead*>(p)->base.err.c_str() : pxi::g_last_error.c_str();
}

int px_hybrid_set_inputs(void* p, const double* u0, const double* f, const double* target, const double* qdag_T,
                         int mem, void* stream) {
  using namespace pxi;
  if (!p || !u0 || !f || !target) return fail(p ? &H(p)->base : nullptr, PX_ERR_ARG, "hybrid inputs: null pointer");
  if (Hybrid2D* h2 = H2(p)) return h2_set_inputs(h2, u0, f, target, qdag_T, mem, (cudaStream_t)stream);
  Hybrid* hy = H(p);
  cudaSetDevice(hy->base.device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t n = hy->nx, B = hy->B;
  PX_TRY(copy_in(hy, hy->u0, u0, B * n, mem, s));
  PX_TRY(copy_in(hy, hy->f, f, B * n, mem, s));
  PX_TRY(copy_in(hy, hy->target, target, (size_t)(hy->S + 1) * hy->target_b * n, mem, s));
  hy->has_qT = qdag_T != nullptr;
  if (qdag_T) PX_TRY(copy_in(hy, hy->qT, qdag_T, B * n, mem, s));
  hy->inputs = true;
  hy->direct_done = hy->adjoint_done = false;
  return PX_OK;
}

int px_hybrid_direct(void* p, int overlap, void* stream) {
  using namespace pxi;
  if (!p) return fail(nullptr, PX_ERR_ARG, "null handle");
  if (Hybrid2D* h2 = H2(p)) return h2_direct(h2, overlap, (cudaStream_t)stream);
  Hybrid* hy = H(p);
  if (!hy->inputs) return fail(&hy->base, PX_ERR_STATE, "hybrid: inputs not set");
  cudaSetDevice(hy->base.device);
  cudaStream_t s = (cudaStream_t)stream;
  px::HybArgs a{};
  a.u0 = hy->u0; a.f = hy->f; a.target = hy->target; a.target_b = hy->target_b;
  a.traj = hy->traj; a.J = hy->J; a.flags = hy->flags; a.offsets = hy->d_offs;
  a.aend = hy->aend; a.zl = hy->zl;
  a.la = hy->law[0]; a.lb = hy->law[1]; a.lc = hy->law[2]; a.lw = hy->law[3];
  a.theta = hy->theta;
  a.D = hy->D; a.hx = hy->hx; a.h = hy->h; a.T = hy->T;
  a.nx = hy->nx; a.B = hy->B; a.P = hy->P; a.S = hy->S;
  // overlap only when every lane CTA and every direct CTA can be resident at once even if each
  // lane took a whole SM (the lanes spin on the flags: a lane waiting for an unscheduled direct
  // CTA must never be possible)
  int sms = 0, per_sm = 0;
  HY_CUDA(hy, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, hy->base.device));
  HY_CUDA(hy, hyb_lanes_occupancy(hy->ppt, hy->lane_smem, &per_sm));
  if (per_sm < 1) return fail(&hy->base, PX_ERR_ARG, "hybrid: the slice kernel does not fit an SM");
  const bool ov = overlap && (long long)hy->B * hy->P + hyb_direct_ctas(hy->nx, hy->B) <= sms;
  HY_CUDA(hy, cudaMemsetAsync(hy->flags, 0, sizeof(int) * hy->B * hy->P, s));
  HY_CUDA(hy, cudaEventRecord(hy->ev[0], s));
  if (ov) {
    HY_CUDA(hy, cudaEventRecord(hy->ev_fork, s));
    HY_CUDA(hy, cudaStreamWaitEvent(hy->side, hy->ev_fork, 0));
    a.wait = 1;
    HY_CUDA(hy, hyb_launch_direct(a, hy->ppt, s));
    HY_CUDA(hy, cudaEventRecord(hy->ev[1], s));
    HY_CUDA(hy, cudaEventRecord(hy->ev[2], hy->side));
    HY_CUDA(hy, hyb_launch_lanes(a, hy->ppt, hy->lane_smem, hy->side));
    HY_CUDA(hy, cudaEventRecord(hy->ev[3], hy->side));
    HY_CUDA(hy, cudaStreamWaitEvent(s, hy->ev[3], 0));  // join
  } else {
    a.wait = 0;
    HY_CUDA(hy, hyb_launch_direct(a, hy->ppt, s));
    HY_CUDA(hy, cudaEventRecord(hy->ev[1], s));
    HY_CUDA(hy, cudaEventRecord(hy->ev[2], s));
    HY_CUDA(hy, hyb_launch_lanes(a, hy->ppt, hy->lane_smem, s));
    HY_CUDA(hy, cudaEventRecord(hy->ev[3], s));
  }
  hy->base.stats.kernel_launches += 2;
  hy->base.stats.rk4_lane_steps += (uint64_t)hy->B * hy->S * 2;
  hy->overlapped = ov ? 1 : 0;
  hy->direct_done = true;
  hy->adjoint_done = false;
  return PX_OK;
}

int px_hybrid_bounds(void* p, double* out3, void* stream) {
  using namespace pxi;
  if (!p || !out3) return fail(p ? &H(p)->base : nullptr, PX_ERR_ARG, "null argument");
  if (Hybrid2D* h2 = H2(p)) return h2_bounds(h2, out3, (cudaStream_t)stream);
  Hybrid* hy = H(p);
  if (!hy->direct_done) return fail(&hy->base, PX_ERR_STATE, "hybrid: run px_hybrid_direct first");
  cudaSetDevice(hy->base.device);
  cudaStream_t s = (cudaStream_t)stream;
  HY_CUDA(hy, hyb_launch_means_bounds(hy->ubar, hy->traj, hy->d_offs, hy->P, hy->B, hy->nx, hy->bpart,
                                      hy->bounds_blocks, hy->bounds, hy->hx, hy->D, s));
  HY_CUDA(hy, cudaMemcpyAsync(out3, hy->bounds, 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
  HY_CUDA(hy, cudaStreamSynchronize(s));
  hy->base.stats.kernel_launches += 3;
  for (int k = 0; k < 3; ++k)
    if (!std::isfinite(out3[k])) return fail(&hy->base, PX_ERR_NONFINITE, "hybrid: non-finite direct trajectory");
  return PX_OK;
}

int px_hybrid_set_slice_plan(void* p, int sl, const px_cheb_plan* plan, const double* gc, const double* gs) {
  using namespace pxi;
  if (!p || !plan || !plan->coef_exp || !plan->coef_phi)
    return fail(p ? &H(p)->base : nullptr, PX_ERR_ARG, "hybrid plan: null argument");
  if (Hybrid2D* h2 = H2(p)) return h2_set_slice_plan(h2, sl, plan, gc, gs);
  Hybrid* hy = H(p);
  if (sl < 0 || sl >= hy->P) return fail(&hy->base, PX_ERR_ARG, "hybrid plan: slice out of range");
  if (plan->substeps < 1 || plan->degree < 1 || !(plan->scale > 0) || (plan->sigma != 1 && plan->sigma != -1))
    return fail(&hy->base, PX_ERR_ARG, "hybrid plan: bad substeps/degree/scale/sigma");
  if (hy->law[3] != 0.0 && (!gc || !gs))
    return fail(&hy->base, PX_ERR_ARG, "hybrid plan: a sine/cosine time law needs the coef_gc / coef_gs series");
  const double span = (hy->offs[sl + 1] - hy->offs[sl]) * hy->h;
  if (std::fabs(plan->span - span) > 1e-12 * std::max(1.0, span))
    return fail(&hy->base, PX_ERR_ARG, "hybrid plan: span does not match the slice width");
  Hybrid::SlicePlan& sp = hy->plans[sl];
  const int K = plan->degree;
  sp.set = true;
  sp.substeps = plan->substeps; sp.degree = K; sp.sigma = plan->sigma;
  sp.c0 = plan->center; sp.d = plan->scale; sp.span = plan->span;
  sp.be.assign(plan->coef_exp, plan->coef_exp + K + 1);
  std::vector<double> bp(plan->coef_phi, plan->coef_phi + K + 1);
  sp.law.assign((size_t)sp.substeps * (K + 1), 0.0);
  const double tau = plan->span / plan->substeps;
  const double t_top = hy->offs[sl + 1] * hy->h;
  for (int j = 0; j < sp.substeps; ++j) law_coef(hy->law, t_top - j * tau, bp, gc, gs, K, sp.law.data() + (size_t)j * (K + 1));
  hy->plans_dirty = true;
  return PX_OK;
}

int px_hybrid_adjoint(void* p, void* stream) {
  using namespace pxi;
  if (!p) return fail(nullptr, PX_ERR_ARG, "null handle");
  if (Hybrid2D* h2 = H2(p)) return h2_adjoint(h2, (cudaStream_t)stream);
  Hybrid* hy = H(p);
  if (!hy->direct_done) return fail(&hy->base, PX_ERR_STATE, "hybrid: run px_hybrid_direct first");
  cudaSetDevice(hy->base.device);
  cudaStream_t s = (cudaStream_t)stream;
  const int top = hy->has_qT ? hy->P - 1 : hy->P - 2;
  for (int q = 0; q <= top; ++q)
    if (!hy->plans[q].set) return fail(&hy->base, PX_ERR_STATE, "hybrid: slice plan " + std::to_string(q) + " not set");
  if (hy->plans_dirty) {
    std::vector<double> pool;
    std::vector<px::HybSlicePlan> table(hy->P);
    for (int q = 0; q < hy->P; ++q) {
      const Hybrid::SlicePlan& sp = hy->plans[q];
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
      HY_CUDA(hy, cudaMalloc(&hy->d_coef, pool.size() * sizeof(double)));
      hy->coef_cap = pool.size();
    }
    HY_CUDA(hy, cudaMemcpy(hy->d_coef, pool.data(), pool.size() * sizeof(double), cudaMemcpyHostToDevice));
    HY_CUDA(hy, cudaMemcpy(hy->d_plans, table.data(), sizeof(px::HybSlicePlan) * hy->P, cudaMemcpyHostToDevice));
    hy->plans_dirty = false;
  }
  px::HybScanArgs a{};
  a.ubar = hy->ubar; a.aend = hy->aend; a.zl = hy->zl; a.qT = hy->has_qT ? hy->qT : nullptr;
  a.plans = hy->d_plans; a.coef = hy->d_coef; a.qdag0 = hy->qdag0; a.grad = hy->grad;
  a.D = hy->D; a.hx = hy->hx; a.T = hy->T; a.nx = hy->nx; a.B = hy->B; a.P = hy->P;
  HY_CUDA(hy, hyb_launch_scan(a, hy->ppt, s));
  hy->base.stats.kernel_launches += 1;
  uint64_t terms = 0;
  for (int q = 0; q <= top; ++q) terms += (uint64_t)hy->plans[q].substeps * hy->plans[q].degree;
  hy->base.stats.exp_terms += terms * hy->B;
  hy->adjoint_done = true;
  return PX_OK;
}

/* Algorithm 2 on the 2D two-field testbed (hybrid2d.cu); the 1D Algorithm 2 is px_nl_*. */
int px_hybrid_nl_init(void* p, void* stream) {
  using namespace pxi;
  if (!p) return fail(nullptr, PX_ERR_ARG, "null handle");
  if (Hybrid2D* h2 = H2(p)) return h2_nl_init(h2, (cudaStream_t)stream);
  return fail(&H(p)->base, PX_ERR_ARG, "px_hybrid_nl_*: the 2D two-field handle (1D: px_nl_init / px_nl_sweep)");
}

int px_hybrid_nl_set_plans(void* p, const px_cheb_plan* slice, const px_cheb_plan* step) {
  using namespace pxi;
  if (!p || !slice || !step) return fail(p ? &H(p)->base : nullptr, PX_ERR_ARG, "null argument");
  if (Hybrid2D* h2 = H2(p)) return h2_nl_set_plans(h2, slice, step);
  return fail(&H(p)->base, PX_ERR_ARG, "px_hybrid_nl_*: the 2D two-field handle");
}

int px_hybrid_nl_sweep(void* p, double* err, void* stream) {
  using namespace pxi;
  if (!p || !err) return fail(p ? &H(p)->base : nullptr, PX_ERR_ARG, "null argument");
  if (Hybrid2D* h2 = H2(p)) return h2_nl_sweep(h2, err, (cudaStream_t)stream);
  return fail(&H(p)->base, PX_ERR_ARG, "px_hybrid_nl_*: the 2D two-field handle");
}

int px_hybrid_nl_finish(void* p, void* stream) {
  using namespace pxi;
  if (!p) return fail(nullptr, PX_ERR_ARG, "null handle");
  if (Hybrid2D* h2 = H2(p)) return h2_nl_finish(h2, (cudaStream_t)stream);
  return fail(&H(p)->base, PX_ERR_ARG, "px_hybrid_nl_*: the 2D two-field handle");
}

int px_hybrid_get(void* p, int field, double* dst, size_t count, int mem, void* stream) {
  using namespace pxi;
  if (!p || !dst) return fail(p ? &H(p)->base : nullptr, PX_ERR_ARG, "null argument");
  if (Hybrid2D* h2 = H2(p)) return h2_get(h2, field, dst, count, mem, (cudaStream_t)stream);
  Hybrid* hy = H(p);
  cudaSetDevice(hy->base.device);
  const size_t n = hy->nx, B = hy->B, P = hy->P, S = hy->S;
  const double* src = nullptr;
  size_t have = 0;
  switch (field) {
    case PX_HFIELD_J: src = hy->J; have = B; break;
    case PX_HFIELD_GRAD: src = hy->grad; have = B * n; break;
    case PX_HFIELD_UT: src = hy->traj + S * B * n; have = B * n; break;
    case PX_HFIELD_QDAG0: src = hy->qdag0; have = B * n; break;
    case PX_HFIELD_TRAJ: src = hy->traj; have = (S + 1) * B * n; break;
    case PX_HFIELD_AEND: src = hy->aend; have = B * P * n; break;
    case PX_HFIELD_ZL: src = hy->zl; have = B * P * n; break;
    case PX_HFIELD_UBAR: src = hy->ubar; have = P * B * n; break;
    default: return fail(&hy->base, PX_ERR_ARG, "hybrid: unknown field");
  }
  const bool needs_adj = field == PX_HFIELD_GRAD || field == PX_HFIELD_QDAG0;
  if ((needs_adj && !hy->adjoint_done) || (!needs_adj && !hy->direct_done))
    return fail(&hy->base, PX_ERR_STATE, "hybrid: field not computed yet");
  if (count != have) return fail(&hy->base, PX_ERR_ARG, "hybrid: count mismatch (" + std::to_string(have) + ")");
  cudaStream_t s = (cudaStream_t)stream;
  HY_CUDA(hy, cudaMemcpyAsync(dst, src, count * sizeof(double),
                              mem == PX_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
  if (mem != PX_MEM_DEVICE) HY_CUDA(hy, cudaStreamSynchronize(s));
  return PX_OK;
}

int px_hybrid_get_timing(void* p, double* ms) {
  using namespace pxi;
  if (!p || !ms) return fail(p ? &H(p)->base : nullptr, PX_ERR_ARG, "null argument");
  if (Hybrid2D* h2 = H2(p)) return h2_get_timing(h2, ms);
  Hybrid* hy = H(p);
  if (!hy->direct_done) return fail(&hy->base, PX_ERR_STATE, "hybrid: no direct sweep timed");
  cudaSetDevice(hy->base.device);
  HY_CUDA(hy, cudaEventSynchronize(hy->ev[3]));
  HY_CUDA(hy, cudaEventSynchronize(hy->ev[1]));
  float a = 0, b = 0, c = 0, e = 0;
  HY_CUDA(hy, cudaEventElapsedTime(&a, hy->ev[0], hy->ev[1]));
  HY_CUDA(hy, cudaEventElapsedTime(&b, hy->ev[2], hy->ev[3]));
  HY_CUDA(hy, cudaEventElapsedTime(&c, hy->ev[0], hy->ev[3]));
  HY_CUDA(hy, cudaEventElapsedTime(&e, hy->ev[1], hy->ev[3]));
  ms[0] = a;
  ms[1] = b;
  ms[2] = std::max(a, c);
  ms[3] = e;  // the slice solves' tail after the serial sweep ended
  ms[4] = hy->overlapped;
  return PX_OK;
}

}  // extern "C"
