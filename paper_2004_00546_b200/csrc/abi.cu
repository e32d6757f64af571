// abi.cu — the C ABI (include/paraexp.h): argument checks, handle lifetime, plans,
// variants, the phase entry points, CUDA-graph capture/replay of the gradient and field
// access. The sweeps themselves are in sweeps.cu / burgers.cu.
#include <cmath>

#include <nvtx3/nvToolsExt.h>

#include "internal.h"

using pxi::Handle;
using pxi::Plan;
using pxi::fail;

namespace {

// the handle's device (the static cudart keeps a per-thread current device)
Handle* bind(void* handle) {
  Handle* h = static_cast<Handle*>(handle);
  if (h) cudaSetDevice(h->device);
  return h;
}

int gradient_phases(Handle* h, void* stream);

int capture_gradient(Handle* h) {
  pxi::drop_segments(h);
  const px_stats before = h->stats;
  h->capturing = true;
  h->cap_error = 0;
  pxi::seg_open(h, -1);
  const int rc = gradient_phases(h, h->gstream);
  pxi::seg_close(h);
  h->capturing = false;
  if (rc != PX_OK || h->cap_error) {
    pxi::drop_segments(h);
    h->stats = before;
    if (rc != PX_OK) return rc;
    return fail(h, PX_ERR_CUDA, "graph capture failed");
  }
  px_stats d{};
  d.rk4_lane_steps = h->stats.rk4_lane_steps - before.rk4_lane_steps;
  d.exp_terms = h->stats.exp_terms - before.exp_terms;
  d.arnoldi_steps = h->stats.arnoldi_steps - before.arnoldi_steps;
  d.kernel_launches = h->stats.kernel_launches - before.kernel_launches;
  d.algorithmic_bytes = h->stats.algorithmic_bytes - before.algorithmic_bytes;
  d.rk4_bytes = h->stats.rk4_bytes - before.rk4_bytes;
  d.exp_bytes = h->stats.exp_bytes - before.exp_bytes;
  h->graph_delta = d;
  h->stats = before;
  h->graph_valid = true;
  return PX_OK;
}

}  // namespace

extern "C" {

int px_abi_version(void) { return PX_ABI_VERSION; }

const char* px_build_info(void) {
  return "paraexp sm_100a fp64 (row-marching Horner RK4, on-chip 1D lanes, Chebyshev fused recurrence, "
         "Arnoldi CGS2, Burgers serial sweep)";
}

const char* px_last_error(const void* handle) {
  const Handle* h = static_cast<const Handle*>(handle);
  if (h && !h->err.empty()) return h->err.c_str();
  return pxi::g_last_error.c_str();
}

int px_create(const px_problem_desc* desc, void** out_handle) {
  if (!desc || !out_handle) return fail(nullptr, PX_ERR_ARG, "null argument");
  const px_problem_desc& d = *desc;
  if (d.nx < 3 || d.ny < 1 || (d.ny > 1 && d.ny < 3)) return fail(nullptr, PX_ERR_ARG, "bad grid");
  if (d.P < 1 || d.nsteps < 1 || d.batch < 1 || d.K < 1) return fail(nullptr, PX_ERR_ARG, "bad sizes");
  if (d.p_begin < 0 || d.p_end > d.P || d.p_begin >= d.p_end) return fail(nullptr, PX_ERR_ARG, "bad slice block");
  if (!(d.T > 0)) return fail(nullptr, PX_ERR_ARG, "T must be positive");
  if (d.kind != PX_KIND_ADVDIFF && d.kind != PX_KIND_BURGERS) return fail(nullptr, PX_ERR_ARG, "bad kind");
  if (d.kind == PX_KIND_BURGERS && d.ny != 1) return fail(nullptr, PX_ERR_ARG, "px_create: Burgers is 1D on this handle (terminal objective); the two-field 2D testbed runs through px_hybrid_* (desc.ny > 1: solve_hybrid_tracking / solve_nonlinear_tracking)");
  if (d.expaction == PX_EXP_KRYLOV && (d.krylov_m < 2 || d.krylov_m > px::KRYLOV_MAX_M))
    return fail(nullptr, PX_ERR_ARG, "krylov_m out of range");
  if (d.basis_rows_x < 1 || d.basis_rows_x > 64 || d.basis_rows_y < 1)
    return fail(nullptr, PX_ERR_ARG, "bad basis table sizes");
  if ((d.flags & PX_FLAG_FIELD_CONTROL) &&
      (d.kind != PX_KIND_ADVDIFF || (size_t)d.K != (size_t)d.nx * d.ny))
    return fail(nullptr, PX_ERR_ARG, "field control: advection–diffusion with K = n");
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return fail(nullptr, PX_ERR_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));

  Handle* h = new Handle();
  h->d = d;
  cudaGetDevice(&h->device);
  h->dim = d.ny == 1 ? 1 : 2;
  h->n = (size_t)d.nx * d.ny;
  h->B = d.batch;
  h->K = d.K;
  h->Pl = d.p_end - d.p_begin;
  h->L = h->B * h->Pl;
  h->rows_x = d.basis_rows_x;
  h->rows_y = d.basis_rows_y;
  h->A = {d.stencil[0], d.stencil[1], d.stencil[2], d.stencil[3], d.stencil[4]};
  h->AT = {d.stencil[0], d.stencil[2], d.stencil[1], d.stencil[4], d.stencil[3]};
  const size_t n = h->n, B = h->B;
  int rc = PX_OK;
  auto A = [&](double** p, size_t cnt) { if (rc == PX_OK) rc = pxi::dalloc_t(h, p, cnt); };
  A(&h->u0, n);
  A(&h->ut, n);
  A(&h->ctrl, B * h->K);
  const bool field_ctl = (d.flags & PX_FLAG_FIELD_CONTROL) != 0;
  A(&h->tx, field_ctl ? 1 : (size_t)h->rows_x * d.nx);
  A(&h->ty, field_ctl ? 1 : (size_t)h->rows_y * d.ny);
  if (rc == PX_OK) rc = pxi::dalloc_t(h, &h->ix, field_ctl ? 1 : h->K);
  if (rc == PX_OK) rc = pxi::dalloc_t(h, &h->iy, field_ctl ? 1 : h->K);
  h->basis_set = field_ctl;  // a field control needs no basis tables
  A(&h->UT, B * n);
  A(&h->QT, B * n);
  A(&h->QDAG0, B * n);
  A(&h->G, B * n);
  A(&h->J, B);
  A(&h->GRAD, B * h->K);
  A(&h->R, field_ctl ? 1 : B * h->rows_x * d.ny);
  h->red_blocks = (int)std::min<size_t>((n + 255) / 256, 1024);
  A(&h->partial, B * h->red_blocks);
  if (rc == PX_OK) rc = pxi::dalloc_t(h, &h->nonfinite, 1);
  for (int i = 0; i < 4; ++i) A(&h->Wk[i], B * n);
  for (int i = 0; i < 2; ++i) A(&h->ACC[i], B * n);
  if (d.kind == PX_KIND_ADVDIFF && h->dim == 2) A(&h->S, B * n);
  if (d.kind == PX_KIND_ADVDIFF) {
    A(&h->g, B * n);
    A(&h->gadj, B * n);
    A(&h->bsrc, B * n);
    A(&h->cz, B * n);
    A(&h->Y0, (size_t)h->L * n);
    A(&h->Y1, (size_t)h->L * n);
    // 2D: the adjoint ∫ in closed form (one FFT solve), no per-lane accumulator in HBM
    h->z_closed = h->dim == 2 && !(d.flags & PX_FLAG_Z_ACCUM);
    if (h->z_closed) {
      A(reinterpret_cast<double**>(&h->fbuf), 2 * B * n);
      A(&h->bsum, B);
      int dims[2] = {d.ny, d.nx};
      if (rc == PX_OK &&
          cufftPlanMany(&h->fft, 2, dims, nullptr, 1, 0, nullptr, 1, 0, CUFFT_Z2Z, (int)B) != CUFFT_SUCCESS) {
        pxi::g_last_error = "cufftPlanMany failed";
        rc = PX_ERR_CUDA;
      }
    } else {
      A(&h->Z, (size_t)h->L * n);
    }
    if ((d.flags & PX_FLAG_BOUNDARY_STATES) && d.p_begin == 0 && d.p_end == d.P)
      A(&h->UBND, B * (size_t)(d.P + 1) * n);
  } else {
    const size_t S = (size_t)d.P * d.nsteps;
    A(&h->traj, (S + 1) * B * n);
    if (d.p_begin == 0 && d.p_end == d.P) {
      A(&h->traj_b, (S + 1) * B * n);
      A(&h->Dc, (size_t)(d.P + 1) * B * n);
      A(&h->nl_err, B * (size_t)d.P);
    }
    A(&h->ubar, (size_t)d.P * B * n);
    h->bounds_blocks = (int)std::min<size_t>(((size_t)d.P * B * n + 255) / 256, 1024);
    A(&h->bpart, 3 * (size_t)h->bounds_blocks);
    A(&h->bounds, 3);
    A(&h->Y0, (size_t)h->L * n);
    A(&h->Y1, (size_t)h->L * n);
    A(&h->Z, (size_t)h->L * n);
  }
  if (rc == PX_OK && d.expaction == PX_EXP_KRYLOV) rc = pxi::krylov_alloc(h->kw, d.krylov_m, n, B, &pxi::g_last_error);
  if (rc != PX_OK) {
    std::string msg = pxi::g_last_error;
    px_destroy(h);
    pxi::g_last_error = msg;
    return rc;
  }
  if (cudaMemset(h->nonfinite, 0, sizeof(int)) != cudaSuccess) {
    px_destroy(h);
    return fail(nullptr, PX_ERR_CUDA, "memset failed");
  }
  *out_handle = h;
  return PX_OK;
}

void px_destroy(void* handle) {
  Handle* h = bind(handle);
  if (!h) return;
  for (void* p : h->allocs) cudaFree(p);
  for (auto& pl : h->plans)
    if (pl.dcoef) cudaFree(pl.dcoef);
  for (auto& m : h->marks) {
    cudaEventDestroy(m.a);
    cudaEventDestroy(m.b);
  }
  for (auto& m : h->kmarks) {
    cudaEventDestroy(m.a);
    cudaEventDestroy(m.b);
  }
  pxi::drop_segments(h);
  if (h->gstream) cudaStreamDestroy(h->gstream);
  if (h->ev_in) cudaEventDestroy(h->ev_in);
  if (h->ev_out) cudaEventDestroy(h->ev_out);
  for (auto e : h->event_pool) cudaEventDestroy(e);
  pxi::krylov_free(h->kw);
  if (h->fft) cufftDestroy(h->fft);
  pxi::free_blocks(h);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  delete h;
}

int px_set_basis(void* handle, const double* tx, const double* ty, const int* ix, const int* iy) {
  Handle* h = bind(handle);
  if (!h || !tx || !ty || !ix || !iy) return fail(h, PX_ERR_ARG, "null argument");
  if (h->d.flags & PX_FLAG_FIELD_CONTROL) return fail(h, PX_ERR_STATE, "field control has no basis tables");
  for (int k = 0; k < h->K; ++k)
    if (ix[k] < 0 || ix[k] >= h->rows_x || iy[k] < 0 || iy[k] >= h->rows_y)
      return fail(h, PX_ERR_ARG, "basis index out of range");
  PX_CUDA(h, cudaMemcpy(h->tx, tx, sizeof(double) * h->rows_x * h->d.nx, cudaMemcpyHostToDevice));
  PX_CUDA(h, cudaMemcpy(h->ty, ty, sizeof(double) * h->rows_y * h->d.ny, cudaMemcpyHostToDevice));
  PX_CUDA(h, cudaMemcpy(h->ix, ix, sizeof(int) * h->K, cudaMemcpyHostToDevice));
  PX_CUDA(h, cudaMemcpy(h->iy, iy, sizeof(int) * h->K, cudaMemcpyHostToDevice));
  h->basis_set = true;
  return PX_OK;
}

int px_set_cheb_plan(void* handle, int slot, const px_cheb_plan* p) {
  Handle* h = bind(handle);
  if (!h || !p) return fail(h, PX_ERR_ARG, "null argument");
  if (slot < 0 || slot >= PX_PLAN_COUNT) return fail(h, PX_ERR_ARG, "bad plan slot");
  if (p->substeps < 1 || p->degree < 1 || !(p->scale > 0) || (p->sigma != 1 && p->sigma != -1) || !p->coef_exp)
    return fail(h, PX_ERR_ARG, "bad Chebyshev plan");
  Plan& pl = h->plans[slot];
  h->graph_valid = false;
  pl.set = true;
  pl.krylov = false;
  pl.span = p->span;
  pl.substeps = p->substeps;
  pl.degree = p->degree;
  pl.center = p->center;
  pl.scale = p->scale;
  pl.sigma = p->sigma;
  pl.be.assign(p->coef_exp, p->coef_exp + p->degree + 1);
  if (p->coef_phi) pl.bp.assign(p->coef_phi, p->coef_phi + p->degree + 1);
  else pl.bp.assign(p->degree + 1, 0.0);
  if (pl.dcoef) cudaFree(pl.dcoef);
  pl.dcoef = nullptr;
  PX_CUDA(h, cudaMalloc(&pl.dcoef, sizeof(double) * 2 * (p->degree + 1)));
  PX_CUDA(h, cudaMemcpy(pl.dcoef, pl.be.data(), sizeof(double) * (p->degree + 1), cudaMemcpyHostToDevice));
  PX_CUDA(h, cudaMemcpy(pl.dcoef + p->degree + 1, pl.bp.data(), sizeof(double) * (p->degree + 1),
                        cudaMemcpyHostToDevice));
  return PX_OK;
}

int px_set_cheb_plan_law(void* handle, int slot, const double* gc, const double* gs) {
  Handle* h = bind(handle);
  if (!h || !gc || !gs) return fail(h, PX_ERR_ARG, "null argument");
  if (slot < 0 || slot >= PX_PLAN_COUNT) return fail(h, PX_ERR_ARG, "bad plan slot");
  Plan& pl = h->plans[slot];
  if (!pl.set || pl.krylov) return fail(h, PX_ERR_STATE, "set the Chebyshev plan of this slot first");
  pl.gc.assign(gc, gc + pl.degree + 1);
  pl.gs.assign(gs, gs + pl.degree + 1);
  h->graph_valid = false;
  return PX_OK;
}

int px_set_time_law(void* handle, const double* law) {
  Handle* h = bind(handle);
  if (!h || !law) return fail(h, PX_ERR_ARG, "null argument");
  for (int k = 0; k < 4; ++k)
    if (!std::isfinite(law[k])) return fail(h, PX_ERR_ARG, "time law: non-finite coefficient");
  if (law[3] < 0) return fail(h, PX_ERR_ARG, "time law: ω must be non-negative");
  const bool constant = law[0] == 1.0 && law[1] == 0.0 && law[2] == 0.0;
  if (!constant && h->d.kind != PX_KIND_ADVDIFF)
    return fail(h, PX_ERR_ARG, "time law: the linear testbed (Burgers: the px_hybrid handle)");
  if (!constant && h->d.expaction != PX_EXP_CHEBYSHEV)
    return fail(h, PX_ERR_ARG, "time law: Chebyshev exp-actions only");
  if (!constant && !h->fctl) PX_TRY(pxi::dalloc_t(h, &h->fctl, (size_t)h->B * h->n));
  for (int k = 0; k < 4; ++k) h->law[k] = law[k];
  h->has_law = !constant;
  if (h->tracking) PX_TRY(pxi::tracking_theta(h));
  // the closed-form adjoint ∫ holds for the time-constant weight only
  h->z_closed = !h->has_law && h->dim == 2 && !(h->d.flags & PX_FLAG_Z_ACCUM);
  if (h->has_law && h->dim == 2 && !h->Z) PX_TRY(pxi::dalloc_t(h, &h->Z, (size_t)h->L * h->n));
  h->graph_valid = false;
  return PX_OK;
}

int px_set_tracking_target(void* handle, const double* target, int per_member, int mem, void* stream) {
  Handle* h = bind(handle);
  if (!h) return fail(h, PX_ERR_ARG, "null handle");
  if (h->d.kind != PX_KIND_ADVDIFF)
    return fail(h, PX_ERR_ARG, "tracking objective: the linear testbed (Burgers: the px_hybrid handle)");
  if (h->d.p_begin != 0 || h->d.p_end != h->d.P) return fail(h, PX_ERR_ARG, "tracking objective: one rank");
  if (per_member != 0 && per_member != 1) return fail(h, PX_ERR_ARG, "per_member must be 0 or 1");
  PX_TRY(pxi::tracking_set(h, target, per_member, mem, static_cast<cudaStream_t>(stream)));
  h->stage = 0;
  return PX_OK;
}

int px_set_krylov_plan(void* handle, int slot, double span, int substeps) {
  Handle* h = bind(handle);
  if (!h) return fail(h, PX_ERR_ARG, "null handle");
  if (slot < 0 || slot >= PX_PLAN_COUNT) return fail(h, PX_ERR_ARG, "bad plan slot");
  if (h->d.expaction != PX_EXP_KRYLOV) return fail(h, PX_ERR_ARG, "handle not created for Krylov");
  if (substeps < 1 || !(span > 0)) return fail(h, PX_ERR_ARG, "bad Krylov plan");
  Plan& pl = h->plans[slot];
  h->graph_valid = false;
  pl.set = true;
  pl.krylov = true;
  pl.span = span;
  pl.substeps = substeps;
  pl.degree = h->d.krylov_m;
  return PX_OK;
}

int px_set_variant(void* handle, int key, int value) {
  Handle* h = bind(handle);
  if (!h) return fail(h, PX_ERR_ARG, "null handle");
  pxi::Variants& v = h->var;
  switch (key) {
    case PX_VAR_MARCH2:
      if (value < 0 || value > 2) return fail(h, PX_ERR_ARG, "PX_VAR_MARCH2 must be 0, 1 or 2");
      v.march2 = value; break;
    case PX_VAR_MARCH_COLS:
      if (value != 2 && value != 3) return fail(h, PX_ERR_ARG, "PX_VAR_MARCH_COLS must be 2 or 3");
      v.march_cols = value; break;
    case PX_VAR_MARCH_BAND:
      if (value < 0) return fail(h, PX_ERR_ARG, "PX_VAR_MARCH_BAND must be ≥ 0");
      v.march_band = value; break;
    case PX_VAR_CHEB_TERMS:
      if (value < 1 || value > 7) return fail(h, PX_ERR_ARG, "PX_VAR_CHEB_TERMS must be 1 … 7");
      v.cheb_terms = value; break;
    case PX_VAR_CHEB_TERMS_PHI:
      if (value < 1 || value > 7) return fail(h, PX_ERR_ARG, "PX_VAR_CHEB_TERMS_PHI must be 1 … 7");
      v.cheb_terms_phi = value; break;
    case PX_VAR_CHEB_STRIP:
      if (value < 0 || (value & 1)) return fail(h, PX_ERR_ARG, "PX_VAR_CHEB_STRIP must be even and ≥ 0");
      v.cheb_strip = value; break;
    case PX_VAR_CHEB_BAND:
      if (value < 0) return fail(h, PX_ERR_ARG, "PX_VAR_CHEB_BAND must be ≥ 0");
      v.cheb_band = value; break;
    case PX_VAR_SCAN1D_CLUSTER: v.scan1d_cluster = value != 0; break;
    case PX_VAR_KRYLOV_ORTHO:
      if (value != 0 && value != 1) return fail(h, PX_ERR_ARG, "PX_VAR_KRYLOV_ORTHO must be 0 or 1");
      v.krylov_ortho = value; break;
    case PX_VAR_BURGERS_CLUSTER: v.burgers_cluster = value != 0; break;
    default: return fail(h, PX_ERR_ARG, "unknown variant key");
  }
  h->graph_valid = false;
  return PX_OK;
}

int px_get_variant(void* handle, int key, int* value) {
  Handle* h = static_cast<Handle*>(handle);
  if (!h || !value) return fail(h, PX_ERR_ARG, "null argument");
  const pxi::Variants& v = h->var;
  switch (key) {
    case PX_VAR_MARCH2: *value = v.march2; break;
    case PX_VAR_MARCH_COLS: *value = v.march_cols; break;
    case PX_VAR_MARCH_BAND: *value = v.march_band; break;
    case PX_VAR_CHEB_TERMS: *value = v.cheb_terms; break;
    case PX_VAR_CHEB_TERMS_PHI: *value = v.cheb_terms_phi; break;
    case PX_VAR_CHEB_STRIP: *value = v.cheb_strip; break;
    case PX_VAR_CHEB_BAND: *value = v.cheb_band; break;
    case PX_VAR_SCAN1D_CLUSTER: *value = v.scan1d_cluster; break;
    case PX_VAR_BURGERS_CLUSTER: *value = v.burgers_cluster; break;
    case PX_VAR_KRYLOV_ORTHO: *value = v.krylov_ortho; break;
    default: return fail(h, PX_ERR_ARG, "unknown variant key");
  }
  return PX_OK;
}

int px_set_adjoint_mode(void* handle, int mode) {
  Handle* h = bind(handle);
  if (!h) return fail(h, PX_ERR_ARG, "null handle");
  if (mode != PX_ADJOINT_ABSORBED && mode != PX_ADJOINT_FROZEN_SPAN) return fail(h, PX_ERR_ARG, "unknown adjoint mode");
  if (mode == PX_ADJOINT_FROZEN_SPAN && h->d.kind != PX_KIND_BURGERS)
    return fail(h, PX_ERR_ARG, "the frozen-span adjoint is the Burgers hybrid's (solve_hybrid)");
  if (mode != h->adjoint_mode) {
    h->adjoint_mode = mode;
    h->graph_valid = false;
  }
  return PX_OK;
}

int px_set_local_blocks(void* handle, int blocks) {
  Handle* h = bind(handle);
  if (!h) return fail(h, PX_ERR_ARG, "null handle");
  if (blocks < 1 || blocks > PX_MAX_LOCAL_BLOCKS || blocks > h->Pl || h->Pl % blocks != 0)
    return fail(h, PX_ERR_ARG, "local blocks must divide the rank's slice count (1 … 16)");
  return pxi::set_local_blocks(h, blocks);
}

int px_set_local_block_sizes(void* handle, int blocks, const int* sizes) {
  Handle* h = bind(handle);
  if (!h || !sizes) return fail(h, PX_ERR_ARG, "null argument");
  if (blocks < 1 || blocks > PX_MAX_LOCAL_BLOCKS || blocks > h->Pl)
    return fail(h, PX_ERR_ARG, "local blocks: 1 … 16 and at most the rank's slice count");
  int sum = 0;
  for (int g = 0; g < blocks; ++g) {
    if (sizes[g] < 1) return fail(h, PX_ERR_ARG, "local blocks: every block needs a slice");
    sum += sizes[g];
  }
  if (sum != h->Pl) return fail(h, PX_ERR_ARG, "local blocks: the sizes must add up to the rank's slices");
  return pxi::set_local_blocks(h, blocks, sizes);
}

int px_set_inputs(void* handle, const double* u0, const double* u_target, const double* ctrl, int mem,
                  void* stream) {
  Handle* h = bind(handle);
  if (!h || !u0 || !u_target || !ctrl) return fail(h, PX_ERR_ARG, "null argument");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const cudaMemcpyKind kind = mem == PX_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  PX_CUDA(h, cudaMemcpyAsync(h->u0, u0, sizeof(double) * h->n, kind, s));
  PX_CUDA(h, cudaMemcpyAsync(h->ut, u_target, sizeof(double) * h->n, kind, s));
  PX_CUDA(h, cudaMemcpyAsync(h->ctrl, ctrl, sizeof(double) * h->B * h->K, kind, s));
  h->inputs_set = true;
  h->stage = 0;
  return PX_OK;
}

int px_direct(void* handle, void* stream) {
  Handle* h = bind(handle);
  if (!h) return fail(h, PX_ERR_ARG, "null handle");
  if (!h->basis_set || !h->inputs_set) return fail(h, PX_ERR_STATE, "basis/inputs not set");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int rc;
  if (h->d.kind == PX_KIND_ADVDIFF) {
    if (h->Pl > 1 && !h->plans[PX_PLAN_SLICE].set) return fail(h, PX_ERR_STATE, "slice plan not set");
    if (h->d.p_end < h->d.P && !h->plans[PX_PLAN_LONG_DIRECT].set)
      return fail(h, PX_ERR_STATE, "long-span direct plan not set");
    rc = pxi::direct_linear(h, s);
  } else {
    const int tm = pxi::tbegin(h, PX_PHASE_RK4_DIRECT, s);
    rc = pxi::burgers_direct(h, s);
    pxi::tend(h, tm, s);
  }
  if (rc == PX_OK) h->stage = 1;
  return rc;
}

int px_finish_direct(void* handle, void* stream) {
  Handle* h = bind(handle);
  if (!h) return fail(h, PX_ERR_ARG, "null handle");
  if (h->stage != 1) return fail(h, PX_ERR_STATE, "px_finish_direct before px_direct");
  int rc = pxi::finish_direct_impl(h, static_cast<cudaStream_t>(stream));
  if (rc == PX_OK) h->stage = 2;
  return rc;
}

int px_nl_init(void* handle, void* stream) {
  Handle* h = bind(handle);
  if (!h) return fail(h, PX_ERR_ARG, "null handle");
  if (h->d.kind != PX_KIND_BURGERS || !h->traj_b) return fail(h, PX_ERR_ARG, "iterative direct: Burgers, one rank");
  if (!h->inputs_set || !h->basis_set) return fail(h, PX_ERR_STATE, "basis/inputs not set");
  PX_TRY(pxi::nl_init(h, static_cast<cudaStream_t>(stream)));
  h->stage = 0;
  return PX_OK;
}

int px_nl_prepare(void* handle, void* stream) {
  Handle* h = bind(handle);
  if (!h || !h->traj_b) return fail(h, PX_ERR_ARG, "iterative direct not available");
  return pxi::nl_means_bounds(h, static_cast<cudaStream_t>(stream));
}

int px_nl_sweep(void* handle, double* err_max, void* stream) {
  Handle* h = bind(handle);
  if (!h || !h->traj_b || !err_max) return fail(h, PX_ERR_ARG, "iterative direct not available");
  return pxi::nl_sweep(h, err_max, static_cast<cudaStream_t>(stream));
}

int px_nl_finish(void* handle, void* stream) {
  Handle* h = bind(handle);
  if (!h || !h->traj_b) return fail(h, PX_ERR_ARG, "iterative direct not available");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t S = (size_t)h->d.P * h->d.nsteps;
  PX_CUDA(h, cudaMemcpyAsync(h->UT, h->traj + S * h->B * h->n, sizeof(double) * h->B * h->n,
                             cudaMemcpyDeviceToDevice, s));
  PX_TRY(pxi::nl_means_bounds(h, s));
  h->stage = 1;
  return PX_OK;
}

int px_set_adjoint_terminal(void* handle, const double* qdag_T, int mem, void* stream) {
  Handle* h = bind(handle);
  if (!h || !qdag_T) return fail(h, PX_ERR_ARG, "null argument");
  if (!h->basis_set) return fail(h, PX_ERR_STATE, "basis not set");
  if (h->d.kind == PX_KIND_BURGERS && h->stage < 1)
    return fail(h, PX_ERR_STATE, "Burgers adjoint needs the direct trajectory (px_direct)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const cudaMemcpyKind kind = mem == PX_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  PX_CUDA(h, cudaMemcpyAsync(h->QT, qdag_T, sizeof(double) * h->B * h->n, kind, s));
  if (h->d.kind == PX_KIND_ADVDIFF)
    PX_TRY(pxi::apply_plus_control(h, h->gadj, h->QT, (long long)h->n, h->AT, false, s));
  h->stage = 2;
  return PX_OK;
}

int px_adjoint(void* handle, void* stream) {
  Handle* h = bind(handle);
  if (!h) return fail(h, PX_ERR_ARG, "null handle");
  if (h->stage != 2) return fail(h, PX_ERR_STATE, "px_adjoint before px_finish_direct");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int rc;
  if (h->d.kind == PX_KIND_ADVDIFF) {
    if (h->d.p_begin > 0 && !h->plans[PX_PLAN_LONG_ADJOINT].set)
      return fail(h, PX_ERR_STATE, "long-span adjoint plan not set");
    rc = pxi::adjoint_linear(h, s);
  } else {
    const int tm = pxi::tbegin(h, PX_PHASE_RK4_ADJOINT, s);
    rc = pxi::burgers_adjoint(h, s);
    pxi::tend(h, tm, s);
    if (rc == PX_OK) rc = pxi::project(h, h->GRAD, h->G, (long long)h->n, 1.0, 0.0, s);
  }
  if (rc == PX_OK) h->stage = 3;
  return rc;
}

int px_finish_adjoint(void* handle, void* stream) {
  Handle* h = bind(handle);
  if (!h) return fail(h, PX_ERR_ARG, "null handle");
  if (h->stage != 3) return fail(h, PX_ERR_STATE, "px_finish_adjoint before px_adjoint");
  int rc = pxi::finish_adjoint_impl(h, static_cast<cudaStream_t>(stream));
  if (rc == PX_OK) h->stage = 4;
  return rc;
}

int px_gradient(void* handle, void* stream) {
  Handle* h = bind(handle);
  if (!h) return fail(h, PX_ERR_ARG, "null handle");
  if (h->d.kind != PX_KIND_ADVDIFF) return fail(h, PX_ERR_ARG, "px_gradient: linear testbed only");
  if (!h->graphs || h->timing >= 2) return gradient_phases(h, stream);
  if (!h->basis_set || !h->inputs_set) return fail(h, PX_ERR_STATE, "basis/inputs not set");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!h->gstream) {
    PX_CUDA(h, cudaStreamCreateWithFlags(&h->gstream, cudaStreamNonBlocking));
    PX_CUDA(h, cudaEventCreateWithFlags(&h->ev_in, cudaEventDisableTiming));
    PX_CUDA(h, cudaEventCreateWithFlags(&h->ev_out, cudaEventDisableTiming));
  }
  if (!h->graph_valid) PX_TRY(capture_gradient(h));
  // order: caller's stream -> graph stream -> caller's stream
  PX_CUDA(h, cudaEventRecord(h->ev_in, s));
  PX_CUDA(h, cudaStreamWaitEvent(h->gstream, h->ev_in, 0));
  nvtxRangePushA("px.gradient(graph)");
  for (auto& sg : h->segs) {
    if (sg.phase >= 0) nvtxRangePushA(pxi::phase_name(sg.phase));
    cudaError_t e;
    if (h->timing && sg.phase >= 0) {
      Handle::TMark m{sg.phase, pxi::take_event(h), pxi::take_event(h), sg.launches, sg.bytes};
      cudaEventRecord(m.a, h->gstream);
      e = cudaGraphLaunch(sg.exec, h->gstream);
      cudaEventRecord(m.b, h->gstream);
      h->marks.push_back(m);
    } else {
      e = cudaGraphLaunch(sg.exec, h->gstream);
    }
    if (sg.phase >= 0) nvtxRangePop();
    if (e != cudaSuccess) {
      nvtxRangePop();
      return fail(h, PX_ERR_CUDA, std::string("cudaGraphLaunch: ") + cudaGetErrorString(e));
    }
  }
  nvtxRangePop();
  PX_CUDA(h, cudaEventRecord(h->ev_out, h->gstream));
  PX_CUDA(h, cudaStreamWaitEvent(s, h->ev_out, 0));
  const px_stats& d = h->graph_delta;
  h->stats.rk4_lane_steps += d.rk4_lane_steps;
  h->stats.exp_terms += d.exp_terms;
  h->stats.arnoldi_steps += d.arnoldi_steps;
  h->stats.kernel_launches += d.kernel_launches;
  h->stats.algorithmic_bytes += d.algorithmic_bytes;
  h->stats.rk4_bytes += d.rk4_bytes;
  h->stats.exp_bytes += d.exp_bytes;
  h->stage = 4;
  return PX_OK;
}

int px_set_graphs(void* handle, int enable) {
  Handle* h = static_cast<Handle*>(handle);
  if (!h) return fail(h, PX_ERR_ARG, "null handle");
  h->graphs = enable != 0;
  h->graph_valid = false;
  return PX_OK;
}

int px_buffer(void* handle, int field, double** dev_ptr, size_t* count) {
  Handle* h = static_cast<Handle*>(handle);
  if (!h || !dev_ptr || !count) return fail(h, PX_ERR_ARG, "null argument");
  const size_t Bn = (size_t)h->B * h->n;
  switch (field) {
    case PX_FIELD_J: *dev_ptr = h->J; *count = h->B; break;
    case PX_FIELD_GRAD: *dev_ptr = h->GRAD; *count = (size_t)h->B * h->K; break;
    case PX_FIELD_UT: *dev_ptr = h->UT; *count = Bn; break;
    case PX_FIELD_QDAG0: *dev_ptr = h->QDAG0; *count = Bn; break;
    case PX_FIELD_G: *dev_ptr = h->G; *count = Bn; break;
    case PX_FIELD_UBND:
      if (!h->UBND) return fail(h, PX_ERR_STATE, "boundary states not enabled");
      *dev_ptr = h->UBND; *count = Bn * (h->d.P + 1); break;
    case PX_FIELD_FROZEN_BOUNDS:
      if (!h->bounds) return fail(h, PX_ERR_STATE, "no frozen bounds (linear testbed)");
      *dev_ptr = h->bounds; *count = 3; break;
    case PX_FIELD_VEND:
      if (!h->vend) return fail(h, PX_ERR_STATE, "direct lanes not computed");
      *dev_ptr = const_cast<double*>(h->vend); *count = (size_t)h->L * h->n; break;
    case PX_FIELD_WEND:
      if (!h->wend) return fail(h, PX_ERR_STATE, "adjoint lanes not computed");
      *dev_ptr = const_cast<double*>(h->wend); *count = (size_t)h->L * h->n; break;
    case PX_FIELD_TRAJ:
      if (!h->traj) return fail(h, PX_ERR_STATE, "no trajectory (linear testbed)");
      *dev_ptr = h->traj; *count = ((size_t)h->d.P * h->d.nsteps + 1) * Bn; break;
    default: return fail(h, PX_ERR_ARG, "bad field");
  }
  return PX_OK;
}

int px_get(void* handle, int field, double* dst, size_t count, int mem, void* stream) {
  Handle* h = bind(handle);
  double* src = nullptr;
  size_t have = 0;
  PX_TRY(px_buffer(handle, field, &src, &have));
  if (count > have) return fail(h, PX_ERR_ARG, "count exceeds field size");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const cudaMemcpyKind kind = mem == PX_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  PX_CUDA(h, cudaMemcpyAsync(dst, src, sizeof(double) * count, kind, s));
  if (mem == PX_MEM_HOST) PX_CUDA(h, cudaStreamSynchronize(s));
  if (field == PX_FIELD_J && mem == PX_MEM_HOST) {
    int flag = 0;
    PX_CUDA(h, cudaMemcpy(&flag, h->nonfinite, sizeof(int), cudaMemcpyDeviceToHost));
    if (flag) {
      cudaMemset(h->nonfinite, 0, sizeof(int));
      return fail(h, PX_ERR_NONFINITE, "non-finite objective (state blew up)");
    }
  }
  return PX_OK;
}

int px_set_timing(void* handle, int enable) {
  Handle* h = static_cast<Handle*>(handle);
  if (!h) return fail(h, PX_ERR_ARG, "null handle");
  if (enable < 0 || enable > 2) return fail(h, PX_ERR_ARG, "timing mode must be 0, 1 or 2");
  h->timing = enable;
  return PX_OK;
}

int px_get_kernel_timing(void* handle, int kclass, double* ms, uint64_t* launches) {
  Handle* h = bind(handle);
  if (!h || !ms || !launches) return fail(h, PX_ERR_ARG, "null argument");
  if (kclass < 0 || kclass >= PX_KCLASS_COUNT) return fail(h, PX_ERR_ARG, "bad kernel class");
  for (auto& m : h->kmarks) {
    PX_CUDA(h, cudaEventSynchronize(m.b));
    float t = 0.f;
    PX_CUDA(h, cudaEventElapsedTime(&t, m.a, m.b));
    h->kms[m.cls] += t;
    h->kcount[m.cls] += 1;
    h->event_pool.push_back(m.a);
    h->event_pool.push_back(m.b);
  }
  h->kmarks.clear();
  *ms = h->kms[kclass];
  *launches = h->kcount[kclass];
  h->kms[kclass] = 0.0;
  h->kcount[kclass] = 0;
  return PX_OK;
}

int px_get_timing(void* handle, px_timing* out) {
  Handle* h = bind(handle);
  if (!h || !out) return fail(h, PX_ERR_ARG, "null argument");
  for (auto& m : h->marks) {
    PX_CUDA(h, cudaEventSynchronize(m.b));
    float ms = 0.f;
    PX_CUDA(h, cudaEventElapsedTime(&ms, m.a, m.b));
    h->tacc.ms[m.phase] += ms;
    h->tacc.launches[m.phase] += m.launches;
    h->tacc.bytes[m.phase] += m.bytes;
    h->event_pool.push_back(m.a);
    h->event_pool.push_back(m.b);
  }
  h->marks.clear();
  *out = h->tacc;
  h->tacc = px_timing{};
  return PX_OK;
}

int px_get_stats(void* handle, px_stats* out) {
  Handle* h = static_cast<Handle*>(handle);
  if (!h || !out) return fail(h, PX_ERR_ARG, "null argument");
  *out = h->stats;
  return PX_OK;
}

int px_reset_stats(void* handle) {
  Handle* h = static_cast<Handle*>(handle);
  if (!h) return fail(h, PX_ERR_ARG, "null handle");
  h->stats = px_stats{};
  return PX_OK;
}

}  // extern "C"

namespace {

int gradient_phases(Handle* h, void* stream) {
  PX_TRY(px_direct(h, stream));
  PX_TRY(px_finish_direct(h, stream));
  PX_TRY(px_adjoint(h, stream));
  PX_TRY(px_finish_adjoint(h, stream));
  return PX_OK;
}

}  // namespace
