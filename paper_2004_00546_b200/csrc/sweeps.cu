// sweeps.cu — one rank's Paraexp sweeps on one GPU (reference structure
// paraexp.py:187-353):
//   direct : g = A·u0 + f                       (absorbed IC, paraexp.py:239-242)
//            v_p = RK4 zero-data solve per slice (all local slices × batch as lanes)
//            D <- v_{p0};  D <- exp(ΔA)·D + v_p  (summed-chain carry; equals the
//                                                 reference's neighbour chains by linearity)
//            D <- exp((P − p1)Δ·A)·D             (blockscan long span, world > 1)
//   adjoint: w' = Aᵀ(w + q†_T), z = ∫w           (absorbed FC, reflected time,
//                                                 paraexp.py:256-295)
//            C <- w_{p1−1};  C <- exp(ΔAᵀ)·C + w_p,  G += Δ·φ₁(ΔAᵀ)·C
//            C <- exp(p0Δ·Aᵀ)·C (+φ₁)            (blockscan long span)
//   outputs: u(T), J, q†(0), G = ∫q†dt, grad_k = ⟨φ_k, G⟩.
// Everything is enqueued on the caller's stream; no host synchronisation.
#include <cmath>

#include "internal.h"

namespace pxi {

int exp_action(Handle* h, int slot, const px::Stencil5& st, const double* src, long long src_bs,
               const double* addend, long long add_bs, double* pacc, double** result, cudaStream_t s,
               double* ssum, double ttop) {
  const Plan& pl = h->plans[slot];
  if (!pl.set) return fail(h, PX_ERR_STATE, "exp-action plan slot " + std::to_string(slot) + " not set");
  if (pl.krylov) {
    if (ssum) return fail(h, PX_ERR_STATE, "carry-input sum: Chebyshev passes only");
    if (pacc && h->has_law) return fail(h, PX_ERR_STATE, "time law: Chebyshev exp-actions only");
    return krylov_action(h, pl, st, src, src_bs, addend, add_bs, pacc, result, s);
  }
  return cheb_action(h, pl, st, src, src_bs, addend, add_bs, pacc, result, s, ssum, ttop);
}

namespace {

// Point the handle's exp-action scratch (Wk, ACC, Krylov work) at a block's own buffers
// while that block's launches are enqueued (kernels capture the pointer values).
struct ScratchSwap {
  Handle* h;
  double* Wk[4];
  double* ACC[2];
  px::KrylovWork kw;
  ScratchSwap(Handle* hh, const Handle::Block& b) : h(hh), kw(hh->kw) {
    for (int i = 0; i < 4; ++i) { Wk[i] = h->Wk[i]; h->Wk[i] = b.Wk[i]; }
    for (int i = 0; i < 2; ++i) { ACC[i] = h->ACC[i]; h->ACC[i] = b.ACC[i]; }
    h->kw = b.kw;
  }
  ~ScratchSwap() {
    for (int i = 0; i < 4; ++i) h->Wk[i] = Wk[i];
    for (int i = 0; i < 2; ++i) h->ACC[i] = ACC[i];
    h->kw = kw;
  }
};

bool use_blocks(const Handle* h) {
  return h->lb > 1 && h->dim == 2 && !(h->d.flags & PX_FLAG_BOUNDARY_STATES) && !h->tracking;
}

// The adjoint's φ₁ integral of the slice carries, Σ_q Δ·φ₁(ΔAᵀ)·C_q, is linear in the carry
// inputs and every carry applies the same operator: it equals ONE φ₁ action on S = Σ_q C_q.
// With the 2D Chebyshev passes the carries accumulate S in their last pass (SS passes, one
// extra stream) instead of carrying a φ₁ accumulator through every pass — which also frees
// the registers for seven-term passes. Krylov and 1D keep the per-carry accumulator.
bool use_ssum(const Handle* h) {
  const Plan& pl = h->plans[PX_PLAN_SLICE];
  return pl.set && !pl.krylov && cheb_has_ssum(h) && !h->has_law;  // a time law weighs each carry differently
}

// start time (physical) of the reflected-time span that propagates a carry through local
// slices q0 … q1−1 down to slice q0's lower edge, i.e. the upper edge of slice q1 − 1
double top_time(const Handle* h, int q1) { return (h->d.p_begin + q1) * (h->d.T / h->d.P); }

// Block-scan of the direct carry inside one handle: block g scans its lanes from a zero
// carry and propagates the result to the rank's last slice edge with one long-span action
// (slot PX_PLAN_BLOCK_LONG + (lb-1-g) - 1); the block results are summed into `out`.
int direct_blocks(Handle* h, const double* vend, double* out, cudaStream_t s) {
  const long long nb = (long long)h->n;
  const long long lane_bs = (long long)h->Pl * nb;
  PX_CUDA(h, cudaEventRecord(h->ev_fork, s));
  for (int g = 0; g < h->lb; ++g) {
    Handle::Block& b = h->blocks[g];
    PX_CUDA(h, cudaStreamWaitEvent(b.st, h->ev_fork, 0));
    ScratchSwap sw(h, b);
    const double* D = vend + (size_t)b.q0 * h->n;
    long long D_bs = lane_bs;
    for (int q = b.q0 + 1; q < b.q1; ++q) {
      double* res = nullptr;
      PX_TRY(exp_action(h, PX_PLAN_SLICE, h->A, D, D_bs, vend + (size_t)q * h->n, lane_bs, nullptr, &res, b.st));
      D = res;
      D_bs = nb;
    }
    if (g < h->lb - 1) {
      double* res = nullptr;
      PX_TRY(exp_action(h, PX_PLAN_BLOCK_LONG + (h->lb - 1 - g) - 1, h->A, D, D_bs, nullptr, 0, nullptr, &res, b.st));
      D = res;
      D_bs = nb;
    }
    PX_TRY(axpby(h, b.D, nb, D, D_bs, 1.0, nullptr, 0, 0.0, b.st));
    PX_CUDA(h, cudaEventRecord(b.ev, b.st));
  }
  for (int g = 0; g < h->lb; ++g) {
    PX_CUDA(h, cudaStreamWaitEvent(s, h->blocks[g].ev, 0));
    PX_TRY(axpby(h, out, nb, h->blocks[g].D, nb, 1.0, g == 0 ? nullptr : out, nb, g == 0 ? 0.0 : 1.0, s));
  }
  return PX_OK;
}

// Adjoint counterpart: block g scans its lanes backwards (φ into its own accumulator) and
// propagates to the rank's first slice edge (slot PX_PLAN_BLOCK_LONG + g - 1); the carries
// are summed into `out` and the φ accumulators added to `gacc`.
int adjoint_blocks(Handle* h, const double* wend, double* out, double* gacc, cudaStream_t s) {
  const long long nb = (long long)h->n;
  const long long lane_bs = (long long)h->Pl * nb;
  PX_CUDA(h, cudaEventRecord(h->ev_fork, s));
  for (int g = 0; g < h->lb; ++g) {
    Handle::Block& b = h->blocks[g];
    PX_CUDA(h, cudaStreamWaitEvent(b.st, h->ev_fork, 0));
    ScratchSwap sw(h, b);
    PX_CUDA(h, cudaMemsetAsync(b.Gp, 0, sizeof(double) * h->B * h->n, b.st));
    const double* C = wend + (size_t)(b.a1 - 1) * h->n;
    long long C_bs = lane_bs;
    const bool ss = use_ssum(h) && b.a1 - b.a0 > 1;
    if (ss) PX_TRY(axpby(h, b.S, nb, C, C_bs, 1.0, nullptr, 0, 0.0, b.st));
    for (int q = b.a1 - 2; q >= b.a0; --q) {
      double* res = nullptr;
      PX_TRY(exp_action(h, PX_PLAN_SLICE, h->AT, C, C_bs, wend + (size_t)q * h->n, lane_bs, ss ? nullptr : b.Gp, &res,
                        b.st, ss && q > b.a0 ? b.S : nullptr, top_time(h, q + 1)));
      C = res;
      C_bs = nb;
    }
    if (g > 0) {
      double* res = nullptr;
      PX_TRY(exp_action(h, PX_PLAN_BLOCK_LONG + g - 1, h->AT, C, C_bs, nullptr, 0, b.Gp, &res, b.st, nullptr,
                        top_time(h, b.a0)));
      C = res;
      C_bs = nb;
    }
    PX_TRY(axpby(h, b.D, nb, C, C_bs, 1.0, nullptr, 0, 0.0, b.st));
    if (ss) {  // Gp += Δ·φ₁(ΔAᵀ)·S (the exp result of this action is not used)
      double* res = nullptr;
      PX_TRY(exp_action(h, PX_PLAN_SLICE, h->AT, b.S, nb, nullptr, 0, b.Gp, &res, b.st));
    }
    PX_CUDA(h, cudaEventRecord(b.ev, b.st));
  }
  for (int g = 0; g < h->lb; ++g) {
    PX_CUDA(h, cudaStreamWaitEvent(s, h->blocks[g].ev, 0));
    PX_TRY(axpby(h, out, nb, h->blocks[g].D, nb, 1.0, g == 0 ? nullptr : out, nb, g == 0 ? 0.0 : 1.0, s));
    PX_TRY(axpby(h, gacc, nb, gacc, nb, 1.0, h->blocks[g].Gp, nb, 1.0, s));
  }
  return PX_OK;
}

}  // namespace

void free_blocks(Handle* h) {
  for (auto& b : h->blocks) {
    for (double* p : b.Wk) cudaFree(p);
    for (double* p : b.ACC) cudaFree(p);
    cudaFree(b.D);
    cudaFree(b.Gp);
    cudaFree(b.S);
    krylov_free(b.kw);
    if (b.st) cudaStreamDestroy(b.st);
    if (b.ev) cudaEventDestroy(b.ev);
  }
  h->blocks.clear();
  h->lb = 1;
}

// Direct blocks take `sizes` (slice order; equal blocks when null); the adjoint uses the mirrored
// partition, so adjoint block g's long span (the blocks before it) has the length of direct block
// G−1−g's (the blocks after it): one set of long-span plans serves both sweeps. Unequal sizes
// balance each block's carries against its long span (the first direct / last adjoint block
// spans the most).
int set_local_blocks(Handle* h, int blocks, const int* sizes) {
  std::vector<int> sz(blocks, blocks > 0 ? h->Pl / blocks : 0);
  if (sizes) sz.assign(sizes, sizes + blocks);
  bool same = blocks == h->lb;
  for (int g = 0; same && g < blocks && blocks > 1; ++g) same = h->blocks[g].q1 - h->blocks[g].q0 == sz[g];
  if (same) return PX_OK;
  free_blocks(h);
  h->graph_valid = false;
  if (blocks == 1) return PX_OK;
  if (!h->ev_fork) PX_CUDA(h, cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
  const size_t Bn = (size_t)h->B * h->n;
  h->blocks.resize(blocks);
  int q = 0, qa = 0;
  for (int g = 0; g < blocks; ++g) {
    Handle::Block& b = h->blocks[g];
    b.q0 = q;
    b.q1 = q + sz[g];
    q = b.q1;
    b.a0 = qa;
    b.a1 = qa + sz[blocks - 1 - g];
    qa = b.a1;
    for (auto& p : b.Wk) PX_CUDA(h, cudaMalloc(&p, sizeof(double) * Bn));
    for (auto& p : b.ACC) PX_CUDA(h, cudaMalloc(&p, sizeof(double) * Bn));
    PX_CUDA(h, cudaMalloc(&b.D, sizeof(double) * Bn));
    PX_CUDA(h, cudaMalloc(&b.Gp, sizeof(double) * Bn));
    PX_CUDA(h, cudaMalloc(&b.S, sizeof(double) * Bn));
    if (h->d.expaction == PX_EXP_KRYLOV) {
      std::string err;
      if (krylov_alloc(b.kw, h->d.krylov_m, h->n, h->B, &err) != PX_OK) {
        free_blocks(h);
        return fail(h, PX_ERR_NOMEM, err);
      }
    }
    PX_CUDA(h, cudaStreamCreateWithFlags(&b.st, cudaStreamNonBlocking));
    PX_CUDA(h, cudaEventCreateWithFlags(&b.ev, cudaEventDisableTiming));
  }
  h->lb = blocks;
  return PX_OK;
}

int direct_linear(Handle* h, cudaStream_t s) {
  const long long nb = (long long)h->n;
  const long long lane_bs = (long long)h->Pl * nb;  // stride between batch members in lanes
  // g = A·u0 + f  (u0 shared by all members); with a time law g = A·u0 and the lanes add θ(t)·f
  if (h->has_law) {
    PX_TRY(apply_plus_control(h, h->g, h->u0, 0, h->A, false, s));
    PX_TRY(apply_plus_control(h, h->fctl, h->u0, 0, px::Stencil5{0.0, 0.0, 0.0, 0.0, 0.0}, true, s));
  } else {
    PX_TRY(apply_plus_control(h, h->g, h->u0, 0, h->A, true, s));
  }
  const double* vend = nullptr;
  int tm = tbegin(h, PX_PHASE_RK4_DIRECT, s);
  PX_TRY(rk4_sweep(h, false, &vend, s));
  tend(h, tm, s);
  h->vend = vend;
  tm = tbegin(h, PX_PHASE_EXP_DIRECT, s);
  if (use_scan1d(h)) {
    PX_TRY(scan1d(h, false, vend, h->UT, nullptr, h->d.p_end < h->d.P ? PX_PLAN_LONG_DIRECT : -1, s));
    tend(h, tm, s);
    return PX_OK;
  }
  const bool bnd = ((h->d.flags & PX_FLAG_BOUNDARY_STATES) || h->tracking) && h->UBND;
  const long long ubs = (long long)(h->d.P + 1) * nb;
  if (bnd) PX_TRY(axpby(h, h->UBND, ubs, h->u0, 0, 1.0, nullptr, 0, 0.0, s));
  if (use_blocks(h)) {
    PX_TRY(direct_blocks(h, vend, h->UT, s));
    if (h->d.p_end < h->d.P) {
      double* res = nullptr;
      PX_TRY(exp_action(h, PX_PLAN_LONG_DIRECT, h->A, h->UT, nb, nullptr, 0, nullptr, &res, s));
      PX_TRY(axpby(h, h->UT, nb, res, nb, 1.0, nullptr, 0, 0.0, s));
    }
    tend(h, tm, s);
    return PX_OK;
  }
  // summed-chain carry over the local block
  const double* D = vend;  // lane p0 of each member
  long long D_bs = lane_bs;
  if (bnd) PX_TRY(axpby(h, h->UBND + nb, ubs, D, D_bs, 1.0, h->u0, 0, 1.0, s));
  for (int q = 1; q < h->Pl; ++q) {
    double* res = nullptr;
    PX_TRY(exp_action(h, PX_PLAN_SLICE, h->A, D, D_bs, vend + (size_t)q * h->n, lane_bs, nullptr, &res, s));
    D = res;
    D_bs = nb;
    if (bnd) PX_TRY(axpby(h, h->UBND + (size_t)(q + 1) * h->n, ubs, D, D_bs, 1.0, h->u0, 0, 1.0, s));
  }
  if (h->d.p_end < h->d.P) {
    double* res = nullptr;
    PX_TRY(exp_action(h, PX_PLAN_LONG_DIRECT, h->A, D, D_bs, nullptr, 0, nullptr, &res, s));
    D = res;
    D_bs = nb;
  }
  PX_TRY(axpby(h, h->UT, nb, D, D_bs, 1.0, nullptr, 0, 0.0, s));
  tend(h, tm, s);
  if (h->tracking) PX_TRY(track_direct(h, s));
  return PX_OK;
}

int adjoint_linear(Handle* h, cudaStream_t s) {
  const long long nb = (long long)h->n;
  const long long lane_bs = (long long)h->Pl * nb;
  const double* wend = nullptr;
  int tm;
  if (h->tracking) {  // lanes with the tracking source from zero data; G <- Σ_p z_p
    PX_TRY(track_adjoint_lanes(h, &wend, s));
    h->wend = wend;
    tm = tbegin(h, PX_PHASE_EXP_ADJOINT, s);
  } else {
    tm = tbegin(h, PX_PHASE_RK4_ADJOINT, s);
    PX_TRY(rk4_sweep(h, true, &wend, s));
    tend(h, tm, s);
    h->wend = wend;
    tm = tbegin(h, PX_PHASE_EXP_ADJOINT, s);
  }
  // G partial <- Σ_p z_p  (z_p = Σ_steps h·w3 + nsteps·c; with a time law the θ-weighted lane
  // integrals and the summed source part in cz, lanes.cu; tracking: summed with its lanes)
  if (!h->tracking) {
    if (h->z_closed) PX_TRY(z_closed_form(h, wend, s));
    else PX_TRY(lane_sum_plus(h, h->G, h->Z, h->cz, h->has_law ? 1.0 : (double)h->Pl * h->d.nsteps, h->z_valid, s));
  }
  if (use_scan1d(h) && !h->has_law) {
    PX_TRY(scan1d(h, true, wend, h->QDAG0, h->G, h->d.p_begin > 0 ? PX_PLAN_LONG_ADJOINT : -1, s));
  } else if (use_blocks(h)) {
    PX_TRY(adjoint_blocks(h, wend, h->QDAG0, h->G, s));
    if (h->d.p_begin > 0) {
      double* res = nullptr;
      PX_TRY(exp_action(h, PX_PLAN_LONG_ADJOINT, h->AT, h->QDAG0, nb, nullptr, 0, h->G, &res, s, nullptr,
                        top_time(h, 0)));
      PX_TRY(axpby(h, h->QDAG0, nb, res, nb, 1.0, nullptr, 0, 0.0, s));
    }
  } else {
    const double* C = wend + (size_t)(h->Pl - 1) * h->n;
    long long C_bs = lane_bs;
    const bool ss = use_ssum(h) && h->Pl > 1;
    if (ss) PX_TRY(axpby(h, h->S, nb, C, C_bs, 1.0, nullptr, 0, 0.0, s));
    for (int q = h->Pl - 2; q >= 0; --q) {
      double* res = nullptr;
      PX_TRY(exp_action(h, PX_PLAN_SLICE, h->AT, C, C_bs, wend + (size_t)q * h->n, lane_bs, ss ? nullptr : h->G, &res,
                        s, ss && q > 0 ? h->S : nullptr, top_time(h, q + 1)));
      C = res;
      C_bs = nb;
    }
    if (h->d.p_begin > 0) {
      double* res = nullptr;
      PX_TRY(exp_action(h, PX_PLAN_LONG_ADJOINT, h->AT, C, C_bs, nullptr, 0, h->G, &res, s, nullptr, top_time(h, 0)));
      C = res;
      C_bs = nb;
    }
    PX_TRY(axpby(h, h->QDAG0, nb, C, C_bs, 1.0, nullptr, 0, 0.0, s));
    if (ss) {  // G += Δ·φ₁(ΔAᵀ)·S (the exp result of this action is not used)
      double* res = nullptr;
      PX_TRY(exp_action(h, PX_PLAN_SLICE, h->AT, h->S, nb, nullptr, 0, h->G, &res, s));
    }
  }
  tend(h, tm, s);
  tm = tbegin(h, PX_PHASE_OTHER, s);
  // tracking: ∂L/∂f = (1/T)∫θ·q† dt (optimization.py:103-112); the terminal objective adds its
  // absorbed final-condition part in finish_adjoint_impl
  if (h->tracking) PX_TRY(axpby(h, h->G, nb, h->G, nb, 1.0 / h->d.T, nullptr, 0, 0.0, s));
  PX_TRY(project(h, h->GRAD, h->G, nb, 1.0, 0.0, s));
  tend(h, tm, s);
  return PX_OK;
}

int finish_direct_impl(Handle* h, cudaStream_t s) {
  const long long nb = (long long)h->n;
  const int tm = tbegin(h, PX_PHASE_OTHER, s);
  // u(T) = u0 + Σ carries (the Burgers sweep writes u(T) itself)
  if (h->d.kind == PX_KIND_ADVDIFF) PX_TRY(axpby(h, h->UT, nb, h->UT, nb, 1.0, h->u0, 0, 1.0, s));
  PX_TRY(axpby(h, h->QT, nb, h->UT, nb, 1.0, h->ut, 0, -1.0, s));
  if (h->tracking) {  // J came with the recording sweep; the adjoint has zero terminal data
    tend(h, tm, s);
    return PX_OK;
  }
  PX_TRY(objective(h, s));
  if (h->d.kind == PX_KIND_ADVDIFF) PX_TRY(apply_plus_control(h, h->gadj, h->QT, nb, h->AT, false, s));
  tend(h, tm, s);
  return PX_OK;
}

int finish_adjoint_impl(Handle* h, cudaStream_t s) {
  const long long nb = (long long)h->n;
  if (h->adjoint_mode == PX_ADJOINT_FROZEN_SPAN) return PX_OK;  // q†_T is not absorbed: nothing to add
  if (h->tracking) return PX_OK;                                  // q†(T) = 0: nothing to add
  const int tm = tbegin(h, PX_PHASE_OTHER, s);
  // absorbed final condition: q† = q†_T + the solved part (paraexp.py:268-270)
  PX_TRY(axpby(h, h->QDAG0, nb, h->QDAG0, nb, 1.0, h->QT, nb, 1.0, s));
  // ∫₀ᵀ θ dt·q†_T (T without a time law)
  double wT = h->d.T;
  if (h->has_law) {
    const double a = h->law[0], b = h->law[1], c = h->law[2], w = h->law[3], T = h->d.T;
    wT = (w == 0.0) ? (a + c) * T : a * T + b * (1.0 - std::cos(w * T)) / w + c * std::sin(w * T) / w;
  }
  PX_TRY(axpby(h, h->G, nb, h->G, nb, 1.0, h->QT, nb, wT, s));
  PX_TRY(project(h, h->GRAD, h->QT, nb, wT, 1.0, s));
  tend(h, tm, s);
  return PX_OK;
}

}  // namespace pxi
