// cheb.cu — Chebyshev exponential actions (cheb_march.cuh, scan1d.cuh): replace the
// reference's Newton–Leja propagator (timestepping.py:306-423) with the host planner's
// a-priori Chebyshev series, the stencil fused into the three-term recurrence.
#include <algorithm>
#include <cmath>
#include <vector>

#include "internal.h"
#include "cheb_march.cuh"
#include "scan1d.cuh"

namespace pxi {

namespace {

// 2D passes: σ = ±1, the φ₁ accumulator and the carry-input sum as template constants
template <int M, int SG, bool PH, bool SS>
int launch_cm_v(Handle* h, const px::ChebMarchArgs& a, unsigned blocks, cudaStream_t s) {
  PX_TRY(smem_attr(h, (const void*)px::k_cheb_march<M, SG, PH, SS>, px::CM_SMEM));
  px::k_cheb_march<M, SG, PH, SS><<<blocks, px::CM_NT, px::CM_SMEM, s>>>(a);
  PX_CHECK_LAUNCH(h);
  return PX_OK;
}
template <int M, int SG>
int launch_cm_s(Handle* h, const px::ChebMarchArgs& a, unsigned blocks, cudaStream_t s) {
  if (a.pacc) return launch_cm_v<M, SG, true, false>(h, a, blocks, s);
  if (a.ssum) return launch_cm_v<M, SG, false, true>(h, a, blocks, s);
  return launch_cm_v<M, SG, false, false>(h, a, blocks, s);
}
template <int M>
int launch_cm(Handle* h, const px::ChebMarchArgs& a, unsigned blocks, cudaStream_t s) {
  return a.sigma < 0 ? launch_cm_s<M, -1>(h, a, blocks, s) : launch_cm_s<M, 1>(h, a, blocks, s);
}

// 2D: Chebyshev action by row-marching passes of up to CM_MAXT fused terms
int cheb_action_march(Handle* h, const Plan& pl, const px::Stencil5& st, const double* src, long long src_bs,
                      const double* addend, long long add_bs, double* pacc, double* ssum, double** result,
                      cudaStream_t s, double ttop) {
  std::vector<double> lawc;  // the time law's series of the current substep (pacc with a law)
  const bool law = pacc && h->has_law;
  const size_t n = h->n;
  const int B = h->B;
  const long long nb = (long long)n;
  const int nx = h->d.nx, ny = h->d.ny;
  px::ChebMarchArgs a{};
  a.st = st;
  a.c0 = pl.center; a.d = pl.scale; a.two_over_d = 2.0 / pl.scale; a.sigma = (double)pl.sigma;
  {
    const double taps[5] = {st.cc - pl.center, st.ce, st.cw, st.cs, st.cn};
    for (int q = 0; q < 5; ++q) {
      a.g[q] = (2.0 / pl.scale) * taps[q];
      a.f[q] = taps[q] / pl.scale;
    }
  }
  a.nx = nx; a.ny = ny; a.B = B;
  // the degree is split into the fewest passes of ≤ cheb_terms terms, sizes balanced
  const int K = pl.degree;
  const int tmax = std::max(1, std::min(px::CM_MAXT, pacc ? h->var.cheb_terms_phi : h->var.cheb_terms));
  const int npass = (K + tmax - 1) / tmax;
  const int cm_terms = (K + npass - 1) / npass;
  if (nx <= 2 * px::CM_NT && h->var.cheb_strip == 0) {
    a.strip_w = nx; a.halo = 0; a.nstrips = 1;
  } else {
    a.halo = (cm_terms + 1) & ~1;  // ≥ the terms of any pass; even (16-byte aligned row segments)
    if (h->var.cheb_strip > 0) {
      a.strip_w = h->var.cheb_strip;
    } else {  // fewest strips of ≤ 2·CM_NT computed columns, useful widths balanced (even)
      const int maxw = 2 * px::CM_NT - 2 * a.halo;
      const int ns = (nx + maxw - 1) / maxw;
      a.strip_w = ((nx + ns - 1) / ns + 1) & ~1;
    }
    a.nstrips = (nx + a.strip_w - 1) / a.strip_w;
  }
  int br;
  if (h->var.cheb_band > 0) {
    br = h->var.cheb_band;
  } else {
    // about one full wave of CM_MINB CTAs per SM
    const size_t per_band_ctas = (size_t)a.nstrips * B;
    const size_t target = (size_t)px::CM_MINB * 148;
    size_t nb_bands = std::max<size_t>(1, target / per_band_ctas);
    br = (int)((ny + nb_bands - 1) / nb_bands);
    if (br < 32) br = std::min(32, ny);
  }
  a.band_rows = br;
  a.nbands = (ny + br - 1) / br;
  const unsigned blocks = (unsigned)((size_t)B * a.nstrips * a.nbands);
  int wsel = 0;  // rotating pair of U output buffers
  for (int sub = 0; sub < pl.substeps; ++sub) {
    if (law) {
      lawc.resize(pl.degree + 1);
      law_coefficients(h, pl, ttop, sub, lawc.data());
    }
    const std::vector<double>& bpv = law ? lawc : pl.bp;
    double* acc = (src == h->ACC[0]) ? h->ACC[1] : h->ACC[0];
    const double* uprev = nullptr;
    long long uprev_bs = 0;
    const double* ucur = src;
    long long ucur_bs = src_bs;
    int k = 0;  // terms done
    bool first = true;
    while (k < K || first) {
      const int M = std::min(cm_terms, K - k);
      a.first = first ? 1 : 0;
      a.u_prev = uprev; a.prev_bs = uprev_bs;
      a.u_cur = ucur; a.cur_bs = ucur_bs;
      a.addend = (first && sub == pl.substeps - 1) ? addend : nullptr;
      a.add_bs = add_bs;
      a.acc = acc;
      a.pacc = pacc;
      const bool last = (k + M >= K);
      double* o0 = h->Wk[2 * wsel];
      double* o1 = h->Wk[2 * wsel + 1];
      a.out_prev = last ? nullptr : o0;
      a.out_cur = last ? nullptr : o1;
      a.ssum = (last && sub == pl.substeps - 1) ? ssum : nullptr;
      for (int j = 0; j <= px::CM_MAXT; ++j) {
        const int term = k + j;
        a.be[j] = (j <= M && term <= K && (j > 0 || first)) ? pl.be[term] : 0.0;
        a.bp[j] = (pacc && j <= M && term <= K && (j > 0 || first)) ? bpv[term] : 0.0;
      }
      int rc;
      const int km = kbegin(h, PX_KCLASS_CHEB, s);
      switch (M) {
        case 1: rc = launch_cm<1>(h, a, blocks, s); break;
        case 2: rc = launch_cm<2>(h, a, blocks, s); break;
        case 3: rc = launch_cm<3>(h, a, blocks, s); break;
        case 4: rc = launch_cm<4>(h, a, blocks, s); break;
        case 5: rc = launch_cm<5>(h, a, blocks, s); break;
        case 6: rc = launch_cm<6>(h, a, blocks, s); break;
        default: rc = launch_cm<7>(h, a, blocks, s); break;
      }
      if (rc != PX_OK) return rc;
      kend(h, km, s);
      // algorithmic bytes: 40n per Chebyshev term (+16n with the φ₁
      // accumulator); the fused pass streams its arrays once for all M terms
      const double bytes = (pacc ? 56.0 : 40.0) * (double)n * B * (double)M;  // Σ M = degree
      h->stats.exp_bytes += bytes;
      h->stats.algorithmic_bytes += bytes;
      uprev = o0; uprev_bs = nb;
      ucur = o1; ucur_bs = nb;
      wsel ^= 1;
      k += M;
      first = false;
    }
    src = acc;
    src_bs = nb;
  }
  h->stats.exp_terms += (uint64_t)pl.substeps * pl.degree * B;
  *result = const_cast<double*>(src);
  return PX_OK;
}

px::Scan1DPlan scan_plan(const Plan& pl) {
  px::Scan1DPlan sp{};
  if (!pl.set) return sp;
  sp.be = pl.dcoef;
  sp.bp = pl.dcoef + pl.degree + 1;
  sp.degree = pl.degree;
  sp.substeps = pl.substeps;
  sp.sigma = pl.sigma;
  sp.c0 = pl.center;
  sp.d = pl.scale;
  return sp;  // f, g filled by scan1d (they need the stencil)
}

}  // namespace

bool cheb_has_ssum(const Handle* h) { return h->dim == 2 && (h->d.nx % 2) == 0; }

// result <- exp(span·M)·src (+ addend);  pacc += span·φ₁(span·M)·src  (if pacc);
// ssum += result (if ssum; the 2D passes only, cheb_has_ssum)
void law_coefficients(const Handle* h, const Plan& pl, double ttop, int sub, double* out) {
  // ∫₀^τ θ(t − s)·e^{sM} ds at t = ttop − sub·τ: α·τφ₁ + A·Gc + B·Gs with
  // A = β sin ωt + γ cos ωt, B = −β cos ωt + γ sin ωt (oracle.config_mode.law_substep_coef)
  const double a = h->law[0], b = h->law[1], c = h->law[2], w = h->law[3];
  const int K = pl.degree;
  if (w == 0.0 || pl.gc.empty()) {
    for (int k = 0; k <= K; ++k) out[k] = (w == 0.0 ? a + c : a) * pl.bp[k];
    return;
  }
  const double t = ttop - sub * (pl.span / pl.substeps);
  const double A = b * std::sin(w * t) + c * std::cos(w * t);
  const double Bc = -b * std::cos(w * t) + c * std::sin(w * t);
  for (int k = 0; k <= K; ++k) out[k] = a * pl.bp[k] + A * pl.gc[k] + Bc * pl.gs[k];
}

int cheb_action(Handle* h, const Plan& pl, const px::Stencil5& st, const double* src, long long src_bs,
                const double* addend, long long add_bs, double* pacc, double** result, cudaStream_t s,
                double* ssum, double ttop) {
  if (!pl.set || pl.krylov) return fail(h, PX_ERR_STATE, "Chebyshev plan not set");
  if (ssum && (pacc || !cheb_has_ssum(h))) return fail(h, PX_ERR_STATE, "carry-input sum: 2D passes without φ₁");
  if (pacc && h->has_law && h->law[3] != 0.0 && pl.gc.empty())
    return fail(h, PX_ERR_STATE, "time law: the plan lacks its law series (px_set_cheb_plan_law)");
  if (h->dim == 2 && (h->d.nx % 2) == 0)
    return cheb_action_march(h, pl, st, src, src_bs, addend, add_bs, pacc, ssum, result, s, ttop);
  const bool law = pacc && h->has_law;
  std::vector<double> lawc(pl.degree + 1);
  const size_t n = h->n;
  const int B = h->B;
  const dim3 grid = grid1(n, B);
  const long long nb = (long long)n;
  for (int sub = 0; sub < pl.substeps; ++sub) {
    if (law) law_coefficients(h, pl, ttop, sub, lawc.data());
    const double* bpv = law ? lawc.data() : pl.bp.data();
    double* acc = (src == h->ACC[0]) ? h->ACC[1] : h->ACC[0];
    px::ChebFirstArgs fa{};
    fa.u0 = src; fa.u0_bstride = src_bs;
    fa.u1 = h->Wk[0];
    fa.acc = acc;
    fa.addend = (sub == pl.substeps - 1) ? addend : nullptr;
    fa.add_bstride = add_bs;
    fa.pacc = pacc;
    fa.st = st;
    fa.c0 = pl.center; fa.d = pl.scale;
    fa.b0 = pl.be[0]; fa.b1 = pl.be[1];
    fa.p0 = pacc ? bpv[0] : 0.0; fa.p1 = pacc ? bpv[1] : 0.0;
    fa.nx = h->d.nx; fa.ny = h->d.ny;
    if (h->dim == 2) px::k_cheb_first<2><<<grid, 256, 0, s>>>(fa);
    else px::k_cheb_first<1><<<grid, 256, 0, s>>>(fa);
    PX_CHECK_LAUNCH(h);
    const double* uprev = src;
    long long uprev_bs = src_bs;
    int cur = 0;
    for (int k = 2; k <= pl.degree; ++k) {
      int nxt = (cur + 1) % 3;
      if (h->Wk[nxt] == uprev) nxt = (nxt + 1) % 3;
      px::ChebTermArgs ta{};
      ta.ucur = h->Wk[cur]; ta.ucur_bstride = nb;
      ta.uprev = uprev; ta.uprev_bstride = uprev_bs;
      ta.unext = h->Wk[nxt];
      ta.acc = acc;
      ta.pacc = pacc;
      ta.st = st;
      ta.c0 = pl.center; ta.two_over_d = 2.0 / pl.scale; ta.sigma = (double)pl.sigma;
      ta.bk = pl.be[k]; ta.pk = pacc ? bpv[k] : 0.0;
      ta.nx = h->d.nx; ta.ny = h->d.ny;
      if (h->dim == 2) px::k_cheb_term<2><<<grid, 256, 0, s>>>(ta);
      else px::k_cheb_term<1><<<grid, 256, 0, s>>>(ta);
      PX_CHECK_LAUNCH(h);
      uprev = h->Wk[cur]; uprev_bs = nb;
      cur = nxt;
    }
    src = acc;
    src_bs = nb;
  }
  const uint64_t terms = (uint64_t)pl.substeps * pl.degree * B;
  h->stats.exp_terms += terms;
  const double bytes = (pacc ? 56.0 : 40.0) * (double)n * terms;
  h->stats.exp_bytes += bytes;
  h->stats.algorithmic_bytes += bytes;
  *result = const_cast<double*>(src);
  return PX_OK;
}

// 1D linear sweeps: the whole carry recursion in one CTA (or one 8-CTA cluster) per member
bool use_scan1d(const Handle* h) {
  const Plan& sl = h->plans[PX_PLAN_SLICE];
  return h->dim == 1 && h->n <= 4096 && (!sl.set || !sl.krylov) && !(h->d.flags & PX_FLAG_BOUNDARY_STATES) &&
         !h->tracking;
}

int scan1d(Handle* h, bool adjoint, const double* lanes, double* out, double* pacc, int long_slot, cudaStream_t s) {
  px::Scan1DArgs a{};
  a.lanes = lanes;
  a.out = out;
  a.pacc = pacc;
  a.st = adjoint ? h->AT : h->A;
  auto prescale = [&](px::Scan1DPlan& sp) {
    const double taps[3] = {a.st.cc - sp.c0, a.st.ce, a.st.cw};
    for (int q = 0; q < 3; ++q) {
      sp.f[q] = sp.d != 0.0 ? taps[q] / sp.d : 0.0;
      sp.g[q] = sp.d != 0.0 ? (2.0 / sp.d) * taps[q] : 0.0;
    }
  };
  a.slice = scan_plan(h->plans[PX_PLAN_SLICE]);
  prescale(a.slice);
  a.use_long = long_slot >= 0 ? 1 : 0;
  if (long_slot >= 0) {
    if (!h->plans[long_slot].set || h->plans[long_slot].krylov)
      return fail(h, PX_ERR_STATE, "long-span Chebyshev plan not set");
    a.lng = scan_plan(h->plans[long_slot]);
    prescale(a.lng);
  }
  a.adjoint = adjoint ? 1 : 0;
  a.n = (int)h->n;
  a.Pl = h->Pl;
  if (h->Pl > 1 && !h->plans[PX_PLAN_SLICE].set) return fail(h, PX_ERR_STATE, "slice plan not set");
  const int ppt = h->n <= 512 ? 1 : (h->n <= 1024 ? 2 : (h->n <= 2048 ? 4 : 8));
  const int nt = (int)((h->n + ppt - 1) / ppt);
  // cluster version (8 CTAs = 8 SMs per member, DSMEM ghost zones of 64 points refreshed
  // every 64 terms — a cluster barrier costs ≈ 4× a CTA barrier; ghost widths 8/16/32 were
  // measured slower) with 2 members per CTA, for the larger 1D grids; one CTA per member
  // otherwise
  constexpr int kCS = 8, kPPT = 4, kG = 64, kMB = 2;
  const int Wc = (int)(h->n / kCS);
  if (h->var.scan1d_cluster && h->n >= 2048 && h->n % (kCS * kPPT) == 0 && Wc >= kG &&
      Wc / kPPT + 2 * (kG / kPPT) <= 256) {
    const int nr = Wc / kPPT + 2 * (kG / kPPT);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(((h->B + kMB - 1) / kMB) * kCS));
    cfg.blockDim = dim3((unsigned)(((nr + 31) / 32) * 32));
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kCS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    PX_CUDA(h, cudaLaunchKernelEx(&cfg, px::k_scan1d_cluster<kPPT, kCS, kG, kMB>, a, h->B));
  } else {
    const bool full = h->n % ppt == 0;
#define PX_S1(PP)                                              \
  do {                                                         \
    if (full) px::k_scan1d<PP, true><<<h->B, nt, 0, s>>>(a);   \
    else px::k_scan1d<PP, false><<<h->B, nt, 0, s>>>(a);       \
  } while (0)
    switch (ppt) {
      case 1: PX_S1(1); break;
      case 2: PX_S1(2); break;
      case 4: PX_S1(4); break;
      default: PX_S1(8); break;
    }
#undef PX_S1
  }
  PX_CHECK_LAUNCH(h);
  uint64_t terms = (uint64_t)(h->Pl - 1) * h->plans[PX_PLAN_SLICE].substeps * h->plans[PX_PLAN_SLICE].degree;
  if (long_slot >= 0) terms += (uint64_t)h->plans[long_slot].substeps * h->plans[long_slot].degree;
  terms *= h->B;
  h->stats.exp_terms += terms;
  const double bytes = (adjoint ? 56.0 : 40.0) * (double)h->n * terms;
  h->stats.exp_bytes += bytes;
  h->stats.algorithmic_bytes += bytes;
  return PX_OK;
}

}  // namespace pxi
