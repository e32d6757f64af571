// lanes.cu — the zero-data RK4 slice solves of all local lanes (rk4.cuh); replaces the
// per-worker rk45_integrate calls of the reference's direct / adjoint workers
// (paraexp.py:193-198, :268-274) with one batched sweep over B members × Pl slices.
#include <algorithm>
#include <cmath>

#include "internal.h"
#include "rk4.cuh"

namespace pxi {

namespace {

// The three-column two-step march (the large-grid default): 64-thread CTAs, 4 per SM,
// b(r−8) from a register ring (two TMA streams); S2 = false is the one-step instantiation
// that runs a sweep's odd remainder step.
int launch_marchc(Handle* h, const px::MarchArgs& a, unsigned blocks, bool one_step, cudaStream_t s) {
  if (one_step) {
    const size_t sm = px::marchc_smem<3, 64, 3>(false);
    PX_TRY(smem_attr(h, (const void*)px::k_rk4_marchc<3, 64, 3, 4, false, false>, sm));
    px::k_rk4_marchc<3, 64, 3, 4, false, false><<<blocks, 64, sm, s>>>(a);
  } else {
    const size_t sm = px::marchc_smem<3, 64, 3>(true);
    PX_TRY(smem_attr(h, (const void*)px::k_rk4_marchc<3, 64, 3, 4, true, true>, sm));
    px::k_rk4_marchc<3, 64, 3, 4, true, true><<<blocks, 64, sm, s>>>(a);
  }
  return PX_OK;
}

// The two-column two-step march: full-row grids (nx ≤ 256), the ∫-accumulating adjoint lanes
// and PX_VAR_MARCH_COLS = 2. 128 threads × 3 CTAs per SM, TMA row ring.
int launch_march2(Handle* h, const px::MarchArgs& a, unsigned blocks, bool zlanes, cudaStream_t s) {
  if (zlanes) {
    const size_t sm = px::march2_smem<128, 3>(true);
    PX_TRY(smem_attr(h, (const void*)px::k_rk4_march2<true, 128, 3, 3>, sm));
    px::k_rk4_march2<true, 128, 3, 3><<<blocks, 128, sm, s>>>(a);
  } else {
    const size_t sm = px::march2_smem<128, 3>(false);
    PX_TRY(smem_attr(h, (const void*)px::k_rk4_march2<false, 128, 3, 3>, sm));
    px::k_rk4_march2<false, 128, 3, 3><<<blocks, 128, sm, s>>>(a);
  }
  return PX_OK;
}

// One RK4 step per launch (small sweeps, PX_VAR_MARCH2 = 0, odd remainders of the two-column march,
// time-law sweeps).
int launch_march1(Handle* h, px::MarchArgs a, int L, bool zlanes, bool remainder, cudaStream_t s) {
  const bool law = h->has_law;
  const int nx = a.nx, ny = a.ny;
  if (nx <= px::MARCH_MAX_CW) {
    a.strip_w = nx; a.halo = 0; a.nstrips = 1;
  } else {
    a.strip_w = px::MARCH_STRIP; a.halo = px::MARCH_HALO;
    a.nstrips = (nx + px::MARCH_STRIP - 1) / px::MARCH_STRIP;
  }
  int br;
  if (remainder) {
    br = std::min(ny, 256);
  } else {
    // bands of rows: enough CTAs for ≥ 4 waves at 2 CTAs/SM, ≥ 32 rows per band
    br = ny;
    while (br > 32 && (size_t)L * a.nstrips * ((ny + br - 1) / br) < 4 * 2 * 148) br = (br + 1) / 2;
    if (ny >= 1024 && br > 256) br = 256;
  }
  a.band_rows = br;
  a.nbands = (ny + br - 1) / br;
  const unsigned blocks = (unsigned)((size_t)L * a.nstrips * a.nbands);
  const size_t smem = px::march_smem(zlanes, law);
  if (zlanes && law) {
    PX_TRY(smem_attr(h, (const void*)px::k_rk4_march<true, true>, smem));
    px::k_rk4_march<true, true><<<blocks, px::MARCH_NT, smem, s>>>(a);
  } else if (zlanes) {
    PX_TRY(smem_attr(h, (const void*)px::k_rk4_march<true>, smem));
    px::k_rk4_march<true><<<blocks, px::MARCH_NT, smem, s>>>(a);
  } else if (law) {
    PX_TRY(smem_attr(h, (const void*)px::k_rk4_march<false, true>, smem));
    px::k_rk4_march<false, true><<<blocks, px::MARCH_NT, smem, s>>>(a);
  } else {
    PX_TRY(smem_attr(h, (const void*)px::k_rk4_march<false>, smem));
    px::k_rk4_march<false><<<blocks, px::MARCH_NT, smem, s>>>(a);
  }
  return PX_OK;
}

}  // namespace

// Zero-data RK4 sweep of all local lanes; returns the final lane buffer.
int rk4_sweep(Handle* h, bool adjoint, const double** final_out, cudaStream_t s) {
  const px::Stencil5 st = adjoint ? h->AT : h->A;
  const double hs = (h->d.T / h->d.P) / h->d.nsteps;
  const double* g = adjoint ? h->gadj : h->g;
  const dim3 grid = grid1(h->n, h->B);
  const int nx = h->d.nx, ny = h->d.ny;
  // Horner constants: t1 = g + (h/4)Mg, t2 = g + (h/3)M t1, b = h(g + (h/2)M t2), c = (h²/2) t2
  auto sax = [&](double* out, const double* x, const double* y, double al, double sc) -> int {
    if (h->dim == 2) px::k_stencil_axpy<2><<<grid, 256, 0, s>>>(out, x, y, st, al, sc, nx, ny);
    else px::k_stencil_axpy<1><<<grid, 256, 0, s>>>(out, x, y, st, al, sc, nx, ny);
    PX_CHECK_LAUNCH(h);
    return PX_OK;
  };
  PX_TRY(sax(h->Wk[0], g, g, 0.25 * hs, 1.0));
  PX_TRY(sax(h->Wk[1], g, h->Wk[0], hs / 3.0, 1.0));
  PX_TRY(sax(h->bsrc, g, h->Wk[1], 0.5 * hs, hs));
  const bool law = h->has_law;
  if (adjoint && !law)
    PX_TRY(axpby(h, h->cz, (long long)h->n, h->Wk[1], (long long)h->n, 0.5 * hs * hs, nullptr, 0, 0.0, s));
  if (adjoint && law) {
    // the source part of the θ-weighted lane integrals summed over every local lane and step:
    // Σ h/6[2θm(Y2 + Y3) + θb·Y4]_source = S0·g + S1·Mg + S2·M²g
    double S0 = 0.0, S1 = 0.0, S2 = 0.0;
    const double delta = h->d.T / h->d.P;
    auto th = [&](double t) { return h->law[0] + h->law[1] * std::sin(h->law[3] * t) + h->law[2] * std::cos(h->law[3] * t); };
    for (int p = h->d.p_begin; p < h->d.p_end; ++p)
      for (int k = 0; k < h->d.nsteps; ++k) {
        const double t = (p + 1) * delta - k * hs;
        const double tm = th(t - 0.5 * hs), tb = th(t - hs);
        S0 += hs * hs * (2.0 * tm + tb) / 6.0;
        S1 += hs * hs * hs * (tm + tb) / 12.0;
        S2 += hs * hs * hs * hs * tb / 24.0;
      }
    const long long nb = (long long)h->n;
    PX_TRY(sax(h->Wk[2], g, g, 1.0, 1.0));                                   // g + Mg
    PX_TRY(axpby(h, h->Wk[3], nb, g, nb, S1 - S2, h->Wk[2], nb, S2, s));     // S1·g + S2·Mg
    PX_TRY(sax(h->Wk[2], g, h->Wk[3], 1.0, 1.0));                            // g + M(S1·g + S2·Mg)
    PX_TRY(axpby(h, h->cz, nb, h->Wk[2], nb, 1.0, g, nb, S0 - 1.0, s));      // + (S0 − 1)·g
  }

  const int nsteps = h->d.nsteps;
  double* cur = nullptr;
  uint64_t launched_steps = 0;
  h->z_valid = false;
  if (h->dim == 1 && h->n <= 4096) {
    // 1D: one CTA per lane runs all the lane's steps on chip
    px::Lane1DArgs a{};
    a.y_out = h->Y0; a.b = h->bsrc; a.z = h->Z; a.st = st; a.h = hs;
    a.n = (int)h->n; a.lanes_per_b = h->Pl; a.nsteps = nsteps;
    a.f = h->fctl; a.delta = h->d.T / h->d.P; a.p_begin = h->d.p_begin;
    for (int k = 0; k < 4; ++k) a.law[k] = h->law[k];
    const int ppt = h->n <= 1024 ? 1 : (h->n <= 2048 ? 2 : 4);
    const int nt = (int)((h->n + ppt - 1) / ppt);
    const bool full = h->n % ppt == 0;
#define PX_L1W(PP, LW)                                                                  \
  do {                                                                                  \
    if (full) {                                                                         \
      if (adjoint) px::k_rk4_lane1d<PP, true, true, LW><<<h->L, nt, 0, s>>>(a);         \
      else px::k_rk4_lane1d<PP, false, true, LW><<<h->L, nt, 0, s>>>(a);                \
    } else {                                                                            \
      if (adjoint) px::k_rk4_lane1d<PP, true, false, LW><<<h->L, nt, 0, s>>>(a);        \
      else px::k_rk4_lane1d<PP, false, false, LW><<<h->L, nt, 0, s>>>(a);               \
    }                                                                                   \
  } while (0)
#define PX_L1(PP)                  \
  do {                             \
    if (law) PX_L1W(PP, true);     \
    else PX_L1W(PP, false);        \
  } while (0)
    if (ppt == 1) PX_L1(1);
    else if (ppt == 2) PX_L1(2);
    else PX_L1(4);
#undef PX_L1
#undef PX_L1W
    PX_CHECK_LAUNCH(h);
    cur = h->Y0;
    launched_steps = nsteps;
    h->z_valid = adjoint;
  } else if (nsteps == 1 && !(law && !adjoint)) {
    px::k_broadcast_lanes<<<dim3((unsigned)std::min<size_t>((h->n + 255) / 256, 1024), h->L), 256, 0, s>>>(
        h->Y0, h->bsrc, h->Pl, h->n);
    PX_CHECK_LAUNCH(h);
    cur = h->Y0;
  } else {
    // adjoint lanes without the ∫ accumulator when it is recovered in closed form
    // afterwards (z_closed: Σ_k h·S(hAᵀ)y_k = (Aᵀ)⁻¹(y_n − n·b), one FFT solve per gradient)
    const bool zlanes = adjoint && !h->z_closed;
    if (h->dim == 2 && (nx & 1)) return fail(h, PX_ERR_ARG, "2D grids need an even nx");
    px::MarchArgs a{};
    a.b = h->bsrc; a.z = h->Z; a.st = st; a.h = hs;
    a.nx = nx; a.ny = ny; a.lanes = h->L; a.lanes_per_b = h->Pl;
    a.f = h->fctl; a.delta = h->d.T / h->d.P; a.p_begin = h->d.p_begin;
    for (int k = 0; k < 4; ++k) a.law[k] = h->law[k];
    {
      const double ks[4] = {0.25 * hs, hs / 3.0, 0.5 * hs, hs};
      const double cf[5] = {st.cc, st.ce, st.cw, st.cs, st.cn};
      for (int j = 0; j < 4; ++j)
        for (int q = 0; q < 5; ++q) a.kc[j][q] = ks[j] * cf[q];
    }
    // two RK4 steps per launch for large sweeps; small sweeps keep one step per launch: the
    // 8-stage pipeline fill (16 rows per band) only pays off when each launch covers ≥ 2^28
    // lane-points
    const int m2 = h->var.march2;
    if (law && !adjoint) {
      // time-law direct lanes: θ·f enters at every stage, so the lanes start from zero (no
      // y₁ = b shortcut) and run one step per launch
      PX_CUDA(h, cudaMemsetAsync(h->Y0, 0, sizeof(double) * h->L * h->n, s));
      cur = h->Y0;
      for (int st_i = 0; st_i < nsteps; ++st_i) {
        double* out = (cur == h->Y0) ? h->Y1 : h->Y0;
        a.y_in = cur;
        a.y_out = out;
        a.step = st_i;
        PX_TRY(launch_march1(h, a, h->L, false, false, s));
        PX_CHECK_LAUNCH(h);
        cur = out;
      }
    } else if (m2 && !law && nsteps >= 3 && (m2 == 2 || (double)h->L * (double)h->n >= 268435456.0)) {
      constexpr int cw2 = 2 * 128;  // computed width of the two-column kernel
      // three columns per thread (k_rk4_marchc): direct lanes, strip mode
      const bool cols3 = !zlanes && h->var.march_cols == 3 && nx > 3 * 64;
      if (cols3) {
        a.halo = 8;
        const int maxu = 3 * 64 - 16;
        const int ns = (nx + maxu - 1) / maxu;
        a.strip_w = (((nx + ns - 1) / ns) + 1) & ~1;
        a.nstrips = (nx + a.strip_w - 1) / a.strip_w;
      } else if (nx <= cw2) {
        a.strip_w = nx; a.halo = 0; a.nstrips = 1;
      } else {
        a.halo = 8; a.strip_w = cw2 - 16;
        a.nstrips = (nx + a.strip_w - 1) / a.strip_w;
      }
      const int band = h->var.march_band ? h->var.march_band : (cols3 ? 1024 : 512);
      // bands of rows (16 rows of pipeline fill each): ≥ 4 waves at 3 CTAs/SM, ≥ 128 rows per band
      int br = std::min(ny, band);
      while (br > 128 && (size_t)h->L * a.nstrips * ((ny + br - 1) / br) < 4 * 3 * 148) br = (br + 1) / 2;
      a.band_rows = br;
      a.nbands = (ny + a.band_rows - 1) / a.band_rows;
      const unsigned blocks = (unsigned)((size_t)h->L * a.nstrips * a.nbands);
      int st_i = 1;
      while (st_i < nsteps) {
        double* out = (cur == h->Y0) ? h->Y1 : h->Y0;
        a.y_in = cur;
        a.y_out = out;
        a.z_zero = (st_i == 1);
        if (nsteps - st_i >= 2) {
          const int km = kbegin(h, PX_KCLASS_MARCH2, s);
          PX_TRY(cols3 ? launch_marchc(h, a, blocks, false, s) : launch_march2(h, a, blocks, zlanes, s));
          kend(h, km, s);
          st_i += 2;
        } else if (cols3) {
          PX_TRY(launch_marchc(h, a, blocks, true, s));  // the three-column kernel, one step
          st_i += 1;
        } else {
          PX_TRY(launch_march1(h, a, h->L, zlanes, true, s));  // odd remainder: one single-step launch
          st_i += 1;
        }
        PX_CHECK_LAUNCH(h);
        cur = out;
      }
    } else {
      for (int st_i = 1; st_i < nsteps; ++st_i) {
        double* out = (cur == h->Y0) ? h->Y1 : h->Y0;
        a.y_in = cur;
        a.y_out = out;
        a.z_zero = (st_i == 1);
        a.step = st_i;
        PX_TRY(launch_march1(h, a, h->L, zlanes, false, s));
        PX_CHECK_LAUNCH(h);
        cur = out;
      }
    }
    launched_steps = (law && !adjoint) ? nsteps : nsteps - 1;
    h->z_valid = zlanes;
  }
  const double bytes_per_point = (adjoint && !h->z_closed) ? 40.0 : 24.0;  // y, b, y' (+ z in/out)
  h->stats.rk4_lane_steps += (uint64_t)h->L * launched_steps;
  // algorithmic bytes: 24n (40n with the ∫ accumulator) per lane and RK4
  // step — per step also when one launch advances two steps (the fused launch streams
  // y, b, y_out once for both, i.e. half the model's bytes: temporal blocking)
  const double bytes = bytes_per_point * (double)h->n * h->L * (double)launched_steps;
  h->stats.rk4_bytes += bytes;
  h->stats.algorithmic_bytes += bytes;
  *final_out = cur;
  return PX_OK;
}

// G[b] = Σ_p Z[b,p] (when with_z) + scale·c[b]: the adjoint lanes' ∫ with the per-lane accumulator
int lane_sum_plus(Handle* h, double* out, const double* lanes, const double* c, double scale, bool with_z,
                  cudaStream_t s) {
  px::k_lane_sum_plus<<<grid_stride(h->n, h->B), 256, 0, s>>>(out, lanes, h->Pl, c, scale, h->n, with_z ? 1 : 0);
  PX_CHECK_LAUNCH(h);
  return PX_OK;
}

}  // namespace pxi
