// cheb_march.cuh — M Chebyshev terms per pass, row-marching (2D).
//
// Replaces the reference's Newton–Leja loop (timestepping.py:343-356: one CSR
// matvec + two norms per term) by the planned Chebyshev series of
// exp(τM)·v (and τφ₁(τM)·v) with the stencil fused into the three-term
// recurrence
//     U_1 = (M − c0)U_0 / d,   U_{j+1} = (2/d)(M − c0)U_j + σ·U_{j−1},
//     acc += b_j U_j,  pacc += p_j U_j.
// A pass computes terms k+1 … k+M for one strip/band of a field: term s of the
// pass works on row r−s while row r of U_k streams in, so only U_{k−1}, U_k,
// acc, pacc are read and U_{k+M−1}, U_{k+M}, acc, pacc written once per pass —
// ≈ (4+4)·8n bytes per M terms instead of 56n per term. The x neighbours of each
// term's input row are exchanged through shared memory (even/odd split arrays,
// double buffered, one barrier per row); vertical neighbours and the per-row
// acc/pacc values live in register queues (the loop is unrolled so the queues
// rotate by renaming).
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"

namespace px {

// ---------------------------------------------------------------------------
// Chebyshev exponential action: stencil fused with the three-term recurrence
// ---------------------------------------------------------------------------

struct ChebFirstArgs {
  const double* u0; long long u0_bstride;     // U_0 (batch-strided)
  double* u1;                                 // U_1 = (M U_0 − c0 U_0)/d  (B × n)
  double* acc;                                // b0 U_0 + b1 U_1 (+ addend)
  const double* addend; long long add_bstride;  // may be nullptr
  double* pacc;                               // += p0 U_0 + p1 U_1 (may be nullptr)
  Stencil5 st;
  double c0, d, b0, b1, p0, p1;
  int nx, ny;
};

template <int DIM>
__global__ void __launch_bounds__(256) k_cheb_first(ChebFirstArgs a) {
  const size_t n = (size_t)a.nx * a.ny;
  const int b = blockIdx.y;
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int y = (int)(i / a.nx), x = (int)(i - (size_t)y * a.nx);
  const double* u0 = a.u0 + b * a.u0_bstride;
  const double u = u0[i];
  const double v1 = (stencil_at<DIM>(u0, a.st, x, y, a.nx, a.ny) - a.c0 * u) / a.d;
  const size_t o = (size_t)b * n + i;
  a.u1[o] = v1;
  double r = a.b0 * u + a.b1 * v1;
  if (a.addend) r += a.addend[b * a.add_bstride + i];
  a.acc[o] = r;
  if (a.pacc) a.pacc[o] += a.p0 * u + a.p1 * v1;
}

struct ChebTermArgs {
  const double* ucur; long long ucur_bstride;
  const double* uprev; long long uprev_bstride;
  double* unext;      // B × n
  double* acc;        // B × n
  double* pacc;       // may be nullptr
  Stencil5 st;
  double c0, two_over_d, sigma, bk, pk;
  int nx, ny;
};

template <int DIM>
__global__ void __launch_bounds__(256) k_cheb_term(ChebTermArgs a) {
  const size_t n = (size_t)a.nx * a.ny;
  const int b = blockIdx.y;
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int y = (int)(i / a.nx), x = (int)(i - (size_t)y * a.nx);
  const double* uc = a.ucur + b * a.ucur_bstride;
  const double* up = a.uprev + b * a.uprev_bstride;
  const double u = uc[i];
  const double un = a.two_over_d * (stencil_at<DIM>(uc, a.st, x, y, a.nx, a.ny) - a.c0 * u) +
                    a.sigma * up[i];
  const size_t o = (size_t)b * n + i;
  a.unext[o] = un;
  a.acc[o] += a.bk * un;
  if (a.pacc) a.pacc[o] += a.pk * un;
}


// CTA size / resident CTAs per SM (compile-time experiment knobs). Measured on config 5 (both scans
// per gradient): 160 × 2 → 106.4 ms, 128 × 3 → 99.0 ms, 96 × 4 → 101.4 ms, 64 × 6 → 102.1 ms, 192 × 2 slower:
// four warps per CTA spread evenly over the SM's four schedulers, 12 resident warps, 168 registers.
#ifndef PX_CM_NT
#define PX_CM_NT 128
#endif
#ifndef PX_CM_MINB
#define PX_CM_MINB 3
#endif
constexpr int CM_NT = PX_CM_NT;  // pairs of columns per thread: computed width ≤ 2·CM_NT
constexpr int CM_MAXT = 7;  // terms per pass (template M ≤ CM_MAXT)
constexpr int CM_DEPTH = 5; // cp.async ring depth (rows)
constexpr int CM_MINB = PX_CM_MINB;  // resident CTAs per SM

struct ChebMarchArgs {
  const double* u_prev; long long prev_bs;  // U_{k−1} (unused on the first pass)
  const double* u_cur; long long cur_bs;    // U_k (first pass: U_0)
  const double* addend; long long add_bs;   // first pass only, may be null
  double* acc;                              // B × n (in/out; first pass: out)
  double* pacc;                             // B × n in/out, may be null
  double* out_prev;                         // U_{k+M−1} (null on the last pass)
  double* out_cur;                          // U_{k+M}
  double* ssum;                             // SS passes: S += acc at every completed row (B × n)
  Stencil5 st;
  double c0, d, two_over_d, sigma;
  double be[CM_MAXT + 1], bp[CM_MAXT + 1];  // coefficients of terms k … k+M
  double g[5];  // (2/d)·(cc − c0, ce, cw, cs, cn): U_{j+1} = Σ g·U_j(stencil) + σ·U_{j−1}
  double f[5];  // (1/d)·(cc − c0, ce, cw, cs, cn): U_1 of the first pass
  int first;
  int nx, ny, B;
  int strip_w, halo, nstrips, band_rows, nbands;
};

template <int M>
struct CmUnroll {  // multiple of 3 (U_k rows), 2 (stage rows) and R
  static constexpr int value = (M == 4) ? 12 : 6;
};
// acc/pacc row slots: M live rows (r−1 … r−M), UN % R == 0. M = 7 keeps M − 1 = 6 slots: the
// new row r−1 (term 1) waits in a temporary until term M has completed and stored row r−M,
// whose slot it then takes (same slot index), so the unroll stays 6.
template <int M>
struct CmRing {
  static constexpr int value = (M <= 3) ? M : (M == 4 ? 4 : 6);
};
template <int M>
struct CmTemp {
  static constexpr bool value = CmRing<M>::value == M - 1;
};

// SG: the recurrence sign σ (±1) as a compile-time constant (0: runtime a.sigma); PH: the φ₁
// accumulator is updated (a.pacc must be non-null), compiled out otherwise; SS (last pass of an
// adjoint carry, not with PH): the completed acc rows (the next carry's input) are also added
// into a.ssum, streamed through the ring's fourth slot at lag M (Σ of the carry inputs: the
// adjoint's φ₁ integral is one action on that sum, sweeps.cu). The
// row ring is filled by per-thread cp.async (a one-thread TMA bulk-copy ring issued after the
// row barrier was measured 15% slower on the scan's short bands).
template <int M, int SG, bool PH, bool SS = false>
__global__ void __launch_bounds__(CM_NT, CM_MINB) k_cheb_march(ChebMarchArgs a) {
  static_assert(!(PH && SS), "the ring has one spare slot: φ accumulator or the carry-input sum");
  __shared__ double pubE[2][M][CM_NT];
  __shared__ double pubO[2][M][CM_NT];
  // ring slots (dynamic smem): [depth][4 arrays: cur(r), prev(r−1), acc(r−1), pacc(r−1)][pairs]
  extern __shared__ double2 cm_ring[];
  constexpr int UN = CmUnroll<M>::value;
  constexpr int R = CmRing<M>::value;
  constexpr bool TEMP = CmTemp<M>::value;

  const int b = blockIdx.x % a.B;
  const int rest = blockIdx.x / a.B;
  const int strip = rest % a.nstrips;
  const int band = rest / a.nstrips;
  const int nx = a.nx, ny = a.ny;
  const size_t n = (size_t)nx * ny;
  const int x0 = strip * a.strip_w;
  const int U = min(a.strip_w, nx - x0);
  const int CW = U + 2 * a.halo;
  const int T = CW >> 1;
  const int t = threadIdx.x;
  const bool active = t < T;
  const int tc = active ? t : 0;
  const int gx = (((x0 - a.halo + 2 * tc) % nx) + nx) % nx;
  const int j0 = band * a.band_rows;
  const int rows_out = min(a.band_rows, ny - j0);
  const int iters = rows_out + 2 * M;
  const bool full_row = a.halo == 0;
  const int tl = (t == 0) ? (full_row ? T - 1 : 0) : t - 1;
  const int tr = (t + 1 >= T) ? (full_row ? 0 : T - 1) : t + 1;
  const bool store_ok = active && (2 * t >= a.halo) && (2 * t + 1 < CW - a.halo);
  const bool first = a.first != 0;
  const bool has_add = first && a.addend != nullptr;
  constexpr bool has_p = PH;
  const bool write_u = a.out_cur != nullptr;

  const double sig = a.sigma;
  auto sgm = [&](double v) -> double {
    if constexpr (SG == 1) return v;
    else if constexpr (SG == -1) return -v;
    else return sig * v;
  };
  const double* __restrict__ cur = a.u_cur + b * a.cur_bs;
  const double* __restrict__ prv = first ? cur : a.u_prev + b * a.prev_bs;
  const double* __restrict__ accin = has_add ? a.addend + b * a.add_bs : a.acc + (size_t)b * n;
  double* __restrict__ accout = a.acc + (size_t)b * n;
  double* __restrict__ pac = has_p ? a.pacc + (size_t)b * n : nullptr;
  double* __restrict__ oprev = write_u ? a.out_prev + (size_t)b * n : nullptr;
  double* __restrict__ ocur = write_u ? a.out_cur + (size_t)b * n : nullptr;
  double* __restrict__ ssm = SS ? a.ssum + (size_t)b * n : nullptr;
  const bool read_acc = !first || has_add;

  auto wrapr = [&](int row) -> int {
    row %= ny;
    return row < 0 ? row + ny : row;
  };
  const int r0 = j0 - M;
  const size_t coloff = (size_t)gx;
  int iss_k = 0, iss_slot = 0;
  // streams: cur row r, lagged rows r−1 (SS: the sum at row r−M, the row completing)
  int rc = wrapr(r0), rl = wrapr(r0 - 1), rm = wrapr(r0 - M);
  auto issue = [&]() {
    if (iss_k < iters) {
      double2* sl = cm_ring + (size_t)iss_slot * 4 * CM_NT;
      cp_async16(sl + t, cur + (size_t)rc * nx + coloff);
      if (!first) cp_async16(sl + CM_NT + t, prv + (size_t)rl * nx + coloff);
      if (read_acc) cp_async16(sl + 2 * CM_NT + t, accin + (size_t)rl * nx + coloff);
      if (has_p) cp_async16(sl + 3 * CM_NT + t, pac + (size_t)rl * nx + coloff);
      if constexpr (SS) cp_async16(sl + 3 * CM_NT + t, ssm + (size_t)rm * nx + coloff);
    }
    cp_async_commit();
    ++iss_k;
    iss_slot = (iss_slot + 1 == CM_DEPTH) ? 0 : iss_slot + 1;
    rc = (rc + 1 == ny) ? 0 : rc + 1;
    if constexpr (SS) rm = (rm + 1 == ny) ? 0 : rm + 1;
    rl = (rl + 1 == ny) ? 0 : rl + 1;
  };
#pragma unroll
  for (int k = 0; k < CM_DEPTH; ++k) issue();
  int rslot = 0;
  int rs = wrapr(r0 - M);  // output row r − M

  double2 q0[3];               // U_k rows (ring by phase mod 3)
  double2 qs[M + 1][2];        // stage-s outputs, last two rows (index 1..M)
  double2 qa[R], qp[PH ? R : 1];  // acc / pacc of rows r−1 … r−M (ring by phase mod R)
#pragma unroll
  for (int k = 0; k < 3; ++k) q0[k] = make_double2(0.0, 0.0);
#pragma unroll
  for (int s = 0; s <= M; ++s) qs[s][0] = qs[s][1] = make_double2(0.0, 0.0);
#pragma unroll
  for (int s = 0; s < R; ++s) qa[s] = make_double2(0.0, 0.0);
#pragma unroll
  for (int s = 0; s < (PH ? R : 1); ++s) qp[s] = make_double2(0.0, 0.0);

  // One Chebyshev term on a column pair: Σ_q coef_q·(stencil tap q) + base, the
  // coefficients pre-scaled on the host (kernel parameters → constant-bank operands);
  // the north neighbour (this iteration's previous term) enters last.
  auto term = [&](const double* cf, double2 base, double2 c, double2 so, double2 nn, double l, double r) -> double2 {
    double x = fma(cf[0], c.x, base.x);
    x = fma(cf[1], c.y, x);
    x = fma(cf[2], l, x);
    x = fma(cf[3], so.x, x);
    double y = fma(cf[0], c.y, base.y);
    y = fma(cf[1], r, y);
    y = fma(cf[2], c.x, y);
    y = fma(cf[3], so.y, y);
    return make_double2(fma(cf[4], nn.x, x), fma(cf[4], nn.y, y));
  };

  // One iteration at ring phase k (compile time); G = guarded (pipeline fill/drain).
  auto iter = [&](auto kc, auto gc, const int i) {
    constexpr int k = decltype(kc)::value % UN;
    constexpr bool G = decltype(gc)::value;
      const int pin = (k + 1) & 1;
      const int pout = k & 1;
      cp_async_wait<CM_DEPTH - 1>();
      const double2* sl = cm_ring + (size_t)rslot * 4 * CM_NT;
      rslot = (rslot + 1 == CM_DEPTH) ? 0 : rslot + 1;
      const double2 ur = sl[t];
      const double2 upv = first ? make_double2(0.0, 0.0) : sl[CM_NT + t];
      const double2 ain = read_acc ? sl[2 * CM_NT + t] : make_double2(0.0, 0.0);
      const double2 pin_v = (has_p || SS) ? sl[3 * CM_NT + t] : make_double2(0.0, 0.0);  // SS: S(r−M)
      issue();
      q0[k % 3] = ur;
      const double2 u0m2 = q0[(k + 1) % 3], u0m1 = q0[(k + 2) % 3];  // rows r−2, r−1
      const int po = k & 1, pp = (k + 1) & 1;  // qs[s][po]: row of iteration i−2, [pp]: i−1
      double2 nq[M + 1];
      nq[0] = ur;
      double2 acc1 = make_double2(0.0, 0.0), pc1 = make_double2(0.0, 0.0);  // TEMP: row r−1's entry
      // term 1 of the pass at row r−1 (creates the acc/pacc entry of that row)
      if (!G || i >= 2) {
        const double l = pubO[pin][0][tl], r = pubE[pin][0][tr];
        double2 u1, acc, pc;
        if (first) {
          u1 = term(a.f, make_double2(0.0, 0.0), u0m1, u0m2, ur, l, r);
          acc.x = a.be[0] * u0m1.x + a.be[1] * u1.x + ain.x;
          acc.y = a.be[0] * u0m1.y + a.be[1] * u1.y + ain.y;
          pc.x = pin_v.x + (a.bp[0] * u0m1.x + a.bp[1] * u1.x);
          pc.y = pin_v.y + (a.bp[0] * u0m1.y + a.bp[1] * u1.y);
        } else {
          u1 = term(a.g, make_double2(sgm(upv.x), sgm(upv.y)), u0m1, u0m2, ur, l, r);
          acc = make_double2(ain.x + a.be[1] * u1.x, ain.y + a.be[1] * u1.y);
          pc = make_double2(pin_v.x + a.bp[1] * u1.x, pin_v.y + a.bp[1] * u1.y);
        }
        nq[1] = u1;
        if constexpr (TEMP) {
          acc1 = acc;
          pc1 = pc;
        } else {
          qa[k % R] = acc;
          if constexpr (PH) qp[k % R] = pc;
        }
      } else {
        nq[1] = make_double2(0.0, 0.0);
      }
      // terms 2 … M of the pass at rows r−s
#pragma unroll
      for (int s = 2; s <= M; ++s) {
        if (!G || i >= 2 * s) {
          const double l = pubO[pin][s - 1][tl], r = pubE[pin][s - 1][tr];
          const double2 c = qs[s - 1][pp];        // row r−s
          const double2 so = qs[s - 1][po];       // row r−s−1
          const double2 pv = (s == 2) ? u0m2 : qs[s - 2][po];  // U_{k+s−2} at row r−s
          const double2 u = term(a.g, make_double2(sgm(pv.x), sgm(pv.y)), c, so, nq[s - 1], l, r);
          nq[s] = u;
          const int ai = (k - s + 1 + 2 * R) % R;  // acc slot of row r−s
          qa[ai].x += a.be[s] * u.x;
          qa[ai].y += a.be[s] * u.y;
          if constexpr (PH) {
            qp[ai].x += a.bp[s] * u.x;
            qp[ai].y += a.bp[s] * u.y;
          }
        } else {
          nq[s] = make_double2(0.0, 0.0);
        }
      }
      // row r−M is complete: acc, pacc, and the pass's last two terms
      if ((!G || i >= 2 * M) && store_ok) {
        const size_t off = (size_t)rs * nx + coloff;
        const int ai = (k - M + 1 + 2 * R) % R;
        __stcs(reinterpret_cast<double2*>(accout + off), qa[ai]);
        if constexpr (PH) __stcs(reinterpret_cast<double2*>(pac + off), qp[ai]);
        if constexpr (SS) __stcs(reinterpret_cast<double2*>(ssm + off), make_double2(pin_v.x + qa[ai].x, pin_v.y + qa[ai].y));
        if (write_u) {
          const double2 up = (M == 1) ? u0m1 : qs[M - 1][pp];
          __stcs(reinterpret_cast<double2*>(oprev + off), up);
          __stcs(reinterpret_cast<double2*>(ocur + off), nq[M]);
        }
      }
      if constexpr (TEMP) {  // row r−M is out: its slot (k mod R) takes row r−1
        qa[k % R] = acc1;
        if constexpr (PH) qp[k % R] = pc1;
      }
      rs = (rs + 1 == ny) ? 0 : rs + 1;
#pragma unroll
      for (int s = 1; s <= M; ++s) qs[s][po] = nq[s];
      if (active) {
#pragma unroll
        for (int s = 0; s < M; ++s) {
          pubE[pout][s][t] = nq[s].x;
          pubO[pout][s][t] = nq[s].y;
        }
      }
      __syncthreads();
  };
  int i0 = 0;
  // fill (stages switch on at i = 2, 4, …, 2M) — guarded groups until every stage is live
  for (; i0 < 2 * M; i0 += UN) {
    if (i0 + UN > iters) break;
    iter(IC<0>{}, BC<true>{}, i0); iter(IC<1>{}, BC<true>{}, i0 + 1); iter(IC<2>{}, BC<true>{}, i0 + 2);
    iter(IC<3>{}, BC<true>{}, i0 + 3); iter(IC<4>{}, BC<true>{}, i0 + 4); iter(IC<5>{}, BC<true>{}, i0 + 5);
    if (UN == 12) {
      iter(IC<6>{}, BC<true>{}, i0 + 6); iter(IC<7>{}, BC<true>{}, i0 + 7); iter(IC<8>{}, BC<true>{}, i0 + 8);
      iter(IC<9>{}, BC<true>{}, i0 + 9); iter(IC<10>{}, BC<true>{}, i0 + 10); iter(IC<11>{}, BC<true>{}, i0 + 11);
    }
  }
  if (i0 >= 2 * M) {
    for (; i0 + UN <= iters; i0 += UN) {  // steady state: no guards
      iter(IC<0>{}, BC<false>{}, i0); iter(IC<1>{}, BC<false>{}, i0 + 1); iter(IC<2>{}, BC<false>{}, i0 + 2);
      iter(IC<3>{}, BC<false>{}, i0 + 3); iter(IC<4>{}, BC<false>{}, i0 + 4); iter(IC<5>{}, BC<false>{}, i0 + 5);
      if (UN == 12) {
        iter(IC<6>{}, BC<false>{}, i0 + 6); iter(IC<7>{}, BC<false>{}, i0 + 7); iter(IC<8>{}, BC<false>{}, i0 + 8);
        iter(IC<9>{}, BC<false>{}, i0 + 9); iter(IC<10>{}, BC<false>{}, i0 + 10); iter(IC<11>{}, BC<false>{}, i0 + 11);
      }
    }
  }
  // drain / short bands
  if (i0 + 0 < iters) iter(IC<0>{}, BC<true>{}, i0);
  if (i0 + 1 < iters) iter(IC<1>{}, BC<true>{}, i0 + 1);
  if (i0 + 2 < iters) iter(IC<2>{}, BC<true>{}, i0 + 2);
  if (i0 + 3 < iters) iter(IC<3>{}, BC<true>{}, i0 + 3);
  if (i0 + 4 < iters) iter(IC<4>{}, BC<true>{}, i0 + 4);
  if (i0 + 5 < iters) iter(IC<5>{}, BC<true>{}, i0 + 5);
  if (UN == 12) {
    if (i0 + 6 < iters) iter(IC<6>{}, BC<true>{}, i0 + 6);
    if (i0 + 7 < iters) iter(IC<7>{}, BC<true>{}, i0 + 7);
    if (i0 + 8 < iters) iter(IC<8>{}, BC<true>{}, i0 + 8);
    if (i0 + 9 < iters) iter(IC<9>{}, BC<true>{}, i0 + 9);
    if (i0 + 10 < iters) iter(IC<10>{}, BC<true>{}, i0 + 10);
    if (i0 + 11 < iters) iter(IC<11>{}, BC<true>{}, i0 + 11);
  }
  cp_async_wait<0>();
}

constexpr size_t CM_SMEM = (size_t)CM_DEPTH * 4 * CM_NT * sizeof(double2);

}  // namespace px
