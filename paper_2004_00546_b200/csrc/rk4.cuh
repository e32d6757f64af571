// rk4.cuh — zero-data RK4 slice solves for the linear testbed, all lanes batched.
//
// For y' = M·y + g with constant g (absorbed initial / final condition,
// paraexp.py:239-242, :268-270) one classical RK4 step is exactly
//     y⁺ = R(hM)·y + b,   R(x) = 1 + x·S(x),   S(x) = 1 + x/2 + x²/6 + x³/24,
//     b  = h·S(hM)·g,
// and the RK4-consistent running integral z = ∫y (RK4 on the augmented system
// (y, z)' = (M y + g, y)) advances by  h·S(hM)·y + c,  c = h²·U(hM)·g,
// U(x) = 1/2 + x/6 + x²/24. The Horner evaluation of R,
//     w1 = y + (h/4)·M·y,  w2 = y + (h/3)·M·w1,  w3 = y + (h/2)·M·w2 (= S(hM)y),
//     y⁺ = y + h·M·w3 + b,
// needs four stencil applications per step like the stage form, but no source
// reads and no stage accumulators, and it yields S(hM)y (= w3) for the integral.
// b and c are formed once per sweep and member (3 stencil passes).
//
// 2D kernel (k_rk4_march): each CTA owns a strip of columns of one lane and
// MARCHES along y; the four Horner stages are pipelined one row apart
// (stage s of iteration i works on row r−s), so the vertical neighbours come
// from per-thread register row queues and only the x neighbours are exchanged
// through shared memory (even/odd split arrays, double buffered: one barrier
// per row). Strips are 512 columns wide with a 4-column recomputed halo (or the
// whole periodic row when nx ≤ 576); bands of rows add 8 pipeline-fill rows.
// HBM traffic ≈ 24n per step (y, b in; y⁺ out) + 16n with z.
//
// Two-step kernels (k_rk4_march2, k_rk4_marchc): the same march with the 8 Horner
// stages of two consecutive steps pipelined (y⁺⁺ at row r−8), so y, b and y_out
// cross DRAM once per two steps. k_rk4_marchc (the large-grid default) gives each
// thread three contiguous columns — the x-neighbour exchange, which bounds these
// kernels on the shared-memory data pipe, costs the same per thread for any column
// count — and streams the rows with 1D bulk copies (TMA) into an mbarrier ring.
//
// 1D kernel (k_rk4_lane1d): a lane (≤ 8192 points) lives on chip; one CTA runs
// all nsteps of its lane, exchanging only the edge values of each thread's run.
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"

namespace px {

constexpr int MARCH_NT = 288;          // 9 warps: pairs of columns per thread
constexpr int MARCH_MAX_CW = 2 * MARCH_NT;
constexpr int MARCH_STRIP = 512;       // useful strip width in strip mode
constexpr int MARCH_HALO = 4;

struct MarchArgs {
  const double* y_in;  // lanes × n; nullptr → y = b (state after the first step from zero)
  double* y_out;       // lanes × n
  const double* b;     // B × n   h·S(hM)·g
  double* z;           // ADJ: lanes × n, z += h·w3
  int z_zero;          // ADJ: treat z_in as 0
  Stencil5 st;
  double h;
  int nx, ny, lanes, lanes_per_b;
  int strip_w;   // useful width per strip (even)
  int halo;      // MARCH_HALO (strips) or 0 (whole periodic row in one CTA)
  int nstrips, band_rows, nbands;
  // k_rk4_march2: stage-scaled stencil k·(cc, ce, cw, cs, cn) for k = h/4, h/3, h/2, h
  double kc[4][5];
  // time law (k_rk4_march<·, true>): forcing θ(t)·f with θ = law[0] + law[1] sin(law[3] t) +
  // law[2] cos(law[3] t); lane p of the rank starts at (p_begin + p)·delta; `step` is the
  // launch's step within the lanes
  const double* f;     // B × n control field (direct lanes)
  double law[4];
  double delta;
  int p_begin, step;
};

__device__ __forceinline__ double law_at(const double* law, double t) {
  return law[0] + law[1] * sin(law[3] * t) + law[2] * cos(law[3] * t);
}

// Per-step scalars of the time law. Direct lanes (forcing θ·f at the stage times of the step
// from t): the Horner stages take +α_s·f and the update +γ·f,
//   α1 = hθ1/4, α2 = h(θ1+θ2)/6, α3 = h(θ1+2θ2)/6, γ = h(θ1+4θ2+θ4)/6
// (θ1 = θ(t), θ2 = θ(t+h/2), θ4 = θ(t+h)) — exactly classical RK4 with a time-dependent source.
// Adjoint lanes (reflected time from t down): the θ-weighted RK4-consistent ∫ of the state,
// h/6[θa·Y1 + 2θm(Y2 + Y3) + θb·Y4], is β0·y + β2·w2 + β3·w3 in the Horner stages
// (Y2 = 2w1 − y, Y3 = 3w2 − 2w1, Y4 = y + 6w3 − 6w2 without the source, whose part is summed
// once per sweep on the host), β0 = h(θa − 2θm + θb)/6, β2 = h(θm − θb), β3 = h·θb.
struct LawStep {
  double c0, c1, c2, c3;  // direct: α1, α2, α3, γ; adjoint: β0, β2, β3, unused
};
__device__ __forceinline__ LawStep law_step(const double* law, bool adjoint, double t, double h) {
  LawStep r;
  if (!adjoint) {
    const double t1 = law_at(law, t), t2 = law_at(law, t + 0.5 * h), t4 = law_at(law, t + h);
    r.c0 = h * t1 * 0.25;
    r.c1 = h * (t1 + t2) / 6.0;
    r.c2 = h * (t1 + 2.0 * t2) / 6.0;
    r.c3 = h * (t1 + 4.0 * t2 + t4) / 6.0;
  } else {
    const double ta = law_at(law, t), tm = law_at(law, t - 0.5 * h), tb = law_at(law, t - h);
    r.c0 = h * (ta - 2.0 * tm + tb) / 6.0;
    r.c1 = h * (tm - tb);
    r.c2 = h * tb;
    r.c3 = 0.0;
  }
  return r;
}

// Row ring: each thread streams its own column pair of the y, b (and z) rows
// MARCH_DEPTH rows ahead with cp.async (LDGSTS) into shared memory, so ~6 rows
// per CTA are in flight without holding registers; a thread only reads back
// the bytes it copied, so the ring needs no barrier.
// ring depth: 6 rows (direct: y, b) / 4 rows (adjoint: y, b, z) keeps two CTAs per SM
template <bool ADJ>
struct MarchDepth {
  static constexpr int value = ADJ ? 4 : 6;
};

// LAW: time-law forcing (direct: a third ring stream f at row r−1, kept four rows deep in
// registers; adjoint: the θ-weighted ∫ instead of z += h·w3)
template <bool ADJ, bool LAW = false>
__global__ void __launch_bounds__(MARCH_NT, 2) k_rk4_march(MarchArgs a) {
  constexpr int NQ = (ADJ || LAW) ? 3 : 2;  // streamed arrays: y, b (, z | f)
  constexpr int MARCH_DEPTH = MarchDepth<ADJ>::value;
  // publish area: [parity][quantity: y, w1, w2, w3][pair] split in even / odd columns
  __shared__ double pubE[2][4][MARCH_NT];
  __shared__ double pubO[2][4][MARCH_NT];
  extern __shared__ double2 ring[];  // [MARCH_DEPTH][NQ][MARCH_NT]

  const int lane = blockIdx.x % a.lanes;
  const int rest = blockIdx.x / a.lanes;
  const int strip = rest % a.nstrips;
  const int band = rest / a.nstrips;
  const int nx = a.nx, ny = a.ny;
  const size_t n = (size_t)nx * ny;
  const int x0 = strip * a.strip_w;
  const int U = min(a.strip_w, nx - x0);
  const int CW = U + 2 * a.halo;
  const int T = CW >> 1;  // active pairs
  const int t = threadIdx.x;
  const bool active = t < T;
  const int tc = active ? t : 0;
  const int gx = (((x0 - a.halo + 2 * tc) % nx) + nx) % nx;  // even
  const int j0 = band * a.band_rows;
  const int rows_out = min(a.band_rows, ny - j0);
  const int iters = rows_out + 8;
  const bool full_row = a.halo == 0;
  const int tl = (t == 0) ? (full_row ? T - 1 : 0) : t - 1;
  const int tr = (t + 1 >= T) ? (full_row ? 0 : T - 1) : t + 1;
  const bool store_ok = active && (2 * t >= a.halo) && (2 * t + 1 < CW - a.halo);

  const Stencil5 st = a.st;
  const double h = a.h, c1 = a.h * 0.25, c2 = a.h / 3.0, c3 = a.h * 0.5;
  const size_t member = (size_t)(lane / a.lanes_per_b);
  const double* __restrict__ bsrc = a.b + member * n;
  const double* __restrict__ ysrc = a.y_in ? a.y_in + (size_t)lane * n : bsrc;
  double* __restrict__ yout = a.y_out + (size_t)lane * n;
  double* __restrict__ zl = ADJ ? a.z + (size_t)lane * n : nullptr;
  const bool zread = ADJ && !a.z_zero;
  const double* __restrict__ fsrc = (LAW && !ADJ) ? a.f + member * n : nullptr;
  LawStep ls{0.0, 0.0, 0.0, 0.0};
  if (LAW) {
    const int p = a.p_begin + lane % a.lanes_per_b;
    ls = ADJ ? law_step(a.law, true, (p + 1) * a.delta - a.step * h, h)
             : law_step(a.law, false, p * a.delta + a.step * h, h);
  }

  // incremental periodic row counters (no per-row integer division)
  auto wrapr = [&](int row) -> int {
    row %= ny;
    return row < 0 ? row + ny : row;
  };
  const int r0 = j0 - 4;
  // issue stream: y row r0+k and b/z rows r0+k-4 for the k-th issued iteration
  int iss_k = 0, iss_slot = 0;
  int ry = wrapr(r0), rb = wrapr(r0 - 4), rf = wrapr(r0 - 1);
  const size_t coloff = (size_t)gx;
  auto issue = [&]() {
    if (iss_k < iters) {
      double2* slot = ring + (size_t)iss_slot * NQ * MARCH_NT;
      cp_async16(slot + t, ysrc + (size_t)ry * nx + coloff);
      cp_async16(slot + MARCH_NT + t, bsrc + (size_t)rb * nx + coloff);
      if (zread) cp_async16(slot + 2 * MARCH_NT + t, zl + (size_t)rb * nx + coloff);
      if (LAW && !ADJ) cp_async16(slot + 2 * MARCH_NT + t, fsrc + (size_t)rf * nx + coloff);
    }
    cp_async_commit();
    ++iss_k;
    iss_slot = (iss_slot + 1 == MARCH_DEPTH) ? 0 : iss_slot + 1;
    ry = (ry + 1 == ny) ? 0 : ry + 1;
    rb = (rb + 1 == ny) ? 0 : rb + 1;
    rf = (rf + 1 == ny) ? 0 : rf + 1;
  };
#pragma unroll
  for (int k = 0; k < MARCH_DEPTH; ++k) issue();
  int rslot = 0;              // ring slot consumed this iteration
  int rs = wrapr(r0 - 4);     // output row (r − 4) of this iteration

  // register row queues as rings indexed by the (unrolled, compile-time) iteration
  // phase k = i mod 6: y rows r-4..r in yq[(k-4..k) mod 6]; w1/w2/w3 keep the last
  // two rows in wq[(k-2) mod 2], wq[(k-1) mod 2]. Unrolling by 6 turns the queue
  // rotation into register renaming (no moves).
  double2 yq[6], w1q[2], w2q[2], w3q[2];
  double2 fq[LAW && !ADJ ? 6 : 1];  // f rows r-1 .. r-4 (ring by phase, like yq)
#pragma unroll
  for (int k = 0; k < 6; ++k) yq[k] = make_double2(0.0, 0.0);
#pragma unroll
  for (int k = 0; k < (LAW && !ADJ ? 6 : 1); ++k) fq[k] = make_double2(0.0, 0.0);
#pragma unroll
  for (int k = 0; k < 2; ++k) w1q[k] = w2q[k] = w3q[k] = make_double2(0.0, 0.0);

  auto apply = [&](double2 c, double2 s, double2 nn, double l, double r) -> double2 {
    double2 o;
    o.x = st.cc * c.x;
    o.x += st.ce * c.y;
    o.x += st.cw * l;
    o.x += st.cn * nn.x;
    o.x += st.cs * s.x;
    o.y = st.cc * c.y;
    o.y += st.ce * r;
    o.y += st.cw * c.x;
    o.y += st.cn * nn.y;
    o.y += st.cs * s.y;
    return o;
  };

  for (int i0 = 0; i0 < iters; i0 += 6) {
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      const int i = i0 + k;
      if (i >= iters) break;
      const int pin = (k + 1) & 1;  // parity published in the previous iteration (i0 even)
      const int pout = k & 1;
      cp_async_wait<MARCH_DEPTH - 1>();
      const double2* slot = ring + (size_t)rslot * NQ * MARCH_NT;
      rslot = (rslot + 1 == MARCH_DEPTH) ? 0 : rslot + 1;
      const double2 yr = slot[t];
      const double2 brow = slot[MARCH_NT + t];  // row r-4
      const double2 zrow = zread ? slot[2 * MARCH_NT + t] : make_double2(0.0, 0.0);
      if constexpr (LAW && !ADJ) fq[k] = slot[2 * MARCH_NT + t];  // f row r-1
      issue();  // refills the slot just consumed (its values are in registers)
      yq[k] = yr;
      // f at the stage rows r-1 .. r-4 (time law; zero otherwise)
      auto frow = [&](int back) -> double2 {
        if constexpr (LAW && !ADJ) return fq[(k + 6 - back) % 6];
        else return make_double2(0.0, 0.0);
      };
      // rows r-4 .. r-1 (yr = row r)
      const double2 y0 = yq[(k + 2) % 6], y1 = yq[(k + 3) % 6], y2 = yq[(k + 4) % 6], y3 = yq[(k + 5) % 6];
      const int po = k & 1, pp = (k + 1) & 1;  // w?q[po]: row of iteration i-2, [pp]: i-1

      double2 nw1 = make_double2(0.0, 0.0), nw2 = nw1, nw3 = nw1;
      if (i >= 2) {  // stage 1 at row r-1: w1 = y + (h/4)·M·y
        const double l = pubO[pin][0][tl], rr = pubE[pin][0][tr];
        const double2 m = apply(y3, y2, yr, l, rr);
        nw1 = make_double2(y3.x + c1 * m.x, y3.y + c1 * m.y);
        if constexpr (LAW && !ADJ) {
          const double2 fv = frow(0);
          nw1.x = fma(ls.c0, fv.x, nw1.x);
          nw1.y = fma(ls.c0, fv.y, nw1.y);
        }
      }
      if (i >= 4) {  // stage 2 at row r-2: w2 = y + (h/3)·M·w1  (w1 rows r-3, r-2, r-1)
        const double l = pubO[pin][1][tl], rr = pubE[pin][1][tr];
        const double2 m = apply(w1q[pp], w1q[po], nw1, l, rr);
        nw2 = make_double2(y2.x + c2 * m.x, y2.y + c2 * m.y);
        if constexpr (LAW && !ADJ) {
          const double2 fv = frow(1);
          nw2.x = fma(ls.c1, fv.x, nw2.x);
          nw2.y = fma(ls.c1, fv.y, nw2.y);
        }
      }
      if (i >= 6) {  // stage 3 at row r-3: w3 = y + (h/2)·M·w2  (w2 rows r-4, r-3, r-2)
        const double l = pubO[pin][2][tl], rr = pubE[pin][2][tr];
        const double2 m = apply(w2q[pp], w2q[po], nw2, l, rr);
        nw3 = make_double2(y1.x + c3 * m.x, y1.y + c3 * m.y);
        if constexpr (LAW && !ADJ) {
          const double2 fv = frow(2);
          nw3.x = fma(ls.c2, fv.x, nw3.x);
          nw3.y = fma(ls.c2, fv.y, nw3.y);
        }
      }
      if (i >= 8) {  // stage 4 at row r-4: y⁺ = y + h·M·w3 + b  (w3 rows r-5, r-4, r-3)
        const double l = pubO[pin][3][tl], rr = pubE[pin][3][tr];
        const double2 w3c = w3q[pp];
        const double2 m = apply(w3c, w3q[po], nw3, l, rr);
        if (store_ok) {
          const size_t off = (size_t)rs * nx + coloff;
          double2 yn;
          yn.x = y0.x + h * m.x + brow.x;
          yn.y = y0.y + h * m.y + brow.y;
          if constexpr (LAW && !ADJ) {
            const double2 fv = frow(3);
            yn.x = fma(ls.c3, fv.x, yn.x);
            yn.y = fma(ls.c3, fv.y, yn.y);
          }
          __stcs(reinterpret_cast<double2*>(yout + off), yn);
          if (ADJ) {
            double2 zn;
            if constexpr (LAW) {  // θ-weighted ∫: β0·y + β2·w2 + β3·w3 at row r-4
              const double2 w2c = w2q[po];
              zn.x = fma(ls.c2, w3c.x, fma(ls.c1, w2c.x, fma(ls.c0, y0.x, zrow.x)));
              zn.y = fma(ls.c2, w3c.y, fma(ls.c1, w2c.y, fma(ls.c0, y0.y, zrow.y)));
            } else {
              zn.x = zrow.x + h * w3c.x;
              zn.y = zrow.y + h * w3c.y;
            }
            __stcs(reinterpret_cast<double2*>(zl + off), zn);
          }
        }
      }
      rs = (rs + 1 == ny) ? 0 : rs + 1;
      w1q[po] = nw1;
      w2q[po] = nw2;
      w3q[po] = nw3;
      if (active) {
        pubE[pout][0][t] = yr.x;  pubO[pout][0][t] = yr.y;
        pubE[pout][1][t] = nw1.x; pubO[pout][1][t] = nw1.y;
        pubE[pout][2][t] = nw2.x; pubO[pout][2][t] = nw2.y;
        pubE[pout][3][t] = nw3.x; pubO[pout][3][t] = nw3.y;
      }
      __syncthreads();
    }
  }
  cp_async_wait<0>();
}

inline size_t march_smem(bool adj, bool law = false) {
  return (size_t)(adj ? MarchDepth<true>::value * 3 : MarchDepth<false>::value * (law ? 3 : 2)) * MARCH_NT *
         sizeof(double2);
}

// ---------------------------------------------------------------------------
// 1D: one CTA per lane, all nsteps on chip
// ---------------------------------------------------------------------------

constexpr int LANE1D_MAX_N = 8192;

struct Lane1DArgs {
  double* y_out;      // lanes × n (lane end states)
  const double* b;    // B × n
  double* z;          // ADJ: lanes × n (written, Σ h·w3 over the steps)
  Stencil5 st;
  double h;
  int n, lanes_per_b, nsteps;
  // LAW (time-law forcing; see law_step): control field, law, slice width, first slice
  const double* f;
  double law[4];
  double delta;
  int p_begin;
};

template <int PPT, bool ADJ, bool FULL = false, bool LAW = false>
__global__ void __launch_bounds__(1024) k_rk4_lane1d(Lane1DArgs a) {
  __shared__ double eL[2][1024];
  __shared__ double eR[2][1024];
  const int n = a.n;
  const int lane = blockIdx.x;
  const int t = threadIdx.x;
  const int NT = blockDim.x;
  const int start = t * PPT;
  const int cnt = max(0, min(PPT, n - start));
  const int last = (n + PPT - 1) / PPT - 1;  // last thread with points
  const int tl = (t == 0) ? last : t - 1;
  const int tr = (t >= last) ? 0 : t + 1;
  const Stencil5 st = a.st;
  const double h = a.h;
  const double cs[4] = {a.h * 0.25, a.h / 3.0, a.h * 0.5, a.h};
  const double* bm = a.b + (size_t)(lane / a.lanes_per_b) * n;
  double y[PPT], b[PPT], w[PPT], z[PPT];
  double fl[LAW && !ADJ ? PPT : 1], w2s[LAW && ADJ ? PPT : 1];
  const int pl = a.p_begin + lane % a.lanes_per_b;
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    y[k] = 0.0;
    z[k] = 0.0;
    b[k] = (k < cnt) ? bm[start + k] : 0.0;
    if constexpr (LAW && !ADJ) fl[k] = (k < cnt) ? a.f[(size_t)(lane / a.lanes_per_b) * n + start + k] : 0.0;
  }
  int par = 0;
  for (int s = 0; s < a.nsteps; ++s) {
    LawStep ls{0.0, 0.0, 0.0, 0.0};
    if constexpr (LAW)
      ls = ADJ ? law_step(a.law, true, (pl + 1) * a.delta - s * h, h) : law_step(a.law, false, pl * a.delta + s * h, h);
    const double lc[4] = {ls.c0, ls.c1, ls.c2, ls.c3};
#pragma unroll
    for (int k = 0; k < PPT; ++k) w[k] = y[k];
#pragma unroll
    for (int stage = 0; stage < 4; ++stage) {
      if (t <= last) {
        // FULL (n a multiple of PPT): static last index; a run-time index would demote w
        // to local memory
        double wlast = w[PPT - 1];
        if (!FULL) {
#pragma unroll
          for (int k = 0; k < PPT; ++k)
            if (k == cnt - 1) wlast = w[k];
        }
        eL[par][t] = w[0];
        eR[par][t] = wlast;
      }
      __syncthreads();
      const double left = eR[par][tl], right = eL[par][tr];
      par ^= 1;
      double m[PPT];
#pragma unroll
      for (int k = 0; k < PPT; ++k) {
        const double wl = (k == 0) ? left : w[k - 1];
        const double wr = (k + 1 == PPT || (!FULL && k + 1 >= cnt)) ? right : w[k + 1];
        double v = st.cc * w[k];
        v += st.ce * wr;
        v += st.cw * wl;
        m[k] = v;
      }
      const double c = cs[stage];
      if (stage < 3) {
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
          if constexpr (LAW && ADJ) {
            if (stage == 2) w2s[k] = w[k];  // w2 (this stage reads it; w becomes w3)
          }
          w[k] = y[k] + c * m[k];
          if constexpr (LAW && !ADJ) w[k] = fma(lc[stage], fl[k], w[k]);
        }
      } else {
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
          if constexpr (LAW && ADJ) z[k] = fma(ls.c2, w[k], fma(ls.c1, w2s[k], fma(ls.c0, y[k], z[k])));
          else if (ADJ) z[k] += h * w[k];
          y[k] = y[k] + h * m[k] + b[k];
          if constexpr (LAW && !ADJ) y[k] = fma(ls.c3, fl[k], y[k]);
        }
      }
    }
  }
  double* yo = a.y_out + (size_t)lane * n;
  double* zo = ADJ ? a.z + (size_t)lane * n : nullptr;
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    if (k < cnt) {
      yo[start + k] = y[k];
      if (ADJ) zo[start + k] = z[k];
    }
  }
  (void)NT;
}

// out = s·(x + α·M·y)  (batch in blockIdx.y)
template <int DIM>
__global__ void k_stencil_axpy(double* out, const double* x, const double* y, Stencil5 st, double alpha,
                               double s, int nx, int ny) {
  const size_t n = (size_t)nx * ny;
  const int b = blockIdx.y;
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int yy = (int)(i / nx), xx = (int)(i - (size_t)yy * nx);
  const size_t o = (size_t)b * n;
  out[o + i] = s * (x[o + i] + alpha * stencil_at<DIM>(y + o, st, xx, yy, nx, ny));
}

// out[b*lanes_per_b + p] = src[b] for every lane (nsteps == 1 corner case)
__global__ void k_broadcast_lanes(double* out, const double* src, int lanes_per_b, size_t n) {
  const int l = blockIdx.y;
  const double* s = src + (size_t)(l / lanes_per_b) * n;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[(size_t)l * n + i] = s[i];
}

// out[b][i] = Σ_p lanes[b*Pl + p][i] + scale·c[b][i]  (fixed order)
__global__ void k_lane_sum_plus(double* out, const double* lanes, int lanes_per_b, const double* c, double scale,
                                size_t n, int with_lanes) {
  const int b = blockIdx.y;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    double r = 0.0;
    if (with_lanes) {
      const double* src = lanes + (size_t)b * lanes_per_b * n + i;
      for (int p = 0; p < lanes_per_b; ++p) r += src[(size_t)p * n];
    }
    if (c) r += scale * c[(size_t)b * n + i];
    out[(size_t)b * n + i] = r;
  }
}

// ---------------------------------------------------------------------------
// Two RK4 steps per launch (temporal blocking of the march): stages 1–4 advance
// y by one step (y⁺ at row r−4), stages 5–8 advance y⁺ by the next (y⁺⁺ at row
// r−8). Halves the per-step DRAM traffic (y, z, y⁺ once per two steps) at the
// cost of 8 pipelined stages of register queues (one CTA per SM). Same
// arithmetic per step as k_rk4_march.
// ---------------------------------------------------------------------------
// NT threads (2 columns each), DEPTH ring rows of y(r), b(r−4), b(r−8), z(r−8)
template <bool ADJ, int M2_NT, int M2_DEPTH, int MINB>
__global__ void __launch_bounds__(M2_NT, MINB) k_rk4_march2(MarchArgs a) {
  constexpr int NQ = ADJ ? 4 : 3;
  extern __shared__ double2 dyn2[];
  double2* ring2 = dyn2;                                                        // [M2_DEPTH][NQ][M2_NT]
  double (*pubE)[8][M2_NT] = reinterpret_cast<double (*)[8][M2_NT]>(dyn2 + M2_DEPTH * NQ * M2_NT);
  double (*pubO)[8][M2_NT] = pubE + 2;
  unsigned long long* mbar = reinterpret_cast<unsigned long long*>(pubE + 4);  // [M2_DEPTH]

  const int lane = blockIdx.x % a.lanes;
  const int rest = blockIdx.x / a.lanes;
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
  const int iters = rows_out + 16;
  const bool full_row = a.halo == 0;
  const int tl = (t == 0) ? (full_row ? T - 1 : 0) : t - 1;
  const int tr = (t + 1 >= T) ? (full_row ? 0 : T - 1) : t + 1;
  const bool store_ok = active && (2 * t >= a.halo) && (2 * t + 1 < CW - a.halo);

  const double h = a.h;
  // stage j: base + k_j·(M·w) as five FMAs with the pre-scaled coefficients (kernel
  // parameters, used as constant-bank operands); the north neighbour (this
  // iteration's previous stage) enters last, so the chain across stages is one DFMA
  auto stage = [&](auto jc, double2 base, double2 c, double2 so, double2 nn, double l, double r) -> double2 {
    constexpr int j = decltype(jc)::value;
    double x = fma(a.kc[j][0], c.x, base.x);
    x = fma(a.kc[j][1], c.y, x);
    x = fma(a.kc[j][2], l, x);
    x = fma(a.kc[j][3], so.x, x);
    double y = fma(a.kc[j][0], c.y, base.y);
    y = fma(a.kc[j][1], r, y);
    y = fma(a.kc[j][2], c.x, y);
    y = fma(a.kc[j][3], so.y, y);
    return make_double2(fma(a.kc[j][4], nn.x, x), fma(a.kc[j][4], nn.y, y));
  };
  const size_t member = (size_t)(lane / a.lanes_per_b);
  const double* __restrict__ bsrc = a.b + member * n;
  const double* __restrict__ ysrc = a.y_in ? a.y_in + (size_t)lane * n : bsrc;
  double* __restrict__ yout = a.y_out + (size_t)lane * n;
  double* __restrict__ zl = ADJ ? a.z + (size_t)lane * n : nullptr;
  const bool zread = ADJ && !a.z_zero;

  auto wrapr = [&](int row) -> int {
    row %= ny;
    return row < 0 ? row + ny : row;
  };
  const int r0 = j0 - 8;
  const size_t coloff = (size_t)gx;
  int iss_k = 0, iss_slot = 0;
  int ry = wrapr(r0), rb4 = wrapr(r0 - 4), rb8 = wrapr(r0 - 8);
  // TMA ring: one thread copies each stream's row segment [x0 − halo, x0 + U + halo) (two
  // pieces when it wraps the periodic x boundary) into the slot; completion on the
  // slot's mbarrier (a per-thread cp.async ring was measured slower).
  const int gx0 = (((x0 - a.halo) % nx) + nx) % nx;
  const int lenA = min(CW, nx - gx0);  // columns before the wrap
  const unsigned row_bytes = (unsigned)CW * 8u;
  auto issue = [&]() {
    if (t == 0 && iss_k < iters) {
      double2* slot = ring2 + (size_t)iss_slot * NQ * M2_NT;
      unsigned long long* bar = mbar + iss_slot;
      const int nq = zread ? 4 : 3;
      mbar_expect_tx(bar, row_bytes * (unsigned)nq);
      const double* rows[4] = {ysrc + (size_t)ry * nx, bsrc + (size_t)rb4 * nx, bsrc + (size_t)rb8 * nx,
                               zread ? zl + (size_t)rb8 * nx : nullptr};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (q < nq) {
          double2* dst = slot + q * M2_NT;
          bulk_g2s(dst, rows[q] + gx0, (unsigned)lenA * 8u, bar);
          if (lenA < CW) bulk_g2s(reinterpret_cast<double*>(dst) + lenA, rows[q], (unsigned)(CW - lenA) * 8u, bar);
        }
      }
    }
    ++iss_k;
    iss_slot = (iss_slot + 1 == M2_DEPTH) ? 0 : iss_slot + 1;
    ry = (ry + 1 == ny) ? 0 : ry + 1;
    rb4 = (rb4 + 1 == ny) ? 0 : rb4 + 1;
    rb8 = (rb8 + 1 == ny) ? 0 : rb8 + 1;
  };
  if (t == 0) {
    for (int k = 0; k < M2_DEPTH; ++k) mbar_init(mbar + k, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

#pragma unroll
  for (int k = 0; k < M2_DEPTH; ++k) issue();
  int rslot = 0;
  unsigned rphase = 0;  // parity of the slot's current fill
  int rs = wrapr(r0 - 8);  // output row r − 8

  // rings (phase k = i mod 6): y rows r-4..r, y⁺ rows r-8..r-4, h·w3 rows r-8..r-3
  double2 yq[6], pq[6];
  double2 zq[6];  // h·w3 rows r-8..r-3 in registers (measured 3% faster than a shared-memory ring)
#pragma unroll
  for (int k = 0; k < 6; ++k) zq[k] = make_double2(0.0, 0.0);
  double2 wq[8][2];  // stage outputs w1,w2,w3 (1..3) and w5,w6,w7 (5..7): last two rows
#pragma unroll
  for (int k = 0; k < 6; ++k) yq[k] = pq[k] = make_double2(0.0, 0.0);
#pragma unroll
  for (int s = 0; s < 8; ++s) wq[s][0] = wq[s][1] = make_double2(0.0, 0.0);


  // One march iteration at ring phase k (compile time); G = guarded (pipeline fill/drain).
  auto iter = [&](auto kc, auto gc, const int i) {
    constexpr int k = decltype(kc)::value;
    constexpr bool G = decltype(gc)::value;
      const int pin = (k + 1) & 1, pout = k & 1;
      const int po = k & 1, pp = (k + 1) & 1;
      mbar_wait(mbar + rslot, rphase);
      const double2* slot = ring2 + (size_t)rslot * NQ * M2_NT;
      rslot = (rslot + 1 == M2_DEPTH) ? 0 : rslot + 1;
      if (rslot == 0) rphase ^= 1u;
      const double2 yr = slot[t];
      const double2 b4 = slot[M2_NT + t];
      const double2 b8 = slot[2 * M2_NT + t];
      const double2 zrow = zread ? slot[3 * M2_NT + t] : make_double2(0.0, 0.0);
      yq[k] = yr;
      const double2 y0 = yq[(k + 2) % 6], y1 = yq[(k + 3) % 6], y2 = yq[(k + 4) % 6], y3 = yq[(k + 5) % 6];
      double2 nw[9];
      if (G) {
#pragma unroll
        for (int s = 0; s < 9; ++s) nw[s] = make_double2(0.0, 0.0);
      }
      // ---- step A (rows r-1 .. r-4) ----
      if (!G || i >= 2) {
        nw[1] = stage(IC<0>{}, y3, y3, y2, yr, pubO[pin][0][tl], pubE[pin][0][tr]);
      }
      if (!G || i >= 4) {
        nw[2] = stage(IC<1>{}, y2, wq[1][pp], wq[1][po], nw[1], pubO[pin][1][tl], pubE[pin][1][tr]);
      }
      if (!G || i >= 6) {
        nw[3] = stage(IC<2>{}, y1, wq[2][pp], wq[2][po], nw[2], pubO[pin][2][tl], pubE[pin][2][tr]);
        if (ADJ) zq[(k + 3) % 6] = make_double2(h * nw[3].x, h * nw[3].y);  // row r-3
      }
      if (!G || i >= 8) {  // y⁺ at row r-4
        nw[4] = stage(IC<3>{}, make_double2(y0.x + b4.x, y0.y + b4.y), wq[3][pp], wq[3][po], nw[3],
                         pubO[pin][3][tl], pubE[pin][3][tr]);
      }
      pq[(k + 2) % 6] = nw[4];  // y⁺ row r-4
      const double2 p4 = nw[4], p5 = pq[(k + 1) % 6], p6 = pq[k % 6], p7 = pq[(k + 5) % 6], p8 = pq[(k + 4) % 6];
      // ---- step B (rows r-5 .. r-8) on y⁺ ----
      if (!G || i >= 10) {
        nw[5] = stage(IC<0>{}, p5, p5, p6, p4, pubO[pin][4][tl], pubE[pin][4][tr]);
      }
      if (!G || i >= 12) {
        nw[6] = stage(IC<1>{}, p6, wq[5][pp], wq[5][po], nw[5], pubO[pin][5][tl], pubE[pin][5][tr]);
      }
      if (!G || i >= 14) {
        nw[7] = stage(IC<2>{}, p7, wq[6][pp], wq[6][po], nw[6], pubO[pin][6][tl], pubE[pin][6][tr]);
      }
      if (!G || i >= 16) {  // y⁺⁺ at row r-8
        const double2 w7c = wq[7][pp];
        const double2 yn = stage(IC<3>{}, make_double2(p8.x + b8.x, p8.y + b8.y), w7c, wq[7][po], nw[7],
                                    pubO[pin][7][tl], pubE[pin][7][tr]);
        if (store_ok) {
          const size_t off = (size_t)rs * nx + coloff;
          __stcs(reinterpret_cast<double2*>(yout + off), yn);
          if (ADJ) {
            const double2 za = zq[(k + 4) % 6];  // h·w3 at row r-8
            double2 zn;
            zn.x = zrow.x + za.x + h * w7c.x;
            zn.y = zrow.y + za.y + h * w7c.y;
            __stcs(reinterpret_cast<double2*>(zl + off), zn);
          }
        }
      }
      rs = (rs + 1 == ny) ? 0 : rs + 1;
#pragma unroll
      for (int s = 1; s <= 7; ++s)
        if (s != 4) wq[s][po] = nw[s];
      if (active) {
        pubE[pout][0][t] = yr.x;     pubO[pout][0][t] = yr.y;
        pubE[pout][1][t] = nw[1].x;  pubO[pout][1][t] = nw[1].y;
        pubE[pout][2][t] = nw[2].x;  pubO[pout][2][t] = nw[2].y;
        pubE[pout][3][t] = nw[3].x;  pubO[pout][3][t] = nw[3].y;
        pubE[pout][4][t] = nw[4].x;  pubO[pout][4][t] = nw[4].y;
        pubE[pout][5][t] = nw[5].x;  pubO[pout][5][t] = nw[5].y;
        pubE[pout][6][t] = nw[6].x;  pubO[pout][6][t] = nw[6].y;
        pubE[pout][7][t] = nw[7].x;  pubO[pout][7][t] = nw[7].y;
      }
      __syncthreads();
      if (t == 0) fence_proxy_async_smem();  // every thread has read this iteration's slot: refill it
      issue();
  };
  int i0 = 0;
  // fill: the first 18 iterations (stages switch on at i = 2, 4, …, 16)
  for (; i0 < 18; i0 += 6) {
    if (i0 + 6 > iters) break;
    iter(IC<0>{}, BC<true>{}, i0); iter(IC<1>{}, BC<true>{}, i0 + 1); iter(IC<2>{}, BC<true>{}, i0 + 2);
    iter(IC<3>{}, BC<true>{}, i0 + 3); iter(IC<4>{}, BC<true>{}, i0 + 4); iter(IC<5>{}, BC<true>{}, i0 + 5);
  }
  if (i0 >= 18) {
    // steady state: every stage live, no guards
    for (; i0 + 6 <= iters; i0 += 6) {
      iter(IC<0>{}, BC<false>{}, i0); iter(IC<1>{}, BC<false>{}, i0 + 1); iter(IC<2>{}, BC<false>{}, i0 + 2);
      iter(IC<3>{}, BC<false>{}, i0 + 3); iter(IC<4>{}, BC<false>{}, i0 + 4); iter(IC<5>{}, BC<false>{}, i0 + 5);
    }
  }
  // drain / short bands: guarded remainder
  if (i0 + 0 < iters) iter(IC<0>{}, BC<true>{}, i0);
  if (i0 + 1 < iters) iter(IC<1>{}, BC<true>{}, i0 + 1);
  if (i0 + 2 < iters) iter(IC<2>{}, BC<true>{}, i0 + 2);
  if (i0 + 3 < iters) iter(IC<3>{}, BC<true>{}, i0 + 3);
  if (i0 + 4 < iters) iter(IC<4>{}, BC<true>{}, i0 + 4);
  if (i0 + 5 < iters) iter(IC<5>{}, BC<true>{}, i0 + 5);
}

// ---------------------------------------------------------------------------
// k_rk4_marchc: the two-step march with NC (≥ 3) contiguous columns per thread.
// The x-neighbour exchange moves 16 B out and 16 B in per thread and stage
// whatever NC is, so its shared-memory bytes per point fall as 2/NC — the
// limiter of the two-column kernel (≈ 70% of its LSU wavefronts). Direct lanes
// only (no ∫ accumulator: the 2D adjoint integral is recovered in closed form),
// strip mode only (halo 8), TMA row ring of y(r), b(r−4), b(r−8).
// ---------------------------------------------------------------------------
template <int NC>
struct ColV {
  double v[NC];
};

template <int NC, int NT, int DEP, int MINB, bool BR = true, bool S2 = true>
__global__ void __launch_bounds__(NT, MINB) k_rk4_marchc(MarchArgs a) {
  // BR: b(r−8) from a register ring of b(r−4) rows (two streams instead of three)
  // (no proxy fence before a slot refill: the slot's generic-proxy reads are complete at
  // the barrier, and write-after-read needs no cross-proxy fence)
  // S2: two RK4 steps per launch; otherwise one (the odd remainder step of a sweep)
  constexpr int NQ = (BR || !S2) ? 2 : 3;
  constexpr int LAG = S2 ? 8 : 4;  // pipeline depth in rows (output row r − LAG)
  constexpr int RW = NT * NC;  // ring row width (doubles)
  using V = ColV<NC>;
  extern __shared__ double dynd[];
  double* ring = dynd;                                                        // [DEP][NQ][RW]
  double (*pubE)[8][NT] = reinterpret_cast<double (*)[8][NT]>(ring + DEP * NQ * RW);
  double (*pubO)[8][NT] = pubE + 2;
  unsigned long long* mbar = reinterpret_cast<unsigned long long*>(pubE + 4);  // [DEP]

  const int lane = blockIdx.x % a.lanes;
  const int rest = blockIdx.x / a.lanes;
  const int strip = rest % a.nstrips;
  const int band = rest / a.nstrips;
  const int nx = a.nx, ny = a.ny;
  const size_t n = (size_t)nx * ny;
  const int x0 = strip * a.strip_w;
  const int U = min(a.strip_w, nx - x0);
  const int CW = U + 2 * a.halo;
  const int t = threadIdx.x;
  const int T = (CW + NC - 1) / NC;
  const int tl = t == 0 ? 0 : t - 1;
  const int tr = t + 1 >= T ? T - 1 : t + 1;
  const int j0 = band * a.band_rows;
  const int rows_out = min(a.band_rows, ny - j0);
  const int iters = rows_out + 2 * LAG;
  const int c0 = NC * t;                                  // first strip column of this thread
  const int gxs = (((x0 - a.halo + c0) % nx) + nx) % nx;  // its global column (no wrap inside a thread's run: nx % 2 == 0, runs are checked below)

  auto stage = [&](auto jc, const V& base, const V& c, const V& so, const V& nn, double l, double r) -> V {
    constexpr int j = decltype(jc)::value;
    V o;
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      const double e = q + 1 < NC ? c.v[q + 1] : r;
      const double w = q > 0 ? c.v[q - 1] : l;
      double x = fma(a.kc[j][0], c.v[q], base.v[q]);
      x = fma(a.kc[j][1], e, x);
      x = fma(a.kc[j][2], w, x);
      x = fma(a.kc[j][3], so.v[q], x);
      o.v[q] = fma(a.kc[j][4], nn.v[q], x);
    }
    return o;
  };
  auto vadd = [](const V& x, const V& y) {
    V o;
#pragma unroll
    for (int q = 0; q < NC; ++q) o.v[q] = x.v[q] + y.v[q];
    return o;
  };
  const size_t member = (size_t)(lane / a.lanes_per_b);
  const double* __restrict__ bsrc = a.b + member * n;
  const double* __restrict__ ysrc = a.y_in ? a.y_in + (size_t)lane * n : bsrc;
  double* __restrict__ yout = a.y_out + (size_t)lane * n;

  auto wrapr = [&](int row) -> int {
    row %= ny;
    return row < 0 ? row + ny : row;
  };
  const int r0 = j0 - LAG;
  int iss_k = 0, iss_slot = 0;
  int ry = wrapr(r0), rb4 = wrapr(r0 - 4), rb8 = wrapr(r0 - 8);
  const int gx0 = (((x0 - a.halo) % nx) + nx) % nx;
  const int lenA = min(CW, nx - gx0);
  const unsigned row_bytes = (unsigned)CW * 8u;
  auto issue = [&]() {
    if (t == 0 && iss_k < iters) {
      double* slot = ring + (size_t)iss_slot * NQ * RW;
      unsigned long long* bar = mbar + iss_slot;
      mbar_expect_tx(bar, row_bytes * (unsigned)NQ);
      const double* rows[3] = {ysrc + (size_t)ry * nx, bsrc + (size_t)rb4 * nx, bsrc + (size_t)rb8 * nx};  // (BR: first two)
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        double* dst = slot + q * RW;
        bulk_g2s(dst, rows[q] + gx0, (unsigned)lenA * 8u, bar);
        if (lenA < CW) bulk_g2s(dst + lenA, rows[q], (unsigned)(CW - lenA) * 8u, bar);
      }
    }
    ++iss_k;
    iss_slot = (iss_slot + 1 == DEP) ? 0 : iss_slot + 1;
    ry = (ry + 1 == ny) ? 0 : ry + 1;
    rb4 = (rb4 + 1 == ny) ? 0 : rb4 + 1;
    rb8 = (rb8 + 1 == ny) ? 0 : rb8 + 1;
  };
  if (t == 0) {
    for (int k = 0; k < DEP; ++k) mbar_init(mbar + k, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < DEP; ++k) issue();
  int rslot = 0;
  unsigned rphase = 0;
  int rs = wrapr(r0 - LAG);
  // columns of this thread that are written back: strip columns [halo, CW − halo)
  bool st_ok[NC];
#pragma unroll
  for (int q = 0; q < NC; ++q) st_ok[q] = (c0 + q >= a.halo) && (c0 + q < CW - a.halo);
  int gxq[NC];
#pragma unroll
  for (int q = 0; q < NC; ++q) gxq[q] = (gxs + q) % nx;

  V yq[6], pq[6];
  V bq[BR ? 6 : 1];  // BR: b(r−4) of the last six iterations
  V wq[8][2];
#pragma unroll
  for (int k = 0; k < 6; ++k)
#pragma unroll
    for (int q = 0; q < NC; ++q) yq[k].v[q] = pq[k].v[q] = 0.0;
#pragma unroll
  for (int k = 0; k < (BR ? 6 : 1); ++k)
#pragma unroll
    for (int q = 0; q < NC; ++q) bq[k].v[q] = 0.0;
#pragma unroll
  for (int s = 0; s < 8; ++s)
#pragma unroll
    for (int q = 0; q < NC; ++q) wq[s][0].v[q] = wq[s][1].v[q] = 0.0;

  auto iter = [&](auto kc, auto gc, const int i) {
    constexpr int k = decltype(kc)::value;
    constexpr bool G = decltype(gc)::value;
    const int pin = (k + 1) & 1, pout = k & 1;
    const int po = k & 1, pp = (k + 1) & 1;
    mbar_wait(mbar + rslot, rphase);
    const double* slot = ring + (size_t)rslot * NQ * RW;
    rslot = (rslot + 1 == DEP) ? 0 : rslot + 1;
    if (rslot == 0) rphase ^= 1u;
    V yr, b4, b8;
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      yr.v[q] = slot[c0 + q];
      b4.v[q] = slot[RW + c0 + q];
      if constexpr (NQ == 3) b8.v[q] = slot[2 * RW + c0 + q];
    }
    if constexpr (BR && S2) {
      bq[k] = b4;
      b8 = bq[(k + 2) % 6];  // b4 of iteration i − 4 = b(r − 8)
    }
    yq[k] = yr;
    const V& y0 = yq[(k + 2) % 6];
    const V& y1 = yq[(k + 3) % 6];
    const V& y2 = yq[(k + 4) % 6];
    const V& y3 = yq[(k + 5) % 6];
    V nw[9];
    if (G) {
#pragma unroll
      for (int s = 0; s < 9; ++s)
#pragma unroll
        for (int q = 0; q < NC; ++q) nw[s].v[q] = 0.0;
    }
    if (!G || i >= 2) nw[1] = stage(IC<0>{}, y3, y3, y2, yr, pubO[pin][0][tl], pubE[pin][0][tr]);
    if (!G || i >= 4) nw[2] = stage(IC<1>{}, y2, wq[1][pp], wq[1][po], nw[1], pubO[pin][1][tl], pubE[pin][1][tr]);
    if (!G || i >= 6) nw[3] = stage(IC<2>{}, y1, wq[2][pp], wq[2][po], nw[2], pubO[pin][2][tl], pubE[pin][2][tr]);
    if (!G || i >= 8) nw[4] = stage(IC<3>{}, vadd(y0, b4), wq[3][pp], wq[3][po], nw[3], pubO[pin][3][tl], pubE[pin][3][tr]);
    if constexpr (!S2) {
      if (!G || i >= 8) {  // y⁺ at row r − 4
        double* orow = yout + (size_t)rs * nx;
#pragma unroll
        for (int q = 0; q < NC; ++q)
          if (st_ok[q]) __stcs(orow + gxq[q], nw[4].v[q]);
      }
    } else {
    pq[(k + 2) % 6] = nw[4];
    const V& p5 = pq[(k + 1) % 6];
    const V& p6 = pq[k % 6];
    const V& p7 = pq[(k + 5) % 6];
    const V& p8 = pq[(k + 4) % 6];
    if (!G || i >= 10) nw[5] = stage(IC<0>{}, p5, p5, p6, nw[4], pubO[pin][4][tl], pubE[pin][4][tr]);
    if (!G || i >= 12) nw[6] = stage(IC<1>{}, p6, wq[5][pp], wq[5][po], nw[5], pubO[pin][5][tl], pubE[pin][5][tr]);
    if (!G || i >= 14) nw[7] = stage(IC<2>{}, p7, wq[6][pp], wq[6][po], nw[6], pubO[pin][6][tl], pubE[pin][6][tr]);
    if (!G || i >= 16) {
      const V yn = stage(IC<3>{}, vadd(p8, b8), wq[7][pp], wq[7][po], nw[7], pubO[pin][7][tl], pubE[pin][7][tr]);
      double* orow = yout + (size_t)rs * nx;
#pragma unroll
      for (int q = 0; q < NC; ++q)
        if (st_ok[q]) __stcs(orow + gxq[q], yn.v[q]);
    }
    }  // S2
    rs = (rs + 1 == ny) ? 0 : rs + 1;
#pragma unroll
    for (int s = 1; s <= (S2 ? 7 : 3); ++s)
      if (s != 4) wq[s][po] = nw[s];
    pubE[pout][0][t] = yr.v[0];     pubO[pout][0][t] = yr.v[NC - 1];
#pragma unroll
    for (int s = 1; s <= (S2 ? 7 : 3); ++s) {
      pubE[pout][s][t] = nw[s].v[0];
      pubO[pout][s][t] = nw[s].v[NC - 1];
    }
    __syncthreads();
    issue();
  };
  int i0 = 0;
  constexpr int FILL = S2 ? 18 : 12;  // guarded groups until every stage is live (i ≥ 2·LAG)
  for (; i0 < FILL; i0 += 6) {
    if (i0 + 6 > iters) break;
    iter(IC<0>{}, BC<true>{}, i0); iter(IC<1>{}, BC<true>{}, i0 + 1); iter(IC<2>{}, BC<true>{}, i0 + 2);
    iter(IC<3>{}, BC<true>{}, i0 + 3); iter(IC<4>{}, BC<true>{}, i0 + 4); iter(IC<5>{}, BC<true>{}, i0 + 5);
  }
  if (i0 >= FILL) {
    for (; i0 + 6 <= iters; i0 += 6) {
      iter(IC<0>{}, BC<false>{}, i0); iter(IC<1>{}, BC<false>{}, i0 + 1); iter(IC<2>{}, BC<false>{}, i0 + 2);
      iter(IC<3>{}, BC<false>{}, i0 + 3); iter(IC<4>{}, BC<false>{}, i0 + 4); iter(IC<5>{}, BC<false>{}, i0 + 5);
    }
  }
  if (i0 + 0 < iters) iter(IC<0>{}, BC<true>{}, i0);
  if (i0 + 1 < iters) iter(IC<1>{}, BC<true>{}, i0 + 1);
  if (i0 + 2 < iters) iter(IC<2>{}, BC<true>{}, i0 + 2);
  if (i0 + 3 < iters) iter(IC<3>{}, BC<true>{}, i0 + 3);
  if (i0 + 4 < iters) iter(IC<4>{}, BC<true>{}, i0 + 4);
  if (i0 + 5 < iters) iter(IC<5>{}, BC<true>{}, i0 + 5);
}

template <int NC, int NT, int DEP>
inline size_t marchc_smem(bool br) {
  return (size_t)DEP * (br ? 2 : 3) * NT * NC * sizeof(double) + 4 * 8 * NT * sizeof(double) +
         DEP * sizeof(unsigned long long);
}

template <int M2_NT, int M2_DEPTH>
inline size_t march2_smem(bool adj) {
  return (size_t)M2_DEPTH * (adj ? 4 : 3) * M2_NT * sizeof(double2) + 4 * 8 * M2_NT * sizeof(double) +
         M2_DEPTH * sizeof(unsigned long long);
}

}  // namespace px
