// hybrid_args.h — kernel argument structs of hybrid.cuh (shared by burgers.cu, which instantiates
// the kernels, and hybrid.cu, the C ABI that drives them).
#pragma once

namespace px {

constexpr int HYB_NT = 256;

struct HybArgs {
  const double* u0;      // B × n
  const double* f;       // B × n forcing fields
  const double* target;  // (S+1) × tb × n tracking target on the nodes (tb = 1: shared)
  int target_b;          // tb
  double* traj;          // (S+1) × B × n
  double* J;             // B
  int* flags;            // B × P progress flags (slice p of member b complete)
  const int* offsets;    // P+1 node offsets (device)
  double* aend;          // (B·P) × n adjoint slice solutions at the slice starts
  double* zl;            // (B·P) × n their θ-weighted integrals
  double la, lb, lc, lw; // time law
  const double* theta;   // θ(k·h/2), k = 0 … 2S (host-evaluated once per handle: no trig per step)
  double D, hx, h, T;
  int nx, B, P, S;
  int wait;              // lanes: wait for the direct's progress flags
};

struct HybSlicePlan {
  int substeps, degree, sigma, exp_off, law_off;
  double c0, d;
};

struct HybScanArgs {
  const double* ubar;          // P × B × n
  const double* aend;          // (B·P) × n
  const double* zl;            // (B·P) × n
  const double* qT;            // B × n terminal data, or null (tracking only)
  const HybSlicePlan* plans;   // P
  const double* coef;          // pool: exp series per slice, law series per (slice, substep)
  double* qdag0;               // B × n
  double* grad;                // B × n  ∂L/∂f = (1/T)∫θ·q† dt
  double D, hx, T;
  int nx, B, P;
};

}  // namespace px
