/*
 * paraexp.h — C ABI of the B200 Paraexp direct-adjoint gradient path.
 *
 * The reference (pkg/src/paradjoint, pure Python) has no native boundary: its
 * hot path is called as Python functions taking CSR operators and callables.
 * This ABI is what a ctypes binding of the reference would call when its
 * existing backend selector (`backend=`, config.py:44,154-156 -> workers.py:335-340)
 * is given "cuda". Each entry point below names the reference interface it
 * replaces. Plain pointers and sizes only; no torch types.
 *
 * Conventions
 *  - One handle per GPU process, bound to the device current at px_create.
 *    Not thread-safe: one host thread drives a handle.
 *  - All work is enqueued on the caller's stream (`stream` is a cudaStream_t;
 *    NULL = legacy default stream). Functions that return host scalars
 *    synchronise that stream.
 *  - Fields are fp64, x fastest (flat index i + nx*j), batch-major: a (B, n)
 *    array holds batch member b at offset b*n (problems.py:48-56).
 *  - Return value 0 = success; otherwise a PX_ERR_* code, with a message from
 *    px_last_error(). The Python layer maps codes onto the reference's
 *    exceptions (errors.py:4-57): PX_ERR_NONFINITE -> IntegrationFailure,
 *    PX_ERR_PLAN -> PropagationFailure, PX_ERR_ARG -> ValueError.
 */
#ifndef PARAEXP_H_
#define PARAEXP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PX_ABI_VERSION 5

enum {
  PX_OK = 0,
  PX_ERR_ARG = 1,
  PX_ERR_CUDA = 2,
  PX_ERR_NONFINITE = 3,
  PX_ERR_PLAN = 4,
  PX_ERR_STATE = 5,
  PX_ERR_NOMEM = 6
};

enum { PX_KIND_ADVDIFF = 0, PX_KIND_BURGERS = 1 };
enum { PX_EXP_CHEBYSHEV = 0, PX_EXP_KRYLOV = 1 };
enum { PX_MEM_HOST = 0, PX_MEM_DEVICE = 1 };

/* plan slots */
enum {
  PX_PLAN_SLICE = 0,        /* slice width Δ, operator A and Aᵀ (same spectrum) */
  PX_PLAN_LONG_DIRECT = 1,  /* span (P - p_end)·Δ, block carry -> T (blockscan) */
  PX_PLAN_LONG_ADJOINT = 2, /* span p_begin·Δ, block carry -> 0 (blockscan) */
  PX_PLAN_FROZEN = 3,       /* Burgers: slice width, frozen J(ū_p)ᵀ */
  PX_PLAN_NL_SLICE = 4,     /* Burgers iterative direct: slice width, J(ū_p) */
  PX_PLAN_NL_STEP = 5,      /* Burgers iterative direct: one RK4 step h, J(ū_p) (node recording) */
  PX_PLAN_BLOCK_LONG = 6,   /* local blocks (px_set_local_blocks): slot 6 + k - 1 holds the span
                               k·(Pl/blocks)·Δ, k = 1 … blocks - 1 (block carry -> block edge) */
  PX_MAX_LOCAL_BLOCKS = 16,
  PX_PLAN_COUNT = PX_PLAN_BLOCK_LONG + PX_MAX_LOCAL_BLOCKS - 1
};

/* fields for px_get / px_buffer */
enum {
  PX_FIELD_J = 0,           /* (B)            objective ½‖u(T) − u_target‖² */
  PX_FIELD_GRAD = 1,        /* (B, K)         ∂J/∂c_k (rank-partial before px_finish_adjoint) */
  PX_FIELD_UT = 2,          /* (B, n)         u(T) (rank-partial carry before px_finish_direct) */
  PX_FIELD_QDAG0 = 3,       /* (B, n)         q†(0) (rank-partial before px_finish_adjoint) */
  PX_FIELD_G = 4,           /* (B, n)         ∫ q† dt (rank-partial before px_finish_adjoint) */
  PX_FIELD_UBND = 5,        /* (B, P+1, n)    direct boundary states u(T_p) (flag, world = 1) */
  PX_FIELD_FROZEN_BOUNDS = 6, /* (3)          Burgers: re_lo, re_hi, im of the frozen-operator FOV union */
  PX_FIELD_VEND = 7,        /* (B, P_local, n) per-slice inhomogeneous end states v_p(T_{p+1}) */
  PX_FIELD_WEND = 8,        /* (B, P_local, n) per-slice adjoint inhomogeneous end states */
  PX_FIELD_TRAJ = 9,        /* (S+1, B, n)    Burgers / tracking direct trajectory (S = P·nsteps) */
  PX_FIELD_COUNT = 10
};

enum {
  PX_FLAG_BOUNDARY_STATES = 1, /* keep u(T_p) for every slice edge (PX_FIELD_UBND; world = 1) */
  PX_FLAG_Z_ACCUM = 2,         /* 2D adjoint ∫: per-lane RK4 accumulator instead of the closed form */
  PX_FLAG_FIELD_CONTROL = 4    /* advection–diffusion: the control is a full spatial field f (B×n, K = n;
                                  no basis tables) and PX_FIELD_GRAD is the field gradient ∫q† dt —
                                  the reference's forcing field f_spatial (problems.py:155-162) */
};

/* Kernel-variant keys for px_set_variant / px_get_variant (per handle; defaults are the
 * measured-best variants, the alternatives exist for parity tests and tuning). */
enum {
  PX_VAR_MARCH2 = 0,          /* 0 one RK4 step per launch; 1 (default) two-step launches for sweeps of
                                 ≥ 2^28 lane-points; 2 two-step launches at any size */
  PX_VAR_MARCH_COLS = 1,      /* columns per thread of the two-step march: 3 (default) or 2 */
  PX_VAR_MARCH_BAND = 2,      /* rows per band of the two-step march (0: automatic) */
  PX_VAR_CHEB_TERMS = 3,      /* most Chebyshev terms fused per 2D pass, 1 … 7 (default 7; passes balanced) */
  PX_VAR_CHEB_STRIP = 4,      /* strip width of the 2D Chebyshev passes (0: balanced) */
  PX_VAR_CHEB_BAND = 5,       /* rows per band of the 2D Chebyshev passes (0: one wave) */
  PX_VAR_SCAN1D_CLUSTER = 6,  /* 1D scans on 8-CTA clusters for n ≥ 2048 (default 1) */
  PX_VAR_BURGERS_CLUSTER = 7, /* Burgers sweeps on 8-CTA clusters for n ≥ 2048 (default 1) */
  PX_VAR_CHEB_TERMS_PHI = 8,  /* as PX_VAR_CHEB_TERMS for passes with the φ₁ accumulator (default 5) */
  PX_VAR_KRYLOV_ORTHO = 9     /* Arnoldi orthogonalisation: 1 (default) delayed reorthogonalisation, one
                                 reduction and two basis passes per step; 0 CGS2, four passes */
};
enum { PX_ADJOINT_ABSORBED = 0, PX_ADJOINT_FROZEN_SPAN = 1 };  /* px_set_adjoint_mode */

typedef struct px_problem_desc {
  int kind;             /* PX_KIND_* */
  int nx, ny;           /* ny == 1: 1D */
  double stencil[5];    /* direct operator (cc, ce, cw, cn, cs); Burgers: D∇² part */
  double D;             /* diffusion (Burgers nonlinear terms use hx and D) */
  double hx;            /* grid spacing in x */
  double T;             /* horizon */
  int P;                /* global slice count (TimePartition.N) */
  int nsteps;           /* RK4 steps per slice, slice rule ⌈Δ/dt⌉ */
  int p_begin, p_end;   /* this rank's contiguous slice block */
  int batch;            /* B independent controls */
  int K;                /* control modes */
  int basis_rows_x;     /* rows of the x factor table */
  int basis_rows_y;     /* rows of the y factor table (1 in 1D) */
  int expaction;        /* PX_EXP_* */
  int krylov_m;         /* Arnoldi vectors (PX_EXP_KRYLOV) */
  int flags;            /* PX_FLAG_* */
} px_problem_desc;

typedef struct px_cheb_plan {
  double span;          /* total span τ = substeps·τ_s */
  int substeps;
  int degree;           /* K: coefficients 0..K */
  double center;        /* c0 */
  double scale;         /* d: X = (M − c0)/d */
  int sigma;            /* +1 imaginary foci, −1 real foci: U_{k+1} = 2X·U_k + σ·U_{k−1} */
  const double* coef_exp;  /* degree+1 host values: e^{τ_s z} */
  const double* coef_phi;  /* degree+1 host values: τ_s·φ₁(τ_s z) (may be NULL) */
} px_cheb_plan;

typedef struct px_stats {
  uint64_t rk4_lane_steps;   /* RK4 steps × lanes executed (one lane = one n-field) */
  uint64_t exp_terms;        /* operator applications inside exp-actions × vectors */
  uint64_t arnoldi_steps;    /* Arnoldi steps × vectors */
  uint64_t kernel_launches;  /* launches of this library's kernels */
  double algorithmic_bytes;  /* Σ units × bytes/unit */
  double rk4_bytes;          /* part of the above in RK4 sweeps */
  double exp_bytes;          /* part of the above in exp-actions */
} px_stats;

/* Library identity (C-ABI version; compiled sm arch string). */
int px_abi_version(void);
const char* px_build_info(void);

/* Problem setup: replaces build_system/System (systems.py:27-117) and the
 * partition (paraexp.py:72-78); allocates device scratch on the current device. */
int px_create(const px_problem_desc* desc, void** out_handle);
void px_destroy(void* handle);
const char* px_last_error(const void* handle);

/* Control basis factor tables (host): tx[rows_x][nx], ty[rows_y][ny], ix[K], iy[K]. */
int px_set_basis(void* handle, const double* tx, const double* ty, const int* ix, const int* iy);

/* Exp-action plans: replace relpm_propagate's adaptive Leja setup
 * (timestepping.py:360-423) by the host planner's a-priori plan. */
int px_set_cheb_plan(void* handle, int slot, const px_cheb_plan* plan);
int px_set_krylov_plan(void* handle, int slot, double span, int substeps);
/* Time-law series of the Chebyshev plan in `slot` (set it first): coef_gc / coef_gs (degree+1 host
 * values each) are the series of ∫₀^τ_s cos(ωs)·e^{sz} ds and ∫₀^τ_s sin(ωs)·e^{sz} ds (ω of the
 * handle's time law). Needed for every adjoint plan when the law has ω > 0. */
int px_set_cheb_plan_law(void* handle, int slot, const double* coef_gc, const double* coef_gs);

/* Forcing time law of the linear testbed: the control field f (from the coefficients and basis,
 * or PX_FLAG_FIELD_CONTROL) is applied as f·θ(t), θ(t) = law[0] + law[1]·sin(law[3]·t) +
 * law[2]·cos(law[3]·t) — the reference's f·sin(ωt) is {0, 1, 0, ω} (problems.py:155-162,
 * systems.py:56-60). Every slice's RK4 lanes evaluate θ at their own stage times; the gradient
 * becomes ∂J/∂f = ∫θ(t)·q†(t) dt (gradient_wrt_forcing, optimization.py:103-112, without the
 * tracking objective's 1/T). {1, 0, 0, 0} restores the time-constant control. Chebyshev only
 * (Krylov plans: PX_ERR_ARG); lanes run one RK4 step per launch and the adjoint keeps a per-lane
 * θ-weighted ∫ accumulator. */
int px_set_time_law(void* handle, const double* law4);

/* Tracking objective of the linear testbed — the reference's linear loop with its own objective
 * (optimization.py:84-112,154-231, algorithm "linear"): J = (1/T)∫‖u − u_t‖² dt (trapezoid on the
 * RK4 nodes), adjoint source 2(u − u_t) with zero terminal data (solve_adjoint_linear with
 * adj_forcing, paraexp.py:298-326), ∂L/∂f = (1/T)∫θ·q† dt. After the Paraexp direct every slice
 * re-marches from its edge state u(T_p) to record the trajectory (PX_FIELD_TRAJ, (S+1, B, n)), and
 * the adjoint lanes read it at their stage times; the carries are the terminal objective's.
 * target: (S+1) × n (per_member 0) or (S+1) × B × n (per_member 1), S = P·nsteps, on the host or the
 * device (mem). nullptr restores the terminal objective ½‖u(T) − u_target‖². One rank (p_begin = 0,
 * p_end = P); local blocks are not used; PX_FIELD_UBND holds the edge states. Replaces: the
 * objective/adjoint-source closures of direct_adjoint_loop for the linear system. */
int px_set_tracking_target(void* handle, const double* target, int per_member, int mem, void* stream);

/* Kernel-variant selection (PX_VAR_*), per handle; invalidates the captured gradient graph. */
int px_set_variant(void* handle, int key, int value);
int px_get_variant(void* handle, int key, int* value);

/* Split this rank's slices into `blocks` equal contiguous blocks whose summed-chain carries
 * run concurrently on side streams of one GPU (the multi-GPU block-scan of SURVEY.md §8(e)
 * inside one handle: block carries meet through one long-span action each, plans in slots
 * PX_PLAN_BLOCK_LONG + k - 1). Pays off when the exp-action kernels leave the GPU idle
 * (Krylov, small fields). 1 = the sequential scan (default). Replaces: the reference's
 * per-worker chains running concurrently (`workers.py:298-346`). */
int px_set_local_blocks(void* handle, int blocks);
/* Local blocks of unequal sizes (slice order, summing to the rank's slices) for the direct sweep;
 * the adjoint uses the mirrored partition. The long-span plan in slot PX_PLAN_BLOCK_LONG + k − 1
 * must then cover the last k direct blocks (= the first k adjoint blocks). */
int px_set_local_block_sizes(void* handle, int blocks, const int* sizes);

/* Burgers adjoint formulation. PX_ADJOINT_ABSORBED (default): the final condition is absorbed
 * into the inhomogeneous solves, exact Jᵀ(u(t)) there and frozen J(ū_p)ᵀ in the carry
 * (solve_adjoint_varying, paraexp.py:329-353 — SURVEY §8(c) Option A, config 3).
 * PX_ADJOINT_FROZEN_SPAN: the reference's solve_hybrid (hybrid.py:194-237, Option B): the
 * inhomogeneous solves start from zero terminal data and, with no adjoint source, vanish;
 * q†_T is propagated over [T, 0] through the frozen J(ū_p)ᵀ (propagate_span, the final span
 * hybrid.py:232-233), ∫q† dt from its φ₁ series. One rank only. Replaces: the choice between
 * direct_adjoint_loop's "hybrid" (solve_hybrid) and "linear"/"nonlinear" (solve_adjoint_varying)
 * adjoints (optimization.py:183-220). */
int px_set_adjoint_mode(void* handle, int mode);

/* Inputs: u0 (n), u_target (n), ctrl (B×K); host or device memory. Replaces the
 * q0 / q_true / f arguments of direct_adjoint_loop (optimization.py:154-169). */
int px_set_inputs(void* handle, const double* u0, const double* u_target, const double* ctrl,
                  int mem, void* stream);

/* Direct sweep (solve_direct_linear, paraexp.py:221-248; Burgers: the hybrid's
 * serial sweep, hybrid.py:185-191): rank-partial u(T) carry in PX_FIELD_UT. */
int px_direct(void* handle, void* stream);
/* After the caller's allreduce of PX_FIELD_UT (world > 1): u(T) = u0 + Σ partials,
 * q†_T = u(T) − u_target, J (cost, optimization.py:84-93 with the terminal objective). */
int px_finish_direct(void* handle, void* stream);
/* Iterative nonlinear direct solve (Algorithm 2, nonlinear.py:69-194), Burgers only,
 * one rank. The host drives the sweeps (it plans the J(ū_p) actions in between):
 *   px_nl_init            iterate ← u0 at every node
 *   loop: px_nl_prepare   slice means ū_p of the iterate + FOV bounds (PX_FIELD_FROZEN_BOUNDS)
 *         [set PX_PLAN_NL_SLICE / PX_PLAN_NL_STEP for that region]
 *         px_nl_sweep     one Jacobian-augmented sweep; *err_max = max_p relative L2 change
 *   px_nl_finish          the converged iterate becomes the direct trajectory (then
 *                         px_finish_direct / the adjoint proceed as after px_direct). */
int px_nl_init(void* handle, void* stream);
int px_nl_prepare(void* handle, void* stream);
int px_nl_sweep(void* handle, double* err_max, void* stream);
int px_nl_finish(void* handle, void* stream);

/* Standalone adjoint terminal data q†_T (B×n): replaces the qdag_T argument of
 * solve_adjoint_linear / solve_adjoint_varying (paraexp.py:298-353) when the
 * adjoint is run without px_finish_direct. Burgers needs px_direct first. */
int px_set_adjoint_terminal(void* handle, const double* qdag_T, int mem, void* stream);
/* Adjoint sweep (solve_adjoint_linear / solve_adjoint_varying, paraexp.py:298-353):
 * rank-partials of q†(0), ∫q† dt and the projected gradient. */
int px_adjoint(void* handle, void* stream);
/* After the caller's allreduce of QDAG0/G/GRAD partials: adds the q†_T terms
 * (gradient_wrt_forcing / initial_condition_gradient, optimization.py:103-117). */
int px_finish_adjoint(void* handle, void* stream);
/* world = 1 convenience: direct + finish + adjoint + finish (one gradient evaluation,
 * direct_adjoint_loop, optimization.py:154-231). Linear testbed only (Burgers needs the
 * host planner between the sweeps). */
int px_gradient(void* handle, void* stream);

/* CUDA-graph replay of px_gradient (default on): the whole gradient is captured
 * once per plan set / timing mode and replayed on an internal stream ordered
 * after the caller's stream. */
int px_set_graphs(void* handle, int enable);

/* Device pointer and element count of a field (for NCCL allreduce by the caller). */
int px_buffer(void* handle, int field, double** dev_ptr, size_t* count);
/* Copy a field out (host or device destination). */
int px_get(void* handle, int field, double* dst, size_t count, int mem, void* stream);

/* Phase timing with CUDA events recorded on the work stream around each sweep
 * phase (enable before the timed region; px_get_timing synchronises the events).
 * Phases: PX_PHASE_*; ms[i] = summed device time, launches[i] = kernel launches
 * inside those phase windows. */
enum {
  PX_PHASE_RK4_DIRECT = 0,
  PX_PHASE_RK4_ADJOINT = 1,
  PX_PHASE_EXP_DIRECT = 2,
  PX_PHASE_EXP_ADJOINT = 3,
  PX_PHASE_OTHER = 4,
  PX_PHASE_COUNT = 5
};
typedef struct px_timing {
  double ms[PX_PHASE_COUNT];
  uint64_t launches[PX_PHASE_COUNT];
  double bytes[PX_PHASE_COUNT];   /* algorithmic bytes executed inside each phase */
} px_timing;
/* enable: 0 off, 1 phase windows (graph replay keeps running), 2 phase windows plus CUDA events
 * around every launch of the kernel classes below (px_gradient then runs eagerly, no graph). */
int px_set_timing(void* handle, int enable);
int px_get_timing(void* handle, px_timing* out);
enum {
  PX_KCLASS_MARCH2 = 0,   /* the two-step fused RK4 march launches (k_rk4_marchc / k_rk4_march2) */
  PX_KCLASS_CHEB = 1,     /* the 2D Chebyshev passes (k_cheb_march) */
  PX_KCLASS_COUNT = 2
};
/* Summed device ms and launch count of one kernel class since the last call (timing mode 2). */
int px_get_kernel_timing(void* handle, int kclass, double* ms, uint64_t* launches);

/* ---- The reference's hybrid algorithm with its own objective (hybrid.py:1-290,
 * optimization.py:84-112,172-189) — a separate handle ----------------
 * 1D Burgers (V ≡ 0), or with desc.ny > 1 the reference's own two-field system (U, V) on an nx×ny
 * grid (problems.py:177-186, 316-343), with the forcing field f(x)·θ(t), θ(t) = law[0] + law[1]·sin(law[3]·t) +
 * law[2]·cos(law[3]·t) (the reference's f·sin(ωt): {0, 1, 0, ω}); tracking objective
 * J = (1/T)∫‖u − u_t‖² dt (trapezoid on the RK4 nodes) against a target given on the nodes;
 * slices of any widths on the serial sweep's uniform node grid (the geometric partition,
 * hybrid.py:35-55); adjoint in the reference's solve_hybrid form (zero terminal data + source
 * s = 2(u − u_t) in every slice, the slice ends through the frozen J(ū_m)ᵀ of all earlier
 * slices); gradient ∂L/∂f = (1/T)∫θ(t)·q†(t) dt (gradient_wrt_forcing). With overlap, each
 * slice's adjoint solve starts on its own SM the moment the serial direct kernel has stored
 * the slice (a progress flag per slice in HBM), i.e. during the serial sweep — the reference's
 * overlapped worker pipeline (hybrid.py:185-204). */
typedef struct px_hybrid_desc {
  int nx;              /* periodic grid; 1D: n = nx points per state */
  double D, hx, T;     /* diffusion, spacing, horizon */
  int batch;           /* B members, one forcing field each */
  int nslices;         /* P */
  const int* offsets;  /* P+1 node offsets 0 = o_0 < … < o_P = S (host); h = T/S */
  double law[4];       /* θ(t) */
  int target_batched;  /* 0: target (S+1)×n shared by the members; 1: (S+1)×B×n */
  /* ny > 1: the reference's own 2D two-field Burgers testbed on an nx×ny grid (problems.py:177-186,
   * 316-343): states, forcing, target and gradient are (U, V) pairs of length n = 2·nx·ny, the U
   * block first, x fastest; hy the y spacing. ny ≤ 1: 1D (V ≡ 0), hy unused. */
  int ny;
  double hy;
} px_hybrid_desc;
enum {
  PX_HFIELD_J = 0,     /* (B)          tracking cost */
  PX_HFIELD_GRAD = 1,  /* (B, n)       ∂L/∂f */
  PX_HFIELD_UT = 2,    /* (B, n)       u(T) */
  PX_HFIELD_QDAG0 = 3, /* (B, n)       q†(0) */
  PX_HFIELD_TRAJ = 4,  /* (S+1, B, n)  direct trajectory */
  PX_HFIELD_AEND = 5,  /* (B, P, n)    slice adjoint solutions at the slice starts */
  PX_HFIELD_ZL = 6,    /* (B, P, n)    their ∫θ·a dt */
  PX_HFIELD_UBAR = 7,  /* (P, B, n)    slice means */
  PX_HFIELD_COUNT = 8
};
int px_hybrid_create(const px_hybrid_desc* desc, void** out_handle);
void px_hybrid_destroy(void* handle);
const char* px_hybrid_last_error(const void* handle);
/* u0 (B×n), f (B×n), target ((S+1)×n or (S+1)×B×n), qdag_T (B×n terminal data, NULL = 0). */
int px_hybrid_set_inputs(void* handle, const double* u0, const double* f, const double* target,
                         const double* qdag_T, int mem, void* stream);
/* Serial direct sweep + J, and every slice's adjoint inhomogeneous solve: overlapped with the
 * sweep when `overlap` and all CTAs fit co-resident (else after it; px_hybrid_get_timing says). */
int px_hybrid_direct(void* handle, int overlap, void* stream);
/* Slice means ū_p and the frozen operators' FOV box (re_lo, re_hi, im) to the host (syncs). */
int px_hybrid_bounds(void* handle, double* out3, void* stream);
/* Slice p's plan for exp(Δ_p J(ū_p)ᵀ) (span Δ_p = (o_{p+1} − o_p)·h) with the time-law series
 * coef_gc / coef_gs (degree+1 each; NULL when law[3] == 0), see expaction.ChebPlan. */
int px_hybrid_set_slice_plan(void* handle, int p, const px_cheb_plan* plan, const double* coef_gc,
                             const double* coef_gs);
/* The frozen-operator carry and the gradient (needs every slice plan). */
int px_hybrid_adjoint(void* handle, void* stream);
/* The reference's loop with algorithm "nonlinear" on the 2D two-field handle (desc.ny > 1, equal
 * slices): the iterative nonlinear direct, Algorithm 2 (nonlinear.py:69-194;
 * optimization.py:206-231). px_hybrid_nl_init: the constant initial guess u0 on every node; then per
 * sweep px_hybrid_bounds (slice means and FOV box of the iterate) → px_hybrid_nl_set_plans (the
 * actions exp(Δ(D∇² + J̄_p)) of slice width and of step width, exp series only) →
 * px_hybrid_nl_sweep (err = max over slices of the relative L2 change, nonlinear.py:44-66; syncs)
 * until err < eps; px_hybrid_nl_finish makes the iterate the direct trajectory (tracking cost, every
 * slice's adjoint solve), after which px_hybrid_bounds / set_slice_plan / adjoint run as for the
 * hybrid (with q†_T = 0 `solve_adjoint_varying`'s absorbed form is the hybrid's). */
int px_hybrid_nl_init(void* handle, void* stream);
int px_hybrid_nl_set_plans(void* handle, const px_cheb_plan* slice, const px_cheb_plan* step);
int px_hybrid_nl_sweep(void* handle, double* err, void* stream);
int px_hybrid_nl_finish(void* handle, void* stream);
int px_hybrid_get(void* handle, int field, double* dst, size_t count, int mem, void* stream);
/* Device ms of the last px_hybrid_direct: ms[0] the serial direct kernel, ms[1] the slice-solve
 * kernel (from its launch, waiting included), ms[2] both (first start to last end), ms[3] the
 * slice solves' tail after the direct ended (the adjoint work the overlap did not hide),
 * ms[4] 1 if the slice solves overlapped the sweep. */
int px_hybrid_get_timing(void* handle, double* ms5);

int px_get_stats(void* handle, px_stats* out);
int px_reset_stats(void* handle);

#ifdef __cplusplus
}
#endif

#endif /* PARAEXP_H_ */
