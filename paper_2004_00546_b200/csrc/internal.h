// internal.h — the native handle and the host-side interfaces between translation units.
//
// Layout of libparaexp.so (one header of kernels per translation unit, so no kernel is
// defined twice):
//   abi.cu      C ABI (include/paraexp.h): argument checks, handle lifetime, CUDA-graph
//               capture/replay of the gradient, field access
//   runtime.cu  errors, allocation, dynamic-smem opt-in, timing windows / NVTX, graph segments
//   sweeps.cu   the Paraexp sweeps of one rank: direct / adjoint (linear), local blocks,
//               finish steps (reference structure paraexp.py:187-353)
//   lanes.cu    rk4.cuh: zero-data RK4 slice solves of all lanes
//   cheb.cu     cheb_march.cuh, scan1d.cuh: Chebyshev exp-actions (2D passes, 1D scans)
//   krylov.cu   krylov.cuh: batched Arnoldi exp-actions
//   burgers.cu  burgers.cuh, burgers_iter.cuh: Burgers serial sweep, adjoint, Algorithm 2
//   ops.cu      kernels.cuh: axpby, projections, reductions, control sources, closed-form ∫
//   tracking.cu tracking.cuh: the linear testbed's tracking objective (recording sweep, cost,
//               adjoint lanes with the source 2(u − u_t))
//   hybrid.cu   C ABI of the reference's hybrid with its tracking objective (px_hybrid_*); its
//               kernels (hybrid.cuh) are instantiated in burgers.cu
//   hybrid2d.cu hybrid2d.cuh: the same entry points on the reference's 2D two-field Burgers testbed
//               (desc.ny > 1), Algorithm 2 on it (px_hybrid_nl_*)
#pragma once
#include <cuda_runtime.h>
#include <cufft.h>

#include <string>
#include <vector>

#include "../../include/paraexp.h"
#include "common.cuh"
#include "hybrid_args.h"

namespace pxi {

// Kernel-variant selection, per handle (px_set_variant). The defaults are the measured-best
// variants; the alternatives stay selectable for the parity tests and the dev tools.
struct Variants {
  int march2 = 1;           // PX_VAR_MARCH2: 0 one RK4 step per launch, 1 two-step launches for
                            // sweeps ≥ 2^28 lane-points, 2 two-step launches at any size
  int march_cols = 3;       // PX_VAR_MARCH_COLS: columns per thread of the two-step march (3: k_rk4_marchc
                            // in strip mode; 2: k_rk4_march2)
  int march_band = 0;       // PX_VAR_MARCH_BAND: rows per band of the two-step march (0: automatic)
  int cheb_terms = 7;       // PX_VAR_CHEB_TERMS: at most this many Chebyshev terms per 2D pass (1 … 7)
  int cheb_terms_phi = 5;   // PX_VAR_CHEB_TERMS_PHI: the same for passes with the φ₁ accumulator (7 spills)
  int cheb_strip = 0;       // PX_VAR_CHEB_STRIP: strip width of the 2D passes (0: balanced)
  int cheb_band = 0;        // PX_VAR_CHEB_BAND: rows per band of the 2D passes (0: one wave)
  int scan1d_cluster = 1;   // PX_VAR_SCAN1D_CLUSTER: 8-CTA cluster scans for 1D n ≥ 2048
  int burgers_cluster = 1;  // PX_VAR_BURGERS_CLUSTER: 8-CTA cluster Burgers sweeps for n ≥ 2048
  int krylov_ortho = 1;     // PX_VAR_KRYLOV_ORTHO: 1 delayed reorthogonalization (two basis passes per
                            // Arnoldi step), 0 CGS2 (four passes)
};

struct Plan {
  bool set = false;
  bool krylov = false;
  double span = 0.0;
  int substeps = 0, degree = 0, sigma = -1;
  double center = 0.0, scale = 1.0;
  std::vector<double> be, bp;
  std::vector<double> gc, gs;  // time-law series (px_set_cheb_plan_law): ∫₀^τ (cos ωs, sin ωs)·e^{sM} ds
  double* dcoef = nullptr;  // device copy: be[0..K], bp[0..K]
};

struct Handle {
  px_problem_desc d{};
  int device = 0;
  int dim = 1;
  size_t n = 0;
  int B = 1, K = 1, Pl = 1, L = 1;
  int rows_x = 1, rows_y = 1;
  px::Stencil5 A{}, AT{};
  Variants var{};

  // inputs
  double *u0 = nullptr, *ut = nullptr, *ctrl = nullptr;
  double *tx = nullptr, *ty = nullptr;
  int *ix = nullptr, *iy = nullptr;
  bool basis_set = false, inputs_set = false;
  // sources and lanes
  double *g = nullptr, *gadj = nullptr;
  double *bsrc = nullptr, *cz = nullptr;  // h·S(hM)·g and h²·U(hM)·g (RK4 Horner constants)
  bool z_valid = false;
  double *Y0 = nullptr, *Y1 = nullptr, *Z = nullptr;
  // closed-form adjoint ∫ (2D circulant operator): Σ_p z_p = (Aᵀ)⁻¹(Σ_p y_n,p − Pl·n·b) + …
  bool z_closed = false;
  int adjoint_mode = PX_ADJOINT_ABSORBED;  // Burgers: PX_ADJOINT_FROZEN_SPAN = reference solve_hybrid
  // forcing time law (px_set_time_law, linear testbed): f·θ(t), θ = law[0] + law[1] sin(law[3] t) +
  // law[2] cos(law[3] t); fctl holds f (B × n), the adjoint's ∫ becomes ∫θ·q† dt
  bool has_law = false;
  double law[4] = {1.0, 0.0, 0.0, 0.0};
  double* fctl = nullptr;
  // tracking objective (px_set_tracking_target, the reference's linear loop): node target
  // (S+1) × n or (S+1) × B × n, θ at the half steps, recording/adjoint lane buffers (tracking.cu)
  bool tracking = false;
  int trk_per_member = 0;
  double *trk_target = nullptr, *trk_theta = nullptr;
  double *trk_y = nullptr, *trk_acc = nullptr, *trk_z = nullptr;
  double* trk_x[2] = {nullptr, nullptr};
  cufftHandle fft = 0;
  double2* fbuf = nullptr;  // B × n complex
  double* bsum = nullptr;   // B: Σ_i b[b][i]
  const double *vend = nullptr, *wend = nullptr;
  // exp-action work
  double* Wk[4] = {nullptr, nullptr, nullptr, nullptr};
  double* ACC[2] = {nullptr, nullptr};
  double* S = nullptr;  // Σ of the adjoint carries' inputs (2D Chebyshev: one φ₁ action on it)
  // outputs
  double *UT = nullptr, *QT = nullptr, *QDAG0 = nullptr, *G = nullptr;
  double *J = nullptr, *GRAD = nullptr, *R = nullptr, *partial = nullptr;
  int* nonfinite = nullptr;
  double* UBND = nullptr;
  int red_blocks = 0;
  // Burgers
  double *traj = nullptr, *ubar = nullptr, *bounds = nullptr, *bpart = nullptr;
  int bounds_blocks = 0;
  // Burgers iterative direct (Algorithm 2)
  double *traj_b = nullptr, *Dc = nullptr, *nl_err = nullptr;
  std::vector<double> nl_err_host;
  // Krylov
  px::KrylovWork kw{};
  // local blocks (px_set_local_blocks): concurrent block carries on side streams
  struct Block {
    double* Wk[4] = {nullptr, nullptr, nullptr, nullptr};
    double* ACC[2] = {nullptr, nullptr};
    px::KrylovWork kw{};
    double* D = nullptr;   // block carry at the block edge (B × n)
    double* Gp = nullptr;  // block φ accumulator (adjoint, B × n)
    double* S = nullptr;   // block's Σ of carry inputs (2D Chebyshev adjoint)
    cudaStream_t st = nullptr;
    cudaEvent_t ev = nullptr;
    int q0 = 0, q1 = 0;  // direct sweep: local slices [q0, q1)
    int a0 = 0, a1 = 0;  // adjoint sweep: the mirrored partition (equal long-span lengths)
  };
  int lb = 1;
  std::vector<Block> blocks;
  cudaEvent_t ev_fork = nullptr;

  Plan plans[PX_PLAN_COUNT];
  px_stats stats{};
  // phase timing (CUDA events on the work stream)
  struct TMark { int phase; cudaEvent_t a, b; uint64_t launches; double bytes; };
  int timing = 0;  // 0 off, 1 phase windows, 2 phase windows + per-launch kernel-class events (eager)
  std::vector<TMark> marks;
  struct KMark { int cls; cudaEvent_t a, b; };
  std::vector<KMark> kmarks;
  double kms[PX_KCLASS_COUNT] = {0.0};
  uint64_t kcount[PX_KCLASS_COUNT] = {0};
  std::vector<cudaEvent_t> event_pool;
  px_timing tacc{};
  // CUDA-graph replay of px_gradient (linear testbed): captured once per
  // (plans, variants, timing mode), replayed on an internal stream ordered after the caller's
  bool graphs = true;
  bool graph_valid = false;
  cudaStream_t gstream = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  px_stats graph_delta{};
  // the captured gradient is a list of segments, one per timing phase (−1: untimed)
  struct Seg { int phase; cudaGraphExec_t exec; uint64_t launches; double bytes; };
  std::vector<Seg> segs;
  bool capturing = false;
  int cap_phase = -1;
  uint64_t cap_launches0 = 0;
  double cap_bytes0 = 0.0;
  int cap_error = 0;
  std::string err;
  int stage = 0;  // 0 none, 1 direct, 2 finished direct, 3 adjoint, 4 finished
  std::vector<void*> allocs;
};

// ---- runtime.cu -----------------------------------------------------------------------
extern thread_local std::string g_last_error;
int fail(Handle* h, int code, const std::string& msg);
int dalloc(Handle* h, void** p, size_t bytes);
template <typename T>
int dalloc_t(Handle* h, T** p, size_t count) {
  return dalloc(h, reinterpret_cast<void**>(p), count * sizeof(T));
}
int smem_attr(Handle* h, const void* kernel, size_t bytes);
// timing windows: tbegin returns −1 (off), −2 (capturing: a graph segment) or a mark index
int tbegin(Handle* h, int phase, cudaStream_t s);
void tend(Handle* h, int idx, cudaStream_t s);
cudaEvent_t take_event(Handle* h);
// per-launch events around one kernel of class `cls` (timing mode 2); kbegin returns −1 when off
int kbegin(Handle* h, int cls, cudaStream_t s);
void kend(Handle* h, int idx, cudaStream_t s);
void seg_open(Handle* h, int phase);
void seg_close(Handle* h);
void drop_segments(Handle* h);
const char* phase_name(int phase);

inline dim3 grid1(size_t n, int B, int nt = 256) {
  size_t blocks = (n + nt - 1) / nt;
  return dim3((unsigned)blocks, (unsigned)B);
}
inline dim3 grid_stride(size_t n, int B) {
  size_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  return dim3((unsigned)blocks, (unsigned)B);
}

// ---- ops.cu ---------------------------------------------------------------------------
int axpby(Handle* h, double* out, long long obs, const double* x, long long xbs, double alpha, const double* y,
          long long ybs, double beta, cudaStream_t s);
int project(Handle* h, double* grad, const double* F, long long Fbs, double alpha, double beta, cudaStream_t s);
int apply_plus_control(Handle* h, double* out, const double* x, long long xbs, const px::Stencil5& st,
                       bool with_control, cudaStream_t s);
int objective(Handle* h, cudaStream_t s);  // J = ½‖QT‖² per member (non-finite flag)
// out[b] = scale·Σ_j partial[b·m + j] (fixed order; non-finite flag)
int finalize_sum(Handle* h, double* out, const double* partial, int m, double scale, cudaStream_t s);
int z_closed_form(Handle* h, const double* wend, cudaStream_t s);

// ---- lanes.cu -------------------------------------------------------------------------
int rk4_sweep(Handle* h, bool adjoint, const double** final_out, cudaStream_t s);
int lane_sum_plus(Handle* h, double* out, const double* lanes, const double* c, double scale, bool with_z,
                  cudaStream_t s);

// ---- cheb.cu / krylov.cu --------------------------------------------------------------
// ttop (time law only): the physical time at which the action's reflected-time span starts;
// pacc then accumulates ∫₀^span θ(ttop − σ)·e^{σM}·src dσ instead of span·φ₁(span·M)·src
int cheb_action(Handle* h, const Plan& pl, const px::Stencil5& st, const double* src, long long src_bs,
                const double* addend, long long add_bs, double* pacc, double** result, cudaStream_t s,
                double* ssum = nullptr, double ttop = 0.0);
// the law series of substep `sub` of plan `pl` started at ttop (K+1 values)
void law_coefficients(const Handle* h, const Plan& pl, double ttop, int sub, double* out);
bool cheb_has_ssum(const Handle* h);
bool use_scan1d(const Handle* h);
int scan1d(Handle* h, bool adjoint, const double* lanes, double* out, double* pacc, int long_slot, cudaStream_t s);
int krylov_action(Handle* h, const Plan& pl, const px::Stencil5& st, const double* src, long long src_bs,
                  const double* addend, long long add_bs, double* pacc, double** result, cudaStream_t s);
int krylov_alloc(px::KrylovWork& kw, int m, size_t n, int B, std::string* err);
void krylov_free(px::KrylovWork& kw);

// ---- sweeps.cu ------------------------------------------------------------------------
int exp_action(Handle* h, int slot, const px::Stencil5& st, const double* src, long long src_bs,
               const double* addend, long long add_bs, double* pacc, double** result, cudaStream_t s,
               double* ssum = nullptr, double ttop = 0.0);
int direct_linear(Handle* h, cudaStream_t s);
int adjoint_linear(Handle* h, cudaStream_t s);
int finish_direct_impl(Handle* h, cudaStream_t s);
int finish_adjoint_impl(Handle* h, cudaStream_t s);
void free_blocks(Handle* h);
int set_local_blocks(Handle* h, int blocks, const int* sizes = nullptr);

// ---- tracking.cu ----------------------------------------------------------------------
int tracking_set(Handle* h, const double* target, int per_member, int mem, cudaStream_t s);
int tracking_theta(Handle* h);  // θ(j·h/2) table from the handle's law
int track_direct(Handle* h, cudaStream_t s);
int track_adjoint_lanes(Handle* h, const double** wend, cudaStream_t s);

// ---- burgers.cu -----------------------------------------------------------------------
int burgers_direct(Handle* h, cudaStream_t s);
int burgers_adjoint(Handle* h, cudaStream_t s);
int nl_init(Handle* h, cudaStream_t s);
int nl_means_bounds(Handle* h, cudaStream_t s);
int nl_sweep(Handle* h, double* err_max, cudaStream_t s);
// the reference's hybrid with its tracking objective (hybrid.cuh, driven by hybrid.cu)
cudaError_t hyb_launch_direct(const px::HybArgs& a, int ppt, cudaStream_t s);
int hyb_direct_ctas(int nx, int B);  // CTAs of the serial sweep (8 per member on a cluster)
cudaError_t hyb_launch_lanes(const px::HybArgs& a, int ppt, size_t smem, cudaStream_t s);
cudaError_t hyb_launch_scan(const px::HybScanArgs& a, int ppt, cudaStream_t s);
cudaError_t hyb_lanes_occupancy(int ppt, size_t smem, int* per_sm);
cudaError_t hyb_launch_means_bounds(double* ubar, const double* traj, const int* offsets, int P, int B, int n,
                                    double* bpart, int bblocks, double* bounds, double hx, double D,
                                    cudaStream_t s);

}  // namespace pxi

#define PX_CUDA(h, call)                                                                  \
  do {                                                                                    \
    cudaError_t _e = (call);                                                              \
    if (_e != cudaSuccess)                                                                \
      return ::pxi::fail((h), _e == cudaErrorMemoryAllocation ? PX_ERR_NOMEM : PX_ERR_CUDA, \
                         std::string(#call) + ": " + cudaGetErrorString(_e));             \
  } while (0)

#define PX_CHECK_LAUNCH(h)                                                                \
  do {                                                                                    \
    cudaError_t _e = cudaGetLastError();                                                  \
    if (_e != cudaSuccess)                                                                \
      return ::pxi::fail((h), PX_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(_e)); \
    (h)->stats.kernel_launches++;                                                         \
  } while (0)

#define PX_TRY(expr)              \
  do {                            \
    int _rc = (expr);             \
    if (_rc != PX_OK) return _rc; \
  } while (0)
