// hybrid2d.h — host-side state of the hybrid handle on the 2D two-field Burgers testbed
// (hybrid2d.cu) and the common head px_hybrid_* dispatches on (hybrid.cu).
#pragma once
#include <string>
#include <vector>

#include "internal.h"

namespace pxi {

constexpr int PX_MAX_CHEB_DEGREE = 2048;  // Algorithm 2's two plans (device coefficient pool)

// Both hybrid handles (1D: hybrid.cu, 2D two-field: hybrid2d.cu) start with this head.
struct HybridHead {
  Handle base;  // device, error text, allocations, stats
  int dim = 1;
};

struct Hybrid2D : HybridHead {
  static constexpr int NSIDE = 4;  // side streams of the overlap pipeline (slice p on stream p mod 4)
  int nx = 0, ny = 0, B = 1, P = 1, S = 1, target_b = 1, max_np = 0;
  double D = 0.0, hx = 0.0, hy = 0.0, T = 1.0, h = 1.0;
  double law[4] = {1.0, 0.0, 0.0, 0.0};
  std::vector<int> offs;
  std::vector<double> theta_host;  // θ(k·h/2), k = 0 … 2S
  int* d_offs = nullptr;
  double* theta = nullptr;
  double *u0 = nullptr, *f = nullptr, *target = nullptr, *qT = nullptr;
  double *traj = nullptr, *J = nullptr, *ubar = nullptr, *qdag0 = nullptr, *grad = nullptr, *G = nullptr;
  double* w[4] = {nullptr, nullptr, nullptr, nullptr};  // direct stages / Chebyshev recurrence (B × 2n each)
  // slice adjoint lanes (B·P × 2n each): a (ends up a_p(T_p)), ∫θa, the RK4 accumulator, two stage inputs
  double *la = nullptr, *lz = nullptr, *lacc = nullptr;
  double* ly[2] = {nullptr, nullptr};
  double *cpart = nullptr, *bpart = nullptr;
  int cost_blocks = 0, bounds_blocks = 0;
  bool has_qT = false, inputs = false, direct_done = false, means_done = false, adjoint_done = false;
  struct SlicePlan {
    bool set = false;
    int substeps = 0, degree = 0, sigma = -1;
    double c0 = 0.0, d = 1.0, span = 0.0;
    std::vector<double> be, law;  // exp series; law series per substep (substeps × (degree+1))
  };
  std::vector<SlicePlan> plans;
  // on-chip variants for small grids (nx·ny ≤ 2048: the whole sweep / every slice solve / the frozen
  // carry as one kernel each, slices released by progress flags); PX_HYB2D_ONCHIP=0 at create forces
  // the per-stage launches
  bool small = false;
  int ppt = 1;
  int* flags = nullptr;
  px::HybSlicePlan* d_plans = nullptr;
  double* d_coef = nullptr;
  size_t coef_cap = 0;
  bool plans_dirty = true;
  // Algorithm 2 (px_hybrid_nl_*): the next iterate, the carried homogeneous parts, per-slice errors,
  // the two plans' exp series (slice width, step width)
  double *Qn = nullptr, *Dc = nullptr, *nl_err = nullptr, *nl_coef = nullptr;
  struct NlPlan { int K = 0, subs = 0, sigma = -1; double c0 = 0.0, d = 1.0; };
  NlPlan nl_s, nl_h;
  std::vector<double> nl_be_s, nl_be_h;  // host copies of the two exp series (per-term launches)
  bool nl_active = false, nl_plans = false;
  cudaStream_t side[NSIDE] = {nullptr, nullptr, nullptr, nullptr};
  std::vector<cudaEvent_t> ev_slice;
  cudaEvent_t ev_join[NSIDE] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  int overlapped = 0;
  Hybrid2D() { dim = 2; }
};

int h2_create(const px_hybrid_desc* d, void** out);
void h2_destroy(Hybrid2D* hy);
int h2_set_inputs(Hybrid2D* hy, const double* u0, const double* f, const double* target, const double* qdag_T, int mem,
                  cudaStream_t s);
int h2_direct(Hybrid2D* hy, int overlap, cudaStream_t s);
int h2_bounds(Hybrid2D* hy, double* out3, cudaStream_t s);
int h2_set_slice_plan(Hybrid2D* hy, int sl, const px_cheb_plan* plan, const double* gc, const double* gs);
int h2_adjoint(Hybrid2D* hy, cudaStream_t s);
int h2_nl_init(Hybrid2D* hy, cudaStream_t s);
int h2_nl_set_plans(Hybrid2D* hy, const px_cheb_plan* slice, const px_cheb_plan* step);
int h2_nl_sweep(Hybrid2D* hy, double* err, cudaStream_t s);
int h2_nl_finish(Hybrid2D* hy, cudaStream_t s);
int h2_get(Hybrid2D* hy, int field, double* dst, size_t count, int mem, cudaStream_t s);
int h2_get_timing(Hybrid2D* hy, double* ms5);

}  // namespace pxi
