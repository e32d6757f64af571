// paraexp_capi.cu — C ABI (include/paraexp.h) and native orchestration of one
// Paraexp direct-adjoint gradient on one GPU (one rank's slice block).
//
// Sweep structure (reference structure paraexp.py:187-353):
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
#include <cuda_runtime.h>
#include <cufft.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges for nsys / Nsight timelines

#include "../../include/paraexp.h"
#include "kernels.cuh"
#include "burgers.cuh"
#include "burgers_iter.cuh"
#include "krylov.cuh"
#include "krylov_coop.cuh"
#include "rk4.cuh"
#include "cheb_march.cuh"
#include "scan1d.cuh"

#include <cstdlib>

namespace {

thread_local std::string g_last_error;

struct Plan {
  bool set = false;
  bool krylov = false;
  double span = 0.0;
  int substeps = 0, degree = 0, sigma = -1;
  double center = 0.0, scale = 1.0;
  std::vector<double> be, bp;
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
  cufftHandle fft = 0;
  double2* fbuf = nullptr;  // B × n complex
  double* bsum = nullptr;   // B: Σ_i b[b][i]
  const double *vend = nullptr, *wend = nullptr;
  // exp-action work
  double* Wk[4] = {nullptr, nullptr, nullptr, nullptr};
  double* ACC[2] = {nullptr, nullptr};
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
    cudaStream_t st = nullptr;
    cudaEvent_t ev = nullptr;
    int q0 = 0, q1 = 0;
  };
  int lb = 1;
  std::vector<Block> blocks;
  cudaEvent_t ev_fork = nullptr;

  Plan plans[PX_PLAN_COUNT];
  px_stats stats{};
  // phase timing (CUDA events on the work stream)
  struct TMark { int phase; cudaEvent_t a, b; uint64_t launches; double bytes; };
  bool timing = false;
  std::vector<TMark> marks;
  std::vector<cudaEvent_t> event_pool;
  px_timing tacc{};
  // CUDA-graph replay of px_gradient (linear testbed): captured once per
  // (plans, timing mode), replayed on an internal stream ordered after the caller's
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

int fail(Handle* h, int code, const std::string& msg) {
  if (h) h->err = msg;
  g_last_error = msg;
  return code;
}

cudaEvent_t take_event(Handle* h) {
  if (!h->event_pool.empty()) {
    cudaEvent_t e = h->event_pool.back();
    h->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

void seg_open(Handle* h, int phase) {
  h->cap_phase = phase;
  h->cap_launches0 = h->stats.kernel_launches;
  h->cap_bytes0 = h->stats.algorithmic_bytes;
  if (cudaStreamBeginCapture(h->gstream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) h->cap_error = 1;
}

void seg_close(Handle* h) {
  cudaGraph_t g = nullptr;
  if (cudaStreamEndCapture(h->gstream, &g) != cudaSuccess || !g) {
    h->cap_error = 1;
    return;
  }
  size_t nn = 0;
  cudaGraphGetNodes(g, nullptr, &nn);
  if (nn > 0) {
    cudaGraphExec_t ex = nullptr;
    if (cudaGraphInstantiate(&ex, g, 0) != cudaSuccess) h->cap_error = 1;
    else
      h->segs.push_back({h->cap_phase, ex, h->stats.kernel_launches - h->cap_launches0,
                         h->stats.algorithmic_bytes - h->cap_bytes0});
  }
  cudaGraphDestroy(g);
}

void drop_segments(Handle* h) {
  for (auto& sg : h->segs) cudaGraphExecDestroy(sg.exec);
  h->segs.clear();
}

const char* phase_name(int phase) {
  static const char* names[] = {"px.rk4_direct", "px.rk4_adjoint", "px.exp_direct", "px.exp_adjoint", "px.other"};
  return (phase >= 0 && phase < PX_PHASE_COUNT) ? names[phase] : "px.phase";
}

// RAII NVTX range (the reference's recorder hooks, `workers.py:26-36`, become timeline ranges)
struct NvtxScope {
  explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
  ~NvtxScope() { nvtxRangePop(); }
  NvtxScope(const NvtxScope&) = delete;
  NvtxScope& operator=(const NvtxScope&) = delete;
};

// Open a timing window for `phase` (returns -1 when timing is off; while capturing a
// graph the window becomes its own graph segment, timed at replay). Eager windows are
// also NVTX ranges.
int tbegin(Handle* h, int phase, cudaStream_t s) {
  if (h->capturing) {
    seg_close(h);
    seg_open(h, phase);
    return -2;
  }
  nvtxRangePushA(phase_name(phase));
  if (!h->timing) return -1;
  Handle::TMark m{phase, take_event(h), take_event(h), h->stats.kernel_launches, h->stats.algorithmic_bytes};
  cudaEventRecord(m.a, s);
  h->marks.push_back(m);
  return (int)h->marks.size() - 1;
}

void tend(Handle* h, int idx, cudaStream_t s) {
  if (idx == -2 && h->capturing) {
    seg_close(h);
    seg_open(h, -1);
    return;
  }
  nvtxRangePop();
  if (idx < 0) return;
  Handle::TMark& m = h->marks[idx];
  cudaEventRecord(m.b, s);
  m.launches = h->stats.kernel_launches - m.launches;
  m.bytes = h->stats.algorithmic_bytes - m.bytes;
}

#define PX_CUDA(h, call)                                                          \
  do {                                                                            \
    cudaError_t _e = (call);                                                      \
    if (_e != cudaSuccess)                                                        \
      return fail((h), _e == cudaErrorMemoryAllocation ? PX_ERR_NOMEM : PX_ERR_CUDA, \
                  std::string(#call) + ": " + cudaGetErrorString(_e));            \
  } while (0)

#define PX_CHECK_LAUNCH(h)                                                        \
  do {                                                                            \
    cudaError_t _e = cudaGetLastError();                                          \
    if (_e != cudaSuccess)                                                        \
      return fail((h), PX_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(_e)); \
    (h)->stats.kernel_launches++;                                                 \
  } while (0)

#define PX_TRY(expr)            \
  do {                          \
    int _rc = (expr);           \
    if (_rc != PX_OK) return _rc; \
  } while (0)

// Opt a kernel into `bytes` of dynamic shared memory once per (kernel, device): the
// attribute belongs to the device's context, so a process driving several GPUs needs it
// on each. The table is shared by all handles (one per device, possibly on different
// host threads), hence the lock.
int smem_attr(Handle* h, const void* kernel, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  PX_CUDA(h, cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = done[{kernel, dev}];
  if (have >= bytes) return PX_OK;
  PX_CUDA(h, cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  have = bytes;
  return PX_OK;
}

int dalloc(Handle* h, void** p, size_t bytes) {
  if (bytes == 0) bytes = 8;
  cudaError_t e = cudaMalloc(p, bytes);
  if (e != cudaSuccess)
    return fail(h, e == cudaErrorMemoryAllocation ? PX_ERR_NOMEM : PX_ERR_CUDA,
                "cudaMalloc(" + std::to_string(bytes) + " B): " + cudaGetErrorString(e));
  h->allocs.push_back(*p);
  return PX_OK;
}

template <typename T>
int dalloc_t(Handle* h, T** p, size_t count) {
  return dalloc(h, reinterpret_cast<void**>(p), count * sizeof(T));
}

inline dim3 grid1(size_t n, int B, int nt = 256) {
  size_t blocks = (n + nt - 1) / nt;
  return dim3((unsigned)blocks, (unsigned)B);
}

inline dim3 grid_stride(size_t n, int B) {
  size_t blocks = std::min<size_t>((n + 255) / 256, 148 * 16);
  return dim3((unsigned)std::max<size_t>(blocks, 1), (unsigned)B);
}

// ---------------------------------------------------------------------------
// RK4 lanes sweep
// ---------------------------------------------------------------------------

int axpby(Handle* h, double* out, long long obs, const double* x, long long xbs, double alpha,
          const double* y, long long ybs, double beta, cudaStream_t s) {
  px::k_axpby<<<grid_stride(h->n, h->B), 256, 0, s>>>(out, obs, x, xbs, alpha, y, ybs, beta, h->n);
  PX_CHECK_LAUNCH(h);
  return PX_OK;
}

// Zero-data RK4 sweep of all local lanes (rk4.cuh); returns the final lane buffer.
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
  if (adjoint)
    PX_TRY(axpby(h, h->cz, (long long)h->n, h->Wk[1], (long long)h->n, 0.5 * hs * hs, nullptr, 0, 0.0, s));

  const int nsteps = h->d.nsteps;
  double* cur = nullptr;
  uint64_t launched_steps = 0;
  h->z_valid = false;
  if (h->dim == 1 && h->n <= 4096) {
    px::Lane1DArgs a{};
    a.y_out = h->Y0; a.b = h->bsrc; a.z = h->Z; a.st = st; a.h = hs;
    a.n = (int)h->n; a.lanes_per_b = h->Pl; a.nsteps = nsteps;
    const int ppt = h->n <= 1024 ? 1 : (h->n <= 2048 ? 2 : 4);
    const int nt = (int)((h->n + ppt - 1) / ppt);
    const bool full = h->n % ppt == 0;
#define PX_L1(PP)                                                                   \
  do {                                                                              \
    if (full) {                                                                     \
      if (adjoint) px::k_rk4_lane1d<PP, true, true><<<h->L, nt, 0, s>>>(a);         \
      else px::k_rk4_lane1d<PP, false, true><<<h->L, nt, 0, s>>>(a);                \
    } else {                                                                        \
      if (adjoint) px::k_rk4_lane1d<PP, true><<<h->L, nt, 0, s>>>(a);               \
      else px::k_rk4_lane1d<PP, false><<<h->L, nt, 0, s>>>(a);                      \
    }                                                                               \
  } while (0)
    if (ppt == 1) PX_L1(1);
    else if (ppt == 2) PX_L1(2);
    else PX_L1(4);
#undef PX_L1
    PX_CHECK_LAUNCH(h);
    cur = h->Y0;
    launched_steps = nsteps;
    h->z_valid = adjoint;
  } else if (nsteps == 1) {
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
    {
      const double ks[4] = {0.25 * hs, hs / 3.0, 0.5 * hs, hs};
      const double cf[5] = {st.cc, st.ce, st.cw, st.cs, st.cn};
      for (int j = 0; j < 4; ++j)
        for (int q = 0; q < 5; ++q) a.kc[j][q] = ks[j] * cf[q];
    }
    // two RK4 steps per launch for large sweeps (PX_MARCH2=0 forces the one-step kernel); small
    // sweeps keep one step per launch: the 8-stage pipeline fill (16 rows per band) and the
    // 1-CTA-per-3-warps occupancy only pay off when each launch covers ≥ 2^28 lane-points
    static const int m2_mode = [] { const char* e = getenv("PX_MARCH2"); return e ? atoi(e) : 1; }();
    if (m2_mode && nsteps >= 3 && (m2_mode == 2 || (double)h->L * (double)h->n >= 268435456.0)) {
      // two steps per launch: halo 8 (one column per stage and side)
      static const int m2_var = [] { const char* e = getenv("PX_M2_VAR"); return e ? atoi(e) : 3; }();
      static const int m2_cols = [] { const char* e = getenv("PX_M2_COLS"); return e ? atoi(e) : 3; }();
      const int m2_nt = m2_var == 2 ? 192 : 128;
      const int cw_max = 2 * m2_nt;
      // NC columns per thread (k_rk4_marchc): direct lanes, strip mode
      const int mc_nc = (!zlanes && m2_cols >= 3) ? m2_cols : 0;
      static const int mc_var = [] { const char* e = getenv("PX_MC_VAR"); return e ? atoi(e) : 6; }();
      const int mc_nt = mc_var >= 3 ? 64 : (mc_nc == 4 ? 96 : 128);
      if (mc_nc && nx > mc_nc * mc_nt) {
        a.halo = 8;
        const int maxu = mc_nc * mc_nt - 16;
        const int ns = (nx + maxu - 1) / maxu;
        a.strip_w = (((nx + ns - 1) / ns) + 1) & ~1;
        a.nstrips = (nx + a.strip_w - 1) / a.strip_w;
      } else if (nx <= cw_max) {
        a.strip_w = nx; a.halo = 0; a.nstrips = 1;
      } else {
        a.halo = 8; a.strip_w = cw_max - 16;
        a.nstrips = (nx + a.strip_w - 1) / a.strip_w;
      }
      static const int m2_band_env = [] { const char* e = getenv("PX_M2_BAND"); return e ? atoi(e) : 0; }();
      const int m2_band = m2_band_env ? m2_band_env : (mc_nc ? 1024 : 512);
      // bands of rows (16 rows of pipeline fill each): ≥ 4 waves at 2 CTAs/SM, ≥ 128 rows per band
      int br = std::min(ny, m2_band);
      while (br > 128 && (size_t)h->L * a.nstrips * ((ny + br - 1) / br) < 4 * 3 * 148) br = (br + 1) / 2;
      a.band_rows = br;
      a.nbands = (ny + a.band_rows - 1) / a.band_rows;
      const unsigned blocks = (unsigned)((size_t)h->L * a.nstrips * a.nbands);
      auto launch2 = [&](bool one_step) -> int {
#define PX_M2(NT, DEP, MB, TM, ...)                                                                            \
  do {                                                                                                     \
    const size_t sm = px::march2_smem<NT, DEP>(zlanes);                                                   \
    if (zlanes) PX_TRY(smem_attr(h, (const void*)px::k_rk4_march2<true, NT, DEP, MB, TM, ##__VA_ARGS__>, sm));  \
    else PX_TRY(smem_attr(h, (const void*)px::k_rk4_march2<false, NT, DEP, MB, TM, ##__VA_ARGS__>, sm));        \
    if (zlanes) px::k_rk4_march2<true, NT, DEP, MB, TM, ##__VA_ARGS__><<<blocks, NT, sm, s>>>(a);                        \
    else px::k_rk4_march2<false, NT, DEP, MB, TM, ##__VA_ARGS__><<<blocks, NT, sm, s>>>(a);                               \
  } while (0)
#define PX_MC(NC, NT, DEP, MB, BR, PF, ...)                                                                   \
  do {                                                                                                     \
    const size_t sm = px::marchc_smem<NC, NT, DEP>(BR);                                                   \
    PX_TRY(smem_attr(h, (const void*)px::k_rk4_marchc<NC, NT, DEP, MB, BR, PF, ##__VA_ARGS__>, sm));      \
    px::k_rk4_marchc<NC, NT, DEP, MB, BR, PF, ##__VA_ARGS__><<<blocks, NT, sm, s>>>(a);                   \
  } while (0)
        if (a.halo > 0 && mc_nc == 3) {
          // default (6): 4 CTAs of 2 warps per SM, b(r−8) from a register ring (two TMA
          // streams), slots refilled after the barrier without a proxy fence (write-after-read
          // only: the generic-proxy reads of the slot are complete at the barrier)
          if (mc_var == 6) {
            if (one_step) PX_MC(3, 64, 3, 4, false, false, false);  // odd remainder step
            else PX_MC(3, 64, 3, 4, true, false);
          } else if (mc_var == 3) PX_MC(3, 64, 3, 4, false, true);  // three streams, proxy fence
          else PX_MC(3, 128, 3, 2, false, true);
          return PX_OK;
        }
        if (a.halo > 0 && mc_nc == 4) {
          if (mc_var >= 3) PX_MC(4, 64, 3, 4, false, true);
          else PX_MC(4, 96, 3, 2, false, true);
          return PX_OK;
        }
#undef PX_MC
        static const int m2_tma = [] { const char* e = getenv("PX_M2_TMA"); return e ? atoi(e) : 1; }();
        if (m2_var == 2) PX_M2(192, 3, 2, false);  // 2 CTAs/SM
        else if (m2_tma == 1) PX_M2(128, 3, 3, true, true);  // 3 CTAs/SM, TMA row ring, h·w3 in registers (default)
        else if (m2_tma) PX_M2(128, 3, 3, true);             // TMA row ring, h·w3 rows in smem
        else PX_M2(128, 3, 3, false);              // 3 CTAs/SM, per-thread cp.async ring
#undef PX_M2
        return PX_OK;
      };
      int st_i = 1;
      while (st_i < nsteps) {
        double* out = (cur == h->Y0) ? h->Y1 : h->Y0;
        a.y_in = cur;
        a.y_out = out;
        a.z_zero = (st_i == 1);
        if (nsteps - st_i >= 2) {
          PX_TRY(launch2(false));
          st_i += 2;
        } else if (a.halo > 0 && mc_nc == 3 && mc_var == 6) {
          PX_TRY(launch2(true));  // the three-column kernel, one step
          st_i += 1;
        } else {
          px::MarchArgs b1 = a;  // odd remainder: one single-step launch
          if (nx <= px::MARCH_MAX_CW) {
            b1.strip_w = nx; b1.halo = 0; b1.nstrips = 1;
          } else {
            b1.strip_w = px::MARCH_STRIP; b1.halo = px::MARCH_HALO;
            b1.nstrips = (nx + px::MARCH_STRIP - 1) / px::MARCH_STRIP;
          }
          b1.band_rows = std::min(ny, 256);
          b1.nbands = (ny + b1.band_rows - 1) / b1.band_rows;
          const unsigned blk1 = (unsigned)((size_t)h->L * b1.nstrips * b1.nbands);
          const size_t sm1 = px::march_smem(zlanes);
          PX_TRY(smem_attr(h, (const void*)px::k_rk4_march<true>, px::march_smem(true)));
          PX_TRY(smem_attr(h, (const void*)px::k_rk4_march<false>, px::march_smem(false)));
          if (zlanes) px::k_rk4_march<true><<<blk1, px::MARCH_NT, sm1, s>>>(b1);
          else px::k_rk4_march<false><<<blk1, px::MARCH_NT, sm1, s>>>(b1);
          st_i += 1;
        }
        PX_CHECK_LAUNCH(h);
        cur = out;
      }
      launched_steps = nsteps - 1;
      h->z_valid = zlanes;
    } else {
    if (nx <= px::MARCH_MAX_CW) {
      a.strip_w = nx; a.halo = 0; a.nstrips = 1;
    } else {
      a.strip_w = px::MARCH_STRIP; a.halo = px::MARCH_HALO;
      a.nstrips = (nx + px::MARCH_STRIP - 1) / px::MARCH_STRIP;
    }
    // bands of rows: enough CTAs for ≥ 4 waves at 2 CTAs/SM, ≥ 32 rows per band
    int br = ny;
    while (br > 32 && (size_t)h->L * a.nstrips * ((ny + br - 1) / br) < 4 * 2 * 148) br = (br + 1) / 2;
    if (ny >= 1024 && br > 256) br = 256;
    a.band_rows = br;
    a.nbands = (ny + br - 1) / br;
    const unsigned blocks = (unsigned)((size_t)h->L * a.nstrips * a.nbands);
    const size_t smem = px::march_smem(zlanes);
    if (zlanes) PX_TRY(smem_attr(h, (const void*)px::k_rk4_march<true>, smem));
    else PX_TRY(smem_attr(h, (const void*)px::k_rk4_march<false>, smem));
    for (int st_i = 1; st_i < nsteps; ++st_i) {
      double* out = (cur == h->Y0) ? h->Y1 : h->Y0;
      a.y_in = cur;
      a.y_out = out;
      a.z_zero = (st_i == 1);
      if (zlanes) px::k_rk4_march<true><<<blocks, px::MARCH_NT, smem, s>>>(a);
      else px::k_rk4_march<false><<<blocks, px::MARCH_NT, smem, s>>>(a);
      PX_CHECK_LAUNCH(h);
      cur = out;
    }
    launched_steps = nsteps - 1;
    h->z_valid = zlanes;
    }
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

// ---------------------------------------------------------------------------
// Chebyshev action over B vectors (batch-strided input)
// ---------------------------------------------------------------------------


// 2D: Chebyshev action by row-marching passes of up to CM_MAXT fused terms (cheb_march.cuh)
template <int M, int SG, bool TM>
int launch_cm_v(Handle* h, const px::ChebMarchArgs& a, unsigned blocks, cudaStream_t s) {
  PX_TRY(smem_attr(h, (const void*)px::k_cheb_march<M, SG, TM>, px::CM_SMEM));
  px::k_cheb_march<M, SG, TM><<<blocks, px::CM_NT, px::CM_SMEM, s>>>(a);
  PX_CHECK_LAUNCH(h);
  return PX_OK;
}
// σ = ±1 as a template constant; PX_CM_VAR: 1 per-thread cp.async ring (default), 0 TMA row
// ring (measured 15% slower here: one-thread issue after the row barrier, short bands)
template <int M>
int launch_cm(Handle* h, const px::ChebMarchArgs& a, unsigned blocks, cudaStream_t s) {
  static const int var = [] { const char* e = getenv("PX_CM_VAR"); return e ? atoi(e) : 1; }();
  const bool neg = a.sigma < 0;
  if (var == 0) return neg ? launch_cm_v<M, -1, true>(h, a, blocks, s) : launch_cm_v<M, 1, true>(h, a, blocks, s);
  return neg ? launch_cm_v<M, -1, false>(h, a, blocks, s) : launch_cm_v<M, 1, false>(h, a, blocks, s);
}

int cheb_action_march(Handle* h, const Plan& pl, const px::Stencil5& st, const double* src, long long src_bs,
                      const double* addend, long long add_bs, double* pacc, double** result, cudaStream_t s) {
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
  static const int cm_terms = [] {  // fused terms per pass (≤ CM_MAXT)
    const char* e = getenv("PX_CM_TERMS");
    const int v = e ? atoi(e) : 6;
    return std::max(1, std::min(px::CM_MAXT, v));
  }();
  static int env_strip = -1, env_band = -1;
  if (env_strip < 0) {
    const char* e1 = getenv("PX_CM_STRIP");
    const char* e2 = getenv("PX_CM_BAND");
    env_strip = e1 ? atoi(e1) : 0;
    env_band = e2 ? atoi(e2) : 0;
  }
  if (nx <= 2 * px::CM_NT && env_strip == 0) {
    a.strip_w = nx; a.halo = 0; a.nstrips = 1;
  } else {
    a.halo = (cm_terms + 1) & ~1;  // ≥ the terms of any pass; even (16-byte aligned row segments)
    if (env_strip > 0) {
      a.strip_w = env_strip;
    } else {  // fewest strips of ≤ 2·CM_NT computed columns, useful widths balanced (even)
      const int maxw = 2 * px::CM_NT - 2 * a.halo;
      const int ns = (nx + maxw - 1) / maxw;
      a.strip_w = ((nx + ns - 1) / ns + 1) & ~1;
    }
    a.nstrips = (nx + a.strip_w - 1) / a.strip_w;
  }
  int br;
  if (env_band > 0) {
    br = env_band;
  } else {
    // about one full wave of 2 CTAs per SM, bands of ≥ 32 rows
    const size_t per_band_ctas = (size_t)a.nstrips * B;
    const size_t target = (size_t)px::CM_MINB * 148;
    size_t nb_bands = std::max<size_t>(1, target / per_band_ctas);
    br = (int)((ny + nb_bands - 1) / nb_bands);
    if (br < 32) br = std::min(32, ny);
  }
  a.band_rows = br;
  a.nbands = (ny + br - 1) / br;
  const unsigned blocks = (unsigned)((size_t)B * a.nstrips * a.nbands);
  const int K = pl.degree;
  int wsel = 0;  // rotating pair of U output buffers
  for (int sub = 0; sub < pl.substeps; ++sub) {
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
      for (int j = 0; j <= px::CM_MAXT; ++j) {
        const int term = k + j;
        a.be[j] = (j <= M && term <= K && (j > 0 || first)) ? pl.be[term] : 0.0;
        a.bp[j] = (pacc && j <= M && term <= K && (j > 0 || first)) ? pl.bp[term] : 0.0;
      }
      int rc;
      switch (M) {
        case 1: rc = launch_cm<1>(h, a, blocks, s); break;
        case 2: rc = launch_cm<2>(h, a, blocks, s); break;
        case 3: rc = launch_cm<3>(h, a, blocks, s); break;
        case 4: rc = launch_cm<4>(h, a, blocks, s); break;
        case 5: rc = launch_cm<5>(h, a, blocks, s); break;
        default: rc = launch_cm<6>(h, a, blocks, s); break;
      }
      if (rc != PX_OK) return rc;
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

// result <- exp(span·M)·src (+ addend);  pacc += span·φ₁(span·M)·src  (if pacc)
int cheb_action(Handle* h, const Plan& pl, const px::Stencil5& st, const double* src, long long src_bs,
                const double* addend, long long add_bs, double* pacc, double** result, cudaStream_t s) {
  if (!pl.set || pl.krylov) return fail(h, PX_ERR_STATE, "Chebyshev plan not set");
  const size_t n = h->n;
  const int B = h->B;
  const dim3 grid = grid1(n, B);
  const long long nb = (long long)n;
  if (h->dim == 2 && (h->d.nx % 2) == 0) return cheb_action_march(h, pl, st, src, src_bs, addend, add_bs, pacc, result, s);
  for (int sub = 0; sub < pl.substeps; ++sub) {
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
    fa.p0 = pacc ? pl.bp[0] : 0.0; fa.p1 = pacc ? pl.bp[1] : 0.0;
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
      ta.bk = pl.be[k]; ta.pk = pacc ? pl.bp[k] : 0.0;
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
  const double bpp = pacc ? 56.0 : 40.0;
  const double bytes = bpp * (double)n * terms;
  h->stats.exp_bytes += bytes;
  h->stats.algorithmic_bytes += bytes;
  *result = const_cast<double*>(src);
  return PX_OK;
}

int exp_action(Handle* h, int slot, const px::Stencil5& st, const double* src, long long src_bs,
               const double* addend, long long add_bs, double* pacc, double** result, cudaStream_t s) {
  const Plan& pl = h->plans[slot];
  if (!pl.set) return fail(h, PX_ERR_STATE, "exp-action plan slot " + std::to_string(slot) + " not set");
  if (pl.krylov) {
    static int coop = -1;
    if (coop < 0) {
      const char* e = getenv("PX_KRYLOV_COOP");
      int dev = 0, ok = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&ok, cudaDevAttrCooperativeLaunch, dev);
      // opt-in: on B200 the grid-wide barriers (3 per Arnoldi step) cost more than the
      // launches they replace at config-4 size (measured 2.25 vs 3.13 gradient evals/s)
      coop = (ok && e && atoi(e) == 1) ? 1 : 0;
    }
    if (coop)
      PX_TRY(px::krylov_action_coop(h->kw, pl.span / pl.substeps, pl.substeps, h->d.krylov_m, st, src, src_bs,
                                    addend, add_bs, pacc, h->ACC, h->B, h->d.nx, h->d.ny, h->dim, result, s,
                                    &h->stats));
    else
      PX_TRY(px::krylov_action(h->kw, pl.span / pl.substeps, pl.substeps, h->d.krylov_m, st, src, src_bs,
                               addend, add_bs, pacc, h->ACC, h->B, h->d.nx, h->d.ny, h->dim, result, s,
                               &h->stats));
    if (cudaGetLastError() != cudaSuccess) return fail(h, PX_ERR_CUDA, "krylov launch failed");
    return PX_OK;
  }
  return cheb_action(h, pl, st, src, src_bs, addend, add_bs, pacc, result, s);
}

int project(Handle* h, double* grad, const double* F, long long Fbs, double alpha, double beta,
            cudaStream_t s) {
  const int rx = h->rows_x;
  if (rx <= 8)
    px::k_project_rows<8><<<dim3(h->d.ny, h->B), 256, 0, s>>>(h->R, F, Fbs, h->tx, rx, h->d.nx, h->d.ny);
  else if (rx <= 16)
    px::k_project_rows<16><<<dim3(h->d.ny, h->B), 256, 0, s>>>(h->R, F, Fbs, h->tx, rx, h->d.nx, h->d.ny);
  else if (rx <= 32)
    px::k_project_rows<32><<<dim3(h->d.ny, h->B), 256, 0, s>>>(h->R, F, Fbs, h->tx, rx, h->d.nx, h->d.ny);
  else
    px::k_project_rows<64><<<dim3(h->d.ny, h->B), 256, 0, s>>>(h->R, F, Fbs, h->tx, rx, h->d.nx, h->d.ny);
  PX_CHECK_LAUNCH(h);
  px::k_project_cols<<<dim3(h->K, h->B), 256, 0, s>>>(grad, h->R, h->ty, h->ix, h->iy, rx, h->K,
                                                      h->d.ny, alpha, beta);
  PX_CHECK_LAUNCH(h);
  return PX_OK;
}

int apply_plus_control(Handle* h, double* out, const double* x, long long xbs, const px::Stencil5& st,
                       bool with_control, cudaStream_t s) {
  const dim3 grid = grid1(h->n, h->B);
  if (h->dim == 2)
    px::k_apply_plus_control<2><<<grid, 256, 0, s>>>(out, x, xbs, st, with_control ? h->ctrl : nullptr,
                                                     h->tx, h->ty, h->ix, h->iy, h->K, h->d.nx, h->d.ny);
  else
    px::k_apply_plus_control<1><<<grid, 256, 0, s>>>(out, x, xbs, st, with_control ? h->ctrl : nullptr,
                                                     h->tx, h->ty, h->ix, h->iy, h->K, h->d.nx, h->d.ny);
  PX_CHECK_LAUNCH(h);
  return PX_OK;
}

// ---------------------------------------------------------------------------
// Linear sweeps
// ---------------------------------------------------------------------------

// 1D linear sweeps: the whole carry recursion in one CTA per member (scan1d.cuh)
bool use_scan1d(const Handle* h) {
  const Plan& sl = h->plans[PX_PLAN_SLICE];
  return h->dim == 1 && h->n <= 4096 && (!sl.set || !sl.krylov) &&
         !(h->d.flags & PX_FLAG_BOUNDARY_STATES);
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

int scan1d(Handle* h, bool adjoint, const double* lanes, double* out, double* pacc, int long_slot,
           cudaStream_t s) {
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
  // cluster version (8 CTAs = 8 SMs per member, DSMEM ghost-zone refresh every G terms)
  // for the larger 1D grids; one CTA per member otherwise
  static const int s1c = [] { const char* e = getenv("PX_SCAN1D_CLUSTER"); return e ? atoi(e) : 1; }();
  constexpr int kCS = 8, kPPT = 4;
  // ghost width G: the cluster refreshes its DSMEM ghost zones every G terms (a cluster barrier
  // costs ≈ 4× a CTA barrier) and recomputes G points per side; 64 measured best (config 2:
  // 8 → 16 → 32 → 64 gave 1814 → 2056 → 2204 → 2300 gradient evals/s)
  static const int kGv = [] {
    const char* e = getenv("PX_SCAN1D_G");
    const int v = e ? atoi(e) : 64;
    return v == 32 ? 32 : (v == 16 ? 16 : (v == 8 ? 8 : 64));
  }();
  const int Wc = (int)(h->n / kCS);
  if (s1c && h->n >= 2048 && h->n % (kCS * kPPT) == 0 && Wc >= kGv && Wc / kPPT + 2 * (kGv / kPPT) <= 256) {
    const int nr = Wc / kPPT + 2 * (kGv / kPPT);
    cudaLaunchConfig_t cfg = {};
    static const int kmb = [] { const char* e = getenv("PX_SCAN1D_MB"); return e ? atoi(e) : 2; }();
    const int mb = kmb >= 4 ? 4 : (kmb >= 2 ? 2 : 1);
    cfg.gridDim = dim3((unsigned)(((h->B + mb - 1) / mb) * kCS));
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
    const int Bm = h->B;
    if (kGv == 64) {
      if (mb == 4) PX_CUDA(h, cudaLaunchKernelEx(&cfg, px::k_scan1d_cluster<kPPT, kCS, 64, 4>, a, Bm));
      else if (mb == 2) PX_CUDA(h, cudaLaunchKernelEx(&cfg, px::k_scan1d_cluster<kPPT, kCS, 64, 2>, a, Bm));
      else PX_CUDA(h, cudaLaunchKernelEx(&cfg, px::k_scan1d_cluster<kPPT, kCS, 64, 1>, a, Bm));
    } else if (kGv == 32) {
      if (mb == 4) PX_CUDA(h, cudaLaunchKernelEx(&cfg, px::k_scan1d_cluster<kPPT, kCS, 32, 4>, a, Bm));
      else if (mb == 2) PX_CUDA(h, cudaLaunchKernelEx(&cfg, px::k_scan1d_cluster<kPPT, kCS, 32, 2>, a, Bm));
      else PX_CUDA(h, cudaLaunchKernelEx(&cfg, px::k_scan1d_cluster<kPPT, kCS, 32, 1>, a, Bm));
    } else if (kGv == 16) {  // ghost zones refreshed every 16 terms (half the cluster barriers)
      if (mb == 4) PX_CUDA(h, cudaLaunchKernelEx(&cfg, px::k_scan1d_cluster<kPPT, kCS, 16, 4>, a, Bm));
      else if (mb == 2) PX_CUDA(h, cudaLaunchKernelEx(&cfg, px::k_scan1d_cluster<kPPT, kCS, 16, 2>, a, Bm));
      else PX_CUDA(h, cudaLaunchKernelEx(&cfg, px::k_scan1d_cluster<kPPT, kCS, 16, 1>, a, Bm));
    } else {
      if (mb == 4) PX_CUDA(h, cudaLaunchKernelEx(&cfg, px::k_scan1d_cluster<kPPT, kCS, 8, 4>, a, Bm));
      else if (mb == 2) PX_CUDA(h, cudaLaunchKernelEx(&cfg, px::k_scan1d_cluster<kPPT, kCS, 8, 2>, a, Bm));
      else PX_CUDA(h, cudaLaunchKernelEx(&cfg, px::k_scan1d_cluster<kPPT, kCS, 8, 1>, a, Bm));
    }
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

void free_blocks(Handle* h) {
  for (auto& b : h->blocks) {
    for (double* p : b.Wk) cudaFree(p);
    for (double* p : b.ACC) cudaFree(p);
    cudaFree(b.D);
    cudaFree(b.Gp);
    px::krylov_free(b.kw);
    if (b.st) cudaStreamDestroy(b.st);
    if (b.ev) cudaEventDestroy(b.ev);
  }
  h->blocks.clear();
  h->lb = 1;
}

bool use_blocks(const Handle* h) {
  return h->lb > 1 && h->dim == 2 && !(h->d.flags & PX_FLAG_BOUNDARY_STATES);
}

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
    const double* C = wend + (size_t)(b.q1 - 1) * h->n;
    long long C_bs = lane_bs;
    for (int q = b.q1 - 2; q >= b.q0; --q) {
      double* res = nullptr;
      PX_TRY(exp_action(h, PX_PLAN_SLICE, h->AT, C, C_bs, wend + (size_t)q * h->n, lane_bs, b.Gp, &res, b.st));
      C = res;
      C_bs = nb;
    }
    if (g > 0) {
      double* res = nullptr;
      PX_TRY(exp_action(h, PX_PLAN_BLOCK_LONG + g - 1, h->AT, C, C_bs, nullptr, 0, b.Gp, &res, b.st));
      C = res;
      C_bs = nb;
    }
    PX_TRY(axpby(h, b.D, nb, C, C_bs, 1.0, nullptr, 0, 0.0, b.st));
    PX_CUDA(h, cudaEventRecord(b.ev, b.st));
  }
  for (int g = 0; g < h->lb; ++g) {
    PX_CUDA(h, cudaStreamWaitEvent(s, h->blocks[g].ev, 0));
    PX_TRY(axpby(h, out, nb, h->blocks[g].D, nb, 1.0, g == 0 ? nullptr : out, nb, g == 0 ? 0.0 : 1.0, s));
    PX_TRY(axpby(h, gacc, nb, gacc, nb, 1.0, h->blocks[g].Gp, nb, 1.0, s));
  }
  return PX_OK;
}

int direct_linear(Handle* h, cudaStream_t s) {
  const long long nb = (long long)h->n;
  const long long lane_bs = (long long)h->Pl * nb;  // stride between batch members in lanes
  // g = A·u0 + f  (u0 shared by all members)
  PX_TRY(apply_plus_control(h, h->g, h->u0, 0, h->A, true, s));
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
  const bool bnd = (h->d.flags & PX_FLAG_BOUNDARY_STATES) && h->UBND;
  const long long ubs = (long long)(h->d.P + 1) * nb;
  if (bnd) {
    PX_TRY(axpby(h, h->UBND, ubs, h->u0, 0, 1.0, nullptr, 0, 0.0, s));
  }
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
  return PX_OK;
}

// G partial <- Σ_p z_p without per-lane accumulators (circulant 2D operator):
// Σ_p z_p = (Aᵀ)⁻¹₀(Σ_p w_n,p − Pl·n·b) + Pl·n·c + Pl·h·b̄·n(n−1)/2, the pseudo-inverse on the
// non-constant Fourier modes by one batched Z2Z FFT solve (kernels.cuh, k_circ_solve).
int z_closed_form(Handle* h, const double* wend, cudaStream_t s) {
  const double hs = (h->d.T / h->d.P) / h->d.nsteps;
  const double ns = (double)h->d.nsteps;
  const dim3 gs = grid_stride(h->n, h->B);
  px::k_zsrc_cplx<<<gs, 256, 0, s>>>(h->fbuf, wend, h->Pl, h->bsrc, (double)h->Pl * ns, h->n);
  PX_CHECK_LAUNCH(h);
  px::k_sum_partial<<<dim3(h->red_blocks, h->B), 256, 0, s>>>(h->partial, h->bsrc, h->n);
  PX_CHECK_LAUNCH(h);
  px::k_finalize_sum<<<h->B, 256, 0, s>>>(h->bsum, h->partial, h->red_blocks, 1.0, nullptr);
  PX_CHECK_LAUNCH(h);
  if (cufftSetStream(h->fft, s) != CUFFT_SUCCESS ||
      cufftExecZ2Z(h->fft, reinterpret_cast<cufftDoubleComplex*>(h->fbuf),
                   reinterpret_cast<cufftDoubleComplex*>(h->fbuf), CUFFT_FORWARD) != CUFFT_SUCCESS)
    return fail(h, PX_ERR_CUDA, "cufft forward failed");
  px::k_circ_solve<<<(unsigned)std::min<size_t>((h->n * h->B + 255) / 256, 148 * 16), 256, 0, s>>>(
      h->fbuf, h->AT, h->d.nx, h->d.ny, h->B);
  PX_CHECK_LAUNCH(h);
  if (cufftExecZ2Z(h->fft, reinterpret_cast<cufftDoubleComplex*>(h->fbuf),
                   reinterpret_cast<cufftDoubleComplex*>(h->fbuf), CUFFT_INVERSE) != CUFFT_SUCCESS)
    return fail(h, PX_ERR_CUDA, "cufft inverse failed");
  const double kconst = (double)h->Pl * hs * ns * (ns - 1.0) / 2.0 / (double)h->n;
  px::k_z_finish<<<gs, 256, 0, s>>>(h->G, h->fbuf, h->cz, (double)h->Pl * ns, h->bsum, kconst, h->n);
  PX_CHECK_LAUNCH(h);
  h->stats.kernel_launches += 2;  // the two cuFFT executions
  return PX_OK;
}

int adjoint_linear(Handle* h, cudaStream_t s) {
  const long long nb = (long long)h->n;
  const long long lane_bs = (long long)h->Pl * nb;
  const double* wend = nullptr;
  int tm = tbegin(h, PX_PHASE_RK4_ADJOINT, s);
  PX_TRY(rk4_sweep(h, true, &wend, s));
  tend(h, tm, s);
  h->wend = wend;
  tm = tbegin(h, PX_PHASE_EXP_ADJOINT, s);
  // G partial <- Σ_p z_p  (z_p = Σ_steps h·w3 + nsteps·c)
  if (h->z_closed) {
    PX_TRY(z_closed_form(h, wend, s));
  } else {
    px::k_lane_sum_plus<<<grid_stride(h->n, h->B), 256, 0, s>>>(h->G, h->Z, h->Pl, h->cz,
                                                                (double)h->Pl * h->d.nsteps, h->n,
                                                                h->z_valid ? 1 : 0);
    PX_CHECK_LAUNCH(h);
  }
  if (use_scan1d(h)) {
    PX_TRY(scan1d(h, true, wend, h->QDAG0, h->G, h->d.p_begin > 0 ? PX_PLAN_LONG_ADJOINT : -1, s));
    tend(h, tm, s);
    tm = tbegin(h, PX_PHASE_OTHER, s);
    PX_TRY(project(h, h->GRAD, h->G, nb, 1.0, 0.0, s));
    tend(h, tm, s);
    return PX_OK;
  }
  if (use_blocks(h)) {
    PX_TRY(adjoint_blocks(h, wend, h->QDAG0, h->G, s));
    if (h->d.p_begin > 0) {
      double* res = nullptr;
      PX_TRY(exp_action(h, PX_PLAN_LONG_ADJOINT, h->AT, h->QDAG0, nb, nullptr, 0, h->G, &res, s));
      PX_TRY(axpby(h, h->QDAG0, nb, res, nb, 1.0, nullptr, 0, 0.0, s));
    }
    tend(h, tm, s);
    tm = tbegin(h, PX_PHASE_OTHER, s);
    PX_TRY(project(h, h->GRAD, h->G, nb, 1.0, 0.0, s));
    tend(h, tm, s);
    return PX_OK;
  }
  const double* C = wend + (size_t)(h->Pl - 1) * h->n;
  long long C_bs = lane_bs;
  for (int q = h->Pl - 2; q >= 0; --q) {
    double* res = nullptr;
    PX_TRY(exp_action(h, PX_PLAN_SLICE, h->AT, C, C_bs, wend + (size_t)q * h->n, lane_bs, h->G, &res, s));
    C = res;
    C_bs = nb;
  }
  if (h->d.p_begin > 0) {
    double* res = nullptr;
    PX_TRY(exp_action(h, PX_PLAN_LONG_ADJOINT, h->AT, C, C_bs, nullptr, 0, h->G, &res, s));
    C = res;
    C_bs = nb;
  }
  PX_TRY(axpby(h, h->QDAG0, nb, C, C_bs, 1.0, nullptr, 0, 0.0, s));
  tend(h, tm, s);
  tm = tbegin(h, PX_PHASE_OTHER, s);
  PX_TRY(project(h, h->GRAD, h->G, nb, 1.0, 0.0, s));
  tend(h, tm, s);
  return PX_OK;
}

int finish_direct_impl(Handle* h, cudaStream_t s) {
  const long long nb = (long long)h->n;
  const int tm = tbegin(h, PX_PHASE_OTHER, s);
  if (h->d.kind == PX_KIND_ADVDIFF) {
    // u(T) = u0 + Σ carries
    PX_TRY(axpby(h, h->UT, nb, h->UT, nb, 1.0, h->u0, 0, 1.0, s));
  }
  PX_TRY(axpby(h, h->QT, nb, h->UT, nb, 1.0, h->ut, 0, -1.0, s));
  px::k_sumsq_partial<<<dim3(h->red_blocks, h->B), 256, 0, s>>>(h->partial, h->QT, h->n);
  PX_CHECK_LAUNCH(h);
  px::k_finalize_sum<<<h->B, 256, 0, s>>>(h->J, h->partial, h->red_blocks, 0.5, h->nonfinite);
  PX_CHECK_LAUNCH(h);
  if (h->d.kind == PX_KIND_ADVDIFF) PX_TRY(apply_plus_control(h, h->gadj, h->QT, nb, h->AT, false, s));
  tend(h, tm, s);
  return PX_OK;
}

int finish_adjoint_impl(Handle* h, cudaStream_t s) {
  const long long nb = (long long)h->n;
  if (h->adjoint_mode == PX_ADJOINT_FROZEN_SPAN) return PX_OK;  // q†_T is not absorbed: nothing to add
  const int tm = tbegin(h, PX_PHASE_OTHER, s);
  // absorbed final condition: q† = q†_T + the solved part (paraexp.py:268-270)
  PX_TRY(axpby(h, h->QDAG0, nb, h->QDAG0, nb, 1.0, h->QT, nb, 1.0, s));
  PX_TRY(axpby(h, h->G, nb, h->G, nb, 1.0, h->QT, nb, h->d.T, s));
  PX_TRY(project(h, h->GRAD, h->QT, nb, h->d.T, 1.0, s));
  tend(h, tm, s);
  return PX_OK;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================

extern "C" {

int px_abi_version(void) { return PX_ABI_VERSION; }

const char* px_build_info(void) {
  return "paraexp sm_100a fp64 (row-marching Horner RK4, on-chip 1D lanes, Chebyshev fused recurrence, "
         "Arnoldi CGS2, Burgers serial sweep)";
}

const char* px_last_error(const void* handle) {
  const Handle* h = static_cast<const Handle*>(handle);
  if (h && !h->err.empty()) return h->err.c_str();
  return g_last_error.c_str();
}

int px_create(const px_problem_desc* desc, void** out_handle) {
  if (!desc || !out_handle) return fail(nullptr, PX_ERR_ARG, "null argument");
  const px_problem_desc& d = *desc;
  if (d.nx < 3 || d.ny < 1 || (d.ny > 1 && d.ny < 3)) return fail(nullptr, PX_ERR_ARG, "bad grid");
  if (d.P < 1 || d.nsteps < 1 || d.batch < 1 || d.K < 1) return fail(nullptr, PX_ERR_ARG, "bad sizes");
  if (d.p_begin < 0 || d.p_end > d.P || d.p_begin >= d.p_end)
    return fail(nullptr, PX_ERR_ARG, "bad slice block");
  if (!(d.T > 0)) return fail(nullptr, PX_ERR_ARG, "T must be positive");
  if (d.kind != PX_KIND_ADVDIFF && d.kind != PX_KIND_BURGERS) return fail(nullptr, PX_ERR_ARG, "bad kind");
  if (d.kind == PX_KIND_BURGERS && d.ny != 1) return fail(nullptr, PX_ERR_ARG, "Burgers path is 1D");
  if (d.expaction == PX_EXP_KRYLOV && (d.krylov_m < 2 || d.krylov_m > px::KRYLOV_MAX_M))
    return fail(nullptr, PX_ERR_ARG, "krylov_m out of range");
  if (d.basis_rows_x < 1 || d.basis_rows_x > 64 || d.basis_rows_y < 1)
    return fail(nullptr, PX_ERR_ARG, "bad basis table sizes");
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
  auto A = [&](double** p, size_t cnt) { if (rc == PX_OK) rc = dalloc_t(h, p, cnt); };
  A(&h->u0, n);
  A(&h->ut, n);
  A(&h->ctrl, B * h->K);
  A(&h->tx, (size_t)h->rows_x * d.nx);
  A(&h->ty, (size_t)h->rows_y * d.ny);
  if (rc == PX_OK) rc = dalloc_t(h, &h->ix, h->K);
  if (rc == PX_OK) rc = dalloc_t(h, &h->iy, h->K);
  A(&h->UT, B * n);
  A(&h->QT, B * n);
  A(&h->QDAG0, B * n);
  A(&h->G, B * n);
  A(&h->J, B);
  A(&h->GRAD, B * h->K);
  A(&h->R, B * h->rows_x * d.ny);
  h->red_blocks = (int)std::min<size_t>((n + 255) / 256, 1024);
  A(&h->partial, B * h->red_blocks);
  if (rc == PX_OK) rc = dalloc_t(h, &h->nonfinite, 1);
  for (int i = 0; i < 4; ++i) A(&h->Wk[i], B * n);
  for (int i = 0; i < 2; ++i) A(&h->ACC[i], B * n);
  if (d.kind == PX_KIND_ADVDIFF) {
    A(&h->g, B * n);
    A(&h->gadj, B * n);
    A(&h->bsrc, B * n);
    A(&h->cz, B * n);
    A(&h->Y0, (size_t)h->L * n);
    A(&h->Y1, (size_t)h->L * n);
    // 2D: the adjoint ∫ in closed form (one FFT solve), no per-lane accumulator in HBM
    static const bool z_accum = [] { const char* e = getenv("PX_Z_ACCUM"); return e && atoi(e) != 0; }();
    h->z_closed = h->dim == 2 && !z_accum;
    if (h->z_closed) {
      A(reinterpret_cast<double**>(&h->fbuf), 2 * B * n);
      A(&h->bsum, B);
      int dims[2] = {d.ny, d.nx};
      if (rc == PX_OK && cufftPlanMany(&h->fft, 2, dims, nullptr, 1, 0, nullptr, 1, 0, CUFFT_Z2Z, (int)B) != CUFFT_SUCCESS) {
        g_last_error = "cufftPlanMany failed";
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
  if (rc == PX_OK && d.expaction == PX_EXP_KRYLOV) rc = px::krylov_alloc(h->kw, d.krylov_m, n, B, &g_last_error);
  if (rc != PX_OK) {
    std::string msg = g_last_error;
    px_destroy(h);
    g_last_error = msg;
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
  Handle* h = static_cast<Handle*>(handle);
  if (!h) return;
  for (void* p : h->allocs) cudaFree(p);
  for (auto& pl : h->plans)
    if (pl.dcoef) cudaFree(pl.dcoef);
  for (auto& m : h->marks) { cudaEventDestroy(m.a); cudaEventDestroy(m.b); }
  drop_segments(h);
  if (h->gstream) cudaStreamDestroy(h->gstream);
  if (h->ev_in) cudaEventDestroy(h->ev_in);
  if (h->ev_out) cudaEventDestroy(h->ev_out);
  for (auto e : h->event_pool) cudaEventDestroy(e);
  px::krylov_free(h->kw);
  if (h->fft) cufftDestroy(h->fft);
  free_blocks(h);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  delete h;
}

int px_set_basis(void* handle, const double* tx, const double* ty, const int* ix, const int* iy) {
  Handle* h = static_cast<Handle*>(handle);
  if (h) cudaSetDevice(h->device);  // the handle's device (static cudart: per-thread current device)
  if (!h || !tx || !ty || !ix || !iy) return fail(h, PX_ERR_ARG, "null argument");
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
  Handle* h = static_cast<Handle*>(handle);
  if (!h || !p) return fail(h, PX_ERR_ARG, "null argument");
  if (slot < 0 || slot >= PX_PLAN_COUNT) return fail(h, PX_ERR_ARG, "bad plan slot");
  if (p->substeps < 1 || p->degree < 1 || !(p->scale > 0) || (p->sigma != 1 && p->sigma != -1) ||
      !p->coef_exp)
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

int px_set_krylov_plan(void* handle, int slot, double span, int substeps) {
  Handle* h = static_cast<Handle*>(handle);
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

int px_set_adjoint_mode(void* handle, int mode) {
  Handle* h = static_cast<Handle*>(handle);
  if (h) cudaSetDevice(h->device);
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
  Handle* h = static_cast<Handle*>(handle);
  if (h) cudaSetDevice(h->device);
  if (!h) return fail(h, PX_ERR_ARG, "null handle");
  if (blocks < 1 || blocks > PX_MAX_LOCAL_BLOCKS || blocks > h->Pl || h->Pl % blocks != 0)
    return fail(h, PX_ERR_ARG, "local blocks must divide the rank's slice count (1 … 16)");
  if (blocks == h->lb) return PX_OK;
  free_blocks(h);
  h->graph_valid = false;
  if (blocks == 1) return PX_OK;
  if (!h->ev_fork) PX_CUDA(h, cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
  const size_t Bn = (size_t)h->B * h->n;
  const int per = h->Pl / blocks;
  h->blocks.resize(blocks);
  for (int g = 0; g < blocks; ++g) {
    Handle::Block& b = h->blocks[g];
    b.q0 = g * per;
    b.q1 = (g + 1) * per;
    for (auto& p : b.Wk) PX_CUDA(h, cudaMalloc(&p, sizeof(double) * Bn));
    for (auto& p : b.ACC) PX_CUDA(h, cudaMalloc(&p, sizeof(double) * Bn));
    PX_CUDA(h, cudaMalloc(&b.D, sizeof(double) * Bn));
    PX_CUDA(h, cudaMalloc(&b.Gp, sizeof(double) * Bn));
    if (h->d.expaction == PX_EXP_KRYLOV) {
      std::string err;
      if (px::krylov_alloc(b.kw, h->d.krylov_m, h->n, h->B, &err) != PX_OK) {
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

int px_set_inputs(void* handle, const double* u0, const double* u_target, const double* ctrl, int mem,
                  void* stream) {
  Handle* h = static_cast<Handle*>(handle);
  if (h) cudaSetDevice(h->device);  // the handle's device (static cudart: per-thread current device)
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
  Handle* h = static_cast<Handle*>(handle);
  if (h) cudaSetDevice(h->device);  // the handle's device (static cudart: per-thread current device)
  if (!h) return fail(h, PX_ERR_ARG, "null handle");
  if (!h->basis_set || !h->inputs_set) return fail(h, PX_ERR_STATE, "basis/inputs not set");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int rc;
  if (h->d.kind == PX_KIND_ADVDIFF) {
    if (h->Pl > 1 && !h->plans[PX_PLAN_SLICE].set) return fail(h, PX_ERR_STATE, "slice plan not set");
    if (h->d.p_end < h->d.P && !h->plans[PX_PLAN_LONG_DIRECT].set)
      return fail(h, PX_ERR_STATE, "long-span direct plan not set");
    rc = direct_linear(h, s);
  } else {
    px::BurgersDirectArgs a{};
    a.u0 = h->u0; a.ctrl = h->ctrl; a.tx = h->tx; a.ix = h->ix; a.K = h->K;
    a.traj = h->traj; a.ubar = h->ubar; a.UT = h->UT;
    a.bpart = h->bpart; a.bounds = h->bounds; a.bounds_blocks = h->bounds_blocks;
    a.D = h->d.D; a.hx = h->d.hx; a.h = (h->d.T / h->d.P) / h->d.nsteps;
    a.nx = h->d.nx; a.B = h->B; a.P = h->d.P; a.nsteps = h->d.nsteps;
    const int tm = tbegin(h, PX_PHASE_RK4_DIRECT, s);
    rc = px::burgers_direct(a, s, &h->stats);
    tend(h, tm, s);
    if (rc != PX_OK) return fail(h, rc, "Burgers direct sweep failed: " + std::string(cudaGetErrorString(cudaGetLastError())));
  }
  if (rc == PX_OK) h->stage = 1;
  return rc;
}

int px_finish_direct(void* handle, void* stream) {
  Handle* h = static_cast<Handle*>(handle);
  if (h) cudaSetDevice(h->device);  // the handle's device (static cudart: per-thread current device)
  if (!h) return fail(h, PX_ERR_ARG, "null handle");
  if (h->stage != 1) return fail(h, PX_ERR_STATE, "px_finish_direct before px_direct");
  int rc = finish_direct_impl(h, static_cast<cudaStream_t>(stream));
  if (rc == PX_OK) h->stage = 2;
  return rc;
}


px::NlPlan nl_plan(const Plan& pl) {
  px::NlPlan p{};
  p.be = pl.dcoef;
  p.degree = pl.degree;
  p.substeps = pl.substeps;
  p.sigma = pl.sigma;
  p.c0 = pl.center;
  p.d = pl.scale;
  return p;
}

int px_nl_init(void* handle, void* stream) {
  Handle* h = static_cast<Handle*>(handle);
  if (h) cudaSetDevice(h->device);  // the handle's device (static cudart: per-thread current device)
  if (!h) return fail(h, PX_ERR_ARG, "null handle");
  if (h->d.kind != PX_KIND_BURGERS || !h->traj_b) return fail(h, PX_ERR_ARG, "iterative direct: Burgers, one rank");
  if (!h->inputs_set || !h->basis_set) return fail(h, PX_ERR_STATE, "basis/inputs not set");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t nodes = (size_t)h->d.P * h->d.nsteps + 1;
  px::k_nl_init<<<1024, 256, 0, s>>>(h->traj, h->u0, nodes, h->B, (int)h->n);
  PX_CHECK_LAUNCH(h);
  h->stage = 0;
  return PX_OK;
}

int nl_means_bounds(Handle* h, cudaStream_t s) {
  const size_t total = (size_t)h->d.P * h->B * h->n;
  px::k_slice_means<<<(unsigned)std::min<size_t>((total + 255) / 256, 4096), 256, 0, s>>>(
      h->ubar, h->traj, h->d.P, h->d.nsteps, h->B, (int)h->n);
  PX_CHECK_LAUNCH(h);
  px::k_frozen_bounds<<<h->bounds_blocks, 256, 0, s>>>(h->bpart, h->ubar, total, (int)h->n, h->d.hx, h->d.D);
  PX_CHECK_LAUNCH(h);
  px::k_frozen_bounds_final<<<1, 256, 0, s>>>(h->bounds, h->bpart, h->bounds_blocks);
  PX_CHECK_LAUNCH(h);
  return PX_OK;
}

int px_nl_prepare(void* handle, void* stream) {
  Handle* h = static_cast<Handle*>(handle);
  if (h) cudaSetDevice(h->device);  // the handle's device (static cudart: per-thread current device)
  if (!h || !h->traj_b) return fail(h, PX_ERR_ARG, "iterative direct not available");
  return nl_means_bounds(h, static_cast<cudaStream_t>(stream));
}

int px_nl_sweep(void* handle, double* err_max, void* stream) {
  Handle* h = static_cast<Handle*>(handle);
  if (h) cudaSetDevice(h->device);  // the handle's device (static cudart: per-thread current device)
  if (!h || !h->traj_b || !err_max) return fail(h, PX_ERR_ARG, "iterative direct not available");
  const Plan& ps = h->plans[PX_PLAN_NL_SLICE];
  const Plan& pt = h->plans[PX_PLAN_NL_STEP];
  if (!ps.set || !pt.set || ps.krylov || pt.krylov) return fail(h, PX_ERR_STATE, "iterative-direct plans not set");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  px::NlArgs a{};
  a.Q = h->traj; a.Qn = h->traj_b; a.ubar = h->ubar; a.u0 = h->u0; a.ctrl = h->ctrl;
  a.tx = h->tx; a.ix = h->ix; a.K = h->K;
  a.yend = h->Y0; a.Dc = h->Dc; a.err = h->nl_err;
  a.slice = nl_plan(ps); a.step = nl_plan(pt);
  a.D = h->d.D; a.hx = h->d.hx; a.h = (h->d.T / h->d.P) / h->d.nsteps;
  a.nx = h->d.nx; a.B = h->B; a.P = h->d.P; a.nsteps = h->d.nsteps;
  const int ppt = (a.nx + px::BURGERS_NT - 1) / px::BURGERS_NT;
  const unsigned lanes = (unsigned)(h->B * h->d.P);
  const size_t sm3 = 3 * (size_t)a.nx * sizeof(double), sm2 = 2 * (size_t)a.nx * sizeof(double);
#define PX_NL(PP)                                                                                          \
  do {                                                                                                     \
    cudaFuncSetAttribute(px::k_nl_inhom<PP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm3);       \
    px::k_nl_inhom<PP><<<lanes, px::BURGERS_NT, sm3, s>>>(a);                                             \
    PX_CHECK_LAUNCH(h);                                                                                    \
    cudaFuncSetAttribute(px::k_nl_scan<PP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);        \
    px::k_nl_scan<PP><<<h->B, px::BURGERS_NT, sm2, s>>>(a);                                               \
    PX_CHECK_LAUNCH(h);                                                                                    \
    cudaFuncSetAttribute(px::k_nl_record<PP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);      \
    px::k_nl_record<PP><<<lanes, px::BURGERS_NT, sm2, s>>>(a);                                            \
    PX_CHECK_LAUNCH(h);                                                                                    \
  } while (0)
  if (ppt <= 1) PX_NL(1);
  else if (ppt <= 2) PX_NL(2);
  else if (ppt <= 4) PX_NL(4);
  else PX_NL(8);
#undef PX_NL
  px::k_nl_error<<<lanes, 256, 0, s>>>(a);
  PX_CHECK_LAUNCH(h);
  h->nl_err_host.resize(lanes);
  PX_CUDA(h, cudaMemcpyAsync(h->nl_err_host.data(), h->nl_err, sizeof(double) * lanes, cudaMemcpyDeviceToHost, s));
  PX_CUDA(h, cudaStreamSynchronize(s));
  double mx = 0.0;
  for (double e : h->nl_err_host) mx = std::max(mx, e);
  *err_max = mx;
  std::swap(h->traj, h->traj_b);
  // stats: one inhomogeneous RK4 sweep + the carry and the node recordings
  const double n = (double)h->n;
  h->stats.rk4_lane_steps += (uint64_t)lanes * h->d.nsteps;
  h->stats.rk4_bytes += 32.0 * n * lanes * h->d.nsteps;
  const uint64_t terms = (uint64_t)h->B * ((h->d.P - 1) * ps.substeps * ps.degree +
                                            (uint64_t)(h->d.P - 1) * (h->d.nsteps - 1) * pt.substeps * pt.degree);
  h->stats.exp_terms += terms;
  h->stats.exp_bytes += 40.0 * n * terms;
  h->stats.algorithmic_bytes += 32.0 * n * lanes * h->d.nsteps + 40.0 * n * terms;
  if (!std::isfinite(mx)) return fail(h, PX_ERR_NONFINITE, "non-finite iterate in the nonlinear sweep");
  return PX_OK;
}

int px_nl_finish(void* handle, void* stream) {
  Handle* h = static_cast<Handle*>(handle);
  if (h) cudaSetDevice(h->device);  // the handle's device (static cudart: per-thread current device)
  if (!h || !h->traj_b) return fail(h, PX_ERR_ARG, "iterative direct not available");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t S = (size_t)h->d.P * h->d.nsteps;
  PX_CUDA(h, cudaMemcpyAsync(h->UT, h->traj + S * h->B * h->n, sizeof(double) * h->B * h->n,
                             cudaMemcpyDeviceToDevice, s));
  PX_TRY(nl_means_bounds(h, s));
  h->stage = 1;
  return PX_OK;
}

int px_set_adjoint_terminal(void* handle, const double* qdag_T, int mem, void* stream) {
  Handle* h = static_cast<Handle*>(handle);
  if (h) cudaSetDevice(h->device);  // the handle's device (static cudart: per-thread current device)
  if (!h || !qdag_T) return fail(h, PX_ERR_ARG, "null argument");
  if (!h->basis_set) return fail(h, PX_ERR_STATE, "basis not set");
  if (h->d.kind == PX_KIND_BURGERS && h->stage < 1)
    return fail(h, PX_ERR_STATE, "Burgers adjoint needs the direct trajectory (px_direct)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const cudaMemcpyKind kind = mem == PX_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  PX_CUDA(h, cudaMemcpyAsync(h->QT, qdag_T, sizeof(double) * h->B * h->n, kind, s));
  if (h->d.kind == PX_KIND_ADVDIFF)
    PX_TRY(apply_plus_control(h, h->gadj, h->QT, (long long)h->n, h->AT, false, s));
  h->stage = 2;
  return PX_OK;
}

int px_adjoint(void* handle, void* stream) {
  Handle* h = static_cast<Handle*>(handle);
  if (h) cudaSetDevice(h->device);  // the handle's device (static cudart: per-thread current device)
  if (!h) return fail(h, PX_ERR_ARG, "null handle");
  if (h->stage != 2) return fail(h, PX_ERR_STATE, "px_adjoint before px_finish_direct");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int rc;
  if (h->d.kind == PX_KIND_ADVDIFF) {
    if (h->d.p_begin > 0 && !h->plans[PX_PLAN_LONG_ADJOINT].set)
      return fail(h, PX_ERR_STATE, "long-span adjoint plan not set");
    rc = adjoint_linear(h, s);
  } else {
    const Plan& pl = h->plans[PX_PLAN_FROZEN];
    const bool span = h->adjoint_mode == PX_ADJOINT_FROZEN_SPAN;
    if (span && (h->d.p_begin != 0 || h->d.p_end != h->d.P))
      return fail(h, PX_ERR_ARG, "the frozen-span adjoint runs on one rank (it is one sequential chain)");
    // one slice and no earlier ranks (the serial loop): no homogeneous carry, no plan needed
    const bool no_carry = h->Pl == 1 && h->d.p_begin == 0 && !span;
    if ((!pl.set || pl.krylov) && !no_carry) return fail(h, PX_ERR_STATE, "frozen-operator plan not set");
    const bool use_plan = pl.set && !pl.krylov;
    px::BurgersAdjointArgs a{};
    a.traj = h->traj; a.ubar = h->ubar; a.QT = h->QT;
    a.W0 = h->Y0; a.W1 = h->Y1; a.Z = h->Z;
    a.G = h->G; a.QDAG0 = h->QDAG0;
    a.Wk[0] = h->Wk[0]; a.Wk[1] = h->Wk[1]; a.Wk[2] = h->Wk[2];
    a.ACC[0] = h->ACC[0]; a.ACC[1] = h->ACC[1];
    a.D = h->d.D; a.hx = h->d.hx; a.h = (h->d.T / h->d.P) / h->d.nsteps;
    a.nx = h->d.nx; a.B = h->B; a.P = h->d.P; a.nsteps = h->d.nsteps;
    a.p_begin = h->d.p_begin; a.p_end = h->d.p_end;
    a.terminal_span = span ? 1 : 0;
    if (use_plan) {
      a.substeps = pl.substeps; a.degree = pl.degree; a.center = pl.center; a.scale = pl.scale;
      a.sigma = pl.sigma; a.be = pl.be.data(); a.bp = pl.bp.data();
    } else {
      a.substeps = 0; a.degree = 0; a.center = 0.0; a.scale = 1.0; a.sigma = 1;
      a.be = a.bp = nullptr;
    }
    const int tm = tbegin(h, PX_PHASE_RK4_ADJOINT, s);
    rc = px::burgers_adjoint(a, s, &h->stats, &h->wend);
    tend(h, tm, s);
    if (rc != PX_OK) return fail(h, rc, "Burgers adjoint sweep failed");
    rc = project(h, h->GRAD, h->G, (long long)h->n, 1.0, 0.0, s);
  }
  if (rc == PX_OK) h->stage = 3;
  return rc;
}

int px_finish_adjoint(void* handle, void* stream) {
  Handle* h = static_cast<Handle*>(handle);
  if (h) cudaSetDevice(h->device);  // the handle's device (static cudart: per-thread current device)
  if (!h) return fail(h, PX_ERR_ARG, "null handle");
  if (h->stage != 3) return fail(h, PX_ERR_STATE, "px_finish_adjoint before px_adjoint");
  int rc = finish_adjoint_impl(h, static_cast<cudaStream_t>(stream));
  if (rc == PX_OK) h->stage = 4;
  return rc;
}

int gradient_phases(Handle* h, void* stream) {
  PX_TRY(px_direct(h, stream));
  PX_TRY(px_finish_direct(h, stream));
  PX_TRY(px_adjoint(h, stream));
  PX_TRY(px_finish_adjoint(h, stream));
  return PX_OK;
}

int capture_gradient(Handle* h) {
  drop_segments(h);
  const px_stats before = h->stats;
  h->capturing = true;
  h->cap_error = 0;
  seg_open(h, -1);
  const int rc = gradient_phases(h, h->gstream);
  seg_close(h);
  h->capturing = false;
  if (rc != PX_OK || h->cap_error) {
    drop_segments(h);
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

int px_gradient(void* handle, void* stream) {
  Handle* h = static_cast<Handle*>(handle);
  if (h) cudaSetDevice(h->device);  // the handle's device (static cudart: per-thread current device)
  if (!h) return fail(h, PX_ERR_ARG, "null handle");
  if (h->d.kind != PX_KIND_ADVDIFF) return fail(h, PX_ERR_ARG, "px_gradient: linear testbed only");
  if (!h->graphs) return gradient_phases(h, stream);
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
  NvtxScope gradient_range("px.gradient(graph)");
  for (auto& sg : h->segs) {
    if (sg.phase >= 0) nvtxRangePushA(phase_name(sg.phase));
    if (h->timing && sg.phase >= 0) {
      Handle::TMark m{sg.phase, take_event(h), take_event(h), sg.launches, sg.bytes};
      PX_CUDA(h, cudaEventRecord(m.a, h->gstream));
      PX_CUDA(h, cudaGraphLaunch(sg.exec, h->gstream));
      PX_CUDA(h, cudaEventRecord(m.b, h->gstream));
      h->marks.push_back(m);
    } else {
      PX_CUDA(h, cudaGraphLaunch(sg.exec, h->gstream));
    }
    if (sg.phase >= 0) nvtxRangePop();
  }
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
  Handle* h = static_cast<Handle*>(handle);
  if (h) cudaSetDevice(h->device);  // the handle's device (static cudart: per-thread current device)
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
  h->timing = enable != 0;
  return PX_OK;
}

int px_get_timing(void* handle, px_timing* out) {
  Handle* h = static_cast<Handle*>(handle);
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
