// kernels.cuh — sm_100a fp64 kernels of the Paraexp direct-adjoint path.
//
// Replaces the reference's per-stage Python/scipy arithmetic:
//   rk45_integrate stage loop (timestepping.py:162-201) + csr_matvec (linalg.py:70-74)
//     -> k_rk4_tile: one fused classical-RK4 step per launch over all (batch × slice)
//        lanes, the four stages computed from one shared-memory tile with a
//        4-point halo (temporal fusion of the stages: 24n algorithmic bytes per
//        step instead of ~160n for stage-by-stage kernels);
//   _LejaInterpolant.step Newton loop (timestepping.py:343-356)
//     -> k_cheb_first / k_cheb_term: stencil fused with the Chebyshev three-term
//        recurrence and the exp and φ₁ accumulators;
//   superposition / cost / gradient quadrature (paraexp.py:202-218,
//   optimization.py:84-112) -> elementwise, reduction and projection kernels with
//   fixed-order (deterministic) reductions.
// No tensor cores: nothing here is a dense contraction; fp64 CUDA-core math.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace px {

struct Stencil5 {
  double cc, ce, cw, cn, cs;
};

// periodic wrap for halo coordinates (tiles may be wider than the grid)
__device__ __forceinline__ int wrapi(int v, int n) {
  v %= n;
  return v < 0 ? v + n : v;
}

// (M u) at flat index i of a periodic nx×ny field (global memory, L1/L2 cached).
template <int DIM>
__device__ __forceinline__ double stencil_at(const double* __restrict__ u, const Stencil5& s,
                                             int x, int y, int nx, int ny) {
  const size_t row = (size_t)y * nx;
  const int xe = (x + 1 == nx) ? 0 : x + 1;
  const int xw = (x == 0) ? nx - 1 : x - 1;
  double r = s.cc * u[row + x];
  r += s.ce * __ldg(u + row + xe);
  r += s.cw * __ldg(u + row + xw);
  if (DIM == 2) {
    const int yn = (y + 1 == ny) ? 0 : y + 1;
    const int ys = (y == 0) ? ny - 1 : y - 1;
    r += s.cn * __ldg(u + (size_t)yn * nx + x);
    r += s.cs * __ldg(u + (size_t)ys * nx + x);
  }
  return r;
}

// ---------------------------------------------------------------------------
// Fused RK4 step over lanes (zero-data inhomogeneous slice solves)
// ---------------------------------------------------------------------------

struct RK4Args {
  const double* y_in;  // lanes × n; nullptr = zero state (first step of a sweep)
  double* y_out;       // lanes × n
  const double* g;     // B × n constant source; lane l uses member l / lanes_per_b
  double* z;           // ADJ: lanes × n running ∫y (in place)
  Stencil5 st;
  double h;
  int nx, ny;
  int lanes, lanes_per_b;
  int tiles_x, tiles_y;
};

// Stage regions: stage s (1..4) computes on the tile grown by (4 - s) points.
// Tile-interior points are owned by fixed threads (accumulators in registers);
// ring points are distributed round-robin.
template <int DIM, int TX, int TY, int NT, bool ADJ>
__global__ void __launch_bounds__(NT) k_rk4_tile(RK4Args a) {
  constexpr int HX = 4;
  constexpr int HY = (DIM == 2) ? 4 : 0;
  constexpr int W = TX + 2 * HX;
  constexpr int H = TY + 2 * HY;
  constexpr int NPT = (TX * TY) / NT;
  static_assert((TX * TY) % NT == 0, "tile must split evenly over threads");
  extern __shared__ double smem[];
  double* s_y = smem;
  double* s_g = s_y + W * H;
  double* s_a = s_g + W * H;
  double* s_b = s_a + W * H;

  const int lane = blockIdx.x % a.lanes;
  const int tile = blockIdx.x / a.lanes;
  const int tx0 = (tile % a.tiles_x) * TX;
  const int ty0 = (tile / a.tiles_x) * TY;
  const int nx = a.nx, ny = a.ny;
  const size_t n = (size_t)nx * ny;
  const double* __restrict__ yin = a.y_in ? a.y_in + (size_t)lane * n : nullptr;
  const double* __restrict__ g = a.g + (size_t)(lane / a.lanes_per_b) * n;
  const Stencil5 st = a.st;
  const double h = a.h, hh = 0.5 * a.h, h6 = a.h / 6.0;

  for (int idx = threadIdx.x; idx < W * H; idx += NT) {
    const int ly = idx / W, lx = idx - ly * W;
    const int gx = wrapi(tx0 + lx - HX, nx);
    const int gy = (DIM == 2) ? wrapi(ty0 + ly - HY, ny) : 0;
    const size_t off = (size_t)gy * nx + gx;
    s_y[idx] = yin ? __ldg(yin + off) : 0.0;
    s_g[idx] = __ldg(g + off);
  }
  __syncthreads();

  auto A = [&](const double* s, int i) -> double {
    double r = st.cc * s[i];
    r += st.ce * s[i + 1];
    r += st.cw * s[i - 1];
    if (DIM == 2) {
      r += st.cn * s[i + W];
      r += st.cs * s[i - W];
    }
    return r;
  };
  auto interior_index = [&](int t) -> int {
    const int q = threadIdx.x + t * NT;
    const int qy = q / TX, qx = q - qy * TX;
    return (qy + HY) * W + (qx + HX);
  };
  // ring of the tile grown by `s`: local index of the idx-th ring point
  auto ring_count = [&](int s) -> int {
    const int sy = (DIM == 2) ? s : 0;
    return (TX + 2 * s) * (TY + 2 * sy) - TX * TY;
  };
  auto ring_index = [&](int s, int idx) -> int {
    const int sy = (DIM == 2) ? s : 0;
    const int rw = TX + 2 * s;
    int r, c;
    if (idx < sy * rw) {
      r = idx / rw; c = idx - r * rw;
    } else if (idx < 2 * sy * rw) {
      idx -= sy * rw;
      r = sy + TY + idx / rw; c = idx % rw;
    } else {
      idx -= 2 * sy * rw;
      r = sy + idx / (2 * s);
      c = idx % (2 * s);
      if (c >= s) c += TX;
    }
    // rectangle origin is (HX - s, HY - sy)
    return (r + HY - sy) * W + (c + HX - s);
  };

  double acc[NPT];
  double zacc[ADJ ? NPT : 1];

  // stage 1: k1 = A y + g, Y2 = y + h/2 k1 (on tile+3)
#pragma unroll
  for (int t = 0; t < NPT; ++t) {
    const int i = interior_index(t);
    const double k = A(s_y, i) + s_g[i];
    const double Y = s_y[i] + hh * k;
    acc[t] = k;
    if (ADJ) zacc[t] = s_y[i] + 2.0 * Y;
    s_a[i] = Y;
  }
  for (int idx = threadIdx.x, m = ring_count(3); idx < m; idx += NT) {
    const int i = ring_index(3, idx);
    s_a[i] = s_y[i] + hh * (A(s_y, i) + s_g[i]);
  }
  __syncthreads();
  // stage 2: k2 = A Y2 + g, Y3 = y + h/2 k2 (on tile+2)
#pragma unroll
  for (int t = 0; t < NPT; ++t) {
    const int i = interior_index(t);
    const double k = A(s_a, i) + s_g[i];
    const double Y = s_y[i] + hh * k;
    acc[t] += 2.0 * k;
    if (ADJ) zacc[t] += 2.0 * Y;
    s_b[i] = Y;
  }
  for (int idx = threadIdx.x, m = ring_count(2); idx < m; idx += NT) {
    const int i = ring_index(2, idx);
    s_b[i] = s_y[i] + hh * (A(s_a, i) + s_g[i]);
  }
  __syncthreads();
  // stage 3: k3 = A Y3 + g, Y4 = y + h k3 (on tile+1), into s_a
#pragma unroll
  for (int t = 0; t < NPT; ++t) {
    const int i = interior_index(t);
    const double k = A(s_b, i) + s_g[i];
    const double Y = s_y[i] + h * k;
    acc[t] += 2.0 * k;
    if (ADJ) zacc[t] += Y;
    s_a[i] = Y;
  }
  for (int idx = threadIdx.x, m = ring_count(1); idx < m; idx += NT) {
    const int i = ring_index(1, idx);
    s_a[i] = s_y[i] + h * (A(s_b, i) + s_g[i]);
  }
  __syncthreads();
  // stage 4: k4 = A Y4 + g; y += h/6 (k1 + 2k2 + 2k3 + k4)
  double* __restrict__ yout = a.y_out + (size_t)lane * n;
  double* __restrict__ z = ADJ ? a.z + (size_t)lane * n : nullptr;
#pragma unroll
  for (int t = 0; t < NPT; ++t) {
    const int q = threadIdx.x + t * NT;
    const int qy = q / TX, qx = q - qy * TX;
    const int gx = tx0 + qx, gy = ty0 + qy;
    const int i = (qy + HY) * W + (qx + HX);
    const double k = A(s_a, i) + s_g[i];
    if (gx < nx && (DIM == 1 || gy < ny)) {
      const size_t off = (size_t)gy * nx + gx;
      yout[off] = s_y[i] + h6 * (acc[t] + k);
      if (ADJ) {
        const double zin = yin ? z[off] : 0.0;
        z[off] = zin + h6 * zacc[t];
      }
    }
  }
}

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

// ---------------------------------------------------------------------------
// Elementwise helpers (batch in blockIdx.y)
// ---------------------------------------------------------------------------

// out[b] = alpha·x[b] + beta·y[b]  (x, y batch-strided; y may be nullptr)
__global__ void k_axpby(double* out, long long out_bstride, const double* x, long long x_bstride,
                        double alpha, const double* y, long long y_bstride, double beta, size_t n) {
  const int b = blockIdx.y;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    double r = alpha * x[b * x_bstride + i];
    if (y) r += beta * y[b * y_bstride + i];
    out[b * out_bstride + i] = r;
  }
}

// out[b] = M x[b] (+ f[b]) with f = Σ_k c[b,k] tx[ix_k][i] ty[iy_k][j] when ctrl != nullptr
template <int DIM>
__global__ void k_apply_plus_control(double* out, const double* src, long long src_bstride, Stencil5 st,
                                     const double* ctrl, const double* tx, const double* ty,
                                     const int* ix, const int* iy, int K, int nx, int ny) {
  const size_t n = (size_t)nx * ny;
  const int b = blockIdx.y;
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int y = (int)(i / nx), x = (int)(i - (size_t)y * nx);
  double r = stencil_at<DIM>(src + b * src_bstride, st, x, y, nx, ny);
  if (ctrl) {
    const double* c = ctrl + (size_t)b * K;
    double f = 0.0;
    for (int k = 0; k < K; ++k) f += c[k] * (tx[(size_t)ix[k] * nx + x] * ty[(size_t)iy[k] * ny + y]);
    r += f;
  }
  out[(size_t)b * n + i] = r;
}

// out[b][i] = Σ_{p<lanes_per_b} lanes[b*lanes_per_b + p][i]  (fixed order)
__global__ void k_lane_sum(double* out, const double* lanes, int lanes_per_b, size_t n) {
  const int b = blockIdx.y;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const double* src = lanes + (size_t)b * lanes_per_b * n + i;
    double r = 0.0;
    for (int p = 0; p < lanes_per_b; ++p) r += src[(size_t)p * n];
    out[(size_t)b * n + i] = r;
  }
}

// ---------------------------------------------------------------------------
// Deterministic reductions
// ---------------------------------------------------------------------------

template <int NT>
__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x < 32) {
    r = (threadIdx.x < NT / 32) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) r += __shfl_down_sync(0xffffffffu, r, o);
  }
  __syncthreads();
  return r;  // valid in thread 0
}

// partial[b][blk] = Σ_{i in blk's grid-stride set} x[b][i]²
__global__ void __launch_bounds__(256) k_sumsq_partial(double* partial, const double* x, size_t n) {
  __shared__ double red[8];
  const int b = blockIdx.y;
  double v = 0.0;
  for (size_t i = (size_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (size_t)gridDim.x * 256) {
    const double t = x[(size_t)b * n + i];
    v += t * t;
  }
  v = block_sum<256>(v, red);
  if (threadIdx.x == 0) partial[(size_t)b * gridDim.x + blockIdx.x] = v;
}

// out[b] = scale · Σ_j partial[b][j]; flag set if non-finite
__global__ void __launch_bounds__(256) k_finalize_sum(double* out, const double* partial, int m,
                                                      double scale, int* nonfinite) {
  __shared__ double red[8];
  const int b = blockIdx.x;
  double v = 0.0;
  for (int j = threadIdx.x; j < m; j += 256) v += partial[(size_t)b * m + j];
  v = block_sum<256>(v, red);
  if (threadIdx.x == 0) {
    const double r = scale * v;
    out[b] = r;
    if (nonfinite && !isfinite(r)) atomicExch(nonfinite, 1);
  }
}

// R[b][a][j] = Σ_i tx[a][i] F[b][j][i] for all x-table rows a (grid: (ny, B))
template <int MAXR>
__global__ void __launch_bounds__(256) k_project_rows(double* R, const double* F, long long F_bstride,
                                                      const double* tx, int rows_x, int nx, int ny) {
  __shared__ double red[8];
  const int j = blockIdx.x, b = blockIdx.y;
  const double* row = F + b * F_bstride + (size_t)j * nx;
  double acc[MAXR];
#pragma unroll
  for (int a = 0; a < MAXR; ++a) acc[a] = 0.0;
  for (int i = threadIdx.x; i < nx; i += 256) {
    const double v = row[i];
#pragma unroll
    for (int a = 0; a < MAXR; ++a)
      if (a < rows_x) acc[a] += tx[(size_t)a * nx + i] * v;
  }
  for (int a = 0; a < rows_x; ++a) {
    const double s = block_sum<256>(acc[a], red);
    if (threadIdx.x == 0) R[((size_t)b * rows_x + a) * ny + j] = s;
  }
}

// grad[b][k] = beta·grad[b][k] + alpha·Σ_j ty[iy_k][j] R[b][ix_k][j]  (grid: (K, B))
__global__ void __launch_bounds__(256) k_project_cols(double* grad, const double* R, const double* ty,
                                                      const int* ix, const int* iy, int rows_x, int K,
                                                      int ny, double alpha, double beta) {
  __shared__ double red[8];
  const int k = blockIdx.x, b = blockIdx.y;
  const double* r = R + ((size_t)b * rows_x + ix[k]) * ny;
  const double* t = ty + (size_t)iy[k] * ny;
  double v = 0.0;
  for (int j = threadIdx.x; j < ny; j += 256) v += t[j] * r[j];
  v = block_sum<256>(v, red);
  if (threadIdx.x == 0) {
    const size_t o = (size_t)b * K + k;
    grad[o] = (beta == 0.0 ? 0.0 : beta * grad[o]) + alpha * v;
  }
}

}  // namespace px
