// Microbenchmark: cost of a per-iteration CTA barrier vs a cluster barrier with a DSMEM edge
// exchange (64-thread CTAs, ~ a row iteration's worth of dependent fp64 work between barriers).
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

template <int MODE>  // 0: __syncthreads + local smem; 1: cluster barrier + remote (DSMEM) store
__global__ void loop(double* out, int iters, int work, long long* cyc) {
  __shared__ double s[2][64];
  cg::cluster_group cl = cg::this_cluster();
  const int t = threadIdx.x;
  double x = t * 1e-3 + blockIdx.x, acc = 0.0;
  int par = 0;
  const unsigned rank = MODE ? cl.block_rank() : 0;
  const unsigned nb = MODE ? cl.num_blocks() : 1;
  double* peer = MODE ? cl.map_shared_rank(&s[0][0], (rank + 1) % nb) : &s[0][0];
  if (MODE) cl.sync();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    for (int k = 0; k < work; ++k) x = fma(x, 1.0000001, 1e-9);
    if (MODE == 0) {
      s[par][t] = x;
      __syncthreads();
      acc += s[par][(t + 1) & 63];
    } else {
      if (t == 0) peer[par * 64 + 63] = x;  // edge value into the neighbour CTA
      s[par][t] = x;
      cl.sync();
      acc += s[par][(t + 1) & 63];
    }
    par ^= 1;
  }
  long long t1 = clock64();
  out[blockIdx.x * 64 + t] = x + acc;
  if (t == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1 << 24); cudaMallocManaged(&cyc, 8);
  const int it = 20000;
  for (int work : {0, 40}) {
    for (int grid : {1, 592}) {
      loop<0><<<grid, 64>>>(out, it, work, cyc); cudaDeviceSynchronize();
      loop<0><<<grid, 64>>>(out, it, work, cyc); cudaDeviceSynchronize();
      printf("work %d grid %d  CTA barrier: %.1f cycles/iter\n", work, grid, (double)cyc[0] / it);
      for (int cs : {2, 4, 8, 16}) {
        if (cs == 16) cudaFuncSetAttribute(loop<1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaLaunchConfig_t cfg{};
        int g = grid < cs ? cs : (grid / cs) * cs;
        cfg.gridDim = dim3(g); cfg.blockDim = dim3(64);
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        cudaError_t e = cudaLaunchKernelEx(&cfg, loop<1>, out, it, work, cyc); cudaDeviceSynchronize();
        e = cudaLaunchKernelEx(&cfg, loop<1>, out, it, work, cyc);
        cudaError_t e2 = cudaDeviceSynchronize();
        printf("work %d grid %d  cluster %2d barrier+DSMEM: %.1f cycles/iter %s\n", work, g, cs, (double)cyc[0] / it,
               (e != cudaSuccess || e2 != cudaSuccess) ? cudaGetErrorString(e != cudaSuccess ? e : e2) : "");
      }
    }
  }
  return 0;
}
