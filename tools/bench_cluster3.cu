// Realistic phase model: C=16 CTAs x 512 threads x big smem; warp 0 of each CTA
// does one "item" (DSMEM operand read of a neighbour CTA + FMAs + smem store),
// then everybody crosses a split cluster barrier.  Variants isolate the costs.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

template <int MODE>
__global__ void __launch_bounds__(512, 1) kphase(int iters, double* sink) {
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ double2 sm[];
  const int r = cl.block_rank(), n = cl.num_blocks();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = make_double2(i, r);
  cl.sync();
  double2 acc = make_double2(0, 0);
  for (int it = 0; it < iters; ++it) {
    if (warp == 0) {
      if (MODE >= 1) {   // DSMEM operand read (8 values per lane)
        const double2* rem = cl.map_shared_rank(sm, (r + 1) % n);
        double2 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = rem[(it & 7) * 256 + k * 32 + lane];
#pragma unroll
        for (int k = 0; k < 8; ++k) { acc.x = fma(v[k].x, 1.0001, acc.x); acc.y = fma(v[k].y, 0.999, acc.y); }
      }
      if (MODE >= 2) sm[1024 + lane] = acc;     // local store of the result
      if (MODE >= 3) {                           // remote store (push) of the result
        double2* rem = cl.map_shared_rank(sm, (r + 1) % n);
        rem[2048 + lane] = acc;
      }
    }
    cl.barrier_arrive();
    cl.barrier_wait();
  }
  if (acc.x == 1.5) sink[0] = acc.y;
}

template <class K>
float run(K kern, int C, int T, int smem, int iters, double* sink) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C * 2); cfg.blockDim = dim3(T); cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaLaunchKernelEx(&cfg, kern, iters, sink);
  cudaEventRecord(a);
  cudaLaunchKernelEx(&cfg, kern, iters, sink);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError(); if (e) printf("err %s\n", cudaGetErrorString(e));
  return ms * 1e3f / iters;
}

int main() {
  double* sink; cudaMalloc(&sink, 8);
  for (int C : {2, 8, 16}) for (int T : {128, 512}) for (int smem : {65536, 200 * 1024}) {
    printf("C=%2d T=%3d smem=%3dK: barrier %.3f | +dsmem read %.3f | +local store %.3f | +remote store %.3f us\n",
           C, T, smem / 1024, run(kphase<0>, C, T, smem, 2000, sink), run(kphase<1>, C, T, smem, 2000, sink),
           run(kphase<2>, C, T, smem, 2000, sink), run(kphase<3>, C, T, smem, 2000, sink));
  }
  return 0;
}
