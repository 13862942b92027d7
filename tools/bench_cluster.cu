// Microbenchmark: cost of a cluster barrier (barrier.cluster arrive+wait) vs
// cluster size and CTA size, and of a dependent L2 load + barrier step.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_sync(int iters, double* sink) {
  cg::cluster_group cl = cg::this_cluster();
  double v = threadIdx.x;
  for (int i = 0; i < iters; ++i) { cl.sync(); v += 1.0; }
  if (v < 0) sink[0] = v;
}

__global__ void k_bar(int iters, double* sink) {
  double v = threadIdx.x;
  for (int i = 0; i < iters; ++i) { __syncthreads(); v += 1.0; }
  if (v < 0) sink[0] = v;
}

// one warp per CTA loads a 4 KB block (L2-hot) per step, then cluster sync
__global__ void k_step(int iters, const double2* __restrict__ m, double* sink) {
  cg::cluster_group cl = cg::this_cluster();
  double2 acc = make_double2(0, 0);
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x < 32) {
      const double2* p = m + ((i * 37 + blockIdx.x) % 64) * 256;
#pragma unroll
      for (int k = 0; k < 8; ++k) { double2 t = __ldg(p + k * 32 + threadIdx.x); acc.x += t.x; acc.y += t.y; }
    }
    cl.sync();
  }
  if (acc.x == 12345.0) sink[0] = acc.y;
}

template <class K, class... A>
float run(K kern, int C, int T, int grid, A... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid); cfg.blockDim = dim3(T);
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaLaunchKernelEx(&cfg, kern, args...);
  cudaEventRecord(a);
  cudaLaunchKernelEx(&cfg, kern, args...);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e) printf("err %s\n", cudaGetErrorString(e));
  return ms;
}

int main() {
  double* sink; cudaMalloc(&sink, 8);
  double2* m; cudaMalloc(&m, 64 * 256 * 16); cudaMemset(m, 0, 64 * 256 * 16);
  const int iters = 2000;
  for (int C : {1, 2, 4, 8, 16})
    for (int T : {128, 256, 512}) {
      float ms = run(k_sync, C, T, C * 2, iters, sink);
      float ms2 = run(k_step, C, T, C * 2, iters, (const double2*)m, sink);
      printf("cluster C=%2d T=%3d: sync %.3f us   l2load+sync %.3f us\n", C, T, ms * 1e3 / iters, ms2 * 1e3 / iters);
    }
  for (int T : {256, 512, 1024}) {
    float ms = run(k_bar, 1, T, 2, iters, sink);
    printf("__syncthreads T=%d: %.3f us\n", T, ms * 1e3 / iters);
  }
  return 0;
}
