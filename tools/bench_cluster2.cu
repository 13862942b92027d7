// Where does a "level" of the cluster BCR spend its time?  Variants of one
// step = (L2-hot 4 KB block load by one warp per CTA) + cluster barrier.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ double2 ld8(const double2* p, int lane) {
  double2 acc = make_double2(0, 0);
#pragma unroll
  for (int k = 0; k < 8; ++k) { double2 t = __ldg(p + k * 32 + lane); acc.x += t.x; acc.y += t.y; }
  return acc;
}

// A: load+use, then cl.sync()
__global__ void kA(int iters, const double2* m, double* sink) {
  cg::cluster_group cl = cg::this_cluster();
  double2 acc = make_double2(0, 0);
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x < 32) { double2 t = ld8(m + ((i * 37 + blockIdx.x) % 64) * 256, threadIdx.x); acc.x += t.x; }
    cl.sync();
  }
  if (acc.x == 1.5) sink[0] = acc.y;
}
// B: arrive; issue next load into regs; wait; use
__global__ void kB(int iters, const double2* m, double* sink) {
  cg::cluster_group cl = cg::this_cluster();
  double2 acc = make_double2(0, 0), reg[8];
  const int lane = threadIdx.x & 31;
  for (int k = 0; k < 8; ++k) reg[k] = __ldg(m + k * 32 + lane);
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x < 32) for (int k = 0; k < 8; ++k) { acc.x += reg[k].x; acc.y += reg[k].y; }
    cl.barrier_arrive();
    if (threadIdx.x < 32) { const double2* p = m + (((i + 1) * 37 + blockIdx.x) % 64) * 256; for (int k = 0; k < 8; ++k) reg[k] = __ldg(p + k * 32 + lane); }
    cl.barrier_wait();
  }
  if (acc.x == 1.5) sink[0] = acc.y;
}
// C: barrier only (arrive/wait split)
__global__ void kC(int iters, const double2* m, double* sink) {
  cg::cluster_group cl = cg::this_cluster();
  double v = 0;
  for (int i = 0; i < iters; ++i) { cl.barrier_arrive(); v += 1; cl.barrier_wait(); }
  if (v < 0) sink[0] = v;
}
// D: smem write + DSMEM read of neighbour after barrier
__global__ void kD(int iters, const double2* m, double* sink) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double2 buf[256];
  double2 acc = make_double2(0, 0);
  const int r = cl.block_rank(), n = cl.num_blocks();
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x < 256) buf[threadIdx.x] = make_double2(i, r);
    cl.sync();
    if (threadIdx.x < 32) {
      const double2* rem = cl.map_shared_rank(buf, (r + 1) % n);
      for (int k = 0; k < 8; ++k) { double2 t = rem[k * 32 + threadIdx.x]; acc.x += t.x; }
    }
    cl.sync();
  }
  if (acc.x == 1.5) sink[0] = acc.y;
}
// E: load only (no barrier), dependent chain of loads per warp
__global__ void kE(int iters, const double2* m, double* sink) {
  double2 acc = make_double2(0, 0);
  int idx = blockIdx.x;
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x < 32) { double2 t = ld8(m + (idx % 64) * 256, threadIdx.x); acc.x += t.x; idx += (int)(t.y) + 37; }
  }
  if (acc.x == 1.5) sink[0] = acc.y;
}

template <class K>
float run(K kern, int C, int T, int iters, const double2* m, double* sink) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C * 2); cfg.blockDim = dim3(T);
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaLaunchKernelEx(&cfg, kern, iters, m, sink);
  cudaEventRecord(a);
  cudaLaunchKernelEx(&cfg, kern, iters, m, sink);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError(); if (e) printf("err %s\n", cudaGetErrorString(e));
  return ms * 1e3f / iters;
}

int main() {
  double* sink; cudaMalloc(&sink, 8);
  double2* m; cudaMalloc(&m, 64 * 256 * 16); cudaMemset(m, 0, 64 * 256 * 16);
  for (int C : {1, 16}) for (int T : {256, 512}) {
    printf("C=%2d T=%3d  A load+use+sync %.3f | B arrive/load/wait %.3f | C split barrier %.3f | D dsmem+2sync %.3f | E load chain %.3f us\n",
           C, T, run(kA, C, T, 2000, m, sink), run(kB, C, T, 2000, m, sink), run(kC, C, T, 2000, m, sink),
           run(kD, C, T, 2000, m, sink), run(kE, C, T, 2000, m, sink));
  }
  return 0;
}
