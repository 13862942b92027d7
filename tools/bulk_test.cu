#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const double2* src, double2* out, int bytes) {
  extern __shared__ __align__(128) double2 sm[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(bytes));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(sm)), "l"(src), "r"(bytes), "r"(su(&bar)) : "memory");
  }
  uint32_t done = 0;
  while (!done) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(done) : "r"(su(&bar)), "r"(0));
  for (int i = threadIdx.x; i < bytes / 16; i += blockDim.x) out[i] = sm[i];
}
int main() {
  for (int bytes : {4096, 16384, 32768, 65536, 131072}) {
    double2 *s, *o; cudaMalloc(&s, bytes); cudaMalloc(&o, bytes);
    double2* h = new double2[bytes / 16]; for (int i = 0; i < bytes / 16; ++i) h[i] = make_double2(i, -i);
    cudaMemcpy(s, h, bytes, cudaMemcpyHostToDevice); cudaMemset(o, 0, bytes);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    k<<<1, 256, bytes>>>(s, o, bytes);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, o, bytes, cudaMemcpyDeviceToHost);
    int bad = 0; for (int i = 0; i < bytes / 16; ++i) bad += (h[i].x != i);
    printf("bytes %d: %s bad=%d\n", bytes, cudaGetErrorString(e), bad);
    if (e) return 1;
  }
}
