// Per-SM TMA streaming rate through an mbarrier ring (no compute): how fast
// can one CTA pull factor blocks, as a function of slot count / size / CTAs.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void __launch_bounds__(512, 1) k(const double2* src, int64_t per_cta_items, int slot_bytes, int ns, unsigned long long* t, int hot_items) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bars = (uint64_t*)sm;
  volatile int* done = (volatile int*)(bars + 64);
  volatile int64_t* seq = (volatile int64_t*)(done + 64);
  unsigned char* ring = sm + 1024;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < ns; ++i) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&bars[i])), "r"(1)); done[i] = i - ns; seq[i] = -1; }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const char* base = (const char*)src + (int64_t)blockIdx.x * per_cta_items * slot_bytes;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  if (warp == 15) {
    for (int64_t i = 0; i < per_cta_items; i += 8) {
      int64_t it = i + lane;
      if (lane < 8 && it < per_cta_items) {
        int sl = it % ns;
        while (done[sl] != it - ns) {}
        uint64_t* bar = &bars[sl];
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(bar)), "r"(slot_bytes));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(su(ring + sl * slot_bytes)), "l"(base + (hot_items ? it % hot_items : it) * slot_bytes), "r"(slot_bytes), "r"(su(bar)) : "memory");
        seq[sl] = it;
      }
      __syncwarp();
    }
  } else {
    double acc = 0;
    for (int64_t it = warp; it < per_cta_items; it += 15) {
      int sl = it % ns;
      uint32_t ph = (it / ns) & 1, ok = 0;
      while (seq[sl] != it) {}
      while (!ok) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(ok) : "r"(su(&bars[sl])), "r"(ph));
      acc += ((const double*)(ring + sl * slot_bytes))[lane];
      __syncwarp();
      if (lane == 0) done[sl] = it;
    }
    if (acc == 12345.0) t[1000] = 1;
  }
  __syncthreads();
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (threadIdx.x == 0) t[blockIdx.x] = t1 - t0;
}
int main() {
  const int64_t total_bytes = 1ll << 32;   // 4 GB arena (cold reads)
  double2* s; cudaMalloc(&s, total_bytes); cudaMemset(s, 0, total_bytes);
  unsigned long long* t; cudaMalloc(&t, 8 * 2048);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  for (int hot : {0, 1}) for (int grid : {1, 32, 148}) for (int slot : {4096, 8192, 16384}) for (int ns : {8, 16, 24}) {
    if (slot * ns > 200 * 1024) continue;
    int64_t per = (int64_t)(8 << 20) / slot;   // 8 MB per CTA
    if (per * slot * grid > total_bytes) per = total_bytes / grid / slot;
    const int hot_items = hot ? (1 << 20) / slot : 0;   // 1 MB per CTA, L2-resident
    k<<<grid, 512, 1024 + slot * ns>>>(s, per, slot, ns, t, hot_items);
    k<<<grid, 512, 1024 + slot * ns>>>(s, per, slot, ns, t, hot_items);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148]; cudaMemcpy(h, t, 8 * grid, cudaMemcpyDeviceToHost);
    double mx = 0; for (int i = 0; i < grid; ++i) mx = mx > h[i] ? mx : h[i];
    double gbs = per * slot / mx;   // bytes per ns = GB/s per CTA
    printf("%s grid %3d slot %5d ns %2d: %6.1f GB/s per CTA, %7.1f GB/s total  %s\n", hot ? "L2 " : "HBM", grid, slot, ns, gbs, gbs * grid, e ? cudaGetErrorString(e) : "");
  }
}
