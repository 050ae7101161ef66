// Micro-benchmark (diagnostics): tcgen05.mma kind::tf32 issue rate when the whole warp runs
// the issue loop (elect.sync inside the asm, warp-uniform descriptors, fully unrolled) versus
// one lane under `if (lane == 0)`.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__host__ __device__ constexpr uint64_t sdesc_c(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_ts_elect(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
               "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d), "r"(a), "l"(bdesc), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d), "r"(a), "l"(bdesc), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void commit_elect(uint32_t bar) {
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool try_wait(uint32_t bar, uint32_t par) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n}" : "=r"(ok) : "r"(bar), "r"(par) : "memory");
  return ok;
}

template <int N, int NM, int MODE>
__global__ void k(long long* out, int reps) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tm;
  const uint32_t sB = (smem_u32(sm) + 1023) & ~1023u;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tm)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm + (sB - smem_u32(sm)))[i] = 0x3f800000u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t t = tm;
  const uint32_t b = smem_u32(&bar);
  const uint64_t d0 = sdesc_c(sB, 16, 1024);
  constexpr uint32_t id = idesc_tf32(128, N);
  if (MODE == 0 ? threadIdx.x < 32 : threadIdx.x == 0) {
    long long acc_issue = 0, acc_done = 0;
    for (int r = 0; r < reps; ++r) {
      long long t0 = clock64();
#pragma unroll
      for (int i = 0; i < NM; ++i) {
        const uint64_t bd = d0 + (uint64_t)((((i & 3) * 32 + ((i >> 2) & 1) * (N * 128)) >> 4));
        if (MODE == 0) mma_ts_elect(t + 256, t + (i & 7) * 8, bd, id, i > 0);
        else mma_ts(t + 256, t + (i & 7) * 8, bd, id, i > 0);
      }
      if (MODE == 0) commit_elect(b); else commit(b);
      long long t1 = clock64();
      while (!try_wait(b, r & 1)) {}
      long long t2 = clock64();
      if (r >= 2) { acc_issue += t1 - t0; acc_done += t2 - t0; }
    }
    if (threadIdx.x == 0) { out[0] = acc_issue / (reps - 2); out[1] = acc_done / (reps - 2); }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t) : "memory");
}

template <int N, int NM, int MODE>
void run(long long* d) {
  cudaFuncSetAttribute(k<N, NM, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  k<N, NM, MODE><<<1, 128, 100 * 1024>>>(d, 20);
  long long h[2];
  cudaError_t e = cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return; }
  printf("%s N=%3d nmma=%2d issue %6lld cyc  done %6lld cyc  (%.1f cyc/mma, floor %d)\n", MODE == 0 ? "warp+elect" : "lane0     ",
         N, NM, h[0], h[1], (double)h[1] / NM, 128 * N / 256);
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  run<64, 16, 0>(d); run<64, 32, 0>(d); run<64, 64, 0>(d);
  run<128, 16, 0>(d); run<128, 32, 0>(d);
  run<256, 16, 0>(d); run<256, 32, 0>(d);
  run<64, 16, 1>(d); run<64, 32, 1>(d); run<64, 64, 1>(d);
  run<256, 32, 1>(d);
  return 0;
}
