// Micro-benchmark (diagnostics, not product): tcgen05.mma kind::tf32 issue->completion time on
// one SM for M=128, N in {64,128,256}, K=8 per instruction, A from TMEM, B from smem (SW128
// K-major), and the commit -> mbarrier -> waiting-thread latency with and without a suspend
// hint.  One CTA, 128 threads; thread 0 issues.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d), "r"(a), "l"(bdesc), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool try_wait(uint32_t bar, uint32_t par) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n}" : "=r"(ok) : "r"(bar), "r"(par) : "memory");
  return ok;
}
__device__ __forceinline__ bool try_wait_hint(uint32_t bar, uint32_t par) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\tselp.u32 %0,1,0,p;\n}" : "=r"(ok) : "r"(bar), "r"(par), "r"(20000u) : "memory");
  return ok;
}
__device__ __forceinline__ bool test_wait(uint32_t bar, uint32_t par) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n}" : "=r"(ok) : "r"(bar), "r"(par) : "memory");
  return ok;
}

// mode: 0 = ts N, 1 = ss N
__global__ void k(long long* out, int N, int nmma, int reps, int waitmode, int ss) {
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
  // zero smem B
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm + (sB - smem_u32(sm)))[i] = 0x3f800000u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t t = tm;
  const uint32_t b = smem_u32(&bar);
  if (threadIdx.x == 0) {
    const uint32_t id = idesc_tf32(128, N);
    long long acc_issue = 0, acc_done = 0;
    for (int r = 0; r < reps; ++r) {
      long long t0 = clock64();
      for (int i = 0; i < nmma; ++i) {
        const uint64_t bd = sdesc(sB + (i & 3) * 32 + ((i >> 2) & 1) * (N * 128), 16, 1024);
        if (ss) {
          const uint64_t ad = sdesc(sB + 32768 + (i & 3) * 32, 16, 1024);
          mma_ss(t + 256, ad, bd, id, i > 0);
        } else {
          mma_ts(t + 256, t + (i & 7) * 8, bd, id, i > 0);
        }
      }
      commit(b);
      long long t1 = clock64();
      if (waitmode == 0) { while (!try_wait(b, r & 1)) {} }
      else if (waitmode == 1) { while (!try_wait_hint(b, r & 1)) {} }
      else { while (!test_wait(b, r & 1)) {} }
      long long t2 = clock64();
      if (r >= 2) { acc_issue += t1 - t0; acc_done += t2 - t0; }
    }
    out[0] = acc_issue / (reps - 2);
    out[1] = acc_done / (reps - 2);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t) : "memory");
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const char* wn[3] = {"try_wait", "try_wait+hint", "test_wait"};
  for (int ss = 0; ss < 2; ++ss)
    for (int N : {64, 128, 256})
      for (int nm : {1, 8, 16, 32, 64})
        for (int w = 0; w < 3; ++w) {
          if (w != 0 && !(nm == 16)) continue;
          k<<<1, 128, 100 * 1024>>>(d, N, nm, 20, w, ss);
          long long h[2];
          cudaError_t e = cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
          if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
          printf("%s N=%3d nmma=%2d %-14s issue %6lld cyc  done %6lld cyc  (%.1f cyc/mma, floor %d)\n", ss ? "ss" : "ts", N, nm,
                 wn[w], h[0], h[1], (double)h[1] / nm, 128 * N / 256);
        }
  return 0;
}
