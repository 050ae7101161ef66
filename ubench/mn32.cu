// Diagnostics: can one V stage serve both MMAs of the streaming kernel if it is stored with the
// 32-byte-atom 128-byte swizzle (Swizzle<2,5,2>: byte bits 5-6 ^= bits 7-8, sm_100 descriptor
// layout type 1, TMA CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)?  V: 64 rows x (tile column) of 64
// bonds (two 32-bond column blocks of 64 x 128 B).  Test 1 (the N/D MMA): B = V MN-major
// (N = 64 bonds, K = 8 rows 8s..8s+7), A[m][x] = (x == m % 8) -> D[m][n] = V[8s + m % 8][n].
// Test 2 (the S MMA): B = V K-major (N = 64 rows, K = 8 bonds 8s..8s+7), A[m][k] = (k == m % 8)
// -> D[m][n] = V[n][8s + m % 8].  Prints mismatches per (layout type, LBO, SBO).
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// byte offset of V[x][k] in the 32-byte-atom swizzled stage
__device__ __forceinline__ int sw32_off(int x, int k, int rows) {
  return (k >> 5) * (rows * 128) + (x >> 3) * 1024 + (x & 7) * 128 + ((((k & 31) >> 3) ^ (x & 3)) << 5) + (k & 7) * 4;
}
__device__ __forceinline__ int sw128_off(int x, int k, int rows) {
  return (k >> 5) * (rows * 128) + (x >> 3) * 1024 + (x & 7) * 128 + ((((k & 31) >> 2) ^ (x & 7)) << 4) + (k & 3) * 4;
}
__global__ void kern(int mode, uint32_t lbo, uint32_t sbo, int step, int swz, int lay, float* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tm;
  const uint32_t base = (smem_u32(sm) + 1023) & ~1023u;
  unsigned char* g = sm + (base - smem_u32(sm));
  const int w = threadIdx.x >> 5;
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tm)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) {
    const int x = i / 64, k = i % 64;
    const int off = lay == 1 ? sw32_off(x, k, 64) : sw128_off(x, k, 64);
    *reinterpret_cast<float*>(g + off) = (float)((x * 37 + k * 11) % 251 + 1);   // exact in TF32
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t t = tm;
  {
    uint32_t r[8];
    const int m = w * 32 + (threadIdx.x & 31);
    for (int j = 0; j < 8; ++j) r[j] = (j == m % 8) ? 0x3f800000u : 0u;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(t + ((uint32_t)(w * 32) << 16)),
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x == 0) {
    // mode 0: MN-major, K step s = 8 rows -> +1024 B; mode 1: K-major, K step s = 8 bonds -> +32 B
    // inside the row (+ 64 rows * 128 B for bonds 32..63)
    const uint32_t addr = mode == 0 ? base + step * 1024 : base + (step & 3) * 32 + (step >> 2) * 64 * 128;
    uint64_t d = ((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) |
                 ((uint64_t)1 << 46) | ((uint64_t)swz << 61);
    uint32_t id = (1u << 4) | (2u << 7) | (2u << 10) | (mode == 0 ? (1u << 16) : 0u) | ((uint32_t)(64 >> 3) << 17) |
                  ((uint32_t)(128 >> 4) << 24);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(t + 64),
                 "r"(t), "l"(d), "r"(id)
                 : "memory");
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n}"
                   : "=r"(ok)
                   : "r"(smem_u32(&bar))
                   : "memory");
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int m = w * 32 + (threadIdx.x & 31);
  for (int n0 = 0; n0 < 64; n0 += 8) {
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(t + 64 + n0 + ((uint32_t)(w * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; ++j) out[m * 64 + n0 + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(t) : "memory");
}
int main(int argc, char** argv) {
  // mn32.bin mode lay swz lbo sbo  (steps 0..7 of one configuration; a fault ends the process)
  const int mode = atoi(argv[1]), lay = atoi(argv[2]), swz = atoi(argv[3]);
  const uint32_t lbo = (uint32_t)atoi(argv[4]), sbo = (uint32_t)atoi(argv[5]);
  float* d;
  cudaMalloc(&d, 128 * 64 * 4);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  static float h[128 * 64];
  for (int step = 0; step < 8; ++step) {
    kern<<<1, 128, 40000>>>(mode, lbo, sbo, step, swz, lay, d);
    cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) { printf("%s lay %d swz %d LBO %u SBO %u step %d: err %s\n", mode == 0 ? "MN" : "K ", lay, swz, lbo, sbo, step, cudaGetErrorString(e)); return 1; }
    int bad = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 64; ++n) {
        const int vx = mode == 0 ? 8 * step + m % 8 : n, vk = mode == 0 ? n : 8 * step + m % 8;
        const float want = (float)((vx * 37 + vk * 11) % 251 + 1);
        if (h[m * 64 + n] != want) ++bad;
      }
    printf("%s lay %d swz %d LBO %5u SBO %5u step %d: mismatches %d  (D[1][0..1] = %g %g)\n", mode == 0 ? "MN" : "K ", lay, swz, lbo,
           sbo, step, bad, h[64], h[65]);
  }
  return 0;
}
