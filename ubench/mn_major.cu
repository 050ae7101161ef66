// Diagnostics: tcgen05.mma kind::tf32 with B read MN-major from an SW128 tile that is stored
// K-major for another MMA (the V stage: rows x = tile columns, 128-byte rows of 32 bond
// values k, 8-row swizzle atoms at 1024 B, second 32-k block at +rows*128).  One MMA with
// M = 128, N = 64 (n = k), K = 8 (x = 8s..8s+7); A[m][x] = (x == m % 8) so D[m][n] =
// V[8s + m % 8][n].  Tries LBO / SBO assignments and reports mismatches.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ int sw128_off(int row, int k, int rows) {
  return (k >> 5) * (rows * 128) + (row >> 3) * 1024 + (row & 7) * 128 + ((((k & 31) >> 2) ^ (row & 7)) << 4) + (k & 3) * 4;
}
__global__ void kern(uint32_t lbo, uint32_t sbo, int step, int swz, float* out) {
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
    *reinterpret_cast<float*>(g + sw128_off(x, k, 64)) = (float)(x * 100 + k);
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
    const uint32_t addr = base + step * 1024;
    uint64_t d = ((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) |
                 ((uint64_t)1 << 46) | ((uint64_t)swz << 61);
    // kind::tf32, D f32, A K-major (from TMEM), B MN-major (bit 16), N = 64, M = 128
    uint32_t id = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 16) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(t + 64), "r"(t), "l"(d), "r"(id) : "memory");
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    uint32_t ok = 0;
    while (!ok) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n}" : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
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
int main() {
  float* d;
  cudaMalloc(&d, 128 * 64 * 4);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  float h[128 * 64];
  uint32_t cand[][2] = {{8192, 1024}, {1024, 8192}, {8192, 128}, {128, 8192}, {16, 1024}, {1024, 16}};
  for (int swz : {2, 1})
    for (auto& c : cand)
      for (int step : {0, 3}) {
        kern<<<1, 128, 40000>>>(c[0], c[1], step, swz, d);
        cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        int bad = 0;
        for (int m = 0; m < 128; ++m)
          for (int n = 0; n < 64; ++n)
            if (h[m * 64 + n] != (float)((8 * step + m % 8) * 100 + n)) ++bad;
        printf("swz %d LBO %5u SBO %5u step %d: mismatches %d / 8192  (D[1][0..3] = %g %g %g %g, D[0][33] = %g)\n", swz, c[0], c[1],
               step, bad, h[64], h[65], h[66], h[67], h[33]);
      }
  return 0;
}
