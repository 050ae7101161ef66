// Micro-benchmark (diagnostics): HBM read rate of the fused kernel's Y streaming patterns with
// no compute - one TMA producer lane and one consumer warp per CTA, NS-stage mbarrier ring,
// grid = row blocks x column chunks as the fused kernel launches for c5 (2048 x 2048 x 1024 fp32).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o ubench/tma_stream ubench/tma_stream.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t b, uint32_t n) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(n)); }
__device__ __forceinline__ void mbar_arrive(uint32_t b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory"); }
__device__ __forceinline__ void mbar_expect(uint32_t b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(n) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint32_t b, uint32_t par) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\tselp.u32 %0, 1, 0, p;\n}"
                 : "=r"(done) : "r"(b), "r"(par), "r"(20000u) : "memory");
}
__device__ __forceinline__ void tma2(uint32_t dst, const CUtensorMap* tm, int c0, int c1, uint32_t bar) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
               ::"r"(dst), "l"((uint64_t)tm), "r"(c0), "r"(c1), "r"(bar) : "memory");
}
__device__ __forceinline__ void tma3(uint32_t dst, const CUtensorMap* tm, int c0, int c1, int c2, uint32_t bar) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
               ::"r"(dst), "l"((uint64_t)tm), "r"(c0), "r"(c1), "r"(c2), "r"(bar) : "memory");
}

struct Args {
  CUtensorMap tm;
  int mode;          // 0: L1 two 2-D boxes {32,128}; 1: L1 one 3-D box {32,2,128}; 2: L1 2-D box {64,128} no swizzle;
                     // 3: L1 3-D box {32,4,128} (two tiles per stage); 4: L0 box {128 rows, 64 cols};
                     // 5: L2 3-D two boxes {32,128,1}
  int ns;            // stages
  int stage_bytes;   // bytes per stage
  int tiles_per_stage;
  long long tiles;   // column tiles per row block
  long long tiles_inner;   // L2: tiles per outer index
  int sink;
};

__global__ void __launch_bounds__(64) stream_kernel(const __grid_constant__ Args a, float* out) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bars[16];
  const uint32_t full = smem_u32(&bars[0]), empty = smem_u32(&bars[8]);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < a.ns; ++i) { mbar_init(full + 8 * i, 1); mbar_init(empty + 8 * i, 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int rb = blockIdx.x;
  const long long per = (a.tiles + gridDim.y - 1) / gridDim.y;
  const long long t0 = blockIdx.y * per;
  long long t1 = t0 + per; if (t1 > a.tiles) t1 = a.tiles;
  const int steps = (int)((t1 - t0 + a.tiles_per_stage - 1) / a.tiles_per_stage);
  const uint32_t sb = smem_u32(base);
  if (warp == 0) {
    if (lane == 0) {
      for (int s = 0; s < steps; ++s) {
        const int st = s % a.ns;
        if (s >= a.ns) mbar_wait(empty + 8 * st, ((s / a.ns) - 1) & 1);
        const uint32_t bar = full + 8 * st, dst = sb + st * a.stage_bytes;
        mbar_expect(bar, a.stage_bytes);
        const long long tile = t0 + (long long)s * a.tiles_per_stage;
        const int row0 = rb * 128;
        switch (a.mode) {
          case 0: tma2(dst, &a.tm, (int)(tile * 64), row0, bar); tma2(dst + a.stage_bytes / 2, &a.tm, (int)(tile * 64 + 32), row0, bar); break;
          case 1: case 3: tma3(dst, &a.tm, 0, (int)(tile * 2), row0, bar); break;
          case 2: tma2(dst, &a.tm, (int)(tile * 64), row0, bar); break;
          case 4: tma2(dst, &a.tm, row0, (int)(tile * 64), bar); break;
          case 5: {
            const long long ti = tile % a.tiles_inner, to = tile / a.tiles_inner;
            tma3(dst, &a.tm, (int)(ti * 64), row0, (int)to, bar);
            tma3(dst + a.stage_bytes / 2, &a.tm, (int)(ti * 64 + 32), row0, (int)to, bar);
          } break;
        }
      }
    }
  } else {
    float acc = 0.f;
    for (int s = 0; s < steps; ++s) {
      const int st = s % a.ns;
      mbar_wait(full + 8 * st, (s / a.ns) & 1);
      acc += reinterpret_cast<const float*>(base + st * a.stage_bytes)[lane * 4];
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + 8 * st);
    }
    if (a.sink) out[blockIdx.x * 1024 + blockIdx.y * 32 + lane] = acc;
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;

int main(int argc, char** argv) {
  const long long I = 2048, J = 2048, K = 1024;
  const size_t n = I * J * K;
  float* Y;
  CK(cudaMalloc(&Y, n * 4));
  CK(cudaMemset(Y, 0, n * 4));
  float* out;
  CK(cudaMalloc(&out, 1 << 22));
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const char* names[] = {"L1 2x box{32,128} SW128 (current ell=0)", "L1 1x 3-D box{32,2,128} SW128",
                         "L1 1x box{64,128} no swizzle", "L1 1x 3-D box{32,4,128} SW128 (2 tiles/stage)",
                         "L0 box{128,64} (current ell=2)", "L2 2x 3-D box{32,128,1} SW128 (current ell=1)"};
  for (int mode = 0; mode < 6; ++mode)
    for (int ns = 2; ns <= 6; ++ns) {
      Args a;
      memset(&a, 0, sizeof(a));
      a.mode = mode;
      a.ns = ns;
      a.tiles_per_stage = mode == 3 ? 2 : 1;
      a.stage_bytes = 32768 * a.tiles_per_stage;
      if ((size_t)a.stage_bytes * ns > 200 * 1024) continue;
      long long rows, cols;
      CUresult r;
      cuuint32_t es[3] = {1, 1, 1};
      if (mode <= 3) {
        rows = I; cols = J * K;
        if (mode == 0) {
          cuuint64_t d[2] = {(cuuint64_t)cols, (cuuint64_t)rows}, s[1] = {(cuuint64_t)cols * 4};
          cuuint32_t b[2] = {32, 128};
          r = enc(&a.tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, Y, d, s, b, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else if (mode == 2) {
          cuuint64_t d[2] = {(cuuint64_t)cols, (cuuint64_t)rows}, s[1] = {(cuuint64_t)cols * 4};
          cuuint32_t b[2] = {64, 128};
          r = enc(&a.tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, Y, d, s, b, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else {
          cuuint64_t d[3] = {32, (cuuint64_t)cols / 32, (cuuint64_t)rows}, s[2] = {128, (cuuint64_t)cols * 4};
          cuuint32_t b[3] = {32, (cuuint32_t)(2 * a.tiles_per_stage), 128};
          r = enc(&a.tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, Y, d, s, b, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        a.tiles = cols / 64;
      } else if (mode == 4) {
        rows = K; cols = I * J;
        cuuint64_t d[2] = {(cuuint64_t)rows, (cuuint64_t)cols}, s[1] = {(cuuint64_t)rows * 4};
        cuuint32_t b[2] = {128, 64};
        r = enc(&a.tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, Y, d, s, b, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        a.tiles = cols / 64;
      } else {
        rows = J;   // rows j, inner cols k, outer i
        cuuint64_t d[3] = {(cuuint64_t)K, (cuuint64_t)J, (cuuint64_t)I}, s[2] = {(cuuint64_t)K * 4, (cuuint64_t)K * J * 4};
        cuuint32_t b[3] = {32, 128, 1};
        r = enc(&a.tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, Y, d, s, b, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        a.tiles_inner = K / 64;
        a.tiles = (K / 64) * I;
      }
      if (r != CUDA_SUCCESS) { printf("%-48s ns=%d encode failed %d\n", names[mode], ns, (int)r); continue; }
      const int rbk = (int)(rows / 128);
      const int chunks = sms / rbk > 0 ? sms / rbk : 1;
      const size_t smem = (size_t)a.stage_bytes * ns + 1024;
      CK(cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      dim3 grid(rbk, chunks);
      for (int w = 0; w < 2; ++w) stream_kernel<<<grid, 64, smem>>>(a, out);
      CK(cudaDeviceSynchronize());
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0); cudaEventCreate(&e1);
      const int reps = 5;
      cudaEventRecord(e0);
      for (int i = 0; i < reps; ++i) stream_kernel<<<grid, 64, smem>>>(a, out);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= reps;
      printf("%-48s ns=%d grid %dx%d  %.3f ms  %.0f GB/s\n", names[mode], ns, grid.x, grid.y, ms, n * 4.0 / ms / 1e6);
    }
  return 0;
}
