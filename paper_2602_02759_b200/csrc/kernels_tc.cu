// sm_100a fused streaming pass on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
// One launch = one factor update ell (Algorithm 1 lines 6-8) over the planner's
// 2-D view Y[row, col] of the data:
//   S   = U V^T               (reconstruction tile, TF32 MMA into TMEM; U split hi+lo)
//   P_a = M ? Y^alpha S^(beta-1) : 0,  P_b = M ? S^(alpha+beta-1) : 0     (registers)
//   N  += P_a V,  D += P_b V  (TF32 MMAs, A operand = P in TMEM, accumulators in TMEM)
// Y and the mask are streamed HBM -> smem by TMA exactly once; Yhat, a and b never leave the SM.
//
// CTA = 128 rows (TMEM lanes) x a contiguous range of 64-column tiles, 23 warps:
//   warps 0-15  elementwise: tcgen05.ld S -> a, b (+ loss) -> tcgen05.st P_a over S, P_b beside
//               it (lane quarter = warp % 4, 16-column group = warp / 4); N / D drains, epilogue
//   warps 16-19 V generators: the tile's 64 direct-V table rows (TMA-loaded) scaled in place by
//               the run's constant-row product, TF32 RN, plus the transposed copy V^T (both in
//               the UMMA SW128 K-major layout: V for the reconstruction, V^T for N / D)
//   warp 20     TMA of the direct-V table rows
//   warp 21     TMA producer of the Y (and mask) tiles
//   warp 22     TMEM allocator + MMA issuer (whole warp, elect.sync)
// TMEM (512 columns): tile buffer[2] (S -> P_a in place | P_b, 2 x 128) | N, D (2xKB) | U_hi, U_lo (2xKB)
// The generated-V path (Khatri-Rao products per tile, warps 16-19) remains for lowerings without
// a direct-V table; the planner routes those to the CUDA-core kernel, so it is not exercised.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "divergence.cuh"
#include "kernels.h"
#include "kernels_tc.h"

namespace nef {
namespace tc {

constexpr int BM = 128, BN = 64;
#ifndef NEF_NS
#define NEF_NS 2   // Y stages without a mask stream (3 measured 2 % slower on the c5 fit)
#endif
#ifndef NEF_NS32
#define NEF_NS32 3   // Y stages of bond <= 32 kernels (2 / 3 / 4 measured within 2 %: 3)
#endif
// Y (/ mask) pipeline stages: 3 with the uint8 mask stream (4 for KB = 32), else NEF_NS (NEF_NS32)
template <int KB, int MM> struct YStages {
  static constexpr int value = MM == 2 ? 2 : KB == 32 ? (MM == 1 ? 4 : NEF_NS32) : (MM == 1 ? 3 : NEF_NS);
};
// V tile stages: 3 with a uint8 mask stream (its stages take the smem), else 4
#ifndef NEF_NV0
#define NEF_NV0 4
#endif
// (MM = 2, the per-entry parameter stream: 2 Y + 2 parameter stages; 3 V stages for bond 64)
template <int KB, int MM> struct VStages { static constexpr int value = MM == 1 ? 3 : (MM == 2 && KB == 64) ? 3 : NEF_NV0; };
#ifndef NEF_ULO_BF16
#define NEF_ULO_BF16 1   // bond 64: the U_lo correction of S as BF16 MMAs (K = 16) on a BF16 copy of V (c5 -4 %)
#endif
#if NEF_ULO_BF16 && NEF_SPLIT_ISSUE
#error "NEF_ULO_BF16 has no split-issue path"
#endif
#ifndef NEF_ND_MN
#define NEF_ND_MN 1   // one V copy (32-byte-atom swizzle) read K-major by S and MN-major by N / D: c5 -3 %, c3 -2.3 %, c4 -5.7 %
#endif
#ifndef NEF_PA_RN
#define NEF_PA_RN 0   // 1: plain RN for P_a in the Euclidean pair too (diagnostics)
#endif
// elementwise warp width: 16 warps of 32 rows x 16 tile columns (default), or (NEF_EW_COLS = 32)
// 8 warps of 32 rows x 32 columns - half the per-tile overhead per entry and 136 registers per
// thread instead of 80, but half the warps to hide the TMEM / shared-memory latencies: measured
// 2-3 % slower on c5 and c3, 3 % faster on c4 (the issue-bound (0.5, 0) pair)
#ifndef NEF_EW_COLS
#define NEF_EW_COLS 16
#endif
constexpr int EWC = NEF_EW_COLS;           // tile columns per elementwise warp
constexpr int EWH = EWC / 16;              // 16-column half-steps per elementwise warp and tile
constexpr int NEW = 4 * (BN / EWC);        // elementwise warps: 4 TMEM lane quarters x BN / EWC column groups
constexpr int NVG = 4;                     // V-generator warps (16 tile columns each)
// warp roles: elementwise warps, 4 V generators, direct-V row loads, TMA producer, MMA issuer.
// The warp schedulers favour higher warp ids, so the producers whose latency is on the critical
// path sit above the elementwise warps (with the producers below, the V generators and the MMA
// issuer starved during the elementwise phase of every tile).
// NEF_SPLIT_ISSUE: the reconstruction MMAs S(t) are issued by a second warp on another
// sub-partition (after the N/D MMAs of the tile whose buffer they overwrite have retired), so the
// sub-partition hosting the N/D issuer carries half the tcgen05.mma issue (experiment)
#ifndef NEF_SPLIT_ISSUE
#define NEF_SPLIT_ISSUE 0
#endif
// NEF_ND_BAR: the N/D issuer waits for P(t) on a named barrier (bar.sync, no polling) that the
// elementwise warps bar.arrive on (experiment)
#ifndef NEF_ND_BAR
#define NEF_ND_BAR 1   // measured: the polling issuer made its sub-partition's elementwise warps lag
                       // ~1 400 cycles per tile (c5 trace); with the barrier ~300
#endif
// NEF_S_WATCH: a watcher warp polls S(t)'s mbarrier and releases the elementwise warps through a
// named barrier, so elementwise warps that finish a tile early sleep instead of polling (experiment)
#ifndef NEF_S_WATCH
#define NEF_S_WATCH 0
#endif
// NEF_WARP_MAP 2 (experiment): the MMA issuer's sub-partition (warp % 4 == 2) hosts no other
// producer - V generators on warps 16, 17, 19, 23, the direct-V loads on 21, warp 18 idle
#ifndef NEF_WARP_MAP
#define NEF_WARP_MAP 3   // measured (ab7): c4 -1.9 %, c3 -0.5 %, c5 -0.2 % against the V generators above the elementwise warps
#endif
#if NEF_WARP_MAP == 3
// V generators below the elementwise warps (the schedulers favour higher warp ids: the V
// generators, which run a tile ahead, take the issue slots the elementwise warps leave idle)
constexpr int W_VG0 = 0, W_EW0 = NVG, W_DV = NEW + 4, W_TMA = NEW + 5, W_MMA = NEW + 6, W_MMA2 = NEW + 7;
constexpr int W_SW = NEW + 7 + NEF_SPLIT_ISSUE;
__device__ __forceinline__ int vg_index(int warp) { return warp < NVG ? warp : -1; }
constexpr int NTHREADS = (NEW + 7 + NEF_SPLIT_ISSUE + NEF_S_WATCH) * 32;
#elif NEF_WARP_MAP == 2
constexpr int W_EW0 = 0, W_VG0 = NEW, W_DV = NEW + 5, W_TMA = NEW + 4, W_MMA = NEW + 6, W_MMA2 = NEW + 8;
constexpr int W_SW = NEW + 8 + NEF_SPLIT_ISSUE;
__device__ __forceinline__ int vg_index(int warp) {
  return warp == NEW ? 0 : warp == NEW + 1 ? 1 : warp == NEW + 3 ? 2 : warp == NEW + 7 ? 3 : -1;
}
constexpr int NTHREADS = (NEW + 8 + NEF_SPLIT_ISSUE + NEF_S_WATCH) * 32;
#else
constexpr int W_EW0 = 0, W_VG0 = NEW, W_DV = NEW + 4, W_TMA = NEW + 5, W_MMA = NEW + 6, W_MMA2 = NEW + 7;
constexpr int W_SW = NEW + 7 + NEF_SPLIT_ISSUE;   // S watcher (NEF_S_WATCH)
__device__ __forceinline__ int vg_index(int warp) { return warp >= W_VG0 && warp < W_VG0 + NVG ? warp - W_VG0 : -1; }
constexpr int NTHREADS = (NEW + 7 + NEF_SPLIT_ISSUE + NEF_S_WATCH) * 32;
#endif
constexpr int Y_STAGE = BM * BN * 4;      // 32 KB
constexpr int M_STAGE = BM * BN;          // 8 KB
// a V stage: V (64 tile columns x KB bonds, SW128 K-major) then its transpose V^T, KB * 256 B each
template <int KB> struct VSt {
  static constexpr int VT_OFF = BN * KB * 4;     // V^T copy after V inside a stage
  static constexpr bool ULB = NEF_ULO_BF16 && KB == 64;   // BF16 copy of V for the U_lo MMAs
  static constexpr int VB_OFF = NEF_ND_MN ? VT_OFF : 2 * VT_OFF;
  static constexpr int SIZE = VB_OFF + (ULB ? BN * KB * 2 : 0);   // (NEF_ND_MN: V only)
};

struct __align__(64) Params {
  CUtensorMap tmY;
  CUtensorMap tmM;
  CUtensorMap tmA;   // MM = 2: per-entry loss parameter stream (phi_i / n_i), Y's geometry
  CUtensorMap tmV[kMaxRestarts];   // direct-V table rows per restart (2-D {K, var_rows}, box {32, 64}, SW128)
  TcArgs a;
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// Wait with a suspend-time hint: the warp sleeps until the phase completes (no issue slots
// burnt on polling).  Bounded: a pipeline bug traps (kernel error) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  for (uint32_t it = 0;; ++it) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(bar), "r"(parity), "r"(20000u)
        : "memory");
    if (done) return;
    if (it > (1u << 22)) __trap();
  }
}
// Spin variant for waits on the critical path (no suspend hint: a suspended waiter was seen to
// wake ~1000 cycles after the phase completed).  Still bounded.
#ifndef NEF_SPIN_HINT
#define NEF_SPIN_HINT 0
#endif
#ifndef NEF_SPIN_BOUND
#define NEF_SPIN_BOUND 2   // 2: eight two-instruction polls per bound check (c3 -2 %, c4 -3 % against 1:
                           // a bound check per poll, five instructions); 0: unbounded (experiment)
#endif
__device__ __forceinline__ void mbar_spin(uint32_t bar, uint32_t parity) {
#if NEF_SPIN_BOUND == 2
  // eight polls of two instructions (try_wait, branch) per bound check; traps after 2^24 rounds
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .u32 c;\n\t"
      "mov.u32 c, 0;\n\t"
      "SPIN_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@p bra DONE_%=;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@p bra DONE_%=;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@p bra DONE_%=;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@p bra DONE_%=;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@p bra DONE_%=;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@p bra DONE_%=;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@p bra DONE_%=;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@p bra DONE_%=;\n\t"
      "add.u32 c, c, 1;\n\t"
      "setp.lt.u32 p, c, 16777216;\n\t"
      "@p bra SPIN_%=;\n\t"
      "trap;\n\t"
      "DONE_%=:\n}" ::"r"(bar), "r"(parity)
      : "memory");
  return;
#endif
#if !NEF_SPIN_BOUND
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "SPIN_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra SPIN_%=;\n}" ::"r"(bar), "r"(parity)
      : "memory");
  return;
#endif
  uint32_t done = 0;
  for (uint32_t it = 0;; ++it) {
#if NEF_SPIN_HINT
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(bar), "r"(parity), "r"(NEF_SPIN_HINT)
        : "memory");
#else
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
#endif
    if (done) return;
    if (it > (1u << 26)) __trap();
  }
}
// Producer-side wait (the producer runs ahead of its consumer): poll with a short sleep
// between tries so the waiting warp leaves the issue slots to the elementwise warps
// (NEF_PROD_HINT=1: suspend-hint try_wait instead, measured 0.5 % slower on c5).
#ifndef NEF_PROD_HINT
#define NEF_PROD_HINT 0
#endif
__device__ __forceinline__ void mbar_wait_relaxed(uint32_t bar, uint32_t parity, uint32_t ns = 256) {
#if NEF_PROD_HINT
  // suspend-hint try_wait: the waiting thread sleeps until the phase completes (or the hint
  // elapses) without polling
  (void)ns;
  mbar_wait(bar, parity);
  return;
#endif
  uint32_t done = 0;
  for (uint32_t it = 0;; ++it) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (done) return;
#ifdef NEF_PROD_NS
    ns = NEF_PROD_NS;   // diagnostics: one sleep length for every producer wait (0: spin)
#endif
    if (ns) __nanosleep(ns);
    if (it > (1u << 26)) __trap();
  }
}
// MMA-issuer wait (NEF_MMA_WAIT: 0 spin - the default, measured 1.5-2 % faster than a 32 ns
// back-off on c5 - else nanoseconds of sleep per failed poll)
#ifndef NEF_MMA_WAIT
#define NEF_MMA_WAIT 0
#endif
__device__ __forceinline__ void mbar_wait_mma(uint32_t bar, uint32_t parity) {
#if NEF_MMA_WAIT == -1
  mbar_wait(bar, parity);   // suspend-time hint: descheduled until the phase completes
#elif NEF_MMA_WAIT
  mbar_wait_relaxed(bar, parity, NEF_MMA_WAIT);
#else
  mbar_spin(bar, parity);
#endif
}
// Elementwise warps waiting for S (NEF_EW_WAIT: 0 spin - the default, measured 1 % faster on
// c5 than a 32 ns back-off once the MMA issuer also spins - 1 suspend-hint wait, else
// nanoseconds of sleep between polls)
#ifndef NEF_EW_WAIT
#define NEF_EW_WAIT 0
#endif
__device__ __forceinline__ void mbar_wait_ew(uint32_t bar, uint32_t parity) {
#if NEF_EW_WAIT == 0
  mbar_spin(bar, parity);
#elif NEF_EW_WAIT == 1
  mbar_wait(bar, parity);
#else
  mbar_wait_relaxed(bar, parity, NEF_EW_WAIT);
#endif
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* tm, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* tm, int c0, int c1, int c2, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// D[tmem] (+)= A[tmem] * B[smem desc], kind::tf32, one CTA
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
// the same, issued by one elected lane of a converged warp (warp-uniform operands)
__device__ __forceinline__ void mma_ts_elect(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
#include "mma_blocks.inc"
// instruction descriptor: kind::f16 with BF16 A and B, D f32, K-major
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// S += U_lo V in BF16 (NEF_ULO_BF16, bond 64): four K = 16 MMAs, A = U_lo packed two per TMEM
// column (alo + 8 s), B = the stage's BF16 copy of V (K-major 128-byte swizzle, +32 B per step)
template <uint32_t IDESC>
__device__ __forceinline__ void mma_slo_bf16_64(uint32_t d, uint32_t alo, uint64_t b) {
  asm volatile(
      "{\n\t"
      ".reg .pred e, t;\n\t"
      ".reg .b32 bl, bh, bk, ak;\n\t"
      ".reg .b64 bd;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.eq.b32 t, %1, %1;\n\t"
      "mov.b64 {bl, bh}, %2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, t;\n\t"
      "add.u32 ak, %1, 8;\n\t"
      "add.u32 bk, bl, 2;\n\t"
      "mov.b64 bd, {bk, bh};\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ak], bd, %3, t;\n\t"
      "add.u32 ak, %1, 16;\n\t"
      "add.u32 bk, bl, 4;\n\t"
      "mov.b64 bd, {bk, bh};\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ak], bd, %3, t;\n\t"
      "add.u32 ak, %1, 24;\n\t"
      "add.u32 bk, bl, 6;\n\t"
      "mov.b64 bd, {bk, bh};\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ak], bd, %3, t;\n\t"
      "}\n" ::"r"(d),
      "r"(alo), "l"(b), "n"(IDESC)
      : "memory");
}
__device__ __forceinline__ void mma_commit_elect(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(bar)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

#define NEF_R16(x)                                                                                              \
  "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]), "=r"(x[4]), "=r"(x[5]), "=r"(x[6]), "=r"(x[7]), "=r"(x[8]), \
      "=r"(x[9]), "=r"(x[10]), "=r"(x[11]), "=r"(x[12]), "=r"(x[13]), "=r"(x[14]), "=r"(x[15])
#define NEF_P16(x)                                                                                              \
  "+r"(x[0]), "+r"(x[1]), "+r"(x[2]), "+r"(x[3]), "+r"(x[4]), "+r"(x[5]), "+r"(x[6]), "+r"(x[7]), "+r"(x[8]), \
      "+r"(x[9]), "+r"(x[10]), "+r"(x[11]), "+r"(x[12]), "+r"(x[13]), "+r"(x[14]), "+r"(x[15])
#define NEF_W16(x)                                                                                                \
  "r"(x[0]), "r"(x[1]), "r"(x[2]), "r"(x[3]), "r"(x[4]), "r"(x[5]), "r"(x[6]), "r"(x[7]), "r"(x[8]), "r"(x[9]), \
      "r"(x[10]), "r"(x[11]), "r"(x[12]), "r"(x[13]), "r"(x[14]), "r"(x[15])

// 16 / 32 consecutive TMEM columns of this thread's lane
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, "
      "[%16];"
      : NEF_R16(r)
      : "r"(taddr));
}
// wait for tcgen05.ld; the registers are tied in so no use can be scheduled above the wait
__device__ __forceinline__ void tmem_ld_wait(uint32_t (&r)[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" : NEF_P16(r) : : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16};" ::"r"(taddr),
      NEF_W16(r)
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}


// UMMA shared-memory descriptor, sm_100 (version 1); layout 2 = SWIZZLE_128B, 1 = SWIZZLE_128B
// with 32-byte atoms (the V stage under NEF_ND_MN)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout = 2) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}
// The V stage (rows = tile columns, 128-byte rows of 32 bonds, a 32-bond column block per
// BN * 128 bytes).  NEF_ND_MN: the 128-byte swizzle with 32-byte atoms (byte bits 5-6 ^= bits 7-8;
// descriptor layout 1, TMA SWIZZLE_128B_ATOM_32B), which the tensor core reads both K-major (the
// reconstruction, B = V with K = bonds; LBO = BN * 128, SBO = 512) and MN-major (numerator /
// denominator, B = V with N = bonds, K = tile columns) - one copy of V serves both MMAs
// (ubench/mn32.cu).  Otherwise the plain 128-byte swizzle, V^T beside it.
// 16-byte chunk j of a V row r: its physical chunk
__device__ __forceinline__ int v_chunk(int j, int r) {
  return NEF_ND_MN ? ((((j >> 1) ^ (r & 3)) << 1) | (j & 1)) : (j ^ (r & 7));
}
__device__ __forceinline__ int v_off(int row, int k, int rows) {
  return (k >> 5) * (rows * 128) + (row >> 3) * 1024 + (row & 7) * 128 + (v_chunk((k & 31) >> 2, row) << 4) + (k & 3) * 4;
}
// instruction descriptor: kind::tf32, D f32, A/B tf32, A and B K-major
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// byte offset of element (row, k) in an SW128 K-major operand whose rows are 128-byte atoms,
// `rows` rows per atom column block (atom column = 32 fp32 along K)
__device__ __forceinline__ int sw128_off(int row, int k, int rows) {
  return (k >> 5) * (rows * 128) + (row >> 3) * 1024 + (row & 7) * 128 + ((((k & 31) >> 2) ^ (row & 7)) << 4) +
         (k & 3) * 4;
}

// ------------------------------------------------------------------ column operand generator
// Table rows of one tile held in registers (software pipelining across tiles).
template <int KB>
struct VTile;

// Lane -> 4x4 block assignment of the V generators.  Lane owns bond chunk c (bonds 4c..4c+3) and,
// for block i, row group rg (rows 4 rg..4 rg+3 of the warp's 16).  A 16-byte shared access is
// served per quarter warp (8 lanes); the 8 lanes of a quarter hit 8 distinct 16-byte chunk slots
// both in V (slot (c & 7) ^ (x0 & 7)) and in V^T (slot (x0 >> 2 & 7) ^ 4 (c & 1)): with q = lane & 3,
// p = lane >> 2 & 1, a quarter with rotation g takes c & 7 = p + 2 ((q + g) & 3) and rg = q ^ 2i.
// (c = lane % C with rg = lane / C would put 8 lanes of one quarter on two V^T slots.)
template <int KB>
__device__ __forceinline__ int vl_c(int lane) {
  static_assert(KB == 32 || KB == 64, "V lane map: KB 32 or 64");
  const int qq = lane >> 3, p = (lane >> 2) & 1, q = lane & 3;
  const int g = KB == 64 ? (qq & 1) : qq;
  const int h = KB == 64 ? (qq >> 1) : 0;
  return 8 * h + p + 2 * ((q + g) & 3);
}
__device__ __forceinline__ int vl_rg(int lane, int i) { return (lane & 3) ^ (2 * i); }

template <int KB>
struct VTile {
  static constexpr int C = KB / 4;          // 16-byte chunks per padded row
  static constexpr int NB = (4 * C) / 32;   // 4x4 blocks per lane (16 rows = 4 row groups per warp)
  float4 ld[NB][4];                         // varying-table rows r of block i, chunk c
  float4 cst;                               // product of the tile-constant rows (chunk c)
  uint32_t vmask;                           // valid tile columns of this warp (16 bits)
  int mode;                                 // 0 fast (<= 1 varying table), 1 general, 2 empty
};

// Mixed-radix odometer of a lane's linear column index over the column modes: advanced by
// the (small, nonnegative) step between consecutive tiles; divides only when a digit wraps.
// Digits live in registers (loops fully unrolled over kMaxModes, guarded by nc).
struct Odo {
  int64_t col = -1;
  int dig[kMaxModes];
};

__device__ __forceinline__ void odo_seek(const TcArgs& a, Odo& o, int64_t col) {
  if (o.col < 0) {
    int64_t rem = col;
#pragma unroll
    for (int d = kMaxModes - 1; d >= 0; --d) {
      if (d >= a.nc) { o.dig[d] = 0; continue; }
      if (d > 0) {
        o.dig[d] = (int)(rem % a.cdim[d]);
        rem /= a.cdim[d];
      } else {
        o.dig[d] = (int)rem;
      }
    }
  } else {
    int carry = (int)(col - o.col);
#pragma unroll
    for (int d = kMaxModes - 1; d >= 0; --d) {
      if (d >= a.nc || carry == 0) continue;
      const int v = o.dig[d] + carry;
      const int n = (int)a.cdim[d];
      if (d == 0 || v < n) {
        o.dig[d] = v;
        carry = 0;
      } else {
        o.dig[d] = v % n;
        carry = v / n;
      }
    }
  }
  o.col = col;
}

// Column offsets of this warp's 16 tile columns (lane & 15), validity, and - on the vector
// path - the loads of the next tile's table rows: lane owns 4x4 blocks (4 rows x 4 bonds).
template <int KB>
__device__ __forceinline__ void vtile_issue(const TcArgs& a, int64_t tile, int xw, int lane, VTile<KB>& v,
                                            int (&toff)[kMaxTabs], Odo& odo) {
  using VT = VTile<KB>;
  const int x = xw + (lane & 15);
  int64_t col;
  bool valid;
  if (a.layout == 0) {
    col = tile * BN + x;
    valid = col < a.CO;
  } else {
    const int64_t ti = tile % a.tiles_inner, to = tile / a.tiles_inner;
    const int64_t ci = ti * BN + x;
    valid = ci < a.CI;
    col = to * a.CI + ci;
  }
  odo_seek(a, odo, col);
#pragma unroll
  for (int q = 0; q < kMaxTabs; ++q) {
    int o = 0;
#pragma unroll
    for (int d = 0; d < kMaxModes; ++d)
      if (q < a.ntab && d < a.nc) o += odo.dig[d] * (int)a.tcs[q][d];
    toff[q] = valid ? o : 0;
  }
  v.vmask = __ballot_sync(0xffffffffu, valid) & 0xffffu;
  if (v.vmask == 0u || !a.vec4) {
    v.mode = v.vmask == 0u ? 2 : 1;
    return;
  }
  const int first = __ffs(v.vmask) - 1;
  const int c = vl_c<KB>(lane);
  const bool kok = c * 4 < a.K;
  int nvar = 0, var_q = -1;
  v.cst = make_float4(1.f, 1.f, 1.f, 1.f);
#pragma unroll
  for (int q = 0; q < kMaxTabs; ++q) {
    if (q >= a.ntab) break;
    const int t0 = __shfl_sync(0xffffffffu, toff[q], first);
    const bool uni = __all_sync(0xffffffffu, !valid || toff[q] == t0);
    if (uni) {
      const float4 r = kok ? __ldg(reinterpret_cast<const float4*>(a.tab[q] + t0) + c) : make_float4(0.f, 0.f, 0.f, 0.f);
      v.cst.x *= r.x; v.cst.y *= r.y; v.cst.z *= r.z; v.cst.w *= r.w;
    } else {
      ++nvar;
      var_q = q;
    }
  }
  if (nvar > 1) {
    v.mode = 1;
    return;
  }
  v.mode = 0;
  if (var_q < 0) {
#pragma unroll
    for (int i = 0; i < VT::NB; ++i)
#pragma unroll
      for (int r = 0; r < 4; ++r) v.ld[i][r] = make_float4(1.f, 1.f, 1.f, 1.f);
    return;
  }
  int tv = toff[0];
#pragma unroll
  for (int q = 1; q < kMaxTabs; ++q)
    if (q == var_q) tv = toff[q];
  const float4* tab = reinterpret_cast<const float4*>(a.tab[var_q]);
#pragma unroll
  for (int i = 0; i < VT::NB; ++i) {
    const int rg = vl_rg(lane, i);   // row group of block i
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int xr = 4 * rg + r;
      const int to = __shfl_sync(0xffffffffu, tv, xr);
      v.ld[i][r] = (((v.vmask >> xr) & 1u) && kok) ? __ldg(tab + (to >> 2) + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
}

// Per-lane smem byte offsets of its 4x4 blocks inside a V stage (constant over tiles).
// Per-lane smem byte offsets of its 4x4 blocks inside a V stage (constant over tiles).  Rows
// x0..x0+3 (x0 % 4 == 0) share one 8-row swizzle group, so row r of V sits at
//   vb + r*128 + ((cx ^ r) << 4)   with cx = (c & 7) ^ (x0 & 7),
// and bond 4c+e of V^T at  vtb + e*128 + ((xc ^ e) << 4)  with xc = ((x0 & 31) >> 2) ^ (4 (c & 1)).
template <int KB>
struct VOff {
  static constexpr int C = KB / 4, NB = (4 * C) / 32;
  int vb[NB], vtb[NB], cx[NB], xc[NB];
  int c16, rowoff[NB], x7[NB];   // (BF16 copy of V: bond chunk, row offset and row & 7 of each block)
  __device__ __forceinline__ void init(int xw, int lane) {
    const int c = vl_c<KB>(lane);
    c16 = c;
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      const int x0 = xw + 4 * vl_rg(lane, i);
      rowoff[i] = (x0 >> 3) * 1024 + (x0 & 7) * 128;
      x7[i] = x0 & 7;
      vb[i] = (c >> 3) * (BN * 128) + (x0 >> 3) * 1024 + (x0 & 7) * 128;
      cx[i] = NEF_ND_MN ? (c & 7) : ((c & 7) ^ (x0 & 7));   // (v_chunk(cx, r): the 4 rows of the block)
      const int k0 = 4 * c;
      vtb[i] = VSt<KB>::VT_OFF + (x0 >> 5) * (KB * 128) + (k0 >> 3) * 1024 + (k0 & 7) * 128;
      xc[i] = ((x0 & 31) >> 2) ^ (k0 & 7);
    }
  }
};

// BF16 copy of V (VSt::ULB, K-major 128-byte swizzle: row x = 64 bonds in 128 bytes): the 4x4 block
// at rows x0..x0+3 (rowoff, x7 = x0 & 7), bonds 4c..4c+3 as four 8-byte stores, RN
template <int KB>
__device__ __forceinline__ void vb16_store(unsigned char* vrow, int rowoff, int x7, int c, const float4 (&p)[4],
                                           uint32_t okbits = 0xfu) {
  if constexpr (VSt<KB>::ULB) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const uint32_t m = ((okbits >> r) & 1u) ? 0xffffffffu : 0u;
      const __nv_bfloat162 lo = __floats2bfloat162_rn(p[r].x, p[r].y), hi = __floats2bfloat162_rn(p[r].z, p[r].w);
      const uint2 v = make_uint2(*reinterpret_cast<const uint32_t*>(&lo) & m, *reinterpret_cast<const uint32_t*>(&hi) & m);
      *reinterpret_cast<uint2*>(vrow + VSt<KB>::VB_OFF + rowoff + r * 128 + ((((c >> 1) ^ ((x7 + r) & 7))) << 4) + (c & 1) * 8) = v;
    }
  }
}
// Store one 4x4 block (rows x0..x0+3, bonds 4c..4c+3): four 16-byte rows of V and four
// 16-byte columns of V^T, TF32 round-to-nearest, zeros where invalid.
template <int KB>
__device__ __forceinline__ void vblock_store(unsigned char* vrow, int vb, int cx, int vtb, int xc, uint32_t okbits,
                                             const float4 (&p)[4]) {
  uint32_t w[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const uint32_t m = ((okbits >> r) & 1u) ? 0xffffffffu : 0u;
    w[r][0] = tf32_bits(p[r].x) & m;
    w[r][1] = tf32_bits(p[r].y) & m;
    w[r][2] = tf32_bits(p[r].z) & m;
    w[r][3] = tf32_bits(p[r].w) & m;
    *reinterpret_cast<uint4*>(vrow + vb + r * 128 + (v_chunk(cx, r) << 4)) = make_uint4(w[r][0], w[r][1], w[r][2], w[r][3]);
  }
  if (!NEF_ND_MN) {
#pragma unroll
    for (int e = 0; e < 4; ++e)
      *reinterpret_cast<uint4*>(vrow + vtb + e * 128 + ((xc ^ e) << 4)) = make_uint4(w[0][e], w[1][e], w[2][e], w[3][e]);
  }
}

// Direct path: bonds beyond K are TMA zero fill times a zero constant row, rows beyond the
// table are zero fill, so no masking; + half a TF32 ulp = RN of what the tensor core truncates
template <int KB>
__device__ __forceinline__ void vblock_store_direct(unsigned char* vrow, int vb, int cx, int vtb, int xc,
                                                    const float4 (&p)[4]) {
  uint32_t w[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    w[r][0] = __float_as_uint(p[r].x) + 0x1000u;
    w[r][1] = __float_as_uint(p[r].y) + 0x1000u;
    w[r][2] = __float_as_uint(p[r].z) + 0x1000u;
    w[r][3] = __float_as_uint(p[r].w) + 0x1000u;
    *reinterpret_cast<uint4*>(vrow + vb + r * 128 + (v_chunk(cx, r) << 4)) = make_uint4(w[r][0], w[r][1], w[r][2], w[r][3]);
  }
  if (!NEF_ND_MN) {
#pragma unroll
    for (int e = 0; e < 4; ++e)
      *reinterpret_cast<uint4*>(vrow + vtb + e * 128 + ((xc ^ e) << 4)) = make_uint4(w[0][e], w[1][e], w[2][e], w[3][e]);
  }
}

// Slow paths (several varying tables, or non-vectorisable tables), out of line so the fast
// path keeps its registers.
template <int KB>
__device__ __noinline__ void vtile_store_slow(const TcArgs& a, int xw, int lane, const VTile<KB>& v,
                                              const int (&toff)[kMaxTabs], unsigned char* vrow, const VOff<KB>& vo) {
  using VT = VTile<KB>;
  const int c = vl_c<KB>(lane);
  const bool kok = c * 4 < a.K;
  if (a.vec4) {
    // general vector path: several varying tables, rows multiplied table by table
#pragma unroll
    for (int i = 0; i < VT::NB; ++i) {
      const int rg = vl_rg(lane, i);
      float4 p[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) p[r] = make_float4(1.f, 1.f, 1.f, 1.f);
      for (int q = 0; q < a.ntab; ++q) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int xr = 4 * rg + r;
          const int to = __shfl_sync(0xffffffffu, toff[q], xr);
          const float4 t = (((v.vmask >> xr) & 1u) && kok) ? __ldg(reinterpret_cast<const float4*>(a.tab[q] + to) + c)
                                                          : make_float4(0.f, 0.f, 0.f, 0.f);
          p[r].x *= t.x; p[r].y *= t.y; p[r].z *= t.z; p[r].w *= t.w;
        }
      }
      const uint32_t ok = kok ? ((v.vmask >> (4 * rg)) & 0xfu) : 0u;
      vblock_store<KB>(vrow, vo.vb[i], vo.cx[i], vo.vtb[i], vo.xc[i], ok, p);
      vb16_store<KB>(vrow, vo.rowoff[i], vo.x7[i], vo.c16, p, ok);
    }
    return;
  }
  {
    // scalar path (bond not contiguous / unaligned rows): lane = bond index k (+32 h)
#pragma unroll 1
    for (int i = 0; i < 16; ++i) {
      const int x = xw + i;
      const bool vi = (v.vmask >> i) & 1u;
#pragma unroll
      for (int h = 0; h < KB / 32; ++h) {
        const int k = h * 32 + lane;
        float p = (vi && k < a.K) ? 1.f : 0.f;
        for (int q = 0; q < a.ntab; ++q) {
          const int to = __shfl_sync(0xffffffffu, toff[q], i);
          if (p != 0.f) p *= __ldg(a.tab[q] + to + a.boff[q][k]);
        }
        const uint32_t w = tf32_bits(p);
        *reinterpret_cast<uint32_t*>(vrow + v_off(x, k, BN)) = w;
        if constexpr (VSt<KB>::ULB)
          *reinterpret_cast<__nv_bfloat16*>(vrow + VSt<KB>::VB_OFF + (x >> 3) * 1024 + (x & 7) * 128 +
                                            (((k >> 3) ^ (x & 7)) << 4) + (k & 7) * 2) = __float2bfloat16_rn(p);
        if (!NEF_ND_MN) *reinterpret_cast<uint32_t*>(vrow + VSt<KB>::VT_OFF + sw128_off(k, x, KB)) = w;
      }
    }
  }
}

template <int KB>
__device__ __forceinline__ void vtile_store(const TcArgs& a, int xw, int lane, const VTile<KB>& v,
                                            const int (&toff)[kMaxTabs], unsigned char* vrow, const VOff<KB>& vo) {
  using VT = VTile<KB>;
  const int c = vl_c<KB>(lane);
  const bool kok = c * 4 < a.K;
  if (v.mode == 1) {
    vtile_store_slow<KB>(a, xw, lane, v, toff, vrow, vo);
    return;
  }
  // fast path (mode 0: constant rows x one varying table) and empty tiles (mode 2: zeros)
#pragma unroll
  for (int i = 0; i < VT::NB; ++i) {
    const int rg = vl_rg(lane, i);
    float4 p[4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
      p[r] = make_float4(v.cst.x * v.ld[i][r].x, v.cst.y * v.ld[i][r].y, v.cst.z * v.ld[i][r].z, v.cst.w * v.ld[i][r].w);
    const uint32_t ok = (v.mode == 0 && kok) ? ((v.vmask >> (4 * rg)) & 0xfu) : 0u;
    vblock_store<KB>(vrow, vo.vb[i], vo.cx[i], vo.vtb[i], vo.xc[i], ok, p);
    vb16_store<KB>(vrow, vo.rowoff[i], vo.x7[i], vo.c16, p, ok);
  }
}

// ------------------------------------------------------------------ elementwise stage
// Row m's 16 Y values of half-step h of column half g (tile columns [32g + 16h, +16)) and
// their mask bytes, four per word (missing values are loaded but only ever feed discarded
// lanes).  Layouts 1 / 2 keep Y in SW128 128-byte lines of 32 columns: line yl at byte yoff,
// 16-byte chunk j stored at chunk j ^ (yl & 7) - two [128 rows][32] boxes (line m of half g)
// or, with a.y3d, one [128 rows][2 halves][32] box (line 2m + g); yoff / yswz are per-warp
// constants computed once (ew_y_line).
__device__ __forceinline__ void ew_y_line(const TcArgs& a, int g, int m, int& yoff, int& yswz) {
  const int yl = a.y3d ? 2 * m + g : m;
  yoff = a.y3d ? yl * 128 : g * (Y_STAGE / 2) + m * 128;
  yswz = yl & 7;
}
__device__ __forceinline__ void ew_load_y(const TcArgs& a, const unsigned char* ys, const unsigned char* ms, int g,
                                          int h, int m, int yoff, int yswz, float (&yv)[16], uint32_t (&mk)[4]) {
  const int c0 = 32 * g + 16 * h;
  if (a.layout == 0) {
    // [64 columns][128 rows] fp32 / uint8, rows contiguous: lane = row, conflict-free
    const float* yf = reinterpret_cast<const float*>(ys) + c0 * BM + m;
#pragma unroll
    for (int j = 0; j < 16; ++j) yv[j] = yf[j * BM];
    if (a.has_mask) {
      const unsigned char* mb = ms + c0 * BM + m;
#pragma unroll
      for (int j4 = 0; j4 < 4; ++j4) {
        uint32_t w = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) w |= (uint32_t)mb[(4 * j4 + e) * BM] << (8 * e);
        mk[j4] = w;
      }
    }
  } else {
    // (a.y3d: rows m and m + 4 share a swizzle phase -> 2-way bank conflict, cheaper than
    // reading the chunk pairs swapped and selecting them back: measured +3 % c5, +5 % c3)
    const unsigned char* sub = ys + yoff;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 f = *reinterpret_cast<const float4*>(sub + (((4 * h + q) ^ yswz) << 4));
      yv[4 * q] = f.x; yv[4 * q + 1] = f.y; yv[4 * q + 2] = f.z; yv[4 * q + 3] = f.w;
    }
    if (a.has_mask) {
      // SW64 [128 rows][64] uint8
      const int q = 2 * g + h;
      const uint4 w = *reinterpret_cast<const uint4*>(ms + m * 64 + ((q ^ ((m >> 1) & 3)) << 4));
      mk[0] = w.x; mk[1] = w.y; mk[2] = w.z; mk[3] = w.w;
    }
  }
}

// TF32 rounding of P_a (R27).  The tensor core reads the top 19 bits of each operand, so adding
// d before it truncates rounds with probability set by d: a constant half ulp (0x1000) is
// round-to-nearest.  For the Euclidean pair a = x is the data itself, and count-like data
// (integers, or integers plus a small offset) above 2^11 sits on or next to the TF32 grid in a
// fixed pattern, so RN errs in one direction on average (measured 1e-4 factor bias on Poisson
// Tucker problems, scripts/emulate_tf32_tucker.py).  There the 16 entries of a half-step take
// 16 stratified offsets (k + 1/2)/16 ulp, unbiased up to 1/32 ulp, at no extra instruction (the
// offsets are immediates).  Every other pair scales x by a continuous factor: plain RN.
template <int KIND>
__host__ __device__ constexpr uint32_t pa_round(int j) {
  return (KIND == EW_EUC && !NEF_PA_RN) ? 0x100u + 0x200u * (uint32_t)j : 0x1000u;
}

// Yhat floor of two reconstructed entries (reading R4: max(S, 1e-30)).  S >= 0 (nonnegative
// operands), so S + 1e-30 is the same value wherever S > 1e-23 (1e-30 is below half an ulp) and
// 1e-30 at S = 0: one packed add on the FMA pipe instead of two max on the (busier) ALU pipe.
// NEF_YH_MAX=1: the max form.
#ifndef NEF_YH_MAX
#define NEF_YH_MAX 0
#endif
__device__ __forceinline__ float2 yhat_floor(uint32_t s0, uint32_t s1) {
#if NEF_YH_MAX
  return make_float2(fmaxf(__uint_as_float(s0), 1e-30f), fmaxf(__uint_as_float(s1), 1e-30f));
#else
  return __fadd2_rn(make_float2(__uint_as_float(s0), __uint_as_float(s1)), make_float2(1e-30f, 1e-30f));
#endif
}

// a, b (and, in loss mode, the loss) of 16 entries: sv holds S on entry and P_a on exit, pb
// receives P_b; zero at missing or out-of-range entries (R5: a select on the observed flag,
// never a multiply).  cv = valid tile columns from the half-step's first column.
// TF32 operands: the tensor core reads only the top 19 bits of each 32-bit container, so
// adding half a TF32 ulp (0x1000) to the bit pattern is round-to-nearest (ties away) of the
// value the MMA consumes; the low 13 bits need not be cleared.
// P_a of one entry in the MM = 1 path (o: training-observed).  SPA (Euclidean pair, bond <= 32):
// P_a = hi + lo, both TF32 - hi the RN of a, lo = a - hi (its own RN error ~2^-22 relative) -
// so the numerator N = P_a_hi V + P_a_lo V carries no TF32 rounding of a (the data itself for
// this pair, R27, R34); lo goes to TMEM columns 384 + 64 b.
template <int KIND, bool SPA>
__device__ __forceinline__ void put_pa(uint32_t (&sv)[16], uint32_t (&pl)[16], int j, bool o, float av) {
  if constexpr (SPA) {
    const uint32_t hi = (__float_as_uint(av) + 0x1000u) & 0xffffe000u;
    sv[j] = o ? hi : 0u;
    pl[j] = o ? __float_as_uint(av - __uint_as_float(hi)) + 0x1000u : 0u;
  } else {
    sv[j] = o ? __float_as_uint(av) + pa_round<KIND>(j) : 0u;
  }
}

template <int KIND, bool SPA>
__device__ __forceinline__ void ew_half(const TcArgs& a, uint32_t (&sv)[16], const float (&yv)[16],
                                        const uint32_t (&mk)[4], int cv, bool row_ok, uint32_t (&pb)[16],
                                        uint32_t (&pl)[16], float (&ls)[3], long long (&cn)[3]) {
  // per-byte valid flags of the tile (row / column in range) as 0x00 / 0xff bytes
  const uint32_t vbits = (!row_ok || cv <= 0) ? 0u : (cv >= 16 ? 0xffffu : ((1u << cv) - 1u));
  uint32_t vb[4];
#pragma unroll
  for (int j4 = 0; j4 < 4; ++j4) {
    const uint32_t b = (vbits >> (4 * j4)) & 0xfu;
    vb[j4] = ((b * 0x00204081u) & 0x01010101u) * 0xffu;   // 4 bits -> 4 bytes of 0x00 / 0xff
  }
  // training-observed bytes: mask byte nonzero (R6), or label == 1 (train) for a split fit (R29)
  uint32_t ob[4], rl[4];
#pragma unroll
  for (int j4 = 0; j4 < 4; ++j4) {
    const uint32_t m = a.has_mask ? mk[j4] : 0x01010101u;
    rl[j4] = m & vb[j4];                                   // labels of in-range entries (split fits)
    ob[j4] = (a.split ? __vcmpeq4(m, 0x01010101u) : m) & vb[j4];
  }
  if (a.mode != 0 && a.split) {   // split fit: train / validation / heldout losses of every labelled entry
#pragma unroll
    for (int j = 0; j < 16; j += 2) {
      const uint32_t r0 = (rl[j >> 2] >> (8 * (j & 3))) & 0xffu;
      const uint32_t r1 = (rl[j >> 2] >> (8 * ((j + 1) & 3))) & 0xffu;
      const float2 yh = yhat_floor(sv[j], sv[j + 1]);
      float2 av, bv, lv;
      Ew<KIND>::abl2(make_float2(r0 ? yv[j] : 1.f, r1 ? yv[j + 1] : 1.f), yh, a.dv, av, bv, lv);
#pragma unroll
      for (int q = 0; q < 3; ++q) ls[q] += (r0 == (uint32_t)(q + 1) ? lv.x : 0.f) + (r1 == (uint32_t)(q + 1) ? lv.y : 0.f);
      put_pa<KIND, SPA>(sv, pl, j, r0 == 1u, av.x);
      put_pa<KIND, SPA>(sv, pl, j + 1, r1 == 1u, av.y);
      pb[j] = r0 == 1u ? __float_as_uint(bv.x) + 0x1000u : 0u;
      pb[j + 1] = r1 == 1u ? __float_as_uint(bv.y) + 0x1000u : 0u;
    }
#pragma unroll
    for (int q = 0; q < 3; ++q)
#pragma unroll
      for (int j4 = 0; j4 < 4; ++j4) cn[q] += __popc(__vcmpeq4(rl[j4], (uint32_t)(q + 1) * 0x01010101u)) >> 3;
    return;
  }
  if (a.mode != 0) {   // loss of the iterate entering the sweep (uniform branch)
#pragma unroll
    for (int j = 0; j < 16; j += 2) {
      const bool o0 = (ob[j >> 2] & (0xffu << (8 * (j & 3)))) != 0u;
      const bool o1 = (ob[j >> 2] & (0xffu << (8 * ((j + 1) & 3)))) != 0u;
      const float2 yh = yhat_floor(sv[j], sv[j + 1]);
      float2 av, bv, lv;
      Ew<KIND>::abl2(make_float2(o0 ? yv[j] : 1.f, o1 ? yv[j + 1] : 1.f), yh, a.dv, av, bv, lv);
      ls[0] += (o0 ? lv.x : 0.f) + (o1 ? lv.y : 0.f);
      put_pa<KIND, SPA>(sv, pl, j, o0, av.x);
      put_pa<KIND, SPA>(sv, pl, j + 1, o1, av.y);
      pb[j] = o0 ? __float_as_uint(bv.x) + 0x1000u : 0u;
      pb[j + 1] = o1 ? __float_as_uint(bv.y) + 0x1000u : 0u;
    }
#pragma unroll
    for (int j4 = 0; j4 < 4; ++j4) cn[0] += __popc(__vcmpne4(ob[j4], 0u)) >> 3;
    return;
  }
#pragma unroll
  for (int j = 0; j < 16; j += 2) {
    const float2 yh = yhat_floor(sv[j], sv[j + 1]);
    const bool o0 = (ob[j >> 2] & (0xffu << (8 * (j & 3)))) != 0u;
    const bool o1 = (ob[j >> 2] & (0xffu << (8 * ((j + 1) & 3)))) != 0u;
    float2 av, bv;
    Ew<KIND>::ab2(make_float2(o0 ? yv[j] : 1.f, o1 ? yv[j + 1] : 1.f), yh, a.dv, av, bv);
    put_pa<KIND, SPA>(sv, pl, j, o0, av.x);
    put_pa<KIND, SPA>(sv, pl, j + 1, o1, av.y);
    pb[j] = o0 ? __float_as_uint(bv.x) + 0x1000u : 0u;
    pb[j + 1] = o1 ? __float_as_uint(bv.y) + 0x1000u : 0u;
  }
}

// P_b bits of one entry in the sentinel path: b > 0 at an observed entry; x * 0 + b is b there and
// NaN at a missing entry (x NaN), and the add-then-max rounds it (TF32 RN) or zeroes it; b == 1 kinds
// (KL, Jensen-Shannon: exact in TF32) are one compare-and-set
template <int KIND>
__device__ __forceinline__ uint32_t pb_sent(float bv, float x) {
  if constexpr (KIND == EW_KL || KIND == EW_JS) return x >= 0.f ? 0x3f800000u : 0u;
  else return (uint32_t)__viaddmax_s32(__float_as_int(__fmaf_rn(x, 0.f, bv)), 0x1000, 0);
}
// two entries: b is made NaN at a missing entry (x NaN) by one packed x * 0 + b, which is b
// exactly at an observed one; the add-then-max then rounds (TF32 RN) or zeroes it
template <int KIND>
__device__ __forceinline__ void pb_sent2(float2 bv, float2 x, uint32_t& p0, uint32_t& p1) {
  if constexpr (KIND == EW_KL || KIND == EW_JS) {
    p0 = pb_sent<KIND>(bv.x, x.x);
    p1 = pb_sent<KIND>(bv.y, x.y);
  } else {
    const float2 q = __ffma2_rn(x, make_float2(0.f, 0.f), bv);
    p0 = (uint32_t)__viaddmax_s32(__float_as_int(q.x), 0x1000, 0);
    p1 = (uint32_t)__viaddmax_s32(__float_as_int(q.y), 0x1000, 0);
  }
}

// P_a bits of one entry in the sentinel path: a >= 0 kinds clamp (a is NaN where x is, so the
// add-then-max both rounds and zeroes a missing entry); signed-a kinds (log forms) select on x.
template <int KIND>
__device__ __forceinline__ uint32_t pa_sent(float av, float x, int j) {
  // (every a >= 0 kind computes a from x - directly or through |x| - so a is NaN at a missing entry)
  if constexpr (Ew<KIND>::kSignedA) return x >= 0.f ? __float_as_uint(av) + pa_round<KIND>(j) : 0u;
  else return (uint32_t)__viaddmax_s32(__float_as_int(av), (int)pa_round<KIND>(j), 0);
}

// The same for the sentinel path (a >= 0 kinds; x NaN = missing): hi = max(RN(a), 0), lo = a - hi
template <int KIND, bool SPA>
__device__ __forceinline__ void put_pa_sent(uint32_t (&sv)[16], uint32_t (&pl)[16], int j, float av, float x) {
  if constexpr (SPA) {
    const uint32_t hi = (uint32_t)__viaddmax_s32(__float_as_int(av), 0x1000, 0) & 0xffffe000u;
    sv[j] = hi;
    pl[j] = x >= 0.f ? __float_as_uint(av - __uint_as_float(hi)) + 0x1000u : 0u;
  } else {
    sv[j] = pa_sent<KIND>(av, x, j);
  }
}

// The same without a mask stream: a missing entry carries the canonical NaN in Y (the sentinel
// copy nef_fit makes once per fit, R5; observed data are >= +0).  a is NaN there (every
// a >= 0 kind computes a from x or |x|) and b is made NaN by x * 0 + b, so one add-then-max per value,
// max(bits + 0x1000, 0), both rounds (TF32 RN of the value the tensor core truncates) and zeroes
// the missing entries.  Entries outside the tile's valid rows / columns (TMA zero fill) are
// turned into the NaN first.
template <int KIND, bool SPA>
__device__ __forceinline__ void ew_half_sent(const TcArgs& a, uint32_t (&sv)[16], float (&yv)[16], int cv, bool row_ok,
                                             uint32_t (&pb)[16], uint32_t (&pl)[16], double& lacc, long long& cnt) {
  if (a.absy) {   // raw unmasked Y (uniform branch): an observed -0.0 must not read as missing
#pragma unroll
    for (int j = 0; j < 16; ++j) yv[j] = fabsf(yv[j]);
  }
  const uint32_t vbits = (!row_ok || cv <= 0) ? 0u : (cv >= 16 ? 0xffffu : ((1u << cv) - 1u));
  if (vbits != 0xffffu) {
#pragma unroll
    for (int j = 0; j < 16; ++j) yv[j] = ((vbits >> j) & 1u) ? yv[j] : __uint_as_float(kSentMissingBits);
  }
  if constexpr (LossOff<KIND>::value) {
    if (a.mode != 0 && a.lconst) {   // loss without its data-only part (R25; count from the sentinel pass)
      float2 l2 = make_float2(0.f, 0.f);
#pragma unroll
      for (int j = 0; j < 16; j += 2) {
        const float2 x = make_float2(yv[j], yv[j + 1]);
        const float2 yh = yhat_floor(sv[j], sv[j + 1]);
        float2 av, bv, rv;
        LossOff<KIND>::abr2(x, yh, av, bv, rv);
        l2 = __fadd2_rn(l2, make_float2(x.x >= 0.f ? rv.x : 0.f, x.y >= 0.f ? rv.y : 0.f));
        sv[j] = (uint32_t)__viaddmax_s32(__float_as_int(av.x), (int)pa_round<KIND>(j), 0);
        sv[j + 1] = (uint32_t)__viaddmax_s32(__float_as_int(av.y), (int)pa_round<KIND>(j + 1), 0);
        pb_sent2<KIND>(bv, x, pb[j], pb[j + 1]);
      }
      lacc += (double)(l2.x + l2.y);   // (inside the uniform loss branch: nothing in update passes)
      return;
    }
  }
  if (a.mode != 0) {   // loss of the iterate entering the sweep (uniform branch)
    // a, b and the loss from |x| (NaN at a missing entry), then x >= 0 selects: the loss of a
    // missing entry is dropped, a and b are zeroed by the add-then-max.
    // The observed count is constant over a fit: only the loss-only pass (mode 2) counts.
    float2 l2 = make_float2(0.f, 0.f);
#pragma unroll
    for (int j = 0; j < 16; j += 2) {
      const float2 x = make_float2(yv[j], yv[j + 1]);
      const float2 yh = yhat_floor(sv[j], sv[j + 1]);
      float2 av, bv, lv;
      Ew<KIND>::abl2(make_float2(fabsf(x.x), fabsf(x.y)), yh, a.dv, av, bv, lv);
      l2 = __fadd2_rn(l2, make_float2(x.x >= 0.f ? lv.x : 0.f, x.y >= 0.f ? lv.y : 0.f));
      if (a.mode == 2) cnt += (x.x >= 0.f ? 1 : 0) + (x.y >= 0.f ? 1 : 0);
      if constexpr (Ew<KIND>::kSignedA) {
        sv[j] = pa_sent<KIND>(av.x, x.x, j);
        sv[j + 1] = pa_sent<KIND>(av.y, x.y, j + 1);
      } else if constexpr (SPA) {
        put_pa_sent<KIND, SPA>(sv, pl, j, av.x, x.x);
        put_pa_sent<KIND, SPA>(sv, pl, j + 1, av.y, x.y);
      } else {
        sv[j] = (uint32_t)__viaddmax_s32(__float_as_int(av.x), (int)pa_round<KIND>(j), 0);
        sv[j + 1] = (uint32_t)__viaddmax_s32(__float_as_int(av.y), (int)pa_round<KIND>(j + 1), 0);
      }
      pb_sent2<KIND>(bv, x, pb[j], pb[j + 1]);
    }
    lacc += (double)(l2.x + l2.y);
    return;
  }
#pragma unroll
  for (int j = 0; j < 16; j += 2) {
    const float2 x = make_float2(yv[j], yv[j + 1]);
    const float2 yh = yhat_floor(sv[j], sv[j + 1]);
    float2 av, bv;
    if (Ew<KIND>::kLinX) {
      Ew<KIND>::ab2(x, yh, a.dv, av, bv);   // a = x * (positive): NaN where x is
    } else {
      Ew<KIND>::ab2(make_float2(fabsf(x.x), fabsf(x.y)), yh, a.dv, av, bv);
    }
    put_pa_sent<KIND, SPA>(sv, pl, j, av.x, x.x);
    put_pa_sent<KIND, SPA>(sv, pl, j + 1, av.y, x.y);
    pb_sent2<KIND>(bv, x, pb[j], pb[j + 1]);
  }
}

// The sentinel-path stage with a per-entry loss parameter (MM = 2: negative binomial phi_i,
// binomial n_i; kLinX kinds): x NaN marks a missing entry (its parameter, possibly garbage or
// TMA zero fill, is replaced by 1 before use), a and b as ew_half_sent.
template <int KIND>
__device__ __forceinline__ void ew_half_aux(const TcArgs& a, uint32_t (&sv)[16], float (&yv)[16], const float (&xa)[16],
                                            int cv, bool row_ok, uint32_t (&pb)[16], double& lacc, long long& cnt) {
  if constexpr (KIND == EW_NB || KIND == EW_BINOM) {
    if (a.absy) {
#pragma unroll
      for (int j = 0; j < 16; ++j) yv[j] = fabsf(yv[j]);
    }
    const uint32_t vbits = (!row_ok || cv <= 0) ? 0u : (cv >= 16 ? 0xffffu : ((1u << cv) - 1u));
    if (vbits != 0xffffu) {
#pragma unroll
      for (int j = 0; j < 16; ++j) yv[j] = ((vbits >> j) & 1u) ? yv[j] : __uint_as_float(kSentMissingBits);
    }
    float l = 0.f;
#pragma unroll
    for (int j = 0; j < 16; j += 2) {
      const float2 yh = yhat_floor(sv[j], sv[j + 1]);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const float x = yv[j + e], y = e ? yh.y : yh.x;
        const float ax = x >= 0.f ? xa[j + e] : 1.f;
        float av, bv;
        Ew<KIND>::ab_aux(x, y, ax, av, bv);
        sv[j + e] = (uint32_t)__viaddmax_s32(__float_as_int(av), 0x1000, 0);
        pb[j + e] = pb_sent<KIND>(bv, x);
        if (a.mode != 0) {
          l += x >= 0.f ? Ew<KIND>::loss_aux(x, y, ax) : 0.f;
          if (a.mode == 2) cnt += x >= 0.f ? 1 : 0;
        }
      }
    }
    if (a.mode != 0) lacc += (double)l;
  }
}

// linear column index of the first column of a tile
// q = x / d, r = x % d for x >= 0, d > 0: the 32-bit divide when both fit (the 64-bit one is a
// ~100-instruction dependent chain; the index arithmetic below sits in front of every launch's
// first V load - timing-neutral on its own, profiles/r02_prologue_trace.txt)
__device__ __forceinline__ void divmod_nn(int64_t x, int64_t d, int64_t& q, int64_t& r) {
  if ((((uint64_t)x | (uint64_t)d) >> 32) == 0) {
    const uint32_t xq = (uint32_t)x / (uint32_t)d;
    q = xq;
    r = (uint32_t)x - xq * (uint32_t)d;
  } else {
    q = x / d;
    r = x - q * d;
  }
}
__device__ __forceinline__ int64_t tile_col0(const TcArgs& a, int64_t tile) {
  if (a.layout == 0) return tile * BN;
  int64_t ti, to;
  divmod_nn(tile, a.tiles_inner, to, ti);
  return to * a.CI + ti * BN;
}

// Direct V: inside a run of vd_E columns (the trailing column modes one table
// stores as consecutive rows), consecutive tiles advance the table row by 64 and the
// tile-constant rows do not change; tiles never straddle runs (vd_E % 64 == 0, or the run is
// the whole column block).  The two functions below recompute from scratch when a new run
// starts (cold, out of line).
__device__ __noinline__ int direct_var_row(const TcArgs& a, int64_t col) {
  int off = 0;
  for (int d = a.nc - 1; d >= 0; --d) {
    int64_t dig = col, rest = 0;
    if (d > 0) divmod_nn(col, a.cdim[d], rest, dig);
    col = rest;
    off += (int)dig * (int)a.tcs[a.var_tab][d];
  }
  return off / a.K;
}
// element offsets of every table's row at linear column col (out of line: divisions)
struct TabOffs { int o[kMaxTabs]; };
__device__ __noinline__ TabOffs direct_offs(const TcArgs& a, int64_t col) {
  TabOffs r;
  for (int q = 0; q < kMaxTabs; ++q) r.o[q] = 0;
  for (int d = a.nc - 1; d >= 0; --d) {
    int64_t dig = col, rest = 0;
    if (d > 0) divmod_nn(col, a.cdim[d], rest, dig);
    col = rest;
    for (int q = 0; q < a.ntab; ++q) r.o[q] += (int)dig * (int)a.tcs[q][d];
  }
  return r;
}
// Tile-constant rows of a run, bond chunk c (4 values) of this lane: loads issued here (all in
// flight together), product formed by cst_product when needed (software-pipelined by the caller).
struct CstLoad { float v[kMaxTabs][4]; };
__device__ __forceinline__ void cst_issue(const TcArgs& a, const float* const* tabs, int64_t col, int c, CstLoad& L) {
  const TabOffs off = direct_offs(a, col);
#pragma unroll
  for (int q = 0; q < kMaxTabs; ++q)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int k = 4 * c + e;
      const bool use = q < a.ntab && q != a.var_tab && k < a.K;
      L.v[q][e] = use ? __ldg(tabs[q] + off.o[q] + k) : 1.f;   // bond stride 1 (planner)
    }
}
__device__ __forceinline__ float4 cst_product(const TcArgs& a, int c, const CstLoad& L) {
  float p[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    p[e] = 4 * c + e < a.K ? 1.f : 0.f;
#pragma unroll
    for (int q = 0; q < kMaxTabs; ++q) p[e] *= L.v[q][e];
  }
  return make_float4(p[0], p[1], p[2], p[3]);
}

// Walk over a chunk's tiles for the direct-V path.  Runs are a fixed number of tiles
// (vd_tpr, host-computed), so a new run is a counter wrap; inside a run the column offset
// advances by 64 per tile, or to the next CI block after a block's (ragged) last tile.  Only
// init (once per CTA) and the callers' work at a new run divide.
struct RunCursor {
  int k, ti, tin, tpr;
  int64_t off, blk_off, tile, ci;
  __device__ __forceinline__ void init(const TcArgs& a, int64_t t0) {
    tpr = (int)a.vd_tpr;
    tin = (int)(a.layout == 0 ? a.tiles : a.tiles_inner);
    ci = a.layout == 0 ? 0 : a.CI;
    tile = t0;
    int64_t qq, rr;
    divmod_nn(t0, tpr, qq, rr);
    k = (int)rr;
    divmod_nn(t0, tin, qq, rr);
    ti = (int)rr;
    off = tile_col0(a, t0) - tile_col0(a, t0 - k);
    blk_off = off - (int64_t)ti * BN;
  }
  // advance to the next tile; true when it starts a new run (then off = 0)
  __device__ __forceinline__ bool next() {
    ++tile;
    const bool wrap = ++ti == tin;
    if (wrap) ti = 0;
    if (++k == tpr) {
      k = 0;
      off = 0;
      blk_off = 0;
      return true;
    }
    if (wrap) {
      blk_off += ci;
      off = blk_off;
    } else {
      off += BN;
    }
    return false;
  }
};

// pipeline timeline (diagnostics): event e of tile t in CTA (0,0)
enum TraceEv : int {
  EV_TMA_ISSUE = 0, EV_VG_START, EV_VG_DONE, EV_MMA1_ISSUE, EV_MMA23_ISSUE, EV_EW_S, EV_EW_Y, EV_EW_HALF,
  EV_EW_DONE, EV_VG_ISSUED, EV_EW_LDW, EV_EW_MATH
};
// compiled in only with -DNEF_TRACE=1 (scripts/build_variants.sh): the checks cost issue slots
#ifndef NEF_TRACE
#define NEF_TRACE 0
#endif
// timing experiments (scripts/build_variants.sh): compiled out of the production build
#ifndef NEF_DBG
#define NEF_DBG 0
#endif
__device__ __forceinline__ void trace_ev(const TcArgs& a, int t, int e) {
#if NEF_TRACE
  if (a.trace && blockIdx.x == 0 && blockIdx.y == 0 && t < 1024) a.trace[t * 32 + e] = (long long)clock64();
#endif
}

#ifndef NEF_UWARP
#define NEF_UWARP 1
#endif
#ifndef NEF_NBUF3
#define NEF_NBUF3 1   // bond <= 32: three TMEM tile buffers (0: two, as for bond 64)
#endif
// TMEM column of tile buffer b: 0 and 128, the third (bond <= 32 only) at 384
__device__ __forceinline__ uint32_t buf_col(int b) { return b == 2 ? 384u : 128u * (uint32_t)b; }

// ------------------------------------------------------------------ the kernel
// TMEM (512 columns x 128 lanes): two tile buffers of 128 columns, each holding S in its first
// 64 columns; the elementwise warps overwrite S in place with P_a and put P_b in the other 64
// (so a tile needs no second buffer and the elementwise stage never waits for the numerator
// MMAs of the previous tile); then N, D (KB each) and U_hi, U_lo (KB each).
//
// Tile t uses buffer t & 1.  Single MMA issuer, in order:
//   S(0), S(1), then for each t: [P(t) ready] N,D += P(t) V(t); [buffer t&1 retired] S(t+2)
// MM: 1 = uint8 mask streamed alongside Y; 0 = no mask stream (no mask, or the NaN-sentinel Y)
template <int KB, int KIND, int MM>
// registers: 80 per thread is the ceiling at 23 warps (the register file is split over the four
// sub-partitions: 16 K registers for the 6 warps of the fullest one; 88 fails to launch)
__global__ void __launch_bounds__(NTHREADS, 1) fused_tc_kernel(const __grid_constant__ Params P) {
  constexpr int NV = VStages<KB, MM>::value;
  constexpr int NS = YStages<KB, MM>::value;
  constexpr int V_STAGE = VSt<KB>::SIZE;
  // Euclidean pair with bond <= 32: numerator operand split hi + lo (put_pa), TMEM 384..511 free
  constexpr bool SPA = (KIND == EW_EUC && KB == 32 && !NEF_PA_RN);
  // TMEM tile buffers: bond <= 32 leaves columns 384..511 free - a third buffer (S(t+3) queued
  // behind the N/D MMAs of tile t, so the elementwise stage of t+1 and t+2 overlap them) unless
  // the split P_a uses them
  constexpr int NBUF = (KB == 32 && MM == 0 && !SPA && NEF_NBUF3) ? 3 : 2;
  extern __shared__ unsigned char smraw[];
  const TcArgs& a = P.a;
  const int tid = threadIdx.x;
#if NEF_UWARP
  // warp index through a shuffle: provably warp-uniform, so every role branch and the code under
  // it (loop counters, stage indices, descriptors) can live in uniform registers
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
#else
  const int warp = tid >> 5;
#endif
  const int lane = tid & 31;

  // 1024-aligned carve-up
  const uint32_t raw = smem_u32(smraw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  unsigned char* gbase = smraw + (base - raw);
  const uint32_t sY = base;                                  // NS x 32 KB
  const uint32_t sM = sY + NS * Y_STAGE;                     // NS x 8 KB
  const uint32_t sV = sM + (MM == 1 ? NS * M_STAGE : MM == 2 ? NS * Y_STAGE : 0);   // NV x (V | V^T)
  const uint32_t sBar = sV + NV * V_STAGE;
  const uint32_t y_full = sBar, y_empty = y_full + 8 * NS;
  const uint32_t v_full = y_empty + 8 * NS, v_empty = v_full + 8 * NV;
  const uint32_t s_full = v_empty + 8 * NV;                  // [NBUF] S(t) in buffer t % NBUF (MMA commit)
  const uint32_t p_full = s_full + 8 * NBUF;                 // [NBUF] P(t) written (16 elementwise warps)
  const uint32_t buf_free = p_full + 8 * NBUF;               // [NBUF] N,D MMAs of tile t retired (commit)
  const uint32_t nd_full = buf_free + 8 * NBUF, u_ready = nd_full + 8;
  const uint32_t vraw_full = u_ready + 8;                    // NV barriers: direct-V rows landed (TMA)
  const uint32_t drain_ready = vraw_full + 8 * NV;           // N/D of a drain group retired (commit)
  const uint32_t sTmem = drain_ready + 8;
  unsigned char* gY = gbase;
  unsigned char* gM = gbase + NS * Y_STAGE;
  unsigned char* gV = gbase + (sV - base);
  uint32_t* gTmem = reinterpret_cast<uint32_t*>(gbase + (sTmem - base));
  // loss reduction scratch: aliases Y stage 0, free once every tile has been consumed
  double* gRed = reinterpret_cast<double*>(gbase);
  long long* gRedC = reinterpret_cast<long long*>(gbase + NEW * 32 * 8);

  const int64_t rb = blockIdx.x;
  const int64_t ch = blockIdx.y;
  const int rs = blockIdx.z;   // restart (N4; 0 unless batched)
  const int64_t t_begin = ch * a.tiles_per_chunk;
  const int64_t t_end = (t_begin + a.tiles_per_chunk < a.tiles) ? t_begin + a.tiles_per_chunk : a.tiles;
  const int T = (int)(t_end > t_begin ? t_end - t_begin : 0);
  const int64_t row0 = rb * BM;
  const int rows_here = (int)((a.n_rows - row0) < BM ? (a.n_rows - row0) : BM);
  // The tensor core's fp32 accumulation truncates (ubench/acc_round.cu), a bias growing with the
  // number of accumulation steps; N and D are therefore drained into the (RN, fp32) partials
  // every G tiles and restarted.
  constexpr int G = kDrainTiles;   // (power of two: t % G is a mask)

  if (tid == 0) trace_ev(a, 1023, 0);   // (trace build: launch phases in row 1023 - entry)
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) { mbar_init(y_full + 8 * i, 1); mbar_init(y_empty + 8 * i, NEW); }
    for (int i = 0; i < NV; ++i) { mbar_init(v_full + 8 * i, NVG); mbar_init(v_empty + 8 * i, 1); }
    for (int i = 0; i < NBUF; ++i) {
      mbar_init(s_full + 8 * i, 1);
      mbar_init(p_full + 8 * i, NEW);
      mbar_init(buf_free + 8 * i, 1);
    }
    mbar_init(nd_full, 1);
    mbar_init(drain_ready, 1);
    mbar_init(u_ready, NEW);
    for (int i = 0; i < NV; ++i) mbar_init(vraw_full + 8 * i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&P.tmY)) : "memory");
    if (a.has_mask) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&P.tmM)) : "memory");
  }
  if (warp == W_MMA) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sTmem) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) trace_ev(a, 1023, 1);   // barriers initialised, TMEM allocated
#if NEF_UWARP
  const uint32_t tmem = __shfl_sync(0xffffffffu, *gTmem, 0);
#else
  const uint32_t tmem = *gTmem;
#endif
  const uint32_t tNa = tmem + 256, tNb = tmem + 256 + KB;
  const uint32_t tUh = tmem + 256 + 2 * KB, tUl = tmem + 256 + 3 * KB;

  if (warp == W_TMA) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      const uint32_t bytes = (uint32_t)Y_STAGE + (a.has_mask ? (uint32_t)M_STAGE : 0u) + (MM == 2 ? (uint32_t)Y_STAGE : 0u);
      for (int t = 0; t < T; ++t) {
        const int st = t % NS;
        mbar_wait_relaxed(y_empty + 8 * st, ((t / NS) & 1) ^ 1);
        trace_ev(a, t, EV_TMA_ISSUE);
        const int64_t tile = t_begin + t;
        const uint32_t bar = y_full + 8 * st;
        mbar_expect_tx(bar, bytes);
        const uint32_t dY = sY + st * Y_STAGE, dM = sM + st * M_STAGE;
        // the Y tile (and, MM = 2, the parameter tile of the same geometry into the second ring)
        auto load_f32 = [&](uint32_t dst, const CUtensorMap* tm) {
          if (a.layout == 0) {
            tma_load_2d(dst, tm, (int)row0, (int)(tile * BN), bar);
          } else {
            const int64_t ti = tile % a.tiles_inner, to = tile / a.tiles_inner;
            if (a.layout == 1) {
              if (a.y3d) {
                tma_load_3d(dst, tm, 0, (int)(ti * 2), (int)row0, bar);
              } else {
                tma_load_2d(dst, tm, (int)(ti * BN), (int)row0, bar);
                tma_load_2d(dst + Y_STAGE / 2, tm, (int)(ti * BN + 32), (int)row0, bar);
              }
            } else {
              tma_load_3d(dst, tm, (int)(ti * BN), (int)row0, (int)to, bar);
              tma_load_3d(dst + Y_STAGE / 2, tm, (int)(ti * BN + 32), (int)row0, (int)to, bar);
            }
          }
        };
        load_f32(dY, &P.tmY);
        if constexpr (MM == 2) load_f32(sM + st * Y_STAGE, &P.tmA);
        if (a.has_mask) {
          if (a.layout == 0) {
            tma_load_2d(dM, &P.tmM, (int)row0, (int)(tile * BN), bar);
          } else {
            const int64_t ti = tile % a.tiles_inner, to = tile / a.tiles_inner;
            if (a.layout == 1) tma_load_2d(dM, &P.tmM, (int)(ti * BN), (int)row0, bar);
            else tma_load_3d(dM, &P.tmM, (int)(ti * BN), (int)row0, (int)to, bar);
          }
        }
      }
    }
  } else if (warp == W_MMA) {
    // ------------------------------------------------------------ MMA issuer
    // The whole warp runs the issue loop (warp-uniform control flow, so descriptors and TMEM
    // addresses stay in uniform registers and every tcgen05.mma is one elected issue; a
    // lane-0-only loop measured ~3x slower issue, starving the N = 64 MMAs).
    if (T > 0) {
      constexpr uint32_t id1 = idesc_tf32(128, BN);   // S = U V^T   : N = 64 tile columns
      constexpr uint32_t id2 = idesc_tf32(128, KB);   // N = P V     : N = bond
      // The tensor pipe executes one thread's MMAs in issue order, so S(t+2) issued right behind
      // the N/D MMAs of tile t cannot overwrite P(t) before they read it (checked: bit-identical
      // factors with and without the explicit wait, scripts/war_check.py).  dbg & 16 restores
      // the explicit wait on the N/D commit.
      const bool war_wait = (NEF_DBG & 16) != 0;
      mbar_wait_mma(u_ready, 0);
      if (lane == 0) trace_ev(a, 1023, 8);   // (trace) U in TMEM
      tc_fence_after();
      // S(t) = U_hi V(t)^T + U_lo V(t)^T into buffer t & 1 (split reconstruction)
      auto mma_s = [&](int t, int b, uint32_t ph) {   // b = t % NBUF, ph = (t / NBUF) & 1
        const int vs = t % NV;
        mbar_wait_mma(v_full + 8 * vs, (t / NV) & 1);
        if (t >= NBUF && war_wait) mbar_wait_mma(buf_free + 8 * b, ph ^ 1);
        tc_fence_after();
        if (lane == 0) trace_ev(a, t, EV_MMA1_ISSUE);
        __syncwarp();
        const uint64_t vd = NEF_ND_MN ? sdesc(sV + vs * V_STAGE, (uint32_t)BN * 128u, 512, 1) : sdesc(sV + vs * V_STAGE, 16, 1024);
        const uint32_t d = tmem + buf_col(b);
        // one asm block, one elect: U_hi and U_lo steps interleaved (tUl = tUh + KB)
        if constexpr ((NEF_DBG & 512) != 0) {   // timing experiment: no U_lo MMAs
          if (KB == 64) mma_s1_block_64<id1>(d, tUh, vd, 0u);
          else mma_s1_block_32<id1>(d, tUh, vd, 0u);
        } else if constexpr (VSt<KB>::ULB) {
          mma_s1_block_64<id1>(d, tUh, vd, 0u);
          mma_slo_bf16_64<idesc_bf16(128, BN)>(d, tUl, sdesc(sV + vs * V_STAGE + VSt<KB>::VB_OFF, 16, 1024));
        } else if (KB == 64) {
          mma_s_block_64<id1>(d, tUh, vd, 0u);
        } else {
          mma_s_block_32<id1>(d, tUh, vd, 0u);
        }
        mma_commit_elect(s_full + 8 * b);
      };
      if (!NEF_SPLIT_ISSUE)
        for (int i = 0; i < NBUF && i < T; ++i) mma_s(i, i, 0);
      int b = 0;                  // buffer of tile u (and of tile u + NBUF's S)
      uint32_t ph = 0;            // (u / NBUF) & 1
      for (int u = 0; u < T; ++u) {
        const int vs = u % NV;
#if NEF_ND_BAR
        // P(u) written by every elementwise warp: a hardware named barrier per tile buffer (the
        // issuer sleeps instead of polling an mbarrier)
        asm volatile("bar.sync %0, %1;" ::"r"(3 + b), "n"((NEW + 1) * 32) : "memory");
#else
        mbar_wait_mma(p_full + 8 * b, ph);
#endif
        tc_fence_after();
        if (lane == 0) trace_ev(a, u, EV_MMA23_ISSUE);
        __syncwarp();
        if (a.mode != 2 && !(NEF_DBG & 64)) {   // NEF_DBG 64: timing experiment without N/D MMAs
          const uint32_t pa = tmem + buf_col(b);   // P_a; P_b at pa + 64
          // the accumulators restart at every drain group (see the elementwise loop)
          const uint32_t acc = (u % G) != 0 ? 1u : 0u;
#if NEF_ND_MN
          // B = V itself read MN-major (32-byte-atom swizzle, see v_chunk): bonds (N) contiguous in
          // its 128-byte rows, the second 32-bond column block BN rows * 128 B further (LBO), 4
          // tile columns (K) per 512 bytes (SBO), 8 per K step
          const uint64_t vtd = sdesc(sV + vs * V_STAGE, (uint32_t)BN * 128u, 512, 1);
          constexpr uint32_t id2m = id2 | (1u << 16);   // B MN-major
          if constexpr (SPA) {
            if (b == 0) mma_nd3_mn_block_32_b0<id2m>(tNa, tNb, pa, vtd, acc);
            else mma_nd3_mn_block_32_b1<id2m>(tNa, tNb, pa, vtd, acc);
          } else if constexpr (KB == 64) {
            mma_nd_mn_block_64<id2m>(tNa, tNb, pa, vtd, acc);
          } else {
            mma_nd_mn_block_32<id2m>(tNa, tNb, pa, vtd, acc);
          }
#else
          // B = V^T, K-major SW128: rows = bond (N), K = tile columns (2 atoms of 32)
          const uint64_t vtd = sdesc(sV + vs * V_STAGE + VSt<KB>::VT_OFF, 16, 1024);
          if constexpr (SPA) {
            if (b == 0) mma_nd3_block_32_b0<id2>(tNa, tNb, pa, vtd, acc);
            else mma_nd3_block_32_b1<id2>(tNa, tNb, pa, vtd, acc);
          } else if constexpr (KB == 64) {
            mma_nd_block_64<id2>(tNa, tNb, pa, vtd, acc);
          } else {
            mma_nd_block_32<id2>(tNa, tNb, pa, vtd, acc);
          }
#endif
        }
        mma_commit_elect(v_empty + 8 * vs);
        mma_commit_elect(buf_free + 8 * b);
        if (u % G == G - 1 && u != T - 1) mma_commit_elect(drain_ready);
        if (!NEF_SPLIT_ISSUE && u + NBUF < T) mma_s(u + NBUF, b, ph ^ 1);
        if (++b == NBUF) { b = 0; ph ^= 1; }
      }
      mma_commit_elect(nd_full);
    }
  } else if (NEF_SPLIT_ISSUE && warp == W_MMA2) {
    // ------------------------------------------------------------ S issuer (NEF_SPLIT_ISSUE)
    if (T > 0) {
      constexpr uint32_t id1 = idesc_tf32(128, BN);
      mbar_wait_mma(u_ready, 0);
      if (lane == 0) trace_ev(a, 1023, 8);   // (trace) U in TMEM
      tc_fence_after();
      int b = 0;
      uint32_t ph = 0;
      for (int t = 0; t < T; ++t) {
        const int vs = t % NV;
        // buffer b is free once the N/D MMAs of tile t - NBUF (the last reader of its P) retired
        if (t >= NBUF) mbar_wait_mma(buf_free + 8 * b, ph ^ 1);
        mbar_wait_mma(v_full + 8 * vs, (t / NV) & 1);
        tc_fence_after();
        if (lane == 0) trace_ev(a, t, EV_MMA1_ISSUE);
        __syncwarp();
        const uint64_t vd = NEF_ND_MN ? sdesc(sV + vs * V_STAGE, (uint32_t)BN * 128u, 512, 1) : sdesc(sV + vs * V_STAGE, 16, 1024);
        const uint32_t d = tmem + buf_col(b);
        if (KB == 64) mma_s_block_64<id1>(d, tUh, vd, 0u);
        else mma_s_block_32<id1>(d, tUh, vd, 0u);
        mma_commit_elect(s_full + 8 * b);
        if (++b == NBUF) { b = 0; ph ^= 1; }
      }
    }
  } else if (NEF_S_WATCH && warp == W_SW) {
    // ------------------------------------------------------------ S watcher (NEF_S_WATCH)
    int b = 0;
    uint32_t ph = 0;
    for (int t = 0; t < T; ++t) {
      mbar_spin(s_full + 8 * b, ph);
      asm volatile("bar.arrive %0, %1;" ::"r"(6 + b), "n"((NEW + 1) * 32) : "memory");
      if (++b == NBUF) { b = 0; ph ^= 1; }
    }
  } else if (warp == W_DV) {
    // ------------------------------------------------------------ direct-V row loads (TMA)
    if (lane == 0 && a.vdirect && T > 0) {
      RunCursor rc;
      trace_ev(a, 1023, 10);   // (trace) loader lane starts
      rc.init(a, t_begin);
      trace_ev(a, 1023, 11);   // (trace) run cursor initialised
      int run_row = direct_var_row(a, tile_col0(a, t_begin) - rc.off);
      trace_ev(a, 1023, 12);   // (trace) first table row known
      for (int t = 0; t < T; ++t) {
        if (t > 0 && rc.next()) run_row = direct_var_row(a, tile_col0(a, rc.tile));
        const int rowv = run_row + (int)rc.off;
        const int vs = t % NV;
        mbar_wait_relaxed(v_empty + 8 * vs, ((t / NV) & 1) ^ 1);
        const uint32_t bar = vraw_full + 8 * vs;
        if (t == 0) trace_ev(a, 1023, 5);   // (trace) first direct-V TMA issued
        mbar_expect_tx(bar, (uint32_t)(KB * BN * 4));
#pragma unroll
        for (int h = 0; h < KB / 32; ++h) tma_load_2d(sV + vs * V_STAGE + h * (BN * 128), &P.tmV[rs], 32 * h, rowv, bar);
      }
    }
  } else if (vg_index(warp) >= 0 && a.vdirect) {
    // ------------------------------------------------------------ direct V: scale rows in place
    // V[x][k] = T_var[row + x][k] * prod_{q != var} T_q[const row][k]; V^T written alongside.
    const int xw = vg_index(warp) * 16;
    const int c = vl_c<KB>(lane);
    VOff<KB> vo;
    vo.init(xw, lane);
    // the next tile's run is looked up one tile ahead so that a new run's constant rows are in
    // flight while the current tile is scaled
    RunCursor rn;
    CstLoad ld;
    float4 cst = make_float4(0.f, 0.f, 0.f, 0.f);
    bool pend = false;
    if (T > 0) {
      rn.init(a, t_begin);
      if (warp == W_VG0 && lane == 0) trace_ev(a, 1023, 9);   // (trace) first constant rows issued
      cst_issue(a, a.tabr[rs], tile_col0(a, t_begin), c, ld);
      cst = cst_product(a, c, ld);
      if (warp == W_VG0 && lane == 0) trace_ev(a, 1023, 6);   // (trace) first constant rows landed
    }
    for (int t = 0; t < T; ++t) {
      if (pend) {
        cst = cst_product(a, c, ld);
        pend = false;
      }
      if (t + 1 < T && rn.next()) {
        cst_issue(a, a.tabr[rs], tile_col0(a, rn.tile), c, ld);
        pend = true;
      }
      const int vs = t % NV;
      mbar_wait_relaxed(vraw_full + 8 * vs, (t / NV) & 1, 96);
      if (warp == W_VG0 && lane == 0) trace_ev(a, t, EV_VG_START);
      unsigned char* vrow = gV + vs * V_STAGE;
#pragma unroll
      for (int i = 0; i < VOff<KB>::NB; ++i) {
        float4 p[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const float4 f = *reinterpret_cast<const float4*>(vrow + vo.vb[i] + r * 128 + (v_chunk(vo.cx[i], r) << 4));
          const float2 lo = __fmul2_rn(make_float2(f.x, f.y), make_float2(cst.x, cst.y));
          const float2 hi = __fmul2_rn(make_float2(f.z, f.w), make_float2(cst.z, cst.w));
          p[r] = make_float4(lo.x, lo.y, hi.x, hi.y);
        }
        if (!(NEF_DBG & 128)) {   // NEF_DBG 128: timing experiment without the V / V^T stores
          vblock_store_direct<KB>(vrow, vo.vb[i], vo.cx[i], vo.vtb[i], vo.xc[i], p);
          vb16_store<KB>(vrow, vo.rowoff[i], vo.x7[i], vo.c16, p);
        }
      }
      if (warp == W_VG0 && lane == 0) trace_ev(a, t, EV_VG_ISSUED);
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(v_full + 8 * vs);
      if (warp == W_VG0 && lane == 0) trace_ev(a, t, EV_VG_DONE);
    }
  } else if (vg_index(warp) >= 0) {
    // ------------------------------------------------------------ column operand V (Khatri-Rao)
    const int xw = vg_index(warp) * 16;
    VTile<KB> cur, nxt;
    int toff_c[kMaxTabs], toff_n[kMaxTabs];
    Odo odo;
    VOff<KB> vo;
    vo.init(xw, lane);
    if (T > 0) vtile_issue<KB>(a, t_begin, xw, lane, cur, toff_c, odo);
    for (int t = 0; t < T; ++t) {
      if (t + 1 < T) vtile_issue<KB>(a, t_begin + t + 1, xw, lane, nxt, toff_n, odo);   // next tile's rows in flight
      if (warp == W_VG0 && lane == 0) trace_ev(a, t, EV_VG_ISSUED);
      const int vs = t % NV;
      mbar_wait_relaxed(v_empty + 8 * vs, ((t / NV) & 1) ^ 1);
      if (warp == W_VG0 && lane == 0) trace_ev(a, t, EV_VG_START);
      vtile_store<KB>(a, xw, lane, cur, toff_c, gV + vs * V_STAGE, vo);
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(v_full + 8 * vs);
      if (warp == W_VG0 && lane == 0) trace_ev(a, t, EV_VG_DONE);
      cur = nxt;
#pragma unroll
      for (int q = 0; q < kMaxTabs; ++q) toff_c[q] = toff_n[q];
    }
  } else if (warp >= W_EW0 && warp < W_EW0 + NEW) {
    // ------------------------------------------------------------ elementwise + epilogue
    const int ew = tid - W_EW0 * 32;       // 0 .. NEW * 32 - 1
    const int gw = (warp - W_EW0) >> 2;    // column group of this warp: tile columns [EWC gw, EWC gw + EWC)
    const int cg0 = gw * EWH;              // its first 16-column group
    const int qd = warp & 3;               // TMEM lane quarter
    const int m = qd * 32 + lane;          // row within the block (= TMEM lane)
    const uint32_t lane_off = (uint32_t)(qd * 32) << 16;
    int yoff[EWH], yswz[EWH];
#pragma unroll
    for (int h = 0; h < EWH; ++h) ew_y_line(a, (cg0 + h) >> 1, m, yoff[h], yswz[h]);
    const int64_t row = row0 + m;
    const bool row_ok = m < rows_here;
    constexpr int NCH = KB / 16;           // 16-column chunks of U_hi (and of U_lo, N, D)
    constexpr int NGW = NEW / 4;           // column groups of elementwise warps
    // U -> TMEM, split hi / lo: the 2 NCH chunks are shared out among the column groups
    {
#pragma unroll 1
      for (int c = gw * (2 * NCH / NGW); c < (gw + 1) * (2 * NCH / NGW); ++c) {
        const bool lo = c >= NCH;
        const int h = lo ? c - NCH : c;
        uint32_t r[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int k = h * 16 + j;
          const float u = (row_ok && k < a.K) ? __ldg(a.Ur[rs] + row * a.K + k) : 0.f;
          const uint32_t hi = tf32_bits(u);
          r[j] = lo ? (VSt<KB>::ULB ? __float_as_uint(u - __uint_as_float(hi)) : tf32_bits(u - __uint_as_float(hi))) : hi;
        }
        if (VSt<KB>::ULB && lo) {   // U_lo as BF16 pairs (k even in the low half): 8 TMEM columns
          uint32_t r2[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const __nv_bfloat162 v = __floats2bfloat162_rn(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1]));
            r2[j] = *reinterpret_cast<const uint32_t*>(&v);
          }
          tmem_st8(tUl + lane_off + h * 8, r2);
        } else {
          tmem_st16((lo ? tUl : tUh) + lane_off + h * 16, r);
        }
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(u_ready);
      if (warp == W_EW0 && lane == 0) trace_ev(a, 1023, 7);   // (trace) this warp's U chunks stored
    }
    // N | D (2 NCH chunks of 16 columns, shared out among the column groups) -> this CTA's split
    // partial of drain group grp (zeros when zero: a chunk with fewer tiles than others)
    auto drain_nd = [&](int64_t grp, bool zero) {
      const int64_t elems = a.n_rows * (int64_t)a.K;
#pragma unroll 1
      for (int c = gw * (2 * NCH / NGW); c < (gw + 1) * (2 * NCH / NGW); ++c) {
        const int which = c >= NCH ? 1 : 0;
        const int h = which ? c - NCH : c;
        float* out = a.Qpartr[rs] + ((ch * a.n_groups + grp) * 2 + which) * elems + row * a.K + h * 16;
        uint32_t r[16];
        if (!zero) {
          tmem_ld16((which ? tNb : tNa) + lane_off + h * 16, r);
          tmem_ld_wait(r);
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) r[j] = 0u;
        }
        if (row_ok && h * 16 < a.K) {
          if (h * 16 + 16 <= a.K && (a.K & 3) == 0) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              reinterpret_cast<uint4*>(out)[q] = make_uint4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (h * 16 + j < a.K) out[j] = __uint_as_float(r[j]);
          }
        }
      }
    };
    double loss_acc[3] = {0.0, 0.0, 0.0};   // [role] (split fits: train / validation / heldout)
    long long cnt[3] = {0, 0, 0};
    // valid columns of a tile: the tile's offset inside its column block, advanced per tile
    // (no 64-bit division in the loop)
    const int64_t cext = a.layout == 0 ? a.CO : a.CI;
    const int tiles_blk = (int)(a.layout == 0 ? a.tiles : a.tiles_inner);
    // only the last tile of a column block can be ragged: its valid columns, computed once
    const int last_tin = tiles_blk - 1;
    const int last_cols = (int)(cext - (int64_t)last_tin * BN);
    int tin = (int)(a.layout == 0 ? t_begin : t_begin % a.tiles_inner);
    int b = 0;           // tile buffer t % NBUF
    uint32_t bph = 0;    // (t / NBUF) & 1
    int st = 0;          // Y stage t % NS
    uint32_t sph = 0;    // (t / NS) & 1
    const uint32_t tlane = tmem + lane_off + 16 * cg0;   // this warp's columns in a tile buffer
    for (int t = 0; t < T; ++t, ++tin) {
      if (tin >= tiles_blk) tin = 0;
      const int cols_here = tin == last_tin ? last_cols : BN;
      const uint32_t tc = tlane + buf_col(b);   // S / P_a columns of this warp
      float lsum[3] = {0.f, 0.f, 0.f};
      uint32_t sv[EWH][16], pb[EWH][16], pl[EWH][16];
      float yv[EWH][16];
      uint32_t mk[EWH][4];
#if NEF_S_WATCH
      asm volatile("bar.sync %0, %1;" ::"r"(6 + b), "n"((NEW + 1) * 32) : "memory");
#else
      mbar_wait_ew(s_full + 8 * b, bph);
#endif
      if (warp == W_EW0 && lane == 0) trace_ev(a, t, EV_EW_S);
      tc_fence_after();
#pragma unroll
      for (int h = 0; h < EWH; ++h) tmem_ld16(tc + 16 * h, sv[h]);
      mbar_spin(y_full + 8 * st, sph);
      if (warp == W_EW0 && lane == 0) trace_ev(a, t, EV_EW_Y);
      float xa[MM == 2 ? EWH : 1][16];   // MM = 2: the per-entry parameters of the entries
#pragma unroll
      for (int h = 0; h < EWH; ++h) {
        mk[h][0] = mk[h][1] = mk[h][2] = mk[h][3] = 0u;
        ew_load_y(a, gY + st * Y_STAGE, gM + st * M_STAGE, (cg0 + h) >> 1, (cg0 + h) & 1, m, yoff[h], yswz[h], yv[h],
                  mk[h]);   // (MM == 0: a.has_mask = 0)
        if constexpr (MM == 2) {
          uint32_t dummy[4];
          ew_load_y(a, gM + st * Y_STAGE, gM, (cg0 + h) >> 1, (cg0 + h) & 1, m, yoff[h], yswz[h], xa[h], dummy);
        }
      }
#pragma unroll
      for (int h = 0; h < EWH; ++h) tmem_ld_wait(sv[h]);
      if (warp == W_EW0 && lane == 0) trace_ev(a, t, EV_EW_LDW);
      __syncwarp();
      if (lane == 0) mbar_arrive(y_empty + 8 * st);  // Y / mask stage read by this warp
#pragma unroll
      for (int h = 0; h < EWH; ++h) {
        const int cv = cols_here - 16 * (cg0 + h);
        if (!(NEF_DBG & 256)) {
          if constexpr (MM == 1) ew_half<KIND, SPA>(a, sv[h], yv[h], mk[h], cv, row_ok, pb[h], pl[h], lsum, cnt);
          else if constexpr (MM == 2) ew_half_aux<KIND>(a, sv[h], yv[h], xa[h], cv, row_ok, pb[h], loss_acc[0], cnt[0]);
          else ew_half_sent<KIND, SPA>(a, sv[h], yv[h], cv, row_ok, pb[h], pl[h], loss_acc[0], cnt[0]);
        } else {   // NEF_DBG 256: timing experiment without the elementwise math (P_b = S + Y)
#pragma unroll
          for (int j = 0; j < 16; ++j) pb[h][j] = sv[h][j] + __float_as_uint(yv[h][j]) + mk[h][j >> 2];
        }
      }
      if (warp == W_EW0 && lane == 0) trace_ev(a, t, EV_EW_MATH);
      if (a.mode != 2) {
#pragma unroll
        for (int h = 0; h < EWH; ++h) {
          tmem_st16(tc + 16 * h, sv[h]);
          tmem_st16(tc + 16 * h + 64, pb[h]);
          if constexpr (SPA) tmem_st16(tmem + 384 + 64 * b + lane_off + 16 * (cg0 + h), pl[h]);
        }
      }
      if (t == 0 && a.debug && blockIdx.x == 0 && blockIdx.y == 0 && rs == 0) {   // test hook (nef_debug_dump)
#pragma unroll
        for (int h = 0; h < EWH; ++h)
#pragma unroll
          for (int j = 0; j < 16; ++j) a.debug[m * 64 + 16 * (cg0 + h) + j] = __uint_as_float(sv[h][j] & 0xffffe000u);
      }
      if (warp == W_EW0 && lane == 0) trace_ev(a, t, EV_EW_HALF);
      if (a.mode != 2) tmem_st_wait();
      if (MM == 1 && a.mode != 0) {
        loss_acc[0] += (double)lsum[0];
        if (a.split) { loss_acc[1] += (double)lsum[1]; loss_acc[2] += (double)lsum[2]; }
      }
      tc_fence_before();
      __syncwarp();
#if NEF_ND_BAR
      asm volatile("bar.arrive %0, %1;" ::"r"(3 + b), "n"((NEW + 1) * 32) : "memory");
#else
      if (lane == 0) mbar_arrive(p_full + 8 * b);      // P(t) in TMEM (or, loss only: S(t) consumed)
#endif
      if (warp == W_EW0 && lane == 0) trace_ev(a, t, EV_EW_DONE);
      if (lane == 0) trace_ev(a, t, 16 + warp - W_EW0);     // per-warp arrival (diagnostics)
      if (a.mode != 2 && t % G == G - 1 && t != T - 1) {
        // drain the group's N / D before any warp can contribute P(t+1) (the N/D MMAs of tile
        // t+1 wait for every warp's P(t+1) and restart the accumulators)
        mbar_wait(drain_ready, (t / G) & 1);
        tc_fence_after();
        drain_nd(t / G, false);
      }
      if (++b == NBUF) { b = 0; bph ^= 1; }
      if (++st == NS) { st = 0; sph ^= 1; }
    }
    // epilogue: the last group's N | D -> split partials (added to the earlier groups' drains)
    if (a.mode != 2) {
      int64_t g0 = 0;
      if (T > 0) {
        mbar_spin(nd_full, 0);
        tc_fence_after();
        if (warp == W_EW0 && lane == 0) trace_ev(a, 1023, 2);   // last N / D MMAs retired
        drain_nd((T - 1) / G, false);
        g0 = (T - 1) / G + 1;
      }
      for (int64_t grp = g0; grp < a.n_groups; ++grp) drain_nd(grp, true);
      if (warp == W_EW0 && lane == 0) trace_ev(a, 1023, 3);     // partials written
    } else if (T > 0) {
      mbar_spin(nd_full, 0);
    }
    if (a.mode != 0) {
      // fixed-order block sums, one per role (split fits: losspart / countpart are [3][parts])
      const int nrole = (MM == 1 && a.split) ? 3 : 1;
      const int64_t parts = (int64_t)gridDim.x * gridDim.y;
      const int64_t id = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
      for (int q = 0; q < nrole; ++q) {
        gRed[ew] = loss_acc[q];
        gRedC[ew] = cnt[q];
        asm volatile("bar.sync 1, %0;" ::"n"(NEW * 32) : "memory");
        for (int w = NEW * 16; w > 0; w >>= 1) {
          if (ew < w) { gRed[ew] += gRed[ew + w]; gRedC[ew] += gRedC[ew + w]; }
          asm volatile("bar.sync 1, %0;" ::"n"(NEW * 32) : "memory");
        }
        if (ew == 0) {
          a.losspartr[rs][q * parts + id] = gRed[0];
          a.countpartr[rs][q * parts + id] = gRedC[0];
        }
        asm volatile("bar.sync 1, %0;" ::"n"(NEW * 32) : "memory");
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (tid == 0) trace_ev(a, 1023, 4);   // every role done
  if (warp == W_MMA) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
// NEF_NO_Y3D=1 (diagnostics): layout 1 with two 2-D boxes per tile
static const bool g_no_y3d = [] { const char* e = std::getenv("NEF_NO_Y3D"); return e && e[0] == '1'; }();

static bool get_encode() {
  if (g_encode) return true;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) return false;
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return true;
}

static bool encode(CUtensorMap* tm, CUtensorMapDataType dt, int rank, const void* ptr, const uint64_t* dims,
                   const uint64_t* strides_bytes, const uint32_t* box, CUtensorMapSwizzle sw) {
  uint32_t es[3] = {1, 1, 1};
  CUresult r = g_encode(tm, dt, (cuuint32_t)rank, const_cast<void*>(ptr), dims, strides_bytes, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

struct TcLauncher {
  const Params& P;
  dim3 grid;
  cudaStream_t s;
  int KB;
  int MM;
  template <int KB_, int KIND, int MM_>
  cudaError_t go() const {
    const size_t smem = smem_bytes(MM_, KB_);
    cudaError_t e = cudaFuncSetAttribute(fused_tc_kernel<KB_, KIND, MM_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    fused_tc_kernel<KB_, KIND, MM_><<<grid, NTHREADS, smem, s>>>(P);
    return cudaGetLastError();
  }
  template <int KIND>
  cudaError_t operator()() const {
#ifdef NEF_SASS_ONLY   // SASS experiments: compile one instantiation (KIND, bond 64, no mask stream)
    if constexpr (KIND != NEF_SASS_ONLY) return cudaErrorInvalidValue;
    else return go<64, KIND, 0>();
#else
    if (MM == 2) {   // per-entry parameter stream: the kinds that have one
      if constexpr (KIND == EW_NB || KIND == EW_BINOM) return KB == 32 ? go<32, KIND, 2>() : go<64, KIND, 2>();
      else return cudaErrorInvalidValue;
    }
    if (KB == 32) return MM ? go<32, KIND, 1>() : go<32, KIND, 0>();
    return MM ? go<64, KIND, 1>() : go<64, KIND, 0>();
#endif
  }
};

size_t smem_bytes(int mm, int kb) {
  const int nv = kb == 32 ? (mm == 1 ? VStages<32, 1>::value : mm == 2 ? VStages<32, 2>::value : VStages<32, 0>::value)
                          : (mm == 1 ? VStages<64, 1>::value : mm == 2 ? VStages<64, 2>::value : VStages<64, 0>::value);
  const int ns = kb == 32 ? (mm == 1 ? YStages<32, 1>::value : mm == 2 ? YStages<32, 2>::value : YStages<32, 0>::value)
                          : (mm == 1 ? YStages<64, 1>::value : mm == 2 ? YStages<64, 2>::value : YStages<64, 0>::value);
  const int vst = kb == 32 ? VSt<32>::SIZE : VSt<64>::SIZE;
  return 1024 + ns * Y_STAGE + (mm == 1 ? ns * M_STAGE : mm == 2 ? ns * Y_STAGE : 0) + nv * vst + 512 + 64;
}

cudaError_t launch(const TcArgs& args, const float* Y, const uint8_t* M, int64_t row_blocks, int64_t chunks,
                   cudaStream_t s, const float* aux) {
  if (!get_encode()) return cudaErrorNotSupported;
  if (aux && M) return cudaErrorInvalidValue;   // the parameter stream runs with the sentinel copy only
  Params P;
  std::memset(&P, 0, sizeof(P));
  P.a = args;
  const int L = args.layout;
  bool ok;
  if (L == 0) {
    uint64_t d[2] = {(uint64_t)args.R, (uint64_t)args.CO};
    uint64_t sy[1] = {(uint64_t)args.R * 4};
    uint32_t by[2] = {128, 64};
    ok = encode(&P.tmY, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, Y, d, sy, by, CU_TENSOR_MAP_SWIZZLE_NONE);
    if (ok && aux) ok = encode(&P.tmA, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, aux, d, sy, by, CU_TENSOR_MAP_SWIZZLE_NONE);
    if (ok && M) {
      uint64_t sm[1] = {(uint64_t)args.R};
      ok = encode(&P.tmM, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, M, d, sm, by, CU_TENSOR_MAP_SWIZZLE_NONE);
    }
  } else if (L == 1) {
    P.a.y3d = (args.CI % 32 == 0 && !g_no_y3d) ? 1 : 0;
    if (P.a.y3d) {
      // {32, CI/32, R}: a box {32, 2, 128} fetches both 128-byte halves of each row back to back
      // (ubench/tma_stream: 7.0 TB/s streaming vs 4.5 TB/s for two {32, 128} boxes per tile)
      uint64_t d[3] = {32, (uint64_t)args.CI / 32, (uint64_t)args.R};
      uint64_t sy[2] = {128, (uint64_t)args.CI * 4};
      uint32_t by[3] = {32, 2, 128};
      ok = encode(&P.tmY, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, Y, d, sy, by, CU_TENSOR_MAP_SWIZZLE_128B);
      if (ok && aux) ok = encode(&P.tmA, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, aux, d, sy, by, CU_TENSOR_MAP_SWIZZLE_128B);
    } else {
      uint64_t d[2] = {(uint64_t)args.CI, (uint64_t)args.R};
      uint64_t sy[1] = {(uint64_t)args.CI * 4};
      uint32_t by[2] = {32, 128};
      ok = encode(&P.tmY, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, Y, d, sy, by, CU_TENSOR_MAP_SWIZZLE_128B);
      if (ok && aux) ok = encode(&P.tmA, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, aux, d, sy, by, CU_TENSOR_MAP_SWIZZLE_128B);
    }
    if (ok && M) {
      uint64_t dm[2] = {(uint64_t)args.CI, (uint64_t)args.R};
      uint64_t sm[1] = {(uint64_t)args.CI};
      uint32_t bm[2] = {64, 128};
      ok = encode(&P.tmM, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, M, dm, sm, bm, CU_TENSOR_MAP_SWIZZLE_64B);
    }
  } else {
    uint64_t d[3] = {(uint64_t)args.CI, (uint64_t)args.R, (uint64_t)args.CO};
    uint64_t sy[2] = {(uint64_t)args.CI * 4, (uint64_t)args.CI * (uint64_t)args.R * 4};
    uint32_t by[3] = {32, 128, 1};
    ok = encode(&P.tmY, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, Y, d, sy, by, CU_TENSOR_MAP_SWIZZLE_128B);
    if (ok && aux) ok = encode(&P.tmA, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, aux, d, sy, by, CU_TENSOR_MAP_SWIZZLE_128B);
    if (ok && M) {
      uint64_t sm[2] = {(uint64_t)args.CI, (uint64_t)args.CI * (uint64_t)args.R};
      uint32_t bm[3] = {64, 128, 1};
      ok = encode(&P.tmM, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, M, d, sm, bm, CU_TENSOR_MAP_SWIZZLE_64B);
    }
  }
  // restart arrays: a single launch is restart 0 = the plain fields
  if (P.a.nrs < 1) {
    P.a.nrs = 1;
    P.a.Ur[0] = args.U;
    for (int q = 0; q < kMaxTabs; ++q) P.a.tabr[0][q] = args.tab[q];
    P.a.Qpartr[0] = args.Qpart;
    P.a.losspartr[0] = args.losspart;
    P.a.countpartr[0] = args.countpart;
    P.a.vdr[0] = args.vd_rows_ptr;
  }
  if (P.a.nrs > 1 && !args.vdirect) return cudaErrorInvalidValue;
  for (int r = 0; ok && args.vdirect && r < P.a.nrs; ++r) {
    // table rows [var_rows][K] -> V stage, two 32-float SW128 boxes (K beyond the row: zeros)
    uint64_t d[2] = {(uint64_t)args.K, (uint64_t)args.var_rows};
    uint64_t sv[1] = {(uint64_t)args.vd_pitch * 4};
    uint32_t bv[2] = {32, 64};
    ok = encode(&P.tmV[r], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, P.a.vdr[r], d, sv, bv,
                NEF_ND_MN ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B);
  }
  if (!ok) return cudaErrorInvalidValue;
  P.a.has_mask = M ? 1 : 0;
  dim3 grid((unsigned)row_blocks, (unsigned)chunks, (unsigned)P.a.nrs);
  return dispatch_ew(args.dv.kind, TcLauncher{P, grid, s, args.KB, M ? 1 : aux ? 2 : 0});
}

}  // namespace tc
}  // namespace nef
