// CUDA-core kernels of the MU sweep (sm_100a):
//   * fused_ffma     : the streamed pass of DESIGN.md §Kernels (K2-FFMA).  For one factor
//                      update it reads each Y / mask entry of the lowering's 2-D view ONCE,
//                      rebuilds the Yhat tile S = U V^T in registers (Alg. 1 line 6, P:165;
//                      never written to memory), forms a = M*Y^alpha*S^(beta-1) and
//                      b = M*S^(alpha+beta-1) (masking P:321) and contracts them with
//                      the column operand: Q_a = P_a V, Q_b = P_b V (Alg. 1 lines 7-8,
//                      P:169-173 via einstr_l).  On the first factor of a sweep it
//                      also accumulates the (alpha,beta)-divergence of that Yhat.
//   * einstep        : one pairwise step of the small-einsum engine (side operands, epilogue)
//   * reduce_q       : deterministic fixed-order sum of split-column partials
//   * update         : Theta <- max(eps, Theta * g^{-1}(A/B)) (eq:explicit-update, P:121;
//                      g table; B == 0 -> multiplier 1, reading R10)
//   * loss_reduce    : fixed-order fp64 sum of per-CTA loss partials
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "divergence.cuh"
#include "kernels.h"

namespace nef {

int pow_code(double p) {
  if (p == 0.0) return POW_0;
  if (p == 1.0) return POW_1;
  if (p == -1.0) return POW_M1;
  if (p == 0.5) return POW_H;
  if (p == -0.5) return POW_MH;
  if (p == -1.5) return POW_M15;
  if (p == 1.5) return POW_15;
  if (p == 2.0) return POW_2;
  if (p == -2.0) return POW_M2;
  return POW_GEN;
}

int ew_kind(double alpha, double beta) {
  if (alpha == 1.0 && beta == 0.0) return EW_KL;
  if (alpha == 1.0 && beta == 1.0) return EW_EUC;
  if (alpha == 1.0 && beta == -0.5) return EW_B_M05;
  if (alpha == 0.5 && beta == 0.0) return EW_A05_B0;
  if (alpha == 1.0 && beta == 0.5) return EW_B05;
  if (alpha == 1.0 && beta == 2.0) return EW_B2;
  if (alpha == 0.5 && beta == 1.0) return EW_A05_B1;
  return EW_GENERIC;
}

DivParams make_div(double alpha, double beta) {
  DivParams d{};
  d.kind = ew_kind(alpha, beta);
  d.alpha = (float)alpha;
  d.beta = (float)beta;
  d.log_case = (alpha == 0.0 && beta == 1.0);
  d.p_xa = (float)alpha;
  d.p_ya = (float)(beta - 1.0);
  d.p_yb = (float)(alpha + beta - 1.0);
  d.c_xa = pow_code(alpha);
  d.c_ya = pow_code(beta - 1.0);
  d.c_yb = pow_code(alpha + beta - 1.0);
  if (alpha == 1.0 && beta == 1.0) d.loss_case = 5;
  else if (alpha != 0 && beta != 0 && alpha + beta != 0) d.loss_case = 0;
  else if (beta == 0 && alpha != 0) d.loss_case = 1;
  else if (alpha == -beta && alpha != 0) d.loss_case = 2;
  else if (alpha == 0 && beta != 0) d.loss_case = 3;
  else d.loss_case = 4;
  return d;
}

DivParams make_div_fam(int fam, double alpha, double beta, double prm) {
  if (fam == FAM_AB) return make_div(alpha, beta);
  DivParams d{};
  d.alpha = 1.f;
  d.beta = 0.f;
  d.prm = (float)prm;
  d.kind = fam == FAM_NEGBIN ? EW_NB : fam == FAM_BERNOULLI ? EW_BERN : fam == FAM_BINOMIAL ? EW_BINOM : EW_JS;
  return d;
}

UpdArgs make_upd_fam(int fam, double alpha, double beta, double eps) {
  if (fam == FAM_AB) return make_upd(alpha, beta, eps);
  // g(lambda) = lambda for NB / Bernoulli / binomial, log for JS
  UpdArgs u{};
  u.eps = eps;
  u.g_case = fam == FAM_JS ? 1 : 0;
  u.inv_expo = 1.0;
  return u;
}

UpdArgs make_upd(double alpha, double beta, double eps) {
  // g(lambda) table
  UpdArgs u{};
  u.eps = eps;
  if (alpha == 0.0 && beta == 1.0) { u.g_case = 1; u.inv_expo = 0; return u; }
  double q = (1.0 - beta) / alpha;
  double expo;
  if (q > 1) expo = 1.0 - beta;
  else if (q < 0) expo = alpha + beta - 1.0;
  else expo = alpha;
  u.g_case = 0;
  u.inv_expo = 1.0 / expo;
  return u;
}

// --------------------------------------------------------------------------------------
// fused streaming pass (CUDA cores)
// --------------------------------------------------------------------------------------
// Row-block height BM_ (64, or 32 when the lowering has <= 32 rows: factors with few rows over
// millions of columns, e.g. the paper's ICEWS / WITS time and action factors); 4 x 4 outputs of
// S per thread, NT = 4 * BM_ threads, 64 columns per tile.
constexpr int BN = 64;

template <int KP, int BM>
struct __align__(16) FSmem {
  static constexpr int PADR = BM + 4;
  float Ut[KP][BM];
  float Vt[KP][BN];
  float V[BN][KP];
  float Pa[BN][PADR];
  float Pb[BN][PADR];
  uint8_t Mk[BN][PADR];
  float Ax[BN][PADR];          // per-entry phi / n (aux losses only)
  long long coff[BN];
  long long roff[BM];
  int toff[kMaxTabs][BN];
};

struct FusedDev {
  FusedArgs a;
  int32_t boff[kMaxTabs][64];
};

template <int KP, int KIND, int BM>
__global__ void __launch_bounds__(4 * BM) fused_ffma_kernel(const __grid_constant__ FusedDev P) {
  constexpr int NT = 4 * BM;     // threads: BM / 4 row groups x 16 column groups
  constexpr int RG = BM / 4;
  extern __shared__ __align__(16) unsigned char smraw[];
  FSmem<KP, BM>& sm = *reinterpret_cast<FSmem<KP, BM>*>(smraw);
  const FusedArgs& a = P.a;
  constexpr int KQ = KP / 16;
  const int t = threadIdx.x;
  const int64_t row0 = (int64_t)blockIdx.x * BM;
  const int rows_here = (int)(a.n_rows - row0 < BM ? a.n_rows - row0 : BM);
  const int K = a.K;

  if (t < BM) {
    long long off = -1;
    if (t < rows_here) {
      int64_t rem = row0 + t;
      off = 0;
      for (int d = a.nr - 1; d >= 0; --d) {
        int64_t i = rem % a.rdim[d];
        rem /= a.rdim[d];
        off += i * a.rys[d];
      }
    }
    sm.roff[t] = off;
  }
  for (int e = t; e < KP * BM; e += NT) {
    int k = e / BM, r = e % BM;
    sm.Ut[k][r] = (k < K && r < rows_here) ? a.U[(row0 + r) * K + k] : 0.f;
  }
  __syncthreads();

  double qa_d[4][KQ], qb_d[4][KQ];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < KQ; ++j) { qa_d[i][j] = 0.0; qb_d[i][j] = 0.0; }
  double loss_acc[3] = {0.0, 0.0, 0.0};   // [role]: split fits keep train / validation / heldout apart
  long long cnt[3] = {0, 0, 0};
  const int rs = (t % RG) * 4;
  const int cs = (t / RG) * 4;
  const int kq = (t / RG) * KQ;

  const int64_t total_tiles = (a.n_cols + BN - 1) / BN;
  const int64_t tb = (int64_t)blockIdx.y * a.tiles_per_chunk;
  const int64_t te = (tb + a.tiles_per_chunk < total_tiles ? tb + a.tiles_per_chunk : total_tiles);
  for (int64_t tile = tb; tile < te; ++tile) {
    const int64_t col0 = tile * BN;
    const int cols_here = (int)(a.n_cols - col0 < BN ? a.n_cols - col0 : BN);
    if (t < BN) {
      long long off = -1;
      int to[kMaxTabs] = {0, 0, 0, 0};
      if (t < cols_here) {
        int64_t rem = col0 + t;
        off = 0;
        for (int d = a.nc - 1; d >= 0; --d) {
          int64_t i = rem % a.cdim[d];
          rem /= a.cdim[d];
          off += i * a.cys[d];
          for (int q = 0; q < a.ntab; ++q) to[q] += (int)(i * a.tcs[q][d]);
        }
      }
      sm.coff[t] = off;
      for (int q = 0; q < kMaxTabs; ++q) sm.toff[q][t] = to[q];
    }
    __syncthreads();
    // Y / mask tile: each entry read once; a missing entry's value is never loaded
#pragma unroll 4
    for (int i = 0; i < BM * BN / NT; ++i) {
      int e = t + i * NT;
      int r, c;
      if (a.row_fast) { r = e % BM; c = e / BM; } else { r = e / BN; c = e % BN; }
      long long ro = sm.roff[r], co = sm.coff[c];
      float y = 0.f, ax = 1.f;
      uint8_t m = 0;
      if (ro >= 0 && co >= 0) {
        long long off = ro + co;
        // mask: observed flag (R6); split fit: the label itself (R29)
        m = a.M ? (a.split ? __ldg(a.M + off) : (uint8_t)(__ldg(a.M + off) != 0)) : (uint8_t)1;
        if (m) {
          y = __ldg(a.Y + off);
          if (a.aux) ax = __ldg(a.aux + off);
        }
      }
      sm.Pa[c][r] = y;
      sm.Mk[c][r] = m;
      if (a.aux) sm.Ax[c][r] = ax;
    }
    // V tile = prod of column tables (Khatri-Rao / side operands), both layouts
    for (int e = t; e < BN * KP; e += NT) {
      int c = e / KP, k = e % KP;
      float v = 0.f;
      if (c < cols_here && k < K) {
        v = 1.f;
        for (int q = 0; q < a.ntab; ++q) v *= __ldg(a.tab[q] + sm.toff[q][c] + P.boff[q][k]);
      }
      sm.V[c][k] = v;
      sm.Vt[k][c] = v;
    }
    __syncthreads();
    // S = U V^T (reconstruction tile, registers only)
    float s[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) s[i][j] = 0.f;
#pragma unroll 8
    for (int k = 0; k < KP; ++k) {
      float4 u = *reinterpret_cast<const float4*>(&sm.Ut[k][rs]);
      float4 v = *reinterpret_cast<const float4*>(&sm.Vt[k][cs]);
      float uu[4] = {u.x, u.y, u.z, u.w}, vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) s[i][j] = fmaf(uu[i], vv[j], s[i][j]);
    }
    // divergence weights a, b (+ loss) in registers
    float lsum[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = cs + j;
      float4 y4 = *reinterpret_cast<const float4*>(&sm.Pa[c][rs]);
      uint32_t m4 = *reinterpret_cast<const uint32_t*>(&sm.Mk[c][rs]);
      float yy[4] = {y4.x, y4.y, y4.z, y4.w};
      float pa[4], pb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t role = (m4 >> (8 * i)) & 0xffu;   // 0 unobserved; 1 train (and any observed entry)
        const bool obs = a.split ? role == 1u : role != 0u;
        const float yh = fmaxf(s[i][j], 1e-30f);       // Yhat floor (reading R4)
        const float x = role ? yy[i] : 1.f;
        float av, bv, lv = 0.f;
        if constexpr (KIND == EW_NB || KIND == EW_BINOM) {
          if (a.aux) {                                   // per-entry phi / n
            const float ax = role ? sm.Ax[c][rs + i] : 1.f;
            Ew<KIND>::ab_aux(x, yh, ax, av, bv);
            if (a.mode != 0 && role) lv = Ew<KIND>::loss_aux(x, yh, ax);
          } else {
            Ew<KIND>::ab(x, yh, a.dv, av, bv);
            if (a.mode != 0 && role) lv = Ew<KIND>::loss(x, yh, a.dv);
          }
        } else {
          Ew<KIND>::ab(x, yh, a.dv, av, bv);
          if (a.mode != 0 && role) lv = Ew<KIND>::loss(x, yh, a.dv);
        }
        pa[i] = obs ? av : 0.f;                          // select, never multiply (R5)
        pb[i] = obs ? bv : 0.f;
        if (a.mode != 0 && role) {
          const int q = a.split ? (int)role - 1 : 0;
          if (q == 0) { lsum[0] += lv; cnt[0] += 1; }
          else if (q == 1) { lsum[1] += lv; cnt[1] += 1; }
          else if (q == 2) { lsum[2] += lv; cnt[2] += 1; }
        }
      }
      if (a.mode != 2) {
        *reinterpret_cast<float4*>(&sm.Pa[c][rs]) = make_float4(pa[0], pa[1], pa[2], pa[3]);
        *reinterpret_cast<float4*>(&sm.Pb[c][rs]) = make_float4(pb[0], pb[1], pb[2], pb[3]);
      }
    }
    loss_acc[0] += (double)lsum[0];
    loss_acc[1] += (double)lsum[1];
    loss_acc[2] += (double)lsum[2];
    __syncthreads();
    if (a.mode != 2) {
      float qa[4][KQ], qb[4][KQ];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < KQ; ++j) { qa[i][j] = 0.f; qb[i][j] = 0.f; }
#pragma unroll 4
      for (int c = 0; c < BN; ++c) {
        float4 p4 = *reinterpret_cast<const float4*>(&sm.Pa[c][rs]);
        float4 q4 = *reinterpret_cast<const float4*>(&sm.Pb[c][rs]);
        float pa[4] = {p4.x, p4.y, p4.z, p4.w}, pb[4] = {q4.x, q4.y, q4.z, q4.w};
        float v[KQ];
#pragma unroll
        for (int j = 0; j < KQ; ++j) v[j] = sm.V[c][kq + j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < KQ; ++j) {
            qa[i][j] = fmaf(pa[i], v[j], qa[i][j]);
            qb[i][j] = fmaf(pb[i], v[j], qb[i][j]);
          }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < KQ; ++j) { qa_d[i][j] += (double)qa[i][j]; qb_d[i][j] += (double)qb[i][j]; }
    }
    __syncthreads();
  }
  if (a.mode != 2) {
    const int64_t elems = a.n_rows * (int64_t)K;
    float* qa_out = a.Qpart + (int64_t)blockIdx.y * 2 * elems;
    float* qb_out = qa_out + elems;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int r = rs + i;
      if (r >= rows_here) continue;
#pragma unroll
      for (int j = 0; j < KQ; ++j) {
        int k = kq + j;
        if (k < K) {
          qa_out[(row0 + r) * K + k] = (float)qa_d[i][j];
          qb_out[(row0 + r) * K + k] = (float)qb_d[i][j];
        }
      }
    }
  }
  if (a.mode != 0) {
    // fixed-order block reduction of the loss (deterministic), one per role on split fits
    __shared__ double red[NT];
    __shared__ long long redc[NT];
    const int64_t parts = (int64_t)gridDim.x * gridDim.y;
    const int64_t id = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
    for (int q = 0; q < (a.split ? 3 : 1); ++q) {
      red[t] = loss_acc[q];
      redc[t] = cnt[q];
      __syncthreads();
      for (int w = NT / 2; w > 0; w >>= 1) {
        if (t < w) { red[t] += red[t + w]; redc[t] += redc[t + w]; }
        __syncthreads();
      }
      if (t == 0) {
        a.losspart[q * parts + id] = red[0];
        a.countpart[q * parts + id] = redc[0];
      }
      __syncthreads();
    }
  }
}

template <int KP, int KIND, int BM>
static cudaError_t launch_kp_bm(const FusedDev& d, cudaStream_t s) {
  size_t smem = sizeof(FSmem<KP, BM>);
  cudaError_t e = cudaFuncSetAttribute(fused_ffma_kernel<KP, KIND, BM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int64_t row_blocks = (d.a.n_rows + BM - 1) / BM;
  dim3 grid((unsigned)row_blocks, (unsigned)d.a.n_chunks);
  fused_ffma_kernel<KP, KIND, BM><<<grid, 4 * BM, smem, s>>>(d);
  return cudaGetLastError();
}
// (<= 32 rows: one row block either way, so the planner's partial layout is unchanged)
template <int KP, int KIND>
static cudaError_t launch_kp(const FusedDev& d, cudaStream_t s) {
  static const bool bm64 = std::getenv("NEF_FFMA_BM64") != nullptr;   // diagnostics
  if (d.a.n_rows <= 32 && !bm64) return launch_kp_bm<KP, KIND, 32>(d, s);
  return launch_kp_bm<KP, KIND, 64>(d, s);
}

struct FfmaLauncher {
  const FusedDev& d;
  cudaStream_t s;
  template <int KIND>
  cudaError_t operator()() const {
    if (d.a.K <= 16) return launch_kp<16, KIND>(d, s);
    if (d.a.K <= 32) return launch_kp<32, KIND>(d, s);
    if (d.a.K <= 64) return launch_kp<64, KIND>(d, s);
    return cudaErrorInvalidValue;
  }
};

cudaError_t launch_fused_ffma(const FusedArgs& a, cudaStream_t s) {
  FusedDev d;
  d.a = a;
  for (int q = 0; q < kMaxTabs; ++q)
    for (int k = 0; k < 64; ++k) d.boff[q][k] = 0;
  for (int q = 0; q < a.ntab; ++q)
    for (int k = 0; k < a.K && k < 64; ++k) d.boff[q][k] = a.boff[q * a.K + k];
  return dispatch_ew(a.dv.kind, FfmaLauncher{d, s});
}

// --------------------------------------------------------------------------------------
// small einsum step
// --------------------------------------------------------------------------------------
struct EinStepDev {
  int nout, nsum;
  long long odim[kMaxDims], as_o[kMaxDims], bs_o[kMaxDims];
  long long sdim[kMaxDims], as_s[kMaxDims], bs_s[kMaxDims];
  long long out_size, sum_size;
};

// Small einsum step C[out] = sum A[..] (* B[..]).  Templated on the index type (32-bit when
// every offset fits) and on the parallelisation: L lanes share one output, each summing a
// contiguous slice of the summed indices (odometer started by one decomposition), partials
// combined with warp shuffles in fp64.  L = 1 for many outputs, 32 for few outputs with long sums
// (e.g. the Tucker core's epilogue: 4096 outputs x 65536 terms).
template <typename I, int L>
__global__ void einstep_kernel(const __grid_constant__ EinStepDev st, const float* __restrict__ A,
                               const float* __restrict__ B, float* __restrict__ C) {
  const long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = (int)(gt % L);
  const long long stride = ((long long)gridDim.x * blockDim.x) / L;
  const I chunk = (I)((st.sum_size + L - 1) / L);
  const I s0 = (I)lane * chunk;
  const I s1 = (I)((long long)s0 + chunk < st.sum_size ? (long long)s0 + chunk : st.sum_size);
  // warp-uniform trip count: the L lanes of an output combine with whole-warp shuffles
  for (long long o = gt / L;; o += stride) {
    const bool valid = o < st.out_size;
    if (L > 1 ? __all_sync(0xffffffffu, !valid) : !valid) break;
    I rem = (I)(valid ? o : 0), ao = 0, bo = 0;
    for (int d = st.nout - 1; d >= 0; --d) {
      const I od = (I)st.odim[d];
      const I i = rem % od;
      rem /= od;
      ao += i * (I)st.as_o[d];
      bo += i * (I)st.bs_o[d];
    }
    I sidx[kMaxDims];
    {
      I r = s0;
      for (int d = st.nsum - 1; d >= 0; --d) {
        const I sd = (I)st.sdim[d];
        sidx[d] = r % sd;
        r /= sd;
        ao += sidx[d] * (I)st.as_s[d];
        bo += sidx[d] * (I)st.bs_s[d];
      }
    }
    double acc = 0.0;
    for (I s = s0; valid && s < s1; ++s) {
      double v = (double)__ldg(A + ao);
      if (B) v *= (double)__ldg(B + bo);
      acc += v;
      for (int d = st.nsum - 1; d >= 0; --d) {
        ao += (I)st.as_s[d];
        bo += (I)st.bs_s[d];
        if (++sidx[d] < (I)st.sdim[d]) break;
        ao -= (I)(st.as_s[d] * st.sdim[d]);
        bo -= (I)(st.bs_s[d] * st.sdim[d]);
        sidx[d] = 0;
      }
    }
    if (L > 1) {
#pragma unroll
      for (int w = L / 2; w > 0; w >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, w);
    }
    if (valid && lane == 0) C[o] = (float)acc;
  }
}

// Fast path for the common step shape: ONE summed index and at most three output indices (the
// side operands and epilogues of CP / Tucker / the paper's custom models, e.g. T[j,k,a] =
// sum_c C[k,c] T1[j,a,c] or the Tucker core's A[a,c,j] = sum_i Q[i,j,c] A[i,a]).  The outputs are
// enumerated in an order chosen on the host (innermost = the output index with the smallest
// stride in the larger operand, so a warp's loads coalesce; C is written through its own
// strides), LANES threads share one output for long sums (interleaved terms, combined by warp
// shuffles), and the terms are summed in blocks of 16 in fp32 (four independent partial sums)
// carried in fp64.  The generic kernel above issued ~300 instructions per output of 16 terms
// (odometer per term, fp64 conversions): ncu 33 us at IPC 3.2 for 1 M outputs on c2.
struct EinStep1Dev {
  int nout;
  int odim[3], as_o[3], bs_o[3], cs_o[3];   // in enumeration order (last = innermost)
  int S, as, bs;
  int out_size;
};
template <bool HASB, int LANES>
__global__ void einstep1_kernel(const __grid_constant__ EinStep1Dev st, const float* __restrict__ A,
                                const float* __restrict__ B, float* __restrict__ C) {
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = gt % LANES;
  const int stride = (gridDim.x * blockDim.x) / LANES;
  // warp-uniform trip count (the lanes of an output shuffle with the whole warp)
  for (int o = gt / LANES;; o += stride) {
    const bool valid = o < st.out_size;
    if (LANES > 1 ? __all_sync(0xffffffffu, !valid) : !valid) break;
    int ao = 0, bo = 0, co = 0, rem = valid ? o : 0;
#pragma unroll
    for (int d = 2; d >= 0; --d) {
      if (d >= st.nout) continue;
      const int n = st.odim[d];
      const int q = d > 0 ? rem / n : 0;
      const int i = rem - q * n;
      rem = q;
      ao += i * st.as_o[d];
      bo += i * st.bs_o[d];
      co += i * st.cs_o[d];
    }
    double tot = 0.0;
    for (int s0 = lane * 16; valid && s0 < st.S; s0 += 16 * LANES) {   // blocks of 16 terms
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      const int s1 = s0 + 16 < st.S ? s0 + 16 : st.S;
      int s = s0;
      for (; s + 4 <= s1; s += 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float a = __ldg(A + ao + (s + u) * st.as);
          acc[u] = HASB ? fmaf(a, __ldg(B + bo + (s + u) * st.bs), acc[u]) : acc[u] + a;
        }
      }
      for (; s < s1; ++s) {
        const float a = __ldg(A + ao + s * st.as);
        acc[0] = HASB ? fmaf(a, __ldg(B + bo + s * st.bs), acc[0]) : acc[0] + a;
      }
      tot += ((double)acc[0] + (double)acc[1]) + ((double)acc[2] + (double)acc[3]);
    }
    if (LANES > 1) {
#pragma unroll
      for (int w = LANES / 2; w > 0; w >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, w);
    }
    if (valid && lane == 0) C[co] = (float)tot;
  }
}

// GEMM-shaped steps: every summed index in both operands, every output index in A only (M),
// in B only (N) or in both (batch).  C[b, m, n] = sum_k A[b, m, k] B[b, n, k] as a shared-memory
// tiled product: a block computes a (16 TM) x (16 TN) output tile with 256 threads (TM x TN
// outputs each), K in chunks of 16 staged through shared memory; fp32 partial sums over 256
// terms carried in fp64 (fixed order: deterministic).  The Tucker side operands and
// epilogues (c2: 1-17 M MAC per step) took 13-23 us per step on the per-output kernels above
// (each thread gathering its own terms, ~20 % of the SMs busy).
struct EinGemmDev {
  int nm, nn, nb, nk;
  int mdim[3], am[3], cm[3];
  int ndim[3], bn[3], cn[3];
  int bdim[2], ab[2], bb[2], cb[2];
  int kdim[2], ak[2], bk[2];
  int M, N, K, NB;
  int a_kfast, b_kfast;   // the operand's innermost summed index has stride 1: load along k
  int ksplit, kc;         // the sum split over ksplit blocks of kc terms (multiple of 16) each
  float* part;            // ksplit > 1: dense partials [ksplit][NB][M][N], summed by einstep_gemm_reduce
};
__device__ __forceinline__ int gemm_koff(const EinGemmDev& g, int k, bool isA) {
  if (g.nk == 1) return k * (isA ? g.ak[0] : g.bk[0]);
  const int k1 = k % g.kdim[1], k0 = k / g.kdim[1];
  return isA ? k0 * g.ak[0] + k1 * g.ak[1] : k0 * g.bk[0] + k1 * g.bk[1];
}
template <int TM, int TN>
__global__ void __launch_bounds__(256) einstep_gemm_kernel(const __grid_constant__ EinGemmDev g, const float* __restrict__ A,
                                                           const float* __restrict__ B, float* __restrict__ C) {
  constexpr int BM = 16 * TM, BN = 16 * TN, BK = 16;
  __shared__ float As[BK][BM + 1], Bs[BK][BN + 1];
  __shared__ int aoff[BM], boff[BN], coff_m[BM], coff_n[BN];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int n0 = blockIdx.x * BN, m0 = blockIdx.y * BM;
  int abo = 0, bbo = 0, cbo = 0;
  const int sp = (int)blockIdx.z % g.ksplit, bz = (int)blockIdx.z / g.ksplit;
  const int kbeg = sp * g.kc, kend = min(g.K, kbeg + g.kc);
  {
    int rem = bz;
    for (int d = g.nb - 1; d >= 0; --d) {
      const int i = rem % g.bdim[d];
      rem /= g.bdim[d];
      abo += i * g.ab[d];
      bbo += i * g.bb[d];
      cbo += i * g.cb[d];
    }
  }
  for (int i = tid; i < BM; i += 256) {
    int rem = m0 + i, ao = 0, co = 0;
    const bool ok = rem < g.M;
    for (int d = g.nm - 1; d >= 0; --d) {
      const int q = rem % g.mdim[d];
      rem /= g.mdim[d];
      ao += q * g.am[d];
      co += q * g.cm[d];
    }
    aoff[i] = ok ? abo + ao : -1;
    coff_m[i] = cbo + co;
  }
  for (int i = tid; i < BN; i += 256) {
    int rem = n0 + i, bo = 0, co = 0;
    const bool ok = rem < g.N;
    for (int d = g.nn - 1; d >= 0; --d) {
      const int q = rem % g.ndim[d];
      rem /= g.ndim[d];
      bo += q * g.bn[d];
      co += q * g.cn[d];
    }
    boff[i] = ok ? bbo + bo : -1;
    coff_n[i] = co;
  }
  __syncthreads();
  float acc[TM][TN];
  double dacc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) { acc[i][j] = 0.f; dacc[i][j] = 0.0; }
  int chunk = 0;
  for (int k0 = kbeg; k0 < kend; k0 += BK, ++chunk) {
    for (int e = tid; e < BM * BK; e += 256) {
      const int mm = g.a_kfast ? e / BK : e % BM, kk = g.a_kfast ? e % BK : e / BM;
      const int k = k0 + kk, ao = aoff[mm];
      As[kk][mm] = (k < kend && ao >= 0) ? __ldg(A + ao + gemm_koff(g, k, true)) : 0.f;
    }
    for (int e = tid; e < BN * BK; e += 256) {
      const int nn = g.b_kfast ? e / BK : e % BN, kk = g.b_kfast ? e % BK : e / BN;
      const int k = k0 + kk, bo = boff[nn];
      Bs[kk][nn] = (k < kend && bo >= 0) ? __ldg(B + bo + gemm_koff(g, k, false)) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float av[TM], bv[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) av[i] = As[kk][ty * TM + i];
#pragma unroll
      for (int j = 0; j < TN; ++j) bv[j] = Bs[kk][tx * TN + j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
    if ((chunk & 15) == 15) {   // every 256 terms: fp32 partial -> fp64
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) { dacc[i][j] += (double)acc[i][j]; acc[i][j] = 0.f; }
    }
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int mm = ty * TM + i;
    if (aoff[mm] < 0) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int nn = tx * TN + j;
      if (boff[nn] < 0) continue;
      const float v = (float)(dacc[i][j] + (double)acc[i][j]);
      if (g.ksplit == 1) C[coff_m[mm] + coff_n[nn]] = v;
      else g.part[(((int64_t)sp * g.NB + bz) * g.M + m0 + mm) * g.N + n0 + nn] = v;
    }
  }
}
// the split partials of einstep_gemm_kernel summed in split order (fp64), written through C's strides
__global__ void einstep_gemm_reduce(const __grid_constant__ EinGemmDev g, float* __restrict__ C) {
  const int64_t tot = (int64_t)g.NB * g.M * g.N;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < tot; o += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int sp = 0; sp < g.ksplit; ++sp) acc += (double)g.part[sp * tot + o];
    int n = (int)(o % g.N), m = (int)((o / g.N) % g.M), b = (int)(o / ((int64_t)g.N * g.M));
    int co = 0;
    for (int d = g.nn - 1; d >= 0; --d) { co += (n % g.ndim[d]) * g.cn[d]; n /= g.ndim[d]; }
    for (int d = g.nm - 1; d >= 0; --d) { co += (m % g.mdim[d]) * g.cm[d]; m /= g.mdim[d]; }
    for (int d = g.nb - 1; d >= 0; --d) { co += (b % g.bdim[d]) * g.cb[d]; b /= g.bdim[d]; }
    C[co] = (float)acc;
  }
}

// Classifies a step for the GEMM kernel (false: not GEMM-shaped, or beyond its limits) and picks
// the tile (tm, tn) and the split of the sum: steps whose output tiles would occupy fewer than
// ~2 blocks per SM split long sums (K > 64) over up to 64 blocks of >= 64 terms.
static bool gemm_classify(const EinStep& st, bool hasB, EinGemmDev& g, int& tm, int& tn, dim3& grid) {
  static const bool off = std::getenv("NEF_EINSTEP_NOGEMM") != nullptr;   // diagnostics
  g = EinGemmDev{};
  if (off || !hasB || st.nsum < 1 || st.nsum > 2 || st.nout > kMaxDims) return false;
  long long cst[kMaxDims];
  long long acc = 1;
  for (int k = st.nout - 1; k >= 0; --k) { cst[k] = acc; acc *= st.odim[k]; }
  long long M = 1, N = 1, NB = 1, K = 1, span_a = 0, span_b = 0;
  for (int k = 0; k < st.nsum; ++k) {
    if (st.as_s[k] == 0 || st.bs_s[k] == 0) return false;
    g.kdim[g.nk] = (int)st.sdim[k]; g.ak[g.nk] = (int)st.as_s[k]; g.bk[g.nk] = (int)st.bs_s[k]; ++g.nk;
    K *= st.sdim[k];
    span_a += (st.sdim[k] - 1) * st.as_s[k];
    span_b += (st.sdim[k] - 1) * st.bs_s[k];
  }
  for (int k = 0; k < st.nout; ++k) {
    const bool ia = st.as_o[k] != 0, ib = st.bs_o[k] != 0;
    if (st.odim[k] == 1) continue;
    if (ia && ib) {
      if (g.nb == 2) return false;
      g.bdim[g.nb] = (int)st.odim[k]; g.ab[g.nb] = (int)st.as_o[k]; g.bb[g.nb] = (int)st.bs_o[k]; g.cb[g.nb] = (int)cst[k]; ++g.nb;
      NB *= st.odim[k];
    } else if (ia) {
      if (g.nm == 3) return false;
      g.mdim[g.nm] = (int)st.odim[k]; g.am[g.nm] = (int)st.as_o[k]; g.cm[g.nm] = (int)cst[k]; ++g.nm;
      M *= st.odim[k];
    } else if (ib) {
      if (g.nn == 3) return false;
      g.ndim[g.nn] = (int)st.odim[k]; g.bn[g.nn] = (int)st.bs_o[k]; g.cn[g.nn] = (int)cst[k]; ++g.nn;
      N *= st.odim[k];
    } else {
      return false;   // an output index in neither operand (broadcast): not a product
    }
    span_a += (st.odim[k] - 1) * st.as_o[k];
    span_b += (st.odim[k] - 1) * st.bs_o[k];
  }
  if (g.nm == 0) { g.nm = 1; g.mdim[0] = 1; }
  if (g.nn == 0) { g.nn = 1; g.ndim[0] = 1; }
  if (span_a >= (1ll << 30) || span_b >= (1ll << 30) || acc >= (1ll << 30) || NB > 65535) return false;
  if (K >= (1ll << 30) || M * N * NB >= (1ll << 30)) return false;
  g.M = (int)M; g.N = (int)N; g.K = (int)K; g.NB = (int)NB;
  g.a_kfast = g.ak[g.nk - 1] == 1;
  g.b_kfast = g.bk[g.nk - 1] == 1;
  tm = M >= 48 ? 4 : M >= 24 ? 2 : 1;
  tn = N >= 48 ? 4 : N >= 24 ? 2 : 1;
  auto ntiles = [&] { return ((N + 16 * tn - 1) / (16 * tn)) * ((M + 16 * tm - 1) / (16 * tm)) * NB; };
  // small outputs: smaller per-thread tiles until the blocks cover the SMs (a 65 536-output
  // step at 4 x 4 ran as 16 blocks on 16 SMs, its latency chain ~4 loads + 16 stores deep)
  while (ntiles() < 148 && (tm > 1 || tn > 1)) {
    if (tm >= tn) tm /= 2;
    else tn /= 2;
  }
  const long long tiles = ntiles();
  long long ks = 1;
  if (K > 64 && tiles < 296) ks = std::min<long long>(std::min<long long>((296 + tiles - 1) / tiles, (K + 63) / 64), 64);
  g.kc = (int)(((K + ks - 1) / ks + 15) / 16 * 16);
  g.ksplit = (int)((K + g.kc - 1) / g.kc);
  grid = dim3((unsigned)((N + 16 * tn - 1) / (16 * tn)), (unsigned)((M + 16 * tm - 1) / (16 * tm)), (unsigned)(NB * g.ksplit));
  return grid.y <= 65535 && grid.z <= 65535;
}

int64_t einstep_scratch_floats(const EinStep& st) {
  EinGemmDev g;
  int tm, tn;
  dim3 grid;
  if (!gemm_classify(st, st.b.kind != BUF_NONE, g, tm, tn, grid) || g.ksplit == 1) return 0;
  return (int64_t)g.ksplit * g.NB * g.M * g.N;
}

static bool einstep_gemm(const EinStep& st, const float* A, const float* B, float* C, cudaStream_t s, float* scratch) {
  EinGemmDev g;
  int tm, tn;
  dim3 grid;
  if (!gemm_classify(st, B != nullptr, g, tm, tn, grid)) return false;
  if (g.ksplit > 1) {
    if (!scratch) return false;   // (no scratch: the per-output kernels)
    g.part = scratch;
  }
#define NEF_GEMM_CASE(A_, B_) \
  if (tm == A_ && tn == B_) einstep_gemm_kernel<A_, B_><<<grid, 256, 0, s>>>(g, A, B, C);
  NEF_GEMM_CASE(4, 4) NEF_GEMM_CASE(4, 2) NEF_GEMM_CASE(4, 1) NEF_GEMM_CASE(2, 4) NEF_GEMM_CASE(2, 2)
  NEF_GEMM_CASE(2, 1) NEF_GEMM_CASE(1, 4) NEF_GEMM_CASE(1, 2) NEF_GEMM_CASE(1, 1)
#undef NEF_GEMM_CASE
  if (g.ksplit > 1) {
    const int64_t tot = (int64_t)g.NB * g.M * g.N;
    einstep_gemm_reduce<<<(unsigned)std::min<int64_t>((tot + 255) / 256, 148 * 8), 256, 0, s>>>(g, C);
  }
  return true;
}

cudaError_t launch_einstep(const EinStep& st, const float* A, const float* B, float* C, cudaStream_t s, float* scratch) {
  if (einstep_gemm(st, A, B, C, s, scratch)) return cudaGetLastError();
  static const bool no_fast = std::getenv("NEF_EINSTEP_GENERIC") != nullptr;   // diagnostics
  {
    // fast path eligibility: one summed index, <= 3 output indices, 32-bit offsets
    bool ok = !no_fast && st.nsum == 1 && st.nout <= 3 && st.out_size < (1ll << 30) && st.sum_size < (1ll << 30);
    long long span_a = (st.sdim[0] - 1) * st.as_s[0], span_b = (st.sdim[0] - 1) * st.bs_s[0];
    for (int k = 0; k < st.nout; ++k) {
      span_a += (st.odim[k] - 1) * st.as_o[k];
      span_b += (st.odim[k] - 1) * st.bs_o[k];
    }
    ok = ok && span_a < (1ll << 30) && span_b < (1ll << 30);
    if (ok) {
      // C strides (row-major over the step's output order), then the enumeration order: the
      // innermost enumerated index is the one with the smallest nonzero stride in the operand
      // spanning more memory (its loads coalesce across a warp)
      long long cst[kMaxDims];
      long long acc = 1;
      for (int k = st.nout - 1; k >= 0; --k) { cst[k] = acc; acc *= st.odim[k]; }
      const bool big_a = !B || span_a >= span_b;
      int order[3] = {0, 1, 2};
      if (st.nout > 1) {
        int inner = st.nout - 1;
        long long best = -1;
        for (int k = 0; k < st.nout; ++k) {
          const long long str = big_a ? st.as_o[k] : st.bs_o[k];
          if (str > 0 && st.odim[k] > 1 && (best < 0 || str < best)) { best = str; inner = k; }
        }
        int w = 0;
        for (int k = 0; k < st.nout; ++k)
          if (k != inner) order[w++] = k;
        order[w] = inner;
      }
      EinStep1Dev d{};
      d.nout = st.nout;
      for (int k = 0; k < st.nout; ++k) {
        const int src = order[k];
        d.odim[k] = (int)st.odim[src];
        d.as_o[k] = (int)st.as_o[src];
        d.bs_o[k] = (int)st.bs_o[src];
        d.cs_o[k] = (int)cst[src];
      }
      d.S = (int)st.sdim[0];
      d.as = (int)st.as_s[0];
      d.bs = (int)st.bs_s[0];
      d.out_size = (int)st.out_size;
      // long sums over few outputs: 8 (or 4) threads per output
      const int lanes = (st.sum_size >= 128 && st.out_size < 148 * 2048) ? 8 : (st.sum_size > 64 ? 4 : 1);
      long long blocks = (st.out_size * lanes + 255) / 256;
      if (blocks > 148 * 32) blocks = 148 * 32;
      if (blocks < 1) blocks = 1;
      const unsigned nb = (unsigned)blocks;
      if (B) {
        if (lanes == 8) einstep1_kernel<true, 8><<<nb, 256, 0, s>>>(d, A, B, C);
        else if (lanes == 4) einstep1_kernel<true, 4><<<nb, 256, 0, s>>>(d, A, B, C);
        else einstep1_kernel<true, 1><<<nb, 256, 0, s>>>(d, A, B, C);
      } else {
        if (lanes == 8) einstep1_kernel<false, 8><<<nb, 256, 0, s>>>(d, A, B, C);
        else if (lanes == 4) einstep1_kernel<false, 4><<<nb, 256, 0, s>>>(d, A, B, C);
        else einstep1_kernel<false, 1><<<nb, 256, 0, s>>>(d, A, B, C);
      }
      return cudaGetLastError();
    }
  }
  EinStepDev d{};
  d.nout = st.nout;
  d.nsum = st.nsum;
  long long span = 1;   // largest offset reached in A or B (bounds the index type)
  long long sa = 0, sb = 0;
  for (int k = 0; k < kMaxDims; ++k) {
    d.odim[k] = st.odim[k]; d.as_o[k] = st.as_o[k]; d.bs_o[k] = st.bs_o[k];
    d.sdim[k] = st.sdim[k]; d.as_s[k] = st.as_s[k]; d.bs_s[k] = st.bs_s[k];
    if (k < st.nout) { sa += (st.odim[k] - 1) * st.as_o[k]; sb += (st.odim[k] - 1) * st.bs_o[k]; }
    if (k < st.nsum) { sa += (st.sdim[k] - 1) * st.as_s[k]; sb += (st.sdim[k] - 1) * st.bs_s[k]; }
  }
  span = std::max(std::max(sa, sb), std::max<long long>(st.out_size, st.sum_size));
  d.out_size = st.out_size;
  d.sum_size = st.sum_size;
  // long sums are split over a warp only for few outputs (a wider split - 65536 outputs x 256
  // terms of the Tucker core's epilogue - measured 14 % slower over a c2 sweep)
  const bool split = st.out_size < 148 * 256 && st.sum_size >= 128;
  const bool small = span < (1ll << 30);
  // too few outputs to fill the GPU with short sums: 4 lanes per output (latency-bound steps of
  // the Tucker side operands, ~20 % occupancy one thread per output)
  static const bool noquad = std::getenv("NEF_EINSTEP_NOQUAD") != nullptr;   // diagnostics
  const bool quad = !split && small && st.out_size < 148 * 1024 && st.sum_size >= 8 && !noquad;
  const int L = split ? 32 : quad ? 4 : 1;
  long long blocks = (st.out_size * L + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  if (blocks < 1) blocks = 1;
  if (quad) einstep_kernel<int, 4><<<(unsigned)blocks, 256, 0, s>>>(d, A, B, C);   // (2 or 8 lanes: slower)
  else if (split && small) einstep_kernel<int, 32><<<(unsigned)blocks, 256, 0, s>>>(d, A, B, C);
  else if (split) einstep_kernel<long long, 32><<<(unsigned)blocks, 256, 0, s>>>(d, A, B, C);
  else if (small) einstep_kernel<int, 1><<<(unsigned)blocks, 256, 0, s>>>(d, A, B, C);
  else einstep_kernel<long long, 1><<<(unsigned)blocks, 256, 0, s>>>(d, A, B, C);
  return cudaGetLastError();
}

// --------------------------------------------------------------------------------------
// Data-only loss term c(x) of an observed entry (R25, LossOff in divergence.cuh)
__device__ __forceinline__ double dterm_c(int dterm, float x) {
  if (dterm == 1) return -4.0 * (double)sqrtf(x);                    // (1, -0.5)
  if (dterm == 2) return x > 0.f ? (double)x * (double)logf(x) - (double)x : 0.0;   // (1, 0)
  if (dterm == 3) {                                                                   // (0.5, 0)
    const double sx = (double)sqrtf(x);
    return x > 0.f ? 2.0 * sx * (double)logf(x) - 4.0 * sx : 0.0;
  }
  return 0.0;
}

// Block sum (fixed order) of (acc, cnt) into dpart[blockIdx.x] / dcpart[blockIdx.x] + slot_off
__device__ __forceinline__ void sent_block_sum(double acc, long long cnt, double* dpart, long long* dcpart, int slot) {
  __shared__ double ra[32];
  __shared__ long long rc[32];
  for (int o = 16; o > 0; o >>= 1) {
    acc += __shfl_down_sync(0xffffffffu, acc, o);
    cnt += __shfl_down_sync(0xffffffffu, cnt, o);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { ra[w] = acc; rc[w] = cnt; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    long long c = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) { a += ra[i]; c += rc[i]; }
    dpart[slot] = a;
    dcpart[slot] = c;
  }
}

// Unmasked fit: data-only loss sum (R25) over every entry, block partials (fixed grid)
__global__ void dterm_kernel(const float* __restrict__ Y, long long n4, long long n, int dterm, double* dpart,
                             long long* dcpart) {
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    const float4 y = __ldcs(reinterpret_cast<const float4*>(Y) + i);
    acc += dterm_c(dterm, y.x) + dterm_c(dterm, y.y) + dterm_c(dterm, y.z) + dterm_c(dterm, y.w);
  }
  for (long long i = n4 * 4 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    acc += dterm_c(dterm, Y[i]);
  sent_block_sum(acc, 0, dpart, dcpart, blockIdx.x);
}


// 4 entries per thread and iteration: one 4-byte mask load and one 16-byte Y load / store, all
// fully coalesced across the warp
// split (R29): M holds labels and only train entries (label 1) count as observed
__global__ void sentinel_kernel(const float* __restrict__ Y, const uint8_t* __restrict__ M, float* __restrict__ out,
                                long long n4, int dterm, double* dpart, long long* dcpart, int split, int sqy) {
  double acc = 0.0;
  long long cnt = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    const uint32_t w0 = M ? __ldcs(reinterpret_cast<const unsigned int*>(M) + i) : 0x01010101u;
    const uint32_t w = split ? __vcmpeq4(w0, 0x01010101u) : w0;
    float4 y = __ldcs(reinterpret_cast<const float4*>(Y) + i);
    if (dpart) {
      cnt += __popc(__vcmpne4(w, 0u)) >> 3;
      if (dterm) {
        if (w & 0xffu) acc += dterm_c(dterm, y.x);
        if (w & 0xff00u) acc += dterm_c(dterm, y.y);
        if (w & 0xff0000u) acc += dterm_c(dterm, y.z);
        if (w & 0xff000000u) acc += dterm_c(dterm, y.w);
      }
    }
    if (sqy) {   // R35: sqrt(y) streamed for (0.5, 0); |y| so that an observed -0 is +0
      y.x = sqrtf(fabsf(y.x)); y.y = sqrtf(fabsf(y.y)); y.z = sqrtf(fabsf(y.z)); y.w = sqrtf(fabsf(y.w));
    }
    // observed: + 0 turns -0 into +0; missing: the canonical NaN (kSentMissingBits)
    const float mis = __uint_as_float(kSentMissingBits);
    y.x = (w & 0xffu) ? y.x + 0.f : mis;
    y.y = (w & 0xff00u) ? y.y + 0.f : mis;
    y.z = (w & 0xff0000u) ? y.z + 0.f : mis;
    y.w = (w & 0xff000000u) ? y.w + 0.f : mis;
    __stcs(reinterpret_cast<float4*>(out) + i, y);
  }
  if (dpart) sent_block_sum(acc, cnt, dpart, dcpart, blockIdx.x);
}
__global__ void sentinel_tail_kernel(const float* __restrict__ Y, const uint8_t* __restrict__ M, float* __restrict__ out,
                                     long long from, long long n, int dterm, double* dpart, long long* dcpart, int slot,
                                     int split, int sqy) {
  double acc = 0.0;
  long long cnt = 0;
  for (long long i = from + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const bool o = !M || (split ? M[i] == 1 : M[i] != 0);
    if (o) { ++cnt; acc += dterm_c(dterm, Y[i]); }
    out[i] = o ? (sqy ? sqrtf(fabsf(Y[i])) : Y[i] + 0.f) : __uint_as_float(kSentMissingBits);
  }
  if (dpart) sent_block_sum(acc, cnt, dpart, dcpart, slot + blockIdx.x);
}

__global__ void set_count_kernel(long long* c, long long n) { *c = n; }

// sweep-graph loss slot: slots[*ctr] = *v, cslots[*ctr] = *c, ++*ctr (one thread)
__global__ void slot_push_kernel(const double* v, const long long* c, double* slots, long long* cslots, long long* ctr) {
  const long long i = *ctr;
  slots[i] = *v;
  cslots[i] = *c;
  *ctr = i + 1;
}
cudaError_t launch_slot_push(const double* v, const long long* c, double* slots, long long* cslots, long long* ctr,
                             cudaStream_t s) {
  slot_push_kernel<<<1, 1, 0, s>>>(v, c, slots, cslots, ctr);
  return cudaGetLastError();
}

__global__ void pad_rows_kernel(const float* __restrict__ src, float* __restrict__ dst, long long rows, int K, int Kp) {
  const long long n = rows * Kp;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / Kp;
    const int k = (int)(i - r * Kp);
    dst[i] = k < K ? src[r * K + k] : 0.f;
  }
}

__global__ void reduce_q_kernel(const float* __restrict__ part, float* __restrict__ Q, long long n_chunks,
                                long long elems) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < elems; e += (long long)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (long long c = 0; c < n_chunks; ++c) acc += (double)part[c * elems + e];
    Q[e] = (float)acc;
  }
}

// Few elements, many partials: warp w of a block sums partials w, w + 8, ... of 32 consecutive
// elements (coalesced), the 8 warp sums are combined in fixed order (deterministic).
__global__ void reduce_q8_kernel(const float* __restrict__ part, float* __restrict__ Q, long long n_chunks,
                                 long long elems) {
  __shared__ double red[8][32];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const long long e = (long long)blockIdx.x * 32 + l;
  double acc = 0.0;
  if (e < elems)
    for (long long c = w; c < n_chunks; c += 8) acc += (double)part[c * elems + e];
  red[w][l] = acc;
  __syncthreads();
  if (w == 0 && e < elems) {
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += red[k][l];
    Q[e] = (float)t;
  }
}

cudaError_t launch_reduce_q(const float* Qpart, float* Q, int64_t n_chunks, int64_t elems2, cudaStream_t s) {
  static const bool q1 = std::getenv("NEF_REDUCE_Q1") != nullptr;   // diagnostics
  if (elems2 <= 148LL * 2048 && n_chunks >= 16 && !q1) {
    reduce_q8_kernel<<<(unsigned)((elems2 + 31) / 32), 256, 0, s>>>(Qpart, Q, n_chunks, elems2);
    return cudaGetLastError();
  }
  long long blocks = (elems2 + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  reduce_q_kernel<<<(unsigned)(blocks < 1 ? 1 : blocks), 256, 0, s>>>(Qpart, Q, n_chunks, elems2);
  return cudaGetLastError();
}

__device__ __forceinline__ float mu_update(float th, double A, double B, const UpdArgs& u) {
  double mult = 1.0;
  if (B > 0.0) {
    const double r = A / B;
    if (u.g_case == 1) mult = exp(r);
    else if (u.inv_expo == 1.0) mult = r;
    else mult = pow(r, u.inv_expo);
  }
  return (float)fmax(u.eps, (double)th * mult);
}

// Fused reduce + update (epilogue-free lowerings on one rank): theta[e] <- update with
// A = sum_c part[c][0][e], B = sum_c part[c][1][e] (fixed order, fp64; the numerator and
// denominator are the factor's own layout).  Few elements with many partials: warp w of a block
// sums partials w, w + 8, ... of 32 consecutive elements (coalesced), combined in fixed order.
__global__ void reduce_update8_kernel(const float* __restrict__ part, float* __restrict__ th, long long n_chunks,
                                      long long n, UpdArgs u) {
  __shared__ double ra[8][32], rb[8][32];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const long long e = (long long)blockIdx.x * 32 + l;
  double a = 0.0, b = 0.0;
  if (e < n)
    for (long long c = w; c < n_chunks; c += 8) {
      a += (double)part[c * 2 * n + e];
      b += (double)part[c * 2 * n + n + e];
    }
  ra[w][l] = a;
  rb[w][l] = b;
  __syncthreads();
  if (w == 0 && e < n) {
    double A = 0.0, B = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) { A += ra[k][l]; B += rb[k][l]; }
    // A and B rounded to fp32 as reduce_q stores them: bit-identical to reduce_q + update
    th[e] = mu_update(th[e], (double)(float)A, (double)(float)B, u);
  }
}
__global__ void reduce_update_kernel(const float* __restrict__ part, float* __restrict__ th, long long n_chunks,
                                     long long n, UpdArgs u) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    double A = 0.0, B = 0.0;
    for (long long c = 0; c < n_chunks; ++c) {
      A += (double)part[c * 2 * n + e];
      B += (double)part[c * 2 * n + n + e];
    }
    th[e] = mu_update(th[e], (double)(float)A, (double)(float)B, u);
  }
}

cudaError_t launch_reduce_update(const float* Qpart, float* theta, int64_t n_chunks, int64_t n, UpdArgs u,
                                 cudaStream_t s) {
  if (n <= 148LL * 1024 && n_chunks >= 16) {
    reduce_update8_kernel<<<(unsigned)((n + 31) / 32), 256, 0, s>>>(Qpart, theta, n_chunks, n, u);
    return cudaGetLastError();
  }
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  reduce_update_kernel<<<(unsigned)(blocks < 1 ? 1 : blocks), 256, 0, s>>>(Qpart, theta, n_chunks, n, u);
  return cudaGetLastError();
}

__global__ void update_kernel(float* __restrict__ th, const float* __restrict__ num, const float* __restrict__ den,
                              long long n, UpdArgs u) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    double A = num[e], B = den[e];
    double mult = 1.0;
    if (B > 0.0) {
      double r = A / B;
      if (u.g_case == 1) mult = exp(r);
      else if (u.inv_expo == 1.0) mult = r;
      else mult = pow(r, u.inv_expo);
    }
    double v = (double)th[e] * mult;
    th[e] = (float)fmax(u.eps, v);
  }
}

cudaError_t launch_update(float* theta, const float* num, const float* den, int64_t n, UpdArgs u, cudaStream_t s) {
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  update_kernel<<<(unsigned)(blocks < 1 ? 1 : blocks), 256, 0, s>>>(theta, num, den, n, u);
  return cudaGetLastError();
}

__global__ void loss_reduce_kernel(const double* __restrict__ part, const long long* __restrict__ cpart, long long n,
                                   double* slot, long long* cslot, double scale, const double* off) {
  __shared__ double red[256];
  __shared__ long long redc[256];
  double acc = 0.0;
  long long c = 0;
  for (long long i = threadIdx.x; i < n; i += 256) { acc += part[i]; c += cpart[i]; }
  red[threadIdx.x] = acc;
  redc[threadIdx.x] = c;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) { red[threadIdx.x] += red[threadIdx.x + w]; redc[threadIdx.x] += redc[threadIdx.x + w]; }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    // off (R25): [data-only loss sum][observed count] of the sentinel pass
    *slot = off ? scale * red[0] + off[0] : red[0];
    *cslot = off ? reinterpret_cast<const long long*>(off)[1] : redc[0];
  }
}

cudaError_t launch_loss_reduce(const double* part, const long long* cpart, int64_t n, double* slot, long long* cslot,
                               cudaStream_t s, double scale, const double* off) {
  loss_reduce_kernel<<<1, 256, 0, s>>>(part, cpart, n, slot, cslot, scale, off);
  return cudaGetLastError();
}

cudaError_t launch_pad_rows(const float* src, float* dst, int64_t rows, int64_t K, int64_t Kp, cudaStream_t s) {
  const long long n = rows * Kp;
  const int blocks = (int)std::min<long long>((n + 255) / 256, 148 * 8);
  pad_rows_kernel<<<blocks > 0 ? blocks : 1, 256, 0, s>>>(src, dst, rows, (int)K, (int)Kp);
  return cudaGetLastError();
}

cudaError_t launch_dterm(const float* Y, int64_t n, int dterm, double* dpart, long long* dcpart, double* dslot,
                         long long* dcslot, cudaStream_t s) {
  const bool vec = (reinterpret_cast<uintptr_t>(Y) & 15) == 0;
  dterm_kernel<<<kSentBlocks, 256, 0, s>>>(Y, vec ? n / 4 : 0, n, dterm, dpart, dcpart);
  loss_reduce_kernel<<<1, 256, 0, s>>>(dpart, dcpart, kSentBlocks, dslot, dcslot, 1.0, nullptr);
  // every entry is observed: the count is n
  set_count_kernel<<<1, 1, 0, s>>>(dcslot, n);
  return cudaGetLastError();
}

cudaError_t launch_sentinel(const float* Y, const uint8_t* M, float* out, int64_t n, int dterm, double* dpart,
                            long long* dcpart, double* dslot, long long* dcslot, cudaStream_t s, int split,
                            int sqy) {
  const bool vec = (((reinterpret_cast<uintptr_t>(Y) | reinterpret_cast<uintptr_t>(out)) & 15) | (reinterpret_cast<uintptr_t>(M) & 3)) == 0;
  const long long n4 = vec ? n / 4 : 0;
  // every one of the kSentBlocks + 1 partials is written (fixed grids), then summed in fixed order
  if (vec) {
    sentinel_kernel<<<kSentBlocks, 256, 0, s>>>(Y, M, out, n4, dterm, dpart, dcpart, split, sqy);
    sentinel_tail_kernel<<<1, 256, 0, s>>>(Y, M, out, n4 * 4, n, dterm, dpart, dcpart, kSentBlocks, split, sqy);
  } else {
    sentinel_tail_kernel<<<kSentBlocks, 256, 0, s>>>(Y, M, out, 0, n, dterm, dpart, dcpart, 0, split, sqy);
    sentinel_tail_kernel<<<1, 256, 0, s>>>(Y, M, out, n, n, dterm, dpart, dcpart, kSentBlocks, split, sqy);
  }
  if (dpart) loss_reduce_kernel<<<1, 256, 0, s>>>(dpart, dcpart, kSentBlocks + 1, dslot, dcslot, 1.0, nullptr);
  return cudaGetLastError();
}

}  // namespace nef
