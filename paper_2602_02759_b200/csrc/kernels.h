// Launch interface of the CUDA kernels (kernels_ffma.cu, kernels_tc.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "nef_internal.h"

namespace nef {

// exponent codes for y^p evaluated in registers ("exponent specialisation")
enum PowCode : int { POW_0 = 0, POW_1, POW_M1, POW_H, POW_MH, POW_M15, POW_15, POW_2, POW_M2, POW_GEN };

int pow_code(double p);

// compile-time specialisations of the elementwise stage (divergence.cuh)
// Missing entries of the sentinel copy of Y (R5): the canonical NaN 0x7fffffff.  Every
// fp32 result that takes it as an input is the same canonical NaN, whose bits + a TF32 rounding
// offset overflow to a negative int32, so the kernels' add-then-max (max(bits + d, 0)) rounds an
// observed weight and zeroes a missing one without a separate select, and x >= 0 is false.
constexpr unsigned kSentMissingBits = 0x7fffffffu;
enum EwKind : int { EW_GENERIC = 0, EW_KL, EW_EUC, EW_B_M05, EW_A05_B0, EW_B05, EW_B2, EW_A05_B1,
                    // App. B losses: negative binomial (scalar phi, or per-entry phi streamed
                    // as aux), Bernoulli odds, binomial odds (scalar n, or per-entry n as aux), Jensen-Shannon
                    EW_NB, EW_BERN, EW_BINOM, EW_JS,
                    // (0.5, 0) streaming sqrt(Y) (nef_fit's once-per-fit copy, R35): Y^alpha precomputed
                    EW_A05_B0_SQ };
int ew_kind(double alpha, double beta);

// loss families (include/nef.h nef_loss_kind)
enum LossFam : int { FAM_AB = 0, FAM_NEGBIN = 1, FAM_BERNOULLI = 2, FAM_BINOMIAL = 3, FAM_JS = 4 };

// Elementwise constants of the (alpha,beta)-divergence
struct DivParams {
  float alpha, beta;
  float p_xa, p_ya, p_yb;       // x^alpha, yhat^(beta-1), yhat^(alpha+beta-1)
  int c_xa, c_ya, c_yb;         // PowCode of the three exponents
  int log_case;                 // (alpha, beta) = (0, 1): a = log(x/yhat), b = 1
  int loss_case;                // 0 generic, 1 beta=0, 2 alpha=-beta, 3 alpha=0, 4 alpha=beta=0, 5 (1,1)
  int kind;                     // EwKind
  float prm;                    // NB dispersion phi / binomial trials n (scalar; per-entry values via aux)
};
DivParams make_div(double alpha, double beta);
DivParams make_div_fam(int fam, double alpha, double beta, double prm);

// Fused streaming pass over Y (and mask) for one lowering.
struct FusedArgs {
  const float* Y;
  const uint8_t* M;            // may be null
  int64_t n_rows, n_cols;
  int K;
  int nr, nc;                   // number of row / col modes
  int64_t rdim[kMaxModes], rys[kMaxModes];
  int64_t cdim[kMaxModes], cys[kMaxModes];
  const float* U;               // [n_rows][K]
  int ntab;
  const float* tab[kMaxTabs];
  int64_t tcs[kMaxTabs][kMaxModes];   // table stride per col mode
  const int32_t* boff;          // [ntab][K]
  int row_fast;
  int64_t n_chunks, tiles_per_chunk;
  float* Qpart;                 // [n_chunks][2][n_rows][K]
  double* losspart;             // [row_blocks * n_chunks] loss sums
  long long* countpart;         // [row_blocks * n_chunks] observed counts
  DivParams dv;
  int mode;                     // 0: update only, 1: update + loss, 2: loss only
  const float* aux;             // per-entry phi (NB) / n (binomial), Y's layout, or null (scalar dv.prm)
  int split;                    // M holds labels 0..3 (R29): train = 1; the loss partials are per role
                                //   (losspart / countpart: [3][row_blocks * n_chunks])
};

cudaError_t launch_fused_ffma(const FusedArgs& a, cudaStream_t s);

// Small einsum step (C = sum A*B, optional B), fp64 accumulation.  GEMM-shaped steps run as a
// tiled product; those with few output tiles and long sums split the sum over blocks and need
// `scratch` (einstep_scratch_floats(st) floats; without it they take the per-output kernels).
cudaError_t launch_einstep(const EinStep& st, const float* A, const float* B, float* C, cudaStream_t s,
                           float* scratch = nullptr);
int64_t einstep_scratch_floats(const EinStep& st);

// out[i] = M[i] ? Y[i] + 0 : -1  (the sentinel copy of Y; M nonzero = observed; observed data >= 0).
// With dpart (kSentBlocks + 1 partials each of dpart / dcpart): also *dslot = sum over observed
// entries of the data-only loss term c(x) (dterm 1: (1,-0.5), 2: (1,0), 3: (0.5,0), 0: none; R25) and
// *dcslot = the observed count, summed in fixed order.
constexpr int kSentBlocks = 148 * 16;
// Unmasked fit (R25): *dslot = sum over all n entries of c(x), *dcslot = n (kSentBlocks partials)
cudaError_t launch_dterm(const float* Y, int64_t n, int dterm, double* dpart, long long* dcpart, double* dslot,
                         long long* dcslot, cudaStream_t s);
cudaError_t launch_sentinel(const float* Y, const uint8_t* M, float* out, int64_t n, int dterm, double* dpart,
                            long long* dcpart, double* dslot, long long* dcslot, cudaStream_t s, int split = 0,
                            int sqrt_y = 0);
// sqrt_y (R35): the copy holds sqrt(y) at observed entries (-1 at missing ones); M may be null (all
// observed).  The data-only loss sum and the observed count still come from y itself.

// dst[r][0..Kp) = src[r][0..K) padded with zeros (16-byte row pitch for TMA)
cudaError_t launch_pad_rows(const float* src, float* dst, int64_t rows, int64_t K, int64_t Kp, cudaStream_t s);

// Q[2][n_rows][K] = sum over chunks of Qpart (fixed order)
cudaError_t launch_reduce_q(const float* Qpart, float* Q, int64_t n_chunks, int64_t elems2, cudaStream_t s);

// theta <- max(eps, theta * g^{-1}(num/den)) (eq:explicit-update; g table)
struct UpdArgs {
  int g_case;       // 0: power 1/expo ; 1: exp (log case)
  double inv_expo;  // 1/expo of the power case
  double eps;
};
UpdArgs make_upd(double alpha, double beta, double eps);
UpdArgs make_upd_fam(int fam, double alpha, double beta, double eps);
cudaError_t launch_update(float* theta, const float* num, const float* den, int64_t n, UpdArgs u, cudaStream_t s);
// the same with the numerator / denominator summed from the split partials Qpart [chunks][2][n]
// (lowerings whose epilogue is the identity, one rank): reduce_q + update in one launch
cudaError_t launch_reduce_update(const float* Qpart, float* theta, int64_t n_chunks, int64_t n, UpdArgs u,
                                 cudaStream_t s);

// Sum CTA loss partials (fixed order) into slot[0] (double) and count into cslot[0].  With off
// (R25): slot[0] = scale * sum + off[0] and cslot[0] = ((long long*)off)[1].
cudaError_t launch_loss_reduce(const double* part, const long long* cpart, int64_t n, double* slot,
                               long long* cslot, cudaStream_t s, double scale = 1.0, const double* off = nullptr);

// Captured sweeps (nef_fit's CUDA graph): slots[*ctr] = *v, cslots[*ctr] = *c, ++*ctr
cudaError_t launch_slot_push(const double* v, const long long* c, double* slots, long long* cslots, long long* ctr,
                             cudaStream_t s);
}  // namespace nef
