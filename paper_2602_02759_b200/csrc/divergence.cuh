// Device-side elementwise math of the (alpha,beta)-divergence shared by the streaming
// kernels: a(x,y) = x^alpha y^(beta-1), b(x,y) = y^(alpha+beta-1) and the loss
// L_{alpha,beta}(x,y) in the cancellation-free u = log(x/y) forms of DESIGN.md §6.
//
// The streaming kernels are templated on an EwKind so that the common (alpha,beta) pairs
// compile to a handful of instructions per entry (exponents folded into rsqrt / rcp / mul);
// the generic pair keeps runtime exponent codes and an out-of-line loss (code size: the
// per-tile loop is unrolled 32x and must stay inside the instruction cache).
#pragma once
#include <cuda_runtime.h>

#include "kernels.h"

namespace nef {

// Single-instruction MUFU forms.  Every argument reaching them is a clamped Yhat (>= 1e-30,
// a normal number) or a data value >= 0, so flush-to-zero never changes a result.
__device__ __forceinline__ float frsqrt(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float frcp(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float fsqrt(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// natural log via MUFU.LG2 (abs. error ~1e-7 in the result; arguments are positive normals or
// are discarded by the callers' selects)
__device__ __forceinline__ float flog(float x) {
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r * 0.69314718055994531f;
}

// f(u) = e^u... series helper on pairs: s(v) with f(v) = v^2 s(v) (see fser below)
__device__ __forceinline__ float2 fser_poly2(float2 v) {
  float2 s = make_float2(1.f / 840.f, 1.f / 840.f);
  s = __ffma2_rn(s, v, make_float2(1.f / 144.f, 1.f / 144.f));
  s = __ffma2_rn(s, v, make_float2(1.f / 30.f, 1.f / 30.f));
  s = __ffma2_rn(s, v, make_float2(1.f / 8.f, 1.f / 8.f));
  s = __ffma2_rn(s, v, make_float2(1.f / 3.f, 1.f / 3.f));
  s = __ffma2_rn(s, v, make_float2(0.5f, 0.5f));
  return __fmul2_rn(__fmul2_rn(v, v), s);
}

// fp32 -> TF32 bit pattern, round to nearest with ties away from zero (= cvt.rna.tf32.f32)
// as two integer ops: add half a TF32 ulp to the magnitude bits, clear the low 13 bits.
__device__ __forceinline__ uint32_t tf32_bits(float x) {
  return (__float_as_uint(x) + 0x1000u) & 0xffffe000u;
}

__device__ __forceinline__ float powc(float y, int code, float p) {
  switch (code) {
    case POW_0: return 1.f;
    case POW_1: return y;
    case POW_M1: return 1.f / y;
    case POW_H: return sqrtf(y);
    case POW_MH: return rsqrtf(y);
    case POW_M15: { float r = rsqrtf(y); return r * r * r; }
    case POW_15: return y * sqrtf(y);
    case POW_2: return y * y;
    case POW_M2: { float r = 1.f / y; return r * r; }
    default: return powf(y, p);
  }
}

// h_p(u) = (e^{pu} - 1 - pu) / p^2, stable near u = 0 (series for |pu| < 0.3)
__device__ __forceinline__ float hfun(float p, float u) {
  float v = p * u;
  if (fabsf(v) < 0.3f) {
    float s = 1.f / 5040.f;
    s = fmaf(s, v, 1.f / 720.f);
    s = fmaf(s, v, 1.f / 120.f);
    s = fmaf(s, v, 1.f / 24.f);
    s = fmaf(s, v, 1.f / 6.f);
    s = fmaf(s, v, 0.5f);
    return u * u * s;
  }
  return (expm1f(v) - v) / (p * p);
}

// f(v) = 1 - e^v + v e^v, stable near v = 0 (series for |v| < 0.3); branch-free
__device__ __forceinline__ float ffun(float v) {
  float s = 1.f / 840.f;
  s = fmaf(s, v, 1.f / 144.f);
  s = fmaf(s, v, 1.f / 30.f);
  s = fmaf(s, v, 1.f / 8.f);
  s = fmaf(s, v, 1.f / 3.f);
  s = fmaf(s, v, 0.5f);
  const float ser = v * v * s;
  const float dir = v * expf(v) - expm1f(v);
  return fabsf(v) < 0.3f ? ser : dir;
}

// L_{alpha,beta}(x, y), x = data, y = max(yhat, 1e-30); out of line (generic pairs only)
static __device__ __noinline__ float loss_entry(float x, float y, const DivParams d) {
  const float a = d.alpha, b = d.beta;
  switch (d.loss_case) {
    case 5: { float r = x - y; return 0.5f * r * r; }
    case 0: {
      float yab = powf(y, a + b);
      if (x <= 0.f) return yab / (a * (a + b));
      float u = logf(x / y);
      return yab / b * ((a + b) * hfun(a + b, u) - a * hfun(a, u));
    }
    case 1: {
      float ya = powc(y, d.c_xa, a);
      if (x <= 0.f) return ya / (a * a);
      float u = logf(x / y);
      return ya / (a * a) * ffun(a * u);
    }
    case 2: return hfun(a, logf(x / y));
    case 3: return powf(y, b) * hfun(b, logf(x / y));
    default: { float u = logf(x / y); return 0.5f * u * u; }
  }
}

// a and b at one entry, runtime exponents (unmasked values; callers select 0 when missing)
__device__ __forceinline__ void ab_entry(float x, float yh, const DivParams& d, float& av, float& bv) {
  if (d.log_case) {
    av = logf(x / yh);
    bv = 1.f;
  } else {
    av = powc(x, d.c_xa, d.p_xa) * powc(yh, d.c_ya, d.p_ya);
    bv = powc(yh, d.c_yb, d.p_yb);
  }
}

// out-of-line variant for the generic kind (keeps the unrolled tile loop small)
static __device__ __noinline__ float2 ab_entry_ool(float x, float yh, const DivParams d) {
  float av, bv;
  ab_entry(x, yh, d, av, bv);
  return make_float2(av, bv);
}

// KL-type loss y f(log(x/y)) for (1, 0): x log(x/y) - x + y, stable near x = y
// f(u) series only (|u| < 0.3), no exponentials
__device__ __forceinline__ float fser(float v) {
  float s = 1.f / 840.f;
  s = fmaf(s, v, 1.f / 144.f);
  s = fmaf(s, v, 1.f / 30.f);
  s = fmaf(s, v, 1.f / 8.f);
  s = fmaf(s, v, 1.f / 3.f);
  s = fmaf(s, v, 0.5f);
  return v * v * s;
}

// x log(x/y) - x + y = y f(u), u = log(x/y): series near u = 0, direct form elsewhere
// (|u| >= 0.3 keeps the direct form's cancellation below ~3e-6 relative); branch-free
__device__ __forceinline__ float kl_loss(float x, float y) {
  const float u = logf(fmaxf(x, 1e-38f) / y);
  const float l = fabsf(u) < 0.3f ? y * fser(u) : fmaf(x, u, y - x);
  return x > 0.f ? l : y;
}

// Compile-time specialisations of (a, b, L) for the (alpha, beta) pairs of the configs
// (paper convention; EW_* in kernels.h).  Ew<EW_GENERIC> defers to the runtime codes.
// ab2 evaluates two entries at once; the specialisations use the packed fp32x2 multiplies of
// sm_100 (FMUL2: one issue slot for two products).
// Traits: kLinX - a = x * (positive factor), so a is NaN where x is the sentinel copy's NaN ("missing");
// kSignedA - a may be negative at an observed entry (log forms: the (0,1) pair, Jensen-Shannon),
// so the sentinel path selects on x instead of clamping a at zero.
template <int KIND>
struct Ew {
  static constexpr bool kLinX = false;   // a = x * (positive factor)
  static constexpr bool kSignedA = true;  // generic pairs include the (0, 1) log case
  static __device__ __forceinline__ void ab(float x, float yh, const DivParams& d, float& av, float& bv) {
    const float2 r = ab_entry_ool(x, yh, d);
    av = r.x;
    bv = r.y;
  }
  static __device__ __forceinline__ void ab2(float2 x, float2 yh, const DivParams& d, float2& av, float2& bv) {
    ab(x.x, yh.x, d, av.x, bv.x);
    ab(x.y, yh.y, d, av.y, bv.y);
  }
  static __device__ __forceinline__ float loss(float x, float yh, const DivParams& d) { return loss_entry(x, yh, d); }
  static __device__ __forceinline__ void abl2(float2 x, float2 yh, const DivParams& d, float2& av, float2& bv,
                                              float2& l) {
    ab2(x, yh, d, av, bv);
    l = make_float2(loss(x.x, yh.x, d), loss(x.y, yh.y, d));
  }
};

template <>
struct Ew<EW_KL> {  // (1, 0): a = x / y, b = 1
  static constexpr bool kLinX = true;   // a = x * (positive factor)
  static constexpr bool kSignedA = false;
  static __device__ __forceinline__ void ab(float x, float yh, const DivParams&, float& av, float& bv) {
    av = x * frcp(yh);
    bv = 1.f;
  }
  static __device__ __forceinline__ void ab2(float2 x, float2 yh, const DivParams&, float2& av, float2& bv) {
    av = __fmul2_rn(x, make_float2(frcp(yh.x), frcp(yh.y)));
    bv = make_float2(1.f, 1.f);
  }
  static __device__ __forceinline__ float loss(float x, float yh, const DivParams&) { return kl_loss(x, yh); }
  // a, b and the loss y f(u), u = log(x/y) = log(a): one rcp and one lg2 per entry
  static __device__ __forceinline__ void abl2(float2 x, float2 yh, const DivParams&, float2& av, float2& bv,
                                              float2& l) {
    av = __fmul2_rn(x, make_float2(frcp(yh.x), frcp(yh.y)));
    bv = make_float2(1.f, 1.f);
    const float2 u = make_float2(flog(fmaxf(av.x, 1e-38f)), flog(fmaxf(av.y, 1e-38f)));
    const float2 ser = __fmul2_rn(yh, fser_poly2(u));
    const float2 dir = __ffma2_rn(x, u, make_float2(yh.x - x.x, yh.y - x.y));
    l.x = x.x > 0.f ? (fabsf(u.x) < 0.3f ? ser.x : dir.x) : yh.x;
    l.y = x.y > 0.f ? (fabsf(u.y) < 0.3f ? ser.y : dir.y) : yh.y;
  }
};

template <>
struct Ew<EW_EUC> {  // (1, 1): a = x, b = y
  static constexpr bool kLinX = true;   // a = x * (positive factor)
  static constexpr bool kSignedA = false;
  static __device__ __forceinline__ void ab(float x, float yh, const DivParams&, float& av, float& bv) {
    av = x;
    bv = yh;
  }
  static __device__ __forceinline__ void ab2(float2 x, float2 yh, const DivParams&, float2& av, float2& bv) {
    av = x;
    bv = yh;
  }
  static __device__ __forceinline__ float loss(float x, float yh, const DivParams&) {
    const float r = x - yh;
    return 0.5f * r * r;
  }
  static __device__ __forceinline__ void abl2(float2 x, float2 yh, const DivParams& d, float2& av, float2& bv,
                                              float2& l) {
    ab2(x, yh, d, av, bv);
    l = make_float2(loss(x.x, yh.x, d), loss(x.y, yh.y, d));
  }
};

template <>
struct Ew<EW_B_M05> {  // (1, -0.5): a = x y^-3/2, b = y^-1/2; L = 2 (sqrt x - sqrt y)^2 / sqrt y
  static constexpr bool kLinX = true;   // a = x * (positive factor)
  static constexpr bool kSignedA = false;
  static __device__ __forceinline__ void ab(float x, float yh, const DivParams&, float& av, float& bv) {
    const float r = frsqrt(yh);
    bv = r;
    av = x * r * r * r;
  }
  static __device__ __forceinline__ void ab2(float2 x, float2 yh, const DivParams&, float2& av, float2& bv) {
    const float2 r = make_float2(frsqrt(yh.x), frsqrt(yh.y));
    bv = r;
    av = __fmul2_rn(__fmul2_rn(x, r), __fmul2_rn(r, r));
  }
  static __device__ __forceinline__ float loss(float x, float yh, const DivParams&) {
    const float r = frsqrt(yh);
    const float d = fsqrt(x) - yh * r;
    return 2.f * d * d * r;
  }
  static __device__ __forceinline__ void abl2(float2 x, float2 yh, const DivParams&, float2& av, float2& bv,
                                              float2& l) {
    // shares rsqrt(yhat) between a, b and the loss 2 (sqrt x - sqrt y)^2 / sqrt y
    const float2 r = make_float2(frsqrt(yh.x), frsqrt(yh.y));
    bv = r;
    av = __fmul2_rn(__fmul2_rn(x, r), __fmul2_rn(r, r));
    const float2 dd = __ffma2_rn(make_float2(-yh.x, -yh.y), r, make_float2(fsqrt(x.x), fsqrt(x.y)));
    const float2 d2 = __fmul2_rn(dd, dd);
    l = __fmul2_rn(__fmul2_rn(d2, r), make_float2(2.f, 2.f));
  }
};

template <>
struct Ew<EW_A05_B0> {  // (0.5, 0): a = sqrt(x) / y, b = y^-1/2; L = 4 y^1/2 f(log(x/y)/2)
  static constexpr bool kLinX = false;   // a = x * (positive factor)
  static constexpr bool kSignedA = false;
  static __device__ __forceinline__ void ab(float x, float yh, const DivParams&, float& av, float& bv) {
    const float r = frsqrt(yh);
    bv = r;
    av = fsqrt(x) * r * r;
  }
  static __device__ __forceinline__ void ab2(float2 x, float2 yh, const DivParams&, float2& av, float2& bv) {
    const float2 r = make_float2(frsqrt(yh.x), frsqrt(yh.y));
    bv = r;
    av = __fmul2_rn(make_float2(fsqrt(x.x), fsqrt(x.y)), __fmul2_rn(r, r));
  }
  static __device__ __forceinline__ float loss(float x, float yh, const DivParams&) {
    // 4 [sqrt y - sqrt x + sqrt x v], v = log(x/y)/2 (= 4 sqrt(y) f(v)); series near v = 0
    const float sy = fsqrt(yh), sx = fsqrt(x);
    const float v = 0.5f * logf(fmaxf(x, 1e-38f) / yh);
    const float l = fabsf(v) < 0.3f ? 4.f * sy * fser(v) : 4.f * (sy - sx + sx * v);
    return x > 0.f ? l : 4.f * sy;
  }
  // shares rsqrt(y), sqrt(x) between a, b and the loss; v = log(x r^2) / 2
  static __device__ __forceinline__ void abl2(float2 x, float2 yh, const DivParams&, float2& av, float2& bv,
                                              float2& l) {
    const float2 r = make_float2(frsqrt(yh.x), frsqrt(yh.y));
    const float2 sx = make_float2(fsqrt(x.x), fsqrt(x.y));
    const float2 r2 = __fmul2_rn(r, r);
    bv = r;
    av = __fmul2_rn(sx, r2);
    const float2 q = __fmul2_rn(x, r2);   // x / y
    const float2 v = make_float2(0.5f * flog(fmaxf(q.x, 1e-38f)), 0.5f * flog(fmaxf(q.y, 1e-38f)));
    const float2 sy = __fmul2_rn(yh, r);
    const float2 ser = __fmul2_rn(__fmul2_rn(sy, make_float2(4.f, 4.f)), fser_poly2(v));
    const float2 dir = __fmul2_rn(make_float2(4.f, 4.f), __ffma2_rn(sx, v, make_float2(sy.x - sx.x, sy.y - sx.y)));
    l.x = x.x > 0.f ? (fabsf(v.x) < 0.3f ? ser.x : dir.x) : 4.f * sy.x;
    l.y = x.y > 0.f ? (fabsf(v.y) < 0.3f ? ser.y : dir.y) : 4.f * sy.y;
  }
};

template <>
struct Ew<EW_B05> {  // (1, 0.5): a = x y^-1/2, b = y^1/2
  static constexpr bool kLinX = true;   // a = x * (positive factor)
  static constexpr bool kSignedA = false;
  static __device__ __forceinline__ void ab(float x, float yh, const DivParams&, float& av, float& bv) {
    const float r = frsqrt(yh);
    av = x * r;
    bv = yh * r;
  }
  static __device__ __forceinline__ void ab2(float2 x, float2 yh, const DivParams& d, float2& av, float2& bv) {
    ab(x.x, yh.x, d, av.x, bv.x);
    ab(x.y, yh.y, d, av.y, bv.y);
  }
  static __device__ __forceinline__ float loss(float x, float yh, const DivParams& d) { return loss_entry(x, yh, d); }
  static __device__ __forceinline__ void abl2(float2 x, float2 yh, const DivParams& d, float2& av, float2& bv,
                                              float2& l) {
    ab2(x, yh, d, av, bv);
    l = make_float2(loss(x.x, yh.x, d), loss(x.y, yh.y, d));
  }
};

template <>
struct Ew<EW_B2> {  // (1, 2): a = x y, b = y^2
  static constexpr bool kLinX = true;   // a = x * (positive factor)
  static constexpr bool kSignedA = false;
  static __device__ __forceinline__ void ab(float x, float yh, const DivParams&, float& av, float& bv) {
    av = x * yh;
    bv = yh * yh;
  }
  static __device__ __forceinline__ void ab2(float2 x, float2 yh, const DivParams& d, float2& av, float2& bv) {
    ab(x.x, yh.x, d, av.x, bv.x);
    ab(x.y, yh.y, d, av.y, bv.y);
  }
  static __device__ __forceinline__ float loss(float x, float yh, const DivParams& d) { return loss_entry(x, yh, d); }
  static __device__ __forceinline__ void abl2(float2 x, float2 yh, const DivParams& d, float2& av, float2& bv,
                                              float2& l) {
    ab2(x, yh, d, av, bv);
    l = make_float2(loss(x.x, yh.x, d), loss(x.y, yh.y, d));
  }
};

template <>
struct Ew<EW_A05_B1> {  // (0.5, 1): a = sqrt(x), b = sqrt(y)
  static constexpr bool kLinX = false;   // a = x * (positive factor)
  static constexpr bool kSignedA = false;
  static __device__ __forceinline__ void ab(float x, float yh, const DivParams&, float& av, float& bv) {
    av = fsqrt(x);
    bv = fsqrt(yh);
  }
  static __device__ __forceinline__ void ab2(float2 x, float2 yh, const DivParams& d, float2& av, float2& bv) {
    ab(x.x, yh.x, d, av.x, bv.x);
    ab(x.y, yh.y, d, av.y, bv.y);
  }
  static __device__ __forceinline__ float loss(float x, float yh, const DivParams& d) { return loss_entry(x, yh, d); }
  static __device__ __forceinline__ void abl2(float2 x, float2 yh, const DivParams& d, float2& av, float2& bv,
                                              float2& l) {
    ab2(x, yh, d, av, bv);
    l = make_float2(loss(x.x, yh.x, d), loss(x.y, yh.y, d));
  }
};

// (0.5, 0) with s = sqrt(x) streamed instead of x (R35: a = x^alpha y^(beta-1) needs x only through
// x^alpha): a = s / y, b = y^-1/2, one MUFU per entry instead of two
template <>
struct Ew<EW_A05_B0_SQ> {
  static constexpr bool kLinX = true;    // a = s * (positive): carries the sentinel's sign
  static constexpr bool kSignedA = false;
  static __device__ __forceinline__ void ab(float s, float yh, const DivParams&, float& av, float& bv) {
    const float r = frsqrt(yh);
    bv = r;
    av = s * r * r;
  }
  static __device__ __forceinline__ void ab2(float2 s, float2 yh, const DivParams&, float2& av, float2& bv) {
    const float2 r = make_float2(frsqrt(yh.x), frsqrt(yh.y));
    bv = r;
    av = __fmul2_rn(s, __fmul2_rn(r, r));
  }
  static __device__ __forceinline__ float loss(float s, float yh, const DivParams& d) {
    return Ew<EW_A05_B0>::loss(s * s, yh, d);
  }
  static __device__ __forceinline__ void abl2(float2 s, float2 yh, const DivParams& d, float2& av, float2& bv,
                                              float2& l) {
    ab2(s, yh, d, av, bv);
    l = make_float2(loss(s.x, yh.x, d), loss(s.y, yh.y, d));
  }
};

// ---- App. B losses; y = max(yhat, 1e-30) is the model (odds for Bernoulli / binomial)
__device__ __forceinline__ float xlogy0(float x, float ly) { return x > 0.f ? x * ly : 0.f; }   // 0 log y = 0 (R8)

// One reciprocal for both weights: r = 1 / (y (c + y)), a = x (c + y) r, b = (c' ...) y r - one MUFU
// per entry instead of two (the two-MUFU forms made these kinds MUFU-bound: 16 k MUFU per tile)
template <>
struct Ew<EW_NB> {  // a = x / y, b = (phi + x) / (phi + y); L = (phi + x) log(phi + y) - x log y
  static constexpr bool kLinX = true;
  static constexpr bool kSignedA = false;
  static __device__ __forceinline__ void ab(float x, float yh, const DivParams& d, float& av, float& bv) {
    const float py = d.prm + yh;
    const float r = frcp(yh * py);
    av = x * py * r;
    bv = (d.prm + x) * yh * r;
  }
  static __device__ __forceinline__ void ab2(float2 x, float2 yh, const DivParams& d, float2& av, float2& bv) {
    ab(x.x, yh.x, d, av.x, bv.x);
    ab(x.y, yh.y, d, av.y, bv.y);
  }
  static __device__ __forceinline__ float loss(float x, float yh, const DivParams& d) {
    return (d.prm + x) * flog(d.prm + yh) - xlogy0(x, flog(yh));
  }
  static __device__ __forceinline__ void abl2(float2 x, float2 yh, const DivParams& d, float2& av, float2& bv,
                                              float2& l) {
    ab2(x, yh, d, av, bv);
    l = make_float2(loss(x.x, yh.x, d), loss(x.y, yh.y, d));
  }
  // per-entry phi (aux): the same forms with phi_i in place of the scalar
  static __device__ __forceinline__ void ab_aux(float x, float yh, float phi, float& av, float& bv) {
    const float py = phi + yh;
    const float r = frcp(yh * py);
    av = x * py * r;
    bv = (phi + x) * yh * r;
  }
  static __device__ __forceinline__ float loss_aux(float x, float yh, float phi) {
    return (phi + x) * flog(phi + yh) - xlogy0(x, flog(yh));
  }
};

template <>
struct Ew<EW_BERN> {  // odds: a = x / y, b = 1 / (1 + y); L = log(1 + y) - x log y
  static constexpr bool kLinX = true;
  static constexpr bool kSignedA = false;
  static __device__ __forceinline__ void ab(float x, float yh, const DivParams&, float& av, float& bv) {
    const float py = 1.f + yh;
    const float r = frcp(yh * py);
    av = x * py * r;
    bv = yh * r;
  }
  static __device__ __forceinline__ void ab2(float2 x, float2 yh, const DivParams& d, float2& av, float2& bv) {
    ab(x.x, yh.x, d, av.x, bv.x);
    ab(x.y, yh.y, d, av.y, bv.y);
  }
  static __device__ __forceinline__ float loss(float x, float yh, const DivParams&) {
    return log1pf(yh) - xlogy0(x, flog(yh));
  }
  static __device__ __forceinline__ void abl2(float2 x, float2 yh, const DivParams& d, float2& av, float2& bv,
                                              float2& l) {
    ab2(x, yh, d, av, bv);
    l = make_float2(loss(x.x, yh.x, d), loss(x.y, yh.y, d));
  }
};

template <>
struct Ew<EW_BINOM> {  // odds with n trials: a = x / y, b = n / (1 + y); L = n log(1 + y) - x log y
  static constexpr bool kLinX = true;
  static constexpr bool kSignedA = false;
  static __device__ __forceinline__ void ab(float x, float yh, const DivParams& d, float& av, float& bv) {
    const float py = 1.f + yh;
    const float r = frcp(yh * py);
    av = x * py * r;
    bv = d.prm * yh * r;
  }
  static __device__ __forceinline__ void ab2(float2 x, float2 yh, const DivParams& d, float2& av, float2& bv) {
    ab(x.x, yh.x, d, av.x, bv.x);
    ab(x.y, yh.y, d, av.y, bv.y);
  }
  static __device__ __forceinline__ float loss(float x, float yh, const DivParams& d) {
    return d.prm * log1pf(yh) - xlogy0(x, flog(yh));
  }
  static __device__ __forceinline__ void abl2(float2 x, float2 yh, const DivParams& d, float2& av, float2& bv,
                                              float2& l) {
    ab2(x, yh, d, av, bv);
    l = make_float2(loss(x.x, yh.x, d), loss(x.y, yh.y, d));
  }
  static __device__ __forceinline__ void ab_aux(float x, float yh, float n, float& av, float& bv) {
    const float py = 1.f + yh;
    const float r = frcp(yh * py);
    av = x * py * r;
    bv = n * yh * r;
  }
  static __device__ __forceinline__ float loss_aux(float x, float yh, float n) {
    return n * log1pf(yh) - xlogy0(x, flog(yh));
  }
};

// Jensen-Shannon: a = log((x + y) / (2y)), b = 1, g = log.  With u = (x - y) / (x + y) the
// loss is m / 2 [(1 + u) log(1 + u) + (1 - u) log(1 - u)], m = (x + y) / 2: the series
// sum_k u^2k / (k (2k - 1)) for |u| < 0.3 (no cancellation near x = y), the direct form elsewhere,
// m log 2 at x = 0.
__device__ __forceinline__ float js_loss(float x, float y) {
  const float m = 0.5f * (x + y);
  const float u = (x - y) / (x + y);
  const float u2 = u * u;
  float s = 1.f / 45.f;                        // k = 5
  s = fmaf(s, u2, 1.f / 28.f);                 // k = 4
  s = fmaf(s, u2, 1.f / 15.f);                 // k = 3
  s = fmaf(s, u2, 1.f / 6.f);                  // k = 2
  s = fmaf(s, u2, 1.f);                        // k = 1
  const float ser = u2 * s;
  const float dir = (1.f + u) * log1pf(u) + (1.f - u) * log1pf(-u);
  const float f = fabsf(u) < 0.3f ? ser : dir;
  return x > 0.f ? 0.5f * m * f : m * 0.69314718055994531f;
}
template <>
struct Ew<EW_JS> {
  static constexpr bool kLinX = false;
  static constexpr bool kSignedA = true;   // a < 0 where x < y
  static __device__ __forceinline__ void ab(float x, float yh, const DivParams&, float& av, float& bv) {
    av = flog(fmaf(x, frcp(yh), 1.f) * 0.5f);   // log((x / y + 1) / 2)
    bv = 1.f;
  }
  static __device__ __forceinline__ void ab2(float2 x, float2 yh, const DivParams& d, float2& av, float2& bv) {
    ab(x.x, yh.x, d, av.x, bv.x);
    ab(x.y, yh.y, d, av.y, bv.y);
  }
  static __device__ __forceinline__ float loss(float x, float yh, const DivParams&) { return js_loss(x, yh); }
  static __device__ __forceinline__ void abl2(float2 x, float2 yh, const DivParams& d, float2& av, float2& bv,
                                              float2& l) {
    ab2(x, yh, d, av, bv);
    l = make_float2(js_loss(x.x, yh.x), js_loss(x.y, yh.y));
  }
};

// Loss with its data-only part split off (R25).  For the pairs below the per-entry divergence
// is  L(x, y) = scale * rem(x, y) + c(x),  with c depending on the data alone:
//   (1, -0.5): 2 (sqrt x - sqrt y)^2 / sqrt y = 2 (x + y) / sqrt y - 4 sqrt x
//   (1, 0)   : x log(x / y) - x + y           = (y - x log y) + (x log x - x)
//   (0.5, 0) : 2 sqrt x log(x / y) - 4 sqrt x + 4 sqrt y = 4 (sqrt y - sqrt x log(y) / 2) + (2 sqrt x log x - 4 sqrt x)
// C = sum_observed c(x) is constant over a fit and is summed once by the sentinel pass
// (launch_sentinel, dterm_c below); the streaming passes then accumulate rem only.  abr2
// takes the SIGNED sentinel value (a carries its sign; rem of a missing entry is discarded by
// the caller's select).
template <int KIND>
struct LossOff {
  static constexpr bool value = false;
  static __device__ __forceinline__ void abr2(float2, float2, float2&, float2&, float2&) {}
};
template <>
struct LossOff<EW_B_M05> {
  static constexpr bool value = true;
  static __device__ __forceinline__ void abr2(float2 x, float2 yh, float2& av, float2& bv, float2& rem) {
    const float2 r = make_float2(frsqrt(yh.x), frsqrt(yh.y));
    bv = r;
    const float2 xr = __fmul2_rn(x, r);
    av = __fmul2_rn(xr, __fmul2_rn(r, r));
    rem = __ffma2_rn(yh, r, xr);   // (x + y) / sqrt y; scale 2
  }
};
template <>
struct LossOff<EW_KL> {
  static constexpr bool value = true;
  static __device__ __forceinline__ void abr2(float2 x, float2 yh, float2& av, float2& bv, float2& rem) {
    av = __fmul2_rn(x, make_float2(frcp(yh.x), frcp(yh.y)));
    bv = make_float2(1.f, 1.f);
    rem = __ffma2_rn(make_float2(-x.x, -x.y), make_float2(flog(yh.x), flog(yh.y)), yh);   // y - x log y; scale 1
  }
};
// (0.5, 0): 4 [sqrt x (log(x/y) / 2) - sqrt x + sqrt y] = 4 (sqrt y - sqrt x log(y) / 2) + (2 sqrt x log x - 4 sqrt x)
template <>
struct LossOff<EW_A05_B0> {
  static constexpr bool value = true;
  static __device__ __forceinline__ void abr2(float2 x, float2 yh, float2& av, float2& bv, float2& rem) {
    const float2 r = make_float2(frsqrt(yh.x), frsqrt(yh.y));
    const float2 sx = make_float2(fsqrt(fabsf(x.x)), fsqrt(fabsf(x.y)));
    bv = r;
    av = __fmul2_rn(sx, __fmul2_rn(r, r));   // sqrt(x) / y (NaN at a missing entry: x is the sentinel NaN)
    const float2 sy = __fmul2_rn(yh, r);
    rem = __ffma2_rn(__fmul2_rn(sx, make_float2(-0.5f, -0.5f)), make_float2(flog(yh.x), flog(yh.y)), sy);   // scale 4
  }
};

template <>
struct LossOff<EW_A05_B0_SQ> {   // the (0.5, 0) split with s = sqrt(x) streamed
  static constexpr bool value = true;
  static __device__ __forceinline__ void abr2(float2 s, float2 yh, float2& av, float2& bv, float2& rem) {
    const float2 r = make_float2(frsqrt(yh.x), frsqrt(yh.y));
    bv = r;
    av = __fmul2_rn(s, __fmul2_rn(r, r));   // NaN at missing entries (the sentinel copy's NaN)
    const float2 sy = __fmul2_rn(yh, r);
    const float2 sa = make_float2(fabsf(s.x), fabsf(s.y));
    rem = __ffma2_rn(__fmul2_rn(sa, make_float2(-0.5f, -0.5f)), make_float2(flog(yh.x), flog(yh.y)), sy);   // scale 4
  }
};

// dispatch helper: calls f.template operator()<KIND>() for the pair's kind
template <typename F>
inline cudaError_t dispatch_ew(int kind, F&& f) {
  switch (kind) {
    case EW_KL: return f.template operator()<EW_KL>();
    case EW_EUC: return f.template operator()<EW_EUC>();
    case EW_B_M05: return f.template operator()<EW_B_M05>();
    case EW_A05_B0: return f.template operator()<EW_A05_B0>();
    case EW_B05: return f.template operator()<EW_B05>();
    case EW_B2: return f.template operator()<EW_B2>();
    case EW_A05_B1: return f.template operator()<EW_A05_B1>();
    case EW_NB: return f.template operator()<EW_NB>();
    case EW_BERN: return f.template operator()<EW_BERN>();
    case EW_BINOM: return f.template operator()<EW_BINOM>();
    case EW_JS: return f.template operator()<EW_JS>();
    case EW_A05_B0_SQ: return f.template operator()<EW_A05_B0_SQ>();
    default: return f.template operator()<EW_GENERIC>();
  }
}

}  // namespace nef
