// Device-side elementwise math of the (alpha,beta)-divergence shared by the streaming
// kernels: a(x,y) = x^alpha y^(beta-1), b(x,y) = y^(alpha+beta-1) and the loss
// L_{alpha,beta}(x,y) in the cancellation-free u = log(x/y) forms of DESIGN.md §6.
#pragma once
#include <cuda_runtime.h>

#include "kernels.h"

namespace nef {

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

// f(v) = 1 - e^v + v e^v, stable near v = 0
__device__ __forceinline__ float ffun(float v) {
  if (fabsf(v) < 0.3f) {
    float s = 1.f / 840.f;
    s = fmaf(s, v, 1.f / 144.f);
    s = fmaf(s, v, 1.f / 30.f);
    s = fmaf(s, v, 1.f / 8.f);
    s = fmaf(s, v, 1.f / 3.f);
    s = fmaf(s, v, 0.5f);
    return v * v * s;
  }
  return v * expf(v) - expm1f(v);
}

// L_{alpha,beta}(x, y), x = data, y = max(yhat, 1e-30)
__device__ __forceinline__ float loss_entry(float x, float y, const DivParams& d) {
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

// a and b at one entry (unmasked values; the caller selects 0 at missing entries)
__device__ __forceinline__ void ab_entry(float x, float yh, const DivParams& d, float& av, float& bv) {
  if (d.log_case) {
    av = logf(x / yh);
    bv = 1.f;
  } else {
    av = powc(x, d.c_xa, d.p_xa) * powc(yh, d.c_ya, d.p_ya);
    bv = powc(yh, d.c_yb, d.p_yb);
  }
}

}  // namespace nef
