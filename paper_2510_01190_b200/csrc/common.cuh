// Shared device helpers for the divergence-uncertainty kernels (sm_100a).
//
// Numerics contract: every product/sum on the analytic
// path is rounded separately, in the reference's order, so the fp64 kernels
// are bit-identical to the reference (stencils.py:64-66, 79-84;
// gaussian.py:41-44).  The helpers below use the _rn intrinsics, which nvcc
// never contracts into FMA, so the translation units need no -fmad=false and
// the Monte Carlo sampler (mc.cu) keeps FMA for Box-Muller.
#pragma once

#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace divuq {

// ---- error word bits (device validation; zero extra HBM bytes) ----------
// Mirrors the reference's construction-time checks: non-finite values
// (grid.py:26-27) and negative sigma (divergence.py:34-35, gaussian.py:28-29).
enum : int { kErrNonFinite = 1, kErrNegativeSigma = 2 };

template <typename T> struct Arith;

template <> struct Arith<double> {
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
  static __device__ __forceinline__ double sqrt_(double a) { return __dsqrt_rn(a); }
};

template <> struct Arith<float> {
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
  static __device__ __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
  static __device__ __forceinline__ float sqrt_(float a) { return __fsqrt_rn(a); }
};

// ---- normal CDF with scipy/cephes ndtr's structure ----------------------
// The reference evaluates both tails with scipy.special.ndtr (lcp.py:66-67).
// Like ndtr we scale the argument by sqrt(1/2) with one multiply and never
// form 1-p for the small tail: small = erfc(|x|)/2 <= 1/2, large = 1 - small.
// (ndtr switches to 0.5 + 0.5*erf(x) for |x| < sqrt(1/2), where both tails are
// ~1/2 and the two forms agree to an ulp; dropping that branch keeps warps
// convergent.)  Within ~1e-13 relative of scipy even at x ~ -37.
// erfc(|x|).  fp32: erfc(a) = exp(-a^2) * h(q) / (a + 2) with q = (a - 2)/(a + 2) and h a
// degree-9 polynomial fitted offline against scipy's erfcx
// (tools/fit_erfc.py; max relative error 3.1e-7 ~ 5 ulp in fp32 evaluation,
// the same class as libdevice erfcf at about half the instructions: one
// reciprocal, one exp, 9 FMA).  exp(-a^2) is corrected for the rounding of
// a*a with one FMA so the deep tail keeps its relative accuracy.
//
// fp64 (round 2): libdevice erfc branches by range (a warp straddling the
// ranges runs several paths) and materialises its rational coefficients with
// UMOV pairs: the fp64 K2 was issue-bound at ~450 instructions per point
// (ncu: 15 % UMOV, 12 % of stalls on branches).  Now branch-free like the LCP
// kernels, but to RELATIVE accuracy over the whole normal range:
// erfc(a) = exp(-a^2) * h(q) / (a + K), q = (a - K) / (a + K), K = 3.75, h a
// degree-18 polynomial fitted against erfcx on [0, 26.6]
// (tools/fit_erfc.py: fit64(3.75, 18, amax=26.6); 5.7e-15 max relative with
// the a*a rounding corrected and exp accurate, checked against mpmath), the
// reciprocal refined twice (2^-92), exp(-a^2) by exp_neg_rel.  erfc(a) for
// a > 26.6 underflows below 2^-1022 (P < 1e-300: returned as 0); erfc(0) = 1.
__constant__ double kErfcRel[19] = {
    0x1.17884282534aap+0, -0x1.eae02d0a14626p-1, 0x1.78fecb4e7fc5cp-1, -0x1.f63dd8118e691p-2,
    0x1.1dc271193b4a5p-2, -0x1.0e3ea225f266ep-3, 0x1.92618b2aa95e2p-5, -0x1.9ac694d9730adp-7,
    0x1.0290567e9387bp-10, 0x1.a0b74c910b513p-11, -0x1.6d9aecf8f4edbp-12, 0x1.63539a4679492p-17,
    0x1.3ad4a1b185870p-15, -0x1.29def7758bfbcp-17, -0x1.c6492fe76ae91p-19, 0x1.ab2c7340f5fc5p-20,
    0x1.8466796e3554ap-22, -0x1.9136493b7ad22p-23, -0x1.cabef9fb414ddp-25};
// e^r Taylor coefficients 1/k!, k = 0..13 (|r| <= ln2/2: truncation < 2e-16)
__constant__ double kExpRel[14] = {
    0x1.0000000000000p+0, 0x1.0000000000000p+0, 0x1.0000000000000p-1, 0x1.5555555555555p-3,
    0x1.5555555555555p-5, 0x1.1111111111111p-7, 0x1.6c16c16c16c17p-10, 0x1.a01a01a01a01ap-13,
    0x1.a01a01a01a01ap-16, 0x1.71de3a556c734p-19, 0x1.27e4fb7789f5cp-22, 0x1.ae64567f544e4p-26,
    0x1.1eed8eff8d898p-29, 0x1.6124613a86d09p-33};

// exp(t) for t in [-708, 0]: k = rint(t log2 e), r = t - k ln2 (fdlibm's hi/lo
// split), e^r by Taylor to r^13, times 2^k built in the exponent bits (k >= -1022)
__device__ __forceinline__ double exp_neg_rel(double t) {
  const double y = fma(t, 0x1.71547652b82fep+0, 0x1.8p52);   // 1.5*2^52 + rint(t*log2(e))
  const double kd = y - 0x1.8p52;
  const int ki = __double2loint(y);
  double r = fma(kd, -6.93147180369123816490e-01, t);
  r = fma(kd, -1.90821492927058770002e-10, r);
  double p = kExpRel[13];
#pragma unroll
  for (int k = 12; k >= 0; --k) p = fma(p, r, kExpRel[k]);
  return p * __hiloint2double((ki + 1023) << 20, 0);
}

__device__ __forceinline__ double erfc_abs(double x) {
  constexpr double K = 3.75;
  const double a = fabs(x);
  const double d = a + K;
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  r = fma(r, fma(-d, r, 1.0), r);
  r = fma(r, fma(-d, r, 1.0), r);
  const double q = (a - K) * r;
  double p = kErfcRel[18];
#pragma unroll
  for (int k = 17; k >= 0; --k) p = fma(p, q, kErfcRel[k]);
  const double s = a * a;
  const double lo = fma(a, a, -s);   // a*a - s exactly
  double y = p * r * exp_neg_rel(fmax(-s, -708.0));
  y = fma(y, -lo, y);                // * exp(-lo) ~ (1 - lo)
  return a > 26.6 ? 0.0 : (a == 0.0 ? 1.0 : y);
}

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ float rsqrt_approx(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ float erfc_abs(float x) {
  const float a = fabsf(x);
  const float r = rcp_approx(a + 2.0f);  // a + 2 in [2, inf]: no special cases
  const float q = __fmul_rn(a - 2.0f, r);
  float p = -4.708851338e-05f;
  p = fmaf(p, q, -5.272014532e-04f);
  p = fmaf(p, q, -7.228796021e-04f);
  p = fmaf(p, q, 3.042218974e-03f);
  p = fmaf(p, q, 6.432665512e-03f);
  p = fmaf(p, q, -2.150291763e-02f);
  p = fmaf(p, q, -3.643533960e-02f);
  p = fmaf(p, q, 2.794715464e-01f);
  p = fmaf(p, q, -6.871609688e-01f);
  p = fmaf(p, q, 1.021582723e+00f);
  const float s = __fmul_rn(a, a);
  const float lo = fmaf(a, a, -s);  // a*a - s exactly
  float y = __fmul_rn(__fmul_rn(p, r), expf(-s));
  y = fmaf(y, -lo, y);              // * exp(-lo) ~ (1 - lo)
  // fp32 erfc underflows past 10.05 (and a = inf); erfc(0) = 1 exactly (both
  // tails 1/2 at a zero argument, as ndtr(0))
  return a > 10.0546875f ? 0.0f : (a == 0.0f ? 1.0f : y);
}

__device__ __forceinline__ double ndtr_(double a) {
  const double x = __dmul_rn(a, 0.70710678118654752440);
  const double y = __dmul_rn(0.5, erfc_abs(x));
  return x > 0.0 ? __dsub_rn(1.0, y) : y;
}

__device__ __forceinline__ float ndtr_(float a) {
  const float x = __fmul_rn(a, 0.70710678118654752440f);
  const float y = __fmul_rn(0.5f, erfc_abs(x));
  return x > 0.0f ? __fsub_rn(1.0f, y) : y;
}

// ---- fp32 ensemble moments: one pass, shifted by the first member ----------
// d_m = x_m - x_0; s = sum d, q = sum d^2 (FMA);  lo = s/M;  mu = x_0 + lo;
// var = (q - s*lo) / (M-1) clamped at 0 (ddof = 1, gaussian.py:41-44).
// Shifting by a member keeps the cancellation benign (|mu - x_0| ~ sigma), and
// a single pass lets the streaming kernels consume each member once without
// holding M values per point.  Every fp32 moment in the library goes through
// this one routine, so the fused, unfused and sharded paths agree bitwise.
//
// The fused kernels also keep the mean's rounding residual r = (x_0 - mu) +
// lo (|r| <= ulp(mu)/2, rounded to bf16 so it packs into 16 bits where shared
// memory is tight) and difference (mu, r) PAIRS in the stencil: rounding mu
// to fp32 before differencing loses ~ulp(mu) per neighbour, which at
// |mu| / sigma ~ 5e3 (config 1: |u| ~ 110, sigma down to 0.02) moves the
// tail argument by ~3e-4 and P(div > 0) by ~1e-4; with the pair the fp32
// fused maps meet |dP| <= 1e-5 P + 1e-6 against the fp64 oracle
// (tests/test_gpu_fullsize.py).
__device__ __forceinline__ float bf16_round(float x) {
  return __bfloat162float(__float2bfloat16_rn(x));
}
__device__ __forceinline__ uint32_t pack_bf16x2(float lo_half, float hi_half) {
  // both already bf16-exact: the conversion is exact
  const __nv_bfloat162 h = __floats2bfloat162_rn(lo_half, hi_half);
  return *reinterpret_cast<const uint32_t*>(&h);
}
__device__ __forceinline__ float unpack_bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float unpack_bf16_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

template <int VEC>
struct ShiftedMoments {
  float x0[VEC], s[VEC], q[VEC];
  __device__ __forceinline__ void add(int m, const float* x) {
    if (m == 0) {
#pragma unroll
      for (int e = 0; e < VEC; ++e) { x0[e] = x[e]; s[e] = 0.0f; q[e] = 0.0f; }
    } else {
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        const float d = x[e] - x0[e];
        s[e] += d;
        q[e] = fmaf(d, d, q[e]);
      }
    }
  }
  // branch-free forms for callers that peel member 0
  __device__ __forceinline__ void first(const float* x) {
#pragma unroll
    for (int e = 0; e < VEC; ++e) { x0[e] = x[e]; s[e] = 0.0f; q[e] = 0.0f; }
  }
  __device__ __forceinline__ void next(const float* x) {
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      const float d = x[e] - x0[e];
      s[e] += d;
      q[e] = fmaf(d, d, q[e]);
    }
  }
  // mu (rounded), its residual r (bf16-exact) and sigma
  __device__ __forceinline__ void finish(int M, float* mu, float* r, float* sg) const {
    const float inv_m = __fdiv_rn(1.0f, float(M));
    const float inv_m1 = __fdiv_rn(1.0f, float(M - 1));
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      const float lo = __fmul_rn(s[e], inv_m);
      mu[e] = __fadd_rn(x0[e], lo);
      if (r != nullptr) r[e] = bf16_round(__fadd_rn(__fsub_rn(x0[e], mu[e]), lo));
      const float var = __fmul_rn(fmaxf(0.0f, fmaf(-s[e], lo, q[e])), inv_m1);
      sg[e] = __fsqrt_rn(var);
    }
  }
  __device__ __forceinline__ void finish(int M, float* mu, float* sg) const {
    finish(M, mu, nullptr, sg);
  }
};

// ---- the stencil: mean and variance of one point ---------------------------
// fp64: the reference's evaluation order bit for bit (stencils.py:64-66,
// 79-84): ((u_hi*c - u_lo*c) + v_hi*c) - v_lo*c [+ w terms], every product
// rounded, variance (s*c)^2 summed hi, lo per axis.
// fp32 (no bitwise bar, 1e-5): the same terms factored per axis --
// c*(hi - lo) and c^2*(s_hi^2 + s_lo^2) with FMAs -- half the instructions and
// no less accurate (one rounding fewer per axis).
template <typename T, bool HAS_W> struct StencilMath;

template <bool HAS_W> struct StencilMath<double, HAS_W> {
  using A = Arith<double>;
  static __device__ __forceinline__ double mean(double uh, double ul, double vh, double vl,
                                                double wh, double wl, double cx, double cy,
                                                double cz) {
    double m = A::sub(A::add(A::sub(A::mul(uh, cx), A::mul(ul, cx)), A::mul(vh, cy)), A::mul(vl, cy));
    if (HAS_W) m = A::sub(A::add(m, A::mul(wh, cz)), A::mul(wl, cz));
    return m;
  }
  static __device__ __forceinline__ double var(double sh, double sl, double svh, double svl,
                                               double swh, double swl, double cx, double cy,
                                               double cz) {
    const double a = A::mul(sh, cx), b = A::mul(sl, cx), c = A::mul(svh, cy), d = A::mul(svl, cy);
    double v = A::add(A::add(A::add(A::mul(a, a), A::mul(b, b)), A::mul(c, c)), A::mul(d, d));
    if (HAS_W) {
      const double f = A::mul(swh, cz), g = A::mul(swl, cz);
      v = A::add(A::add(v, A::mul(f, f)), A::mul(g, g));
    }
    return v;
  }
};

template <bool HAS_W> struct StencilMath<float, HAS_W> {
  static __device__ __forceinline__ float mean(float uh, float ul, float vh, float vl, float wh,
                                               float wl, float cx, float cy, float cz) {
    const float z = HAS_W ? cz * (wh - wl) : 0.0f;
    return fmaf(cx, uh - ul, fmaf(cy, vh - vl, z));
  }
  // (mu, r) pairs (ShiftedMoments): each difference is (hi_h - hi_l) + (r_h - r_l)
  static __device__ __forceinline__ float dpair(float h, float l, float rh, float rl) {
    return __fadd_rn(__fsub_rn(h, l), __fsub_rn(rh, rl));
  }
  static __device__ __forceinline__ float mean_r(float uh, float ul, float ruh, float rul, float vh,
                                                 float vl, float rvh, float rvl, float wh, float wl,
                                                 float rwh, float rwl, float cx, float cy, float cz) {
    const float z = HAS_W ? __fmul_rn(cz, dpair(wh, wl, rwh, rwl)) : 0.0f;
    return fmaf(cx, dpair(uh, ul, ruh, rul), fmaf(cy, dpair(vh, vl, rvh, rvl), z));
  }
  static __device__ __forceinline__ float var(float sh, float sl, float svh, float svl, float swh,
                                              float swl, float cx, float cy, float cz) {
    const float z = HAS_W ? (cz * cz) * fmaf(swh, swh, swl * swl) : 0.0f;
    return fmaf(cx * cx, fmaf(sh, sh, sl * sl), fmaf(cy * cy, fmaf(svh, svh, svl * svl), z));
  }
};

// ---- sigma = sqrt(var) and the tails P(div > t), P(div < -t) -------------
// fp64: IEEE sqrt and division (sigma bitwise equal to the reference).
// fp32: branch-free -- one approximate rsqrt gives sigma = var * rsqrt(var)
// and 1/sigma (|err| <= ~3 ulp, well inside the 1e-5 fp32 bar), so the VEC
// points of a lane interleave without slow-path branches.
// Both: reference semantics of _tail_probs (lcp.py:48-68) -- sigma == 0 is a
// step with mu == theta counted "below"; otherwise both tails evaluated
// directly; theta = t for the source map, -t for the sink map.
template <typename T> struct Tails;

template <> struct Tails<double> {
  static __device__ __forceinline__ void eval(double m, double var, double t, bool t_zero,
                                              double& sg, double& ps, double& pk);
};
template <> struct Tails<float> {
  static __device__ __forceinline__ void eval(float m, float var, float t, bool t_zero,
                                              float& sg, float& ps, float& pk);
};

// P(X > theta) and P(X <= theta) exactly as _tail_probs (lcp.py:48-68):
// sigma == 0 is a step with mu == theta counted as "below"; otherwise
// t = (theta - mu) / sigma (overflow to +-inf allowed), below = ndtr(t),
// above = ndtr(-t).
template <typename T>
__device__ __forceinline__ T prob_above(T mu, T sigma, T theta) {
  if (sigma == T(0)) return mu <= theta ? T(0) : T(1);
  T t = Arith<T>::div(Arith<T>::sub(theta, mu), sigma);
  return ndtr_(-t);
}
template <typename T>
__device__ __forceinline__ T prob_below(T mu, T sigma, T theta) {
  if (sigma == T(0)) return mu <= theta ? T(1) : T(0);
  T t = Arith<T>::div(Arith<T>::sub(theta, mu), sigma);
  return ndtr_(t);
}

// below = P(X <= t_arg quantile) = ndtr(q), above = ndtr(-q) from one erfc
// (ndtr structure: x = q*sqrt(1/2); small tail erfc(|x|)/2, never 1 - p).
template <typename T>
__device__ __forceinline__ void ndtr_pair(T q, T& below, T& above) {
  using A = Arith<T>;
  const T x = A::mul(q, T(0.70710678118654752440));
  const T y = A::mul(T(0.5), erfc_abs(x));
  const T c = A::sub(T(1), y);
  below = x > T(0) ? c : y;
  above = x > T(0) ? y : c;
}

// (below, above) of one point from ONE erfc: bitwise equal to
// (prob_below, prob_above) -- ndtr(-t) negates ndtr(t)'s scaled argument
// exactly, so both evaluate the same erfc(|x|) (lcp.py:48-68).
template <typename T>
__device__ __forceinline__ void tail_pair(T mu, T sigma, T theta, T& below, T& above) {
  if (sigma == T(0)) {
    below = mu <= theta ? T(1) : T(0);
    above = T(1) - below;
    return;
  }
  ndtr_pair(Arith<T>::div(Arith<T>::sub(theta, mu), sigma), below, above);
}

// n / d for d > 0 finite, branch-free: reciprocal (rcp.approx, two Newton
// steps) and one residual correction (<= 1 ulp).  The reference divides with
// overflow allowed (lcp.py:62-65): a tiny d (rcp.approx.ftz flushes
// subnormals; 1/d overflows below 2^-1022) is scaled by 2^128 together with n
// (exact), and a quotient that overflows stays +-inf (the residual step would
// turn it into NaN).
// (NEWTON = 1: ~2^-46 before the correction -- enough for the LCP's
// absolute bar; the relative fp64 maps use 2)
template <int NEWTON = 2>
__device__ __forceinline__ double div_pos(double n, double d) {
  const bool tiny = d < 0x1p-896;
  const double sc = tiny ? 0x1p128 : 1.0;
  const double dd = d * sc, nn = n * sc;
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(dd));
#pragma unroll
  for (int k = 0; k < NEWTON; ++k) r = fma(r, fma(-dd, r, 1.0), r);
  const double q = nn * r;
  const double c = fma(fma(-dd, q, nn), r, q);
  return isinf(q) ? q : c;
}

// fp64 tails, branch-free: sigma = 0 (the step function) is selected after
// the erfc instead of branched around (0/0 and x/0 quotients are discarded)
__device__ __forceinline__ void Tails<double>::eval(double m, double var, double t, bool t_zero,
                                                    double& sg, double& ps, double& pk) {
  using A = Arith<double>;
  sg = A::sqrt_(var);                        // IEEE: sigma bitwise equal to the reference
  const bool z = sg == 0.0;
  const double d = z ? 1.0 : sg;
  double b1, a1, b2, a2;
  ndtr_pair(div_pos(A::sub(t, m), d), b1, a1);
  if (t_zero) {  // theta = +0 and -0 give the same quotient: one erfc serves both
    b2 = b1;
  } else {
    ndtr_pair(div_pos(A::sub(-t, m), d), b2, a2);
  }
  ps = z ? (m <= t ? 0.0 : 1.0) : a1;
  pk = z ? (m <= -t ? 1.0 : 0.0) : b2;
}

__device__ __forceinline__ void Tails<float>::eval(float m, float var, float t, bool t_zero,
                                                   float& sg, float& ps, float& pk) {
  // rsqrt.approx flushes subnormals: a variance below FLT_MIN (sigma < 1.1e-19)
  // is evaluated as FLT_MIN; the tails are then 0/1 to fp32 precision anyway
  const float vs = fmaxf(var, 1.17549435e-38f);
  const float r = rsqrt_approx(vs);
  sg = var == 0.0f ? 0.0f : vs * r;
  float b1, a1, b2, a2;
  ndtr_pair((t - m) * r, b1, a1);
  if (t_zero) {
    b2 = b1;
  } else {
    ndtr_pair((-t - m) * r, b2, a2);
  }
  ps = var == 0.0f ? (m <= t ? 0.0f : 1.0f) : a1;
  pk = var == 0.0f ? (m <= -t ? 1.0f : 0.0f) : b2;
}

// ---- vector types: VEC consecutive x-points per thread ------------------
template <typename T, int VEC> struct alignas(sizeof(T) * VEC) Vec { T v[VEC]; };

template <typename T, int VEC>
__device__ __forceinline__ Vec<T, VEC> ldg_vec(const T* p) {
  return *reinterpret_cast<const Vec<T, VEC>*>(p);
}
// streaming (evict-first) loads/stores for data touched exactly once
template <typename T, int VEC>
__device__ __forceinline__ Vec<T, VEC> ld_stream(const T* p) {
  Vec<T, VEC> r;
  if constexpr (sizeof(Vec<T, VEC>) == 16) {
    int4 q = __ldcs(reinterpret_cast<const int4*>(p));
    r = *reinterpret_cast<Vec<T, VEC>*>(&q);
  } else if constexpr (sizeof(Vec<T, VEC>) == 8) {
    int2 q = __ldcs(reinterpret_cast<const int2*>(p));
    r = *reinterpret_cast<Vec<T, VEC>*>(&q);
  } else {
    r.v[0] = __ldcs(p);
  }
  return r;
}
template <typename T, int VEC>
__device__ __forceinline__ void st_stream(T* p, const Vec<T, VEC>& x) {
  if constexpr (sizeof(Vec<T, VEC>) == 16) {
    __stcs(reinterpret_cast<int4*>(p), *reinterpret_cast<const int4*>(&x));
  } else if constexpr (sizeof(Vec<T, VEC>) == 8) {
    __stcs(reinterpret_cast<int2*>(p), *reinterpret_cast<const int2*>(&x));
  } else {
    __stcs(p, x.v[0]);
  }
}

template <typename T>
__device__ __forceinline__ int check_value(T x) { return isfinite(x) ? 0 : kErrNonFinite; }
template <typename T>
__device__ __forceinline__ int check_sigma(T s) {
  return (isfinite(s) ? 0 : kErrNonFinite) | (s < T(0) ? kErrNegativeSigma : 0);
}

// one atomic per warp at most
__device__ __forceinline__ void flush_error(int* err, int bits) {
  if (err == nullptr) return;
  unsigned m = __ballot_sync(0xffffffffu, bits != 0);
  if (m == 0) return;
  int all = bits;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) all |= __shfl_xor_sync(0xffffffffu, all, o);
  if ((threadIdx.x & 31) == (__ffs(m) - 1)) atomicOr(err, all);
}

}  // namespace divuq
