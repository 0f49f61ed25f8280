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
// ndtr scales the argument by sqrt(1/2) with one multiply, uses erf near zero
// and erfc in the tails, and never forms 1-p for the small tail; keeping that
// structure keeps us within ~1e-13 relative of scipy even at x ~ -37.
__device__ __forceinline__ double ndtr_(double a) {
  const double kSqrtHalf = 0.70710678118654752440;
  double x = __dmul_rn(a, kSqrtHalf);
  double z = fabs(x);
  if (z < kSqrtHalf) return __dadd_rn(0.5, __dmul_rn(0.5, erf(x)));
  double y = __dmul_rn(0.5, erfc(z));
  return x > 0.0 ? __dsub_rn(1.0, y) : y;
}

__device__ __forceinline__ float ndtr_(float a) {
  const float kSqrtHalf = 0.70710678118654752440f;
  float x = __fmul_rn(a, kSqrtHalf);
  float z = fabsf(x);
  if (z < kSqrtHalf) return __fadd_rn(0.5f, __fmul_rn(0.5f, erff(x)));
  float y = __fmul_rn(0.5f, erfcf(z));
  return x > 0.0f ? __fsub_rn(1.0f, y) : y;
}

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
