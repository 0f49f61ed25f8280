// Velocity-magnitude-gradient prologue.
//
// Replaces velocity_magnitude (gaussian.py:48-50: hypot(u, v)), gradient
// (gaussian.py:53-58 -> stencils.py:87-96: f[hi]*c - f[lo]*c per axis, the
// same one-sided boundary rule as the divergence) and gradient_ensemble
// (gaussian.py:61-66: every member mapped through both) -- the Red Sea
// vortex-core pipeline.  The ensemble kernel is fused: each output point
// recomputes the four neighbour magnitudes it needs (hypot is cheap next to
// the 16 bytes it reads per point per member), so members go HBM -> gradient
// in one pass with no magnitude field in between.
#pragma once

#include "common.cuh"

namespace divuq {

template <typename T> __device__ __forceinline__ T hypot_(T a, T b);
template <> __device__ __forceinline__ double hypot_(double a, double b) { return hypot(a, b); }
template <> __device__ __forceinline__ float hypot_(float a, float b) { return hypotf(a, b); }

template <typename T>
__global__ void vmag_kernel(const T* __restrict__ u, const T* __restrict__ v, int64_t n,
                            T* __restrict__ out, int* err) {
  int errbits = 0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const T a = u[i], b = v[i];
    errbits |= check_value(a) | check_value(b);
    out[i] = hypot_(a, b);
  }
  flush_error(err, errbits);
}

// One axis of the reference stencil at coordinate a of n (stencils.py:46-50).
struct AxisRule {
  int64_t lo, hi;
  bool bd;
};
__device__ __forceinline__ AxisRule axis_rule(int64_t a, int64_t n) {
  return AxisRule{a > 0 ? a - 1 : 0, a < n - 1 ? a + 1 : n - 1, a == 0 || a == n - 1};
}

// gradient of a scalar field, or (MAG) of |(u, v)| computed on the fly.
// planes: `members` planes of (u[, v]) with stride `pstride` between member
// blocks; outputs (gx, gy) per member with the same strides.
template <typename T, bool MAG>
__global__ void gradient2d_kernel(const T* __restrict__ in, int64_t members, int64_t in_mstride,
                                  int64_t nx, int64_t ny, T cx_in, T cx_bd, T cy_in, T cy_bd,
                                  T* __restrict__ out, int64_t out_mstride, int* err) {
  using A = Arith<T>;
  const int64_t n = nx * ny;
  int errbits = 0;
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < members * n;
       t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t m = t / n, p = t % n;
    const int64_t i = p % nx, j = p / nx;
    const T* f = in + m * in_mstride;
    auto val = [&](int64_t q) -> T {
      if constexpr (MAG) return hypot_(f[q], f[n + q]);
      else return f[q];
    };
    const AxisRule rx = axis_rule(i, nx), ry = axis_rule(j, ny);
    const T cx = rx.bd ? cx_bd : cx_in, cy = ry.bd ? cy_bd : cy_in;
    const T gx = A::sub(A::mul(val(j * nx + rx.hi), cx), A::mul(val(j * nx + rx.lo), cx));
    const T gy = A::sub(A::mul(val(ry.hi * nx + i), cy), A::mul(val(ry.lo * nx + i), cy));
    errbits |= check_value(f[p]);
    if constexpr (MAG) errbits |= check_value(f[n + p]);
    out[m * out_mstride + p] = gx;
    out[m * out_mstride + n + p] = gy;
  }
  flush_error(err, errbits);
}

}  // namespace divuq
