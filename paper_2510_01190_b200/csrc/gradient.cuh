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

// gradient of a scalar field, or (MAG) of |(u, v)| computed on the fly.
// A CTA of 32 x 8 threads owns a 64 x 16 tile of one member (2 x 2 points per
// thread): it loads the tile plus a one-point halo with all of a thread's
// loads in flight at once (coalesced row segments; halo re-reads, 16 %, hit
// L2), evaluates the field (the magnitude, for MAG) ONCE per loaded point into
// shared memory, then every thread forms its points' one-axis differences.
// planes: `members` blocks of (u[, v]) with stride in_mstride; outputs
// (gx, gy) per member.
constexpr int kGrTX = 64, kGrTY = 16, kGrBX = 32, kGrBY = 8;
constexpr int kGrV = (kGrTX + 2) * (kGrTY + 2);
constexpr int kGrNQ = (kGrV + kGrBX * kGrBY - 1) / (kGrBX * kGrBY);

template <typename T, bool MAG>
__global__ void __launch_bounds__(kGrBX * kGrBY, 3)
gradient2d_kernel(const T* __restrict__ in, int64_t members, int64_t in_mstride, int64_t nx,
                  int64_t ny, T cx_in, T cx_bd, T cy_in, T cy_bd, T* __restrict__ out,
                  int64_t out_mstride, int* err) {
  using A = Arith<T>;
  __shared__ T f[kGrTY + 2][kGrTX + 2];
  const int64_t n = nx * ny;
  const int tid = threadIdx.y * kGrBX + threadIdx.x;
  const int64_t i0 = int64_t(blockIdx.x) * kGrTX, j0 = int64_t(blockIdx.y) * kGrTY;
  int errbits = 0;
  for (int64_t m = blockIdx.z; m < members; m += gridDim.z) {
    const T* src = in + m * in_mstride;
    // (tile + halo) with clamped coordinates: a clamped slot is only read as
    // the one-sided boundary neighbour, which IS the clamped point
    T a[kGrNQ], b[kGrNQ];
#pragma unroll
    for (int k = 0; k < kGrNQ; ++k) {
      const int q = min(tid + k * kGrBX * kGrBY, kGrV - 1);
      const int qy = q / (kGrTX + 2), qx = q % (kGrTX + 2);
      const int64_t gi = min(max(i0 + qx - 1, int64_t(0)), nx - 1);
      const int64_t gj = min(max(j0 + qy - 1, int64_t(0)), ny - 1);
      const int64_t p = gj * nx + gi;
      a[k] = src[p];
      if constexpr (MAG) b[k] = src[n + p];
    }
#pragma unroll
    for (int k = 0; k < kGrNQ; ++k) {
      const int q = tid + k * kGrBX * kGrBY;
      if (q < kGrV) {
        if constexpr (MAG) f[q / (kGrTX + 2)][q % (kGrTX + 2)] = hypot_(a[k], b[k]);
        else f[q / (kGrTX + 2)][q % (kGrTX + 2)] = a[k];
      }
    }
    __syncthreads();
#pragma unroll
    for (int ry = 0; ry < kGrTY; ry += kGrBY) {
#pragma unroll
      for (int rx = 0; rx < kGrTX; rx += kGrBX) {
        const int64_t i = i0 + threadIdx.x + rx, j = j0 + threadIdx.y + ry;
        if (i < nx && j < ny) {
          const int x = threadIdx.x + rx + 1, y = threadIdx.y + ry + 1;
          const bool bx = i == 0 || i == nx - 1, by = j == 0 || j == ny - 1;
          const T cx = bx ? cx_bd : cx_in, cy = by ? cy_bd : cy_in;
          const int xh = i < nx - 1 ? x + 1 : x, xl = i > 0 ? x - 1 : x;
          const int yh = j < ny - 1 ? y + 1 : y, yl = j > 0 ? y - 1 : y;
          const T gx = A::sub(A::mul(f[y][xh], cx), A::mul(f[y][xl], cx));
          const T gy = A::sub(A::mul(f[yh][x], cy), A::mul(f[yl][x], cy));
          const int64_t p = j * nx + i;
          out[m * out_mstride + p] = gx;
          out[m * out_mstride + n + p] = gy;
        }
      }
    }
    // validation word: every loaded interior slot is some point's own value
#pragma unroll
    for (int k = 0; k < kGrNQ; ++k) {
      errbits |= check_value(a[k]);
      if constexpr (MAG) errbits |= check_value(b[k]);
    }
    __syncthreads();
  }
  flush_error(err, errbits);
}

}  // namespace divuq
