// Level-crossing probability per grid cell.
//
// Replaces lcp() / cell_crossing_probability (lcp.py:71-100): for cell
// (ci, cj) with corners v00 = cj*nx + ci, v00+1, v00+nx, v00+nx+1 (that
// order, lcp.py:88-91), LCP = clip(1 - (prod_k below_k + prod_k above_k), 0, 1)
// with (below, above) = _tail_probs(mu, sigma, theta) per corner
// (lcp.py:48-68) and np.prod's sequential order ((c0*c1)*c2)*c3.
//
// Layout of the work: a CTA of 32 x 8 threads owns a 64 x 16 tile of cells
// (2 x 2 cells per thread).  It loads the tile's 65 x 17 corner vertices with
// all of a thread's loads in flight at once, evaluates each vertex's tail pair
// ONCE into shared memory (one erfc per vertex, 1.08 per cell -- the fp64 erfc
// is the kernel's bound, not HBM), then every thread forms its cells' products.
#pragma once

#include "common.cuh"

namespace divuq {

constexpr int kLcpTX = 64, kLcpTY = 16, kLcpBX = 32, kLcpBY = 8;
constexpr int kLcpV = (kLcpTX + 1) * (kLcpTY + 1);
constexpr int kLcpNQ = (kLcpV + kLcpBX * kLcpBY - 1) / (kLcpBX * kLcpBY);

template <typename T>
__global__ void __launch_bounds__(kLcpBX * kLcpBY)
lcp2d_kernel(const T* __restrict__ mu, const T* __restrict__ sigma, int64_t nx, int64_t ny,
             T theta, T* __restrict__ out, int* err) {
  using A = Arith<T>;
  __shared__ T below[kLcpTY + 1][kLcpTX + 1];
  __shared__ T above[kLcpTY + 1][kLcpTX + 1];
  const int tid = threadIdx.y * kLcpBX + threadIdx.x;
  const int64_t ci0 = int64_t(blockIdx.x) * kLcpTX, cj0 = int64_t(blockIdx.y) * kLcpTY;
  int errbits = 0;
  T mv[kLcpNQ], sv[kLcpNQ];
#pragma unroll
  for (int k = 0; k < kLcpNQ; ++k) {  // all loads first: kLcpNQ x 2 in flight per thread
    const int v = tid + k * kLcpBX * kLcpBY;
    const int vy = v / (kLcpTX + 1), vx = v % (kLcpTX + 1);
    const int64_t i = ci0 + vx, j = cj0 + vy;
    mv[k] = T(0);
    sv[k] = T(1);
    if (v < kLcpV && i < nx && j < ny) {
      mv[k] = mu[j * nx + i];
      sv[k] = sigma[j * nx + i];
    }
  }
#pragma unroll
  for (int k = 0; k < kLcpNQ; ++k) {
    const int v = tid + k * kLcpBX * kLcpBY;
    if (v < kLcpV) {
      const int vy = v / (kLcpTX + 1), vx = v % (kLcpTX + 1);
      errbits |= check_value(mv[k]) | check_sigma(sv[k]);
      T b, a;
      tail_pair(mv[k], sv[k], theta, b, a);
      below[vy][vx] = b;
      above[vy][vx] = a;
    }
  }
  __syncthreads();
#pragma unroll
  for (int ry = 0; ry < kLcpTY; ry += kLcpBY) {
#pragma unroll
    for (int rx = 0; rx < kLcpTX; rx += kLcpBX) {
      const int x = threadIdx.x + rx, y = threadIdx.y + ry;
      const int64_t ci = ci0 + x, cj = cj0 + y;
      if (ci < nx - 1 && cj < ny - 1) {
        // corners in lcp.py order: v00, v00+1, v00+nx, v00+nx+1
        const T pb = A::mul(A::mul(A::mul(below[y][x], below[y][x + 1]), below[y + 1][x]), below[y + 1][x + 1]);
        const T pa = A::mul(A::mul(A::mul(above[y][x], above[y][x + 1]), above[y + 1][x]), above[y + 1][x + 1]);
        const T r = A::sub(T(1), A::add(pb, pa));
        out[cj * (nx - 1) + ci] = r < T(0) ? T(0) : (r > T(1) ? T(1) : r);
      }
    }
  }
  flush_error(err, errbits);
}

// stacked cells: mu4 / sigma4 are (n, 4) row-major, corners in order
template <typename T>
__global__ void cell_crossing_kernel(const T* __restrict__ mu4, const T* __restrict__ sigma4,
                                     int64_t n, T theta, T* __restrict__ out, int* err) {
  using A = Arith<T>;
  int errbits = 0;
  for (int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < n;
       c += int64_t(gridDim.x) * blockDim.x) {
    T pb = T(1), pa = T(1);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const T m = mu4[c * 4 + k], s = sigma4[c * 4 + k];
      errbits |= check_value(m) | check_sigma(s);
      T b, a;
      tail_pair(m, s, theta, b, a);
      pb = k == 0 ? b : A::mul(pb, b);
      pa = k == 0 ? a : A::mul(pa, a);
    }
    const T r = A::sub(T(1), A::add(pb, pa));
    out[c] = r < T(0) ? T(0) : (r > T(1) ? T(1) : r);
  }
  flush_error(err, errbits);
}

}  // namespace divuq
