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

// ---- branch-free fp64 erfc for the level-crossing kernels ----------------
// libdevice's erfc takes different code paths by range, so a warp whose
// vertices straddle the ranges runs several of them (ncu: the LCP kernel was
// issue-bound at ~330 instructions per cell).  Here: erfc(a) =
// exp(-a^2) * h(q) / (a + K), q = (a - K) / (a + K), K = 3.75, h a degree-20
// polynomial fitted offline against scipy's erfcx (tools/fit_erfc.py: fit64;
// max relative error 3.8e-15 on [0, 26.5]), one reciprocal, one branch-free
// exp, and the a*a rounding corrected by one FMA.  The LCP bar is absolute (1e-12) on
// products of tail probabilities, far above this.  Past a = 26.6 erfc is
// below the smallest normal double: 0 (also for a = inf, sigma -> 0+).
__constant__ double kErfcLcp[21] = {
    0x1.17884282534a6p+0, -0x1.eae02d0a14575p-1, 0x1.78fecb4e81911p-1, -0x1.f63dd81197172p-2,
    0x1.1dc27118a572ap-2, -0x1.0e3ea22487d15p-3, 0x1.92618b748e0dbp-5, -0x1.9ac695838042dp-7,
    0x1.02900c1cc2f87p-10, 0x1.a0b7617bbe006p-11, -0x1.6d95991270bd9p-12, 0x1.63741a4632739p-17,
    0x1.3a61910987620p-15, -0x1.2ab497b501b66p-17, -0x1.bb2922abacccep-19, 0x1.bb2c732d1672ap-20,
    0x1.3f8939719327ap-22, -0x1.1066ac54efe96p-22, -0x1.6288b0af8129ap-25, 0x1.f6c45f0bc1fb5p-26,
    0x1.1081b6baf64d4p-27};

// exp(t) for t in [-708, 0] (the caller discards t < -707): k = rint(t/ln2),
// r = t - k ln2 (fdlibm's hi/lo split), e^r by its Taylor series to r^12
// (|r| <= 0.347: truncation < 2e-16), times 2^k built in the exponent bits.
// Coefficients come from constant memory (no UMOV-materialised literals), no
// range branches.
__constant__ double kExpTaylor[13] = {
    0x1.0000000000000p+0, 0x1.0000000000000p+0, 0x1.0000000000000p-1, 0x1.5555555555555p-3,
    0x1.5555555555555p-5, 0x1.1111111111111p-7, 0x1.6c16c16c16c17p-10, 0x1.a01a01a01a01ap-13,
    0x1.a01a01a01a01ap-16, 0x1.71de3a556c734p-19, 0x1.27e4fb7789f5cp-22, 0x1.ae64567f544e4p-26,
    0x1.1eed8eff8d898p-29};

__device__ __forceinline__ double exp_neg_lcp(double t) {
  const double y = fma(t, 0x1.71547652b82fep+0, 0x1.8p52);   // 1.5*2^52 + rint(t*log2(e))
  const double kd = y - 0x1.8p52;
  const int ki = __double2loint(y);
  double r = fma(kd, -6.93147180369123816490e-01, t);
  r = fma(kd, -1.90821492927058770002e-10, r);
  double p = kExpTaylor[12];
#pragma unroll
  for (int k = 11; k >= 0; --k) p = fma(p, r, kExpTaylor[k]);
  return p * __hiloint2double((ki + 1023) << 20, 0);
}

__device__ __forceinline__ double erfc_abs_lcp(double x) {
  constexpr double K = 3.75;
  const double a = fabs(x);
  const double d = a + K;
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  const double q = (a - K) * r;
  double p = kErfcLcp[20];
#pragma unroll
  for (int k = 19; k >= 0; --k) p = fma(p, q, kErfcLcp[k]);
  const double s = a * a;
  const double lo = fma(a, a, -s);   // a*a - s exactly
  double y = p * r * exp_neg_lcp(fmax(-s, -707.0));
  y = fma(y, -lo, y);                // * exp(-lo) ~ (1 - lo)
  return a > 26.6 ? 0.0 : y;
}
__device__ __forceinline__ float erfc_abs_lcp(float x) { return erfc_abs(x); }

// (theta - mu) / sigma: fp64 by reciprocal + two Newton steps (<= 1 ulp; no
// IEEE-division slow path: sigma > 0 and finite here); fp32 IEEE as before
__device__ __forceinline__ double lcp_div(double n, double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  const double q = n * r;
  return fma(fma(-d, q, n), r, q);   // one residual correction
}
__device__ __forceinline__ float lcp_div(float n, float d) { return __fdiv_rn(n, d); }

// tail pair of one vertex for the LCP kernels: _tail_probs semantics
// (lcp.py:48-68) with the branch-free erfc above (fp32: the shared fp32 erfc)
template <typename T>
__device__ __forceinline__ void tail_pair_lcp(T mu, T sigma, T theta, T& below, T& above) {
  using A = Arith<T>;
  if (sigma == T(0)) {
    below = mu <= theta ? T(1) : T(0);
    above = T(1) - below;
    return;
  }
  const T x = A::mul(lcp_div(A::sub(theta, mu), sigma), T(0.70710678118654752440));
  const T y = A::mul(T(0.5), erfc_abs_lcp(x));
  const T c = A::sub(T(1), y);
  below = x > T(0) ? c : y;
  above = x > T(0) ? y : c;
}

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
  T* const bl = &below[0][0];
  T* const ab = &above[0][0];
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
  // park (mu, sigma) in the tile's own slots (flat slot v = vy*(TX+1) + vx), so
  // the tail pairs run as a rolled loop: the erfc / exp coefficients stay in
  // uniform registers across iterations instead of being reloaded per copy
#pragma unroll
  for (int k = 0; k < kLcpNQ; ++k) {
    const int v = tid + k * kLcpBX * kLcpBY;
    if (v < kLcpV) { bl[v] = mv[k]; ab[v] = sv[k]; }
  }
#pragma unroll 1
  for (int v = tid; v < kLcpV; v += kLcpBX * kLcpBY) {   // own slots only: no barrier needed
    const T m = bl[v], sg = ab[v];
    errbits |= check_value(m) | check_sigma(sg);
    T b, a;
    tail_pair_lcp(m, sg, theta, b, a);
    bl[v] = b;
    ab[v] = a;
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
      tail_pair_lcp(m, s, theta, b, a);
      pb = k == 0 ? b : A::mul(pb, b);
      pa = k == 0 ? a : A::mul(pa, a);
    }
    const T r = A::sub(T(1), A::add(pb, pa));
    out[c] = r < T(0) ? T(0) : (r > T(1) ? T(1) : r);
  }
  flush_error(err, errbits);
}

}  // namespace divuq
