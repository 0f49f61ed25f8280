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
#include "tma.cuh"

namespace divuq {

// ---- branch-free fp64 erfc for the level-crossing kernels ----------------
// libdevice's erfc takes different code paths by range, so a warp whose
// vertices straddle the ranges runs several of them (ncu: the LCP kernel was
// issue-bound at ~330 instructions per cell).  Here: erfc(a) =
// exp(-a^2) * h(q) / (a + K), q = (a - K) / (a + K), K = 3, h a degree-16
// polynomial fitted offline against scipy's erfcx on [0, 6.2]
// (tools/fit_erfc.py: fit64(3.0, 16, amax=6.2); max error 1.3e-15 absolute,
// 2.9e-15 relative), one reciprocal (one Newton step), one branch-free exp,
// and the a*a rounding corrected by one FMA.  The LCP bar is ABSOLUTE
// (1e-12 on products of tail probabilities): past a = 6.2 erfc(a) < 1.9e-18,
// returned as 0 (also for a = inf, sigma -> 0+).  (The first version fitted
// degree 20 on [0, 26.5] to 3.8e-15 relative: 4 more FMAs per vertex.)
__constant__ double kErfcLcp[17] = {
    0x1.12f21ddd9f5e1p+0, -0x1.c44c471baa268p-1, 0x1.2e326945de38ap-1, -0x1.3deb21416ca90p-2,
    0x1.e995f11b16886p-4, -0x1.b78993b5e4be8p-6, -0x1.3dd3e5fc26ebfp-10, 0x1.8dae28f56a401p-9,
    -0x1.1f7943276e395p-11, -0x1.2234c8a90349bp-12, 0x1.c350cc2d97cf3p-14, 0x1.fd736047b47bdp-16,
    -0x1.28c763237c059p-16, -0x1.4c4280ee09a7ap-18, 0x1.9657f8bc02840p-19, 0x1.d4b67a91621acp-20,
    0x1.2479dd117d25fp-22};

// exp(t) for t in [-39, 0] (a <= 6.2): k = rint(t/ln2), r = t - k ln2
// (fdlibm's hi/lo split), e^r by its Taylor series to r^11 (|r| <= 0.347:
// truncation < 7e-15 relative), times 2^k built in the exponent bits.
// Coefficients come from constant memory (no UMOV-materialised literals), no
// range branches.
__constant__ double kExpTaylor[12] = {
    0x1.0000000000000p+0, 0x1.0000000000000p+0, 0x1.0000000000000p-1, 0x1.5555555555555p-3,
    0x1.5555555555555p-5, 0x1.1111111111111p-7, 0x1.6c16c16c16c17p-10, 0x1.a01a01a01a01ap-13,
    0x1.a01a01a01a01ap-16, 0x1.71de3a556c734p-19, 0x1.27e4fb7789f5cp-22, 0x1.ae64567f544e4p-26};

__device__ __forceinline__ double exp_neg_lcp(double t) {
  const double y = fma(t, 0x1.71547652b82fep+0, 0x1.8p52);   // 1.5*2^52 + rint(t*log2(e))
  const double kd = y - 0x1.8p52;
  const int ki = __double2loint(y);
  double r = fma(kd, -6.93147180369123816490e-01, t);
  r = fma(kd, -1.90821492927058770002e-10, r);
  double p = kExpTaylor[11];
#pragma unroll
  for (int k = 10; k >= 0; --k) p = fma(p, r, kExpTaylor[k]);
  return p * __hiloint2double((ki + 1023) << 20, 0);
}

// 1/d: rcp.approx (~2^-23) and one Newton step (~2^-46 relative) -- ample for
// the absolute 1e-12 LCP bar; lcp_div below adds a residual correction
__device__ __forceinline__ double rcp_lcp(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  return fma(r, fma(-d, r, 1.0), r);
}

__device__ __forceinline__ double erfc_abs_lcp(double x) {
  constexpr double K = 3.0;
  const double a = fabs(x);
  const double r = rcp_lcp(a + K);
  const double q = (a - K) * r;
  double p = kErfcLcp[16];
#pragma unroll
  for (int k = 15; k >= 0; --k) p = fma(p, q, kErfcLcp[k]);
  const double s = a * a;
  const double lo = fma(a, a, -s);   // a*a - s exactly
  double y = p * r * exp_neg_lcp(fmax(-s, -39.0));
  y = fma(y, -lo, y);                // * exp(-lo) ~ (1 - lo)
  // erfc(0) = 1 exactly, so a tail argument of exactly 0 gives 1/2 on both
  // sides like ndtr(0) -- the reference's exact negation symmetry of the
  // LCP (test_lcp.py:53-62) needs it (the fit is ~1e-15 off at 0)
  return a > 6.2 ? 0.0 : (a == 0.0 ? 1.0 : y);
}
__device__ __forceinline__ float erfc_abs_lcp(float x) { return erfc_abs(x); }

// erfc(a) / 2 for a = |x| >= 0: erfc_abs_lcp with the 1/2 folded into the
// coefficients (every Horner step, product and the FMA correction are the
// halved values exactly: bitwise 0.5 * erfc_abs_lcp(a)) and without the
// exponent clamp -- past a = 6.2 (and for a = inf) the exp's garbage is
// discarded by the final select, never propagated.
__constant__ double kErfcLcpHalf[17] = {
    0x1.12f21ddd9f5e1p-1, -0x1.c44c471baa268p-2, 0x1.2e326945de38ap-2, -0x1.3deb21416ca90p-3,
    0x1.e995f11b16886p-5, -0x1.b78993b5e4be8p-7, -0x1.3dd3e5fc26ebfp-11, 0x1.8dae28f56a401p-10,
    -0x1.1f7943276e395p-12, -0x1.2234c8a90349bp-13, 0x1.c350cc2d97cf3p-15, 0x1.fd736047b47bdp-17,
    -0x1.28c763237c059p-17, -0x1.4c4280ee09a7ap-19, 0x1.9657f8bc02840p-20, 0x1.d4b67a91621acp-21,
    0x1.2479dd117d25fp-23};
__device__ __forceinline__ double half_erfc_lcp(double a) {
  constexpr double K = 3.0;
  const double r = rcp_lcp(a + K);
  const double q = (a - K) * r;
  double p = kErfcLcpHalf[16];
#pragma unroll
  for (int k = 15; k >= 0; --k) p = fma(p, q, kErfcLcpHalf[k]);
  const double s = a * a;
  const double lo = fma(a, a, -s);
  double y = p * r * exp_neg_lcp(-s);
  y = fma(y, -lo, y);
  return a > 6.2 ? 0.0 : (a == 0.0 ? 0.5 : y);
}

// the tail argument (theta - mu) / sigma * sqrt(1/2) for the LCP kernels,
// rounded as before (lcp_div, then the multiply): the CLI's LCP CSV must stay
// within 1e-12 relative + 1e-15 absolute of the reference's (tests/test_cli.py),
// which a one-Newton quotient without the residual step (~2^-46) misses
__device__ __forceinline__ double lcp_arg(double n, double sigma) {
  return div_pos<1>(n, sigma) * 0.70710678118654752440;
}

// (theta - mu) / sigma: fp64 by reciprocal + one Newton step + one residual
// correction (~1 ulp; no IEEE-division slow path: sigma > 0 and finite
// here).  Two edges follow the reference's "overflow allowed" division
// (lcp.py:62-65) exactly: a tiny sigma (rcp.approx.ftz flushes subnormals and
// 1/sigma overflows below 2^-1022) takes the IEEE division, and a quotient
// that overflows stays +-inf (the residual step would turn inf into NaN).
// Both found by the reference's own test_lcp.py run through the drop-in hook
// (tests/test_reference_boundary.py).
__device__ __forceinline__ double lcp_div(double n, double d) { return div_pos<1>(n, d); }
__device__ __forceinline__ float lcp_div(float n, float d) { return __fdiv_rn(n, d); }

// tail pair of one vertex for the LCP kernels: _tail_probs semantics
// (lcp.py:48-68) with the branch-free erfc above (fp32: the shared fp32 erfc)
// fp64, branch-free: sigma = 0 (the reference's step function, lcp.py:58-61:
// below = mu <= theta) becomes x = +inf for theta - mu >= 0 and -inf below,
// which the erfc maps to exactly (1, 0) / (0, 1)
__device__ __forceinline__ void tail_pair_lcp(double mu, double sigma, double theta, double& below,
                                              double& above) {
  const double n = theta - mu;
  const double xs = lcp_arg(n, sigma);
  const double x = sigma == 0.0 ? (n >= 0.0 ? __longlong_as_double(0x7ff0000000000000ll)
                                            : __longlong_as_double(0xfff0000000000000ll))
                                : xs;
  const double y = half_erfc_lcp(fabs(x));
  const double c = 1.0 - y;
  below = x > 0.0 ? c : y;
  above = x > 0.0 ? y : c;
}

// the pair stored in place: the larger tail c goes to `below` when x > 0 and
// to `above` otherwise -- the store addresses are selected (2 integer selects)
// instead of the two fp64 values (4 FSEL)
__device__ __forceinline__ void tail_store_lcp(double mu, double sigma, double theta, double* below,
                                               double* above) {
  const double n = theta - mu;
  const double xs = lcp_arg(n, sigma);
  const double x = sigma == 0.0 ? (n >= 0.0 ? __longlong_as_double(0x7ff0000000000000ll)
                                            : __longlong_as_double(0xfff0000000000000ll))
                                : xs;
  const double y = half_erfc_lcp(fabs(x));
  const bool pos = x > 0.0;
  *(pos ? above : below) = y;
  *(pos ? below : above) = 1.0 - y;
}
__device__ __forceinline__ void tail_store_lcp(float mu, float sigma, float theta, float* below, float* above);

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

__device__ __forceinline__ void tail_store_lcp(float mu, float sigma, float theta, float* below, float* above) {
  float b, a;
  tail_pair_lcp(mu, sigma, theta, b, a);
  *below = b;
  *above = a;
}

#ifndef DIVUQ_LCP_UNROLL
#define DIVUQ_LCP_UNROLL 2   // with 6 CTAs/SM (40 regs): 123.3 -> 121.3 us; 5 + 4 CTAs: 179 us
#endif
constexpr int kLcpUnroll = DIVUQ_LCP_UNROLL;
#ifndef DIVUQ_LCP_MINB
#define DIVUQ_LCP_MINB 6
#endif
constexpr int kLcpTX = 64, kLcpTY = 16, kLcpBX = 32, kLcpBY = 8;
#ifndef DIVUQ_LCP_TMA_TY
#define DIVUQ_LCP_TMA_TY 40   // 16: 121.5 us, 24: 114.8, 32: 113.7, 40: 112.6 (4096^2)
#endif
constexpr int kLcpTYT = DIVUQ_LCP_TMA_TY;   // cell rows per CTA of lcp2d_tma_kernel

// max(r, 0) keeping NaN: r = 1 - (pb + pa) is never -0, and the GPU's NaN
// is positive, so the sign bit alone says r < 0 (fp32: the plain compare)
__device__ __forceinline__ double lcp_clip0(double r) { return __double2hiint(r) < 0 ? 0.0 : r; }
__device__ __forceinline__ float lcp_clip0(float r) { return r < 0.0f ? 0.0f : r; }

// the tile's cells from its tail tables (row pitch W): lcp.py:88-100, corners
// v00, v00+1, v00+nx, v00+nx+1, np.prod's order.  clip(r, 0, 1): r <= 1 always
// (1 minus a sum of products of tails in [0, 1]; the erfc fit is relative, so
// no tail is ever below 0), so only the lower clip is evaluated; NaN passes
// through both ways like np.clip.  Bounds and addressing in 32-bit per tile.
template <typename T, int W, int TY = kLcpTY>
__device__ __forceinline__ void lcp_tile_cells(const T* below, const T* above, int64_t ci0, int64_t cj0,
                                               int64_t nx, int64_t ny, T* __restrict__ out) {
  using A = Arith<T>;
  const int xl = int(min(nx - 1 - ci0, int64_t(kLcpTX))), yl = int(min(ny - 1 - cj0, int64_t(TY)));
  const int64_t ld = nx - 1;
  T* const o = out + cj0 * ld + ci0;
#pragma unroll
  for (int ry = 0; ry < TY; ry += kLcpBY) {
#pragma unroll
    for (int rx = 0; rx < kLcpTX; rx += kLcpBX) {
      const int x = threadIdx.x + rx, y = threadIdx.y + ry;
      if (x < xl && y < yl) {
        const T* b = below + y * W + x;
        const T* a = above + y * W + x;
        const T pb = A::mul(A::mul(A::mul(b[0], b[1]), b[W]), b[W + 1]);
        const T pa = A::mul(A::mul(A::mul(a[0], a[1]), a[W]), a[W + 1]);
        const T r = A::sub(T(1), A::add(pb, pa));
        o[int64_t(y) * ld + x] = lcp_clip0(r);
      }
    }
  }
}
constexpr int kLcpV = (kLcpTX + 1) * (kLcpTY + 1);
constexpr int kLcpNQ = (kLcpV + kLcpBX * kLcpBY - 1) / (kLcpBX * kLcpBY);

template <typename T>
__global__ void __launch_bounds__(kLcpBX * kLcpBY, DIVUQ_LCP_MINB)
lcp2d_kernel(const T* __restrict__ mu, const T* __restrict__ sigma, int64_t nx, int64_t ny,
             T theta, T* __restrict__ out, int* err) {
  using A = Arith<T>;
  __shared__ T below[kLcpTY + 1][kLcpTX + 1];
  __shared__ T above[kLcpTY + 1][kLcpTX + 1];
  const int tid = threadIdx.y * kLcpBX + threadIdx.x;
  const int64_t ci0 = int64_t(blockIdx.x) * kLcpTX, cj0 = int64_t(blockIdx.y) * kLcpTY;
  int nonfinite = 0, negative = 0;   // validation flags (check_value / check_sigma)
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
    nonfinite |= int(!isfinite(m)) | int(!isfinite(sg));
    negative |= int(sg < T(0));
    tail_store_lcp(m, sg, theta, bl + v, ab + v);
  }
  const int errbits = (nonfinite ? kErrNonFinite : 0) | (negative ? kErrNegativeSigma : 0);
  __syncthreads();
  lcp_tile_cells<T, kLcpTX + 1>(&below[0][0], &above[0][0], ci0, cj0, nx, ny, out);
  flush_error(err, errbits);
}

// TMA variant (nx * sizeof(T) % 16 == 0): one thread stages the tile's
// (mu, sigma) boxes of 17 x (64 + 16 B) vertices straight into the two tables
// with cp.async.bulk.tensor (out-of-grid vertices arrive as 0, 0: a finite
// step-function tail pair in cells that are never written), so the per-vertex
// index arithmetic, bounds checks and parking of the register-loaded kernel
// disappear (~40 of its ~200 instructions per vertex); the tail-pair loop runs
// over every table slot without coordinates.  Same arithmetic as above.
template <typename T>
struct LcpTma {
  static constexpr int W = kLcpTX + 16 / int(sizeof(T));   // box width: 16-byte multiple
  static constexpr int H = kLcpTYT + 1;
};

template <typename T>
__global__ void __launch_bounds__(kLcpBX * kLcpBY, DIVUQ_LCP_MINB)
lcp2d_tma_kernel(const __grid_constant__ CUtensorMap map_mu, const __grid_constant__ CUtensorMap map_sg,
                 int64_t nx, int64_t ny, T theta, T* __restrict__ out, int* err) {
  using A = Arith<T>;
  using L = LcpTma<T>;
  __shared__ __align__(128) T below[L::H][L::W];
  __shared__ __align__(128) T above[L::H][L::W];
  __shared__ uint64_t bar;
  const int tid = threadIdx.y * kLcpBX + threadIdx.x;
  const int64_t ci0 = int64_t(blockIdx.x) * kLcpTX, cj0 = int64_t(blockIdx.y) * kLcpTYT;
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
    mbar_expect_tx(&bar, 2 * L::H * L::W * sizeof(T));
    tma_load_3d(&below[0][0], &map_mu, &bar, int(ci0), int(cj0), 0);
    tma_load_3d(&above[0][0], &map_sg, &bar, int(ci0), int(cj0), 0);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  int nonfinite = 0, negative = 0;   // validation flags (check_value / check_sigma)
  T* const bl = &below[0][0];
  T* const ab = &above[0][0];
#pragma unroll kLcpUnroll
  for (int v = tid; v < L::H * L::W; v += kLcpBX * kLcpBY) {   // own slots only: no barrier needed
    const T m = bl[v], sg = ab[v];
    nonfinite |= int(!isfinite(m)) | int(!isfinite(sg));
    negative |= int(sg < T(0));
    tail_store_lcp(m, sg, theta, bl + v, ab + v);
  }
  const int errbits = (nonfinite ? kErrNonFinite : 0) | (negative ? kErrNegativeSigma : 0);
  __syncthreads();
  lcp_tile_cells<T, L::W, kLcpTYT>(&below[0][0], &above[0][0], ci0, cj0, nx, ny, out);
  flush_error(err, errbits);
}

// Odd nx (fp64 rows not 16-byte aligned: no tiled tensor map): the same tile
// on 1D tensor maps over the flat arrays, one row box per vertex row.  A box
// must start on a 16-byte boundary, so row y's box starts one element early
// when its offset is odd and the row sits at shift sh(y) = ((cj0 + y) nx) & 1
// in its table row (cj0 + y parity for odd nx; ci0 is even).  Out-of-range
// parts arrive as 0; a row's last two table columns hold the next row's
// first values, read only by cells that are never written.
constexpr int kLcpFTY = 32;   // cell rows per CTA (2 x 33 x 640 B tables: static shared memory)
struct LcpFlat {
  static constexpr int W = kLcpTX + 2;    // vertices per row used (65) rounded to even
  static constexpr int BOX = W + 2;       // row box: + 1 element of start slack, even
  static constexpr int P = 80;            // table pitch (640 B: 128-byte aligned rows)
  static constexpr int H = kLcpFTY + 1;
};

__global__ void __launch_bounds__(kLcpBX * kLcpBY, DIVUQ_LCP_MINB)
lcp2d_flat_kernel(const __grid_constant__ CUtensorMap map_mu, const __grid_constant__ CUtensorMap map_sg,
                  int64_t nx, int64_t ny, double theta, double* __restrict__ out, int* err) {
  using A = Arith<double>;
  using L = LcpFlat;
  __shared__ __align__(128) double below[L::H][L::P];
  __shared__ __align__(128) double above[L::H][L::P];
  __shared__ uint64_t bar;
  const int tid = threadIdx.y * kLcpBX + threadIdx.x;
  const int64_t ci0 = int64_t(blockIdx.x) * kLcpTX, cj0 = int64_t(blockIdx.y) * kLcpFTY;
  const int odd = int(nx & 1);
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
    mbar_expect_tx(&bar, 2u * L::H * L::BOX * sizeof(double));
  }
  __syncthreads();
  if (tid == 0 || tid == 32) {   // two issuing threads: one 1D load every ~72 cycles each
    const CUtensorMap* map = tid == 0 ? &map_mu : &map_sg;
    double* tab = tid == 0 ? &below[0][0] : &above[0][0];
    for (int r = 0; r < L::H; ++r) {
      const int64_t off = (cj0 + r) * nx + ci0;
      tma_load_1d(tab + r * L::P, map, &bar, int(off & ~int64_t(1)));
    }
  }
  mbar_wait(&bar, 0);
  int nonfinite = 0, negative = 0;
  double* const bl = &below[0][0];
  double* const ab = &above[0][0];
#pragma unroll kLcpUnroll
  for (int v = tid; v < L::H * L::W; v += kLcpBX * kLcpBY) {
    const int y = v / L::W, x = v - y * L::W;
    const int idx = y * L::P + (odd & int(cj0 + y)) + x;
    const double m = bl[idx], sg = ab[idx];
    nonfinite |= int(!isfinite(m)) | int(!isfinite(sg));
    negative |= int(sg < 0.0);
    tail_store_lcp(m, sg, theta, bl + idx, ab + idx);
  }
  const int errbits = (nonfinite ? kErrNonFinite : 0) | (negative ? kErrNegativeSigma : 0);
  __syncthreads();
  const int xl = int(min(nx - 1 - ci0, int64_t(kLcpTX))), yl = int(min(ny - 1 - cj0, int64_t(kLcpFTY)));
  const int64_t ld = nx - 1;
  double* const o = out + cj0 * ld + ci0;
#pragma unroll
  for (int ry = 0; ry < kLcpFTY; ry += kLcpBY) {
#pragma unroll
    for (int rx = 0; rx < kLcpTX; rx += kLcpBX) {
      const int x = threadIdx.x + rx, y = threadIdx.y + ry;
      if (x < xl && y < yl) {
        const int r0 = y * L::P + (odd & int(cj0 + y)) + x;
        const int r1 = (y + 1) * L::P + (odd & int(cj0 + y + 1)) + x;
        // corners in lcp.py order: v00, v00+1, v00+nx, v00+nx+1
        const double pb = A::mul(A::mul(A::mul(bl[r0], bl[r0 + 1]), bl[r1]), bl[r1 + 1]);
        const double pa = A::mul(A::mul(A::mul(ab[r0], ab[r0 + 1]), ab[r1]), ab[r1 + 1]);
        o[int64_t(y) * ld + x] = lcp_clip0(A::sub(1.0, A::add(pb, pa)));
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

namespace divuq {

// ---------------------------------------------------------------------------
// propagate_divergence -> lcp fused ("fused into the K2
// epilogue"): the (u, v) moments of a tile's 65 x 17 vertices plus their
// stencil halo are TMA-staged, every vertex's divergence (mu, sigma) is
// evaluated with K2's arithmetic (StencilMath<double>: the reference order,
// stencils.py:64-84, IEEE sqrt -- bitwise equal to propagate_divergence),
// its tail pair with the LCP kernels' tail_pair_lcp, and the cells' crossing
// probability with lcp.py:71-100's corner order -- so the result is bitwise
// K2 followed by lcp2d_tma_kernel, without writing (mu, sigma) to HBM and
// reading them back unless the caller asks for them.
// Boxes (fp64, 16-byte aligned starts): u moments rows j0..j0+16, columns
// i0-2..i0+65 (68 wide); v moments rows j0-1..j0+17, columns i0..i0+65
// (66 wide).  Out-of-grid slots arrive as 0 and feed only vertices that are
// never written and cells that are never written.
// ---------------------------------------------------------------------------
#ifndef DIVUQ_LCPF_TY
#define DIVUQ_LCPF_TY 16
#endif
#ifndef DIVUQ_LCPF_ALIAS
#define DIVUQ_LCPF_ALIAS 0
#endif
constexpr int kLcpFY = DIVUQ_LCPF_TY;           // cell rows per CTA of the fused kernel
constexpr bool kLcpFAlias = DIVUQ_LCPF_ALIAS;   // tail tables over the u boxes (tails held in registers)
struct LcpFused {
  static constexpr int UW = kLcpTX + 4, UH = kLcpFY + 1;   // u box: x from i0 - 2
  static constexpr int VW = kLcpTX + 2, VH = kLcpFY + 3;   // v box: y from j0 - 1
  static constexpr int W = kLcpTX + 2, H = kLcpFY + 1;     // vertex / tail tables
  static constexpr int NV = (H * (kLcpTX + 1) + kLcpBX * kLcpBY - 1) / (kLcpBX * kLcpBY);
  static constexpr uint32_t kBytes = uint32_t(2 * UW * UH + 2 * VW * VH) * 8u;
  static_assert(H * W <= UH * UW, "a tail table fits in a u box");
};

struct LcpFusedSmem {
  alignas(128) double mu_u[LcpFused::UH][LcpFused::UW];
  alignas(128) double s_u[LcpFused::UH][LcpFused::UW];
  alignas(128) double mu_v[LcpFused::VH][LcpFused::VW];
  alignas(128) double s_v[LcpFused::VH][LcpFused::VW];
#if !DIVUQ_LCPF_ALIAS
  alignas(16) double below[LcpFused::H][LcpFused::W];
  alignas(16) double above[LcpFused::H][LcpFused::W];
#endif
  uint64_t bar;
};

struct LcpFusedParams {
  int64_t nx, ny;
  double cx_in, cx_bd, cy_in, cy_bd, theta;
  double *out_mu, *out_sigma, *out_lcp;
  int* err;
};

// vertices (x, y) of the tile, x in [0, 65), y in [0, 17): global (i0 + x,
// j0 + y) -> (mu, sigma) with K2's arithmetic -> tail pair into the tables
template <bool EDGE>
__device__ __forceinline__ int lcpf_vertices(LcpFusedSmem& s, const LcpFusedParams& p, int tid,
                                             int64_t i0, int64_t j0, double* tb, double* ta) {
  using A = Arith<double>;
  using F = LcpFused;
  using SM = StencilMath<double, false>;
  const int64_t nx = p.nx, ny = p.ny;
  int nonfinite = 0, negative = 0;
  double rb[kLcpFAlias ? F::NV : 1], ra[kLcpFAlias ? F::NV : 1];   // tails held until the boxes are free
#pragma unroll
  for (int k = 0; k < (kLcpFAlias ? F::NV : 1); ++k) { rb[k] = 0.0; ra[k] = 0.0; }
#pragma unroll (kLcpFAlias ? F::NV : 1)
  for (int k = 0; k < F::NV; ++k) {
    const int v = tid + k * kLcpBX * kLcpBY;
    if (v >= F::H * (kLcpTX + 1)) break;
    const int y = v / (kLcpTX + 1), x = v - y * (kLcpTX + 1);
    const int64_t i = i0 + x, j = j0 + y;
    if (EDGE && (i >= nx || j >= ny)) continue;
    // stencils.py:46-51: the point itself at the global faces, c = 1/h there
    const bool ilo = EDGE && i == 0, ihi = EDGE && i == nx - 1;
    const bool jlo = EDGE && j == 0, jhi = EDGE && j == ny - 1;
    const int ux = x + 2, vy = y + 1;            // this vertex in the u / v boxes
    const double cx = (ilo || ihi) ? p.cx_bd : p.cx_in;
    const double cy = (jlo || jhi) ? p.cy_bd : p.cy_in;
    const int xl = ilo ? ux : ux - 1, xh = ihi ? ux : ux + 1;
    const int yl = jlo ? vy : vy - 1, yh = jhi ? vy : vy + 1;
    const double m = SM::mean(s.mu_u[y][xh], s.mu_u[y][xl], s.mu_v[yh][x], s.mu_v[yl][x], 0.0, 0.0,
                              cx, cy, 0.0);
    const double var = SM::var(s.s_u[y][xh], s.s_u[y][xl], s.s_v[yh][x], s.s_v[yl][x], 0.0, 0.0,
                               cx, cy, 0.0);
    const double sg = A::sqrt_(var);
    // validation: every in-grid input point is some tile's vertex exactly once
    const bool owned = (x < kLcpTX || (EDGE && i == nx - 1)) && (y < kLcpFY || (EDGE && j == ny - 1));
    if (owned) {
      const double mu = s.mu_u[y][ux], mv = s.mu_v[vy][x], su = s.s_u[y][ux], sv = s.s_v[vy][x];
      nonfinite |= int(!isfinite(mu)) | int(!isfinite(mv)) | int(!isfinite(su)) | int(!isfinite(sv));
      negative |= int(su < 0.0) | int(sv < 0.0);
      if (p.out_mu || p.out_sigma) {
        const int64_t o = j * nx + i;
        if (p.out_mu) p.out_mu[o] = m;
        if (p.out_sigma) p.out_sigma[o] = sg;
      }
    }
    if constexpr (kLcpFAlias) {
      tail_pair_lcp(m, sg, p.theta, rb[k], ra[k]);
    } else {
      tail_store_lcp(m, sg, p.theta, tb + y * F::W + x, ta + y * F::W + x);
    }
  }
  if constexpr (kLcpFAlias) {
    __syncthreads();   // every box read is done: the tables take over the u boxes
#pragma unroll
    for (int k = 0; k < F::NV; ++k) {
      const int v = tid + k * kLcpBX * kLcpBY;
      if (v >= F::H * (kLcpTX + 1)) break;
      const int y = v / (kLcpTX + 1), x = v - y * (kLcpTX + 1);
      tb[y * F::W + x] = rb[k];
      ta[y * F::W + x] = ra[k];
    }
  }
  return (nonfinite ? kErrNonFinite : 0) | (negative ? kErrNegativeSigma : 0);
}

__global__ void __launch_bounds__(kLcpBX * kLcpBY)
lcp2d_fused_kernel(const __grid_constant__ CUtensorMap m_mu_u, const __grid_constant__ CUtensorMap m_s_u,
                   const __grid_constant__ CUtensorMap m_mu_v, const __grid_constant__ CUtensorMap m_s_v,
                   const LcpFusedParams p) {
  using A = Arith<double>;
  using F = LcpFused;
  using SM = StencilMath<double, false>;
  extern __shared__ __align__(128) unsigned char lf_smem[];
  LcpFusedSmem& s = *reinterpret_cast<LcpFusedSmem*>(lf_smem);
  const int tid = threadIdx.y * kLcpBX + threadIdx.x;
  const int64_t i0 = int64_t(blockIdx.x) * kLcpTX, j0 = int64_t(blockIdx.y) * kLcpFY;
  if (tid == 0) {
    mbar_init(&s.bar, 1);
    mbar_fence_init();
    mbar_expect_tx(&s.bar, F::kBytes);
    tma_load_3d(&s.mu_u[0][0], &m_mu_u, &s.bar, int(i0) - 2, int(j0), 0);
    tma_load_3d(&s.s_u[0][0], &m_s_u, &s.bar, int(i0) - 2, int(j0), 0);
    tma_load_3d(&s.mu_v[0][0], &m_mu_v, &s.bar, int(i0), int(j0) - 1, 0);
    tma_load_3d(&s.s_v[0][0], &m_s_v, &s.bar, int(i0), int(j0) - 1, 0);
  }
  __syncthreads();
  mbar_wait(&s.bar, 0);
  const int64_t nx = p.nx, ny = p.ny;
  // tiles clear of the global faces and of the grid's end take the path
  // without boundary logic (CTA-uniform branch; same arithmetic)
  const bool interior = i0 >= 1 && i0 + kLcpTX <= nx - 2 && j0 >= 1 && j0 + kLcpFY <= ny - 2;
#if DIVUQ_LCPF_ALIAS
  double* const tb = &s.mu_u[0][0];
  double* const ta = &s.s_u[0][0];
#else
  double* const tb = &s.below[0][0];
  double* const ta = &s.above[0][0];
#endif
  const int errbits = interior ? lcpf_vertices<false>(s, p, tid, i0, j0, tb, ta)
                               : lcpf_vertices<true>(s, p, tid, i0, j0, tb, ta);
  __syncthreads();
  lcp_tile_cells<double, F::W, kLcpFY>(tb, ta, i0, j0, nx, ny, p.out_lcp);
  flush_error(p.err, errbits);
}

}  // namespace divuq
