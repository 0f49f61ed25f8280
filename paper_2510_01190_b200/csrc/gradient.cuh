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
#include "tma.cuh"

namespace divuq {

template <typename T> __device__ __forceinline__ T hypot_(T a, T b);
template <> __device__ __forceinline__ double hypot_(double a, double b) { return hypot(a, b); }
// fp32 (1e-5 bar): sqrt(a^2 + b^2) as r * rsqrt(r) -- 5 instructions instead
// of hypotf's ~25 with its scaling branches; |err| ~2 ulp.  No overflow guard:
// |a|, |b| must stay below ~1.8e19 (velocities).  r < FLT_MIN (|v| < 1.1e-19)
// evaluates to <= 1.1e-19 instead of sqrt(r).
__device__ __forceinline__ float sqrt_of_sq(float r) {   // r = a^2 + b^2 >= 0
  return r * rsqrt_approx(fmaxf(r, 1.17549435e-38f));
}
template <> __device__ __forceinline__ float hypot_(float a, float b) {
  return sqrt_of_sq(fmaf(a, a, b * b));
}

// fp32 magnitude as a (hi, lo) pair.  Differencing fp32-rounded magnitudes
// loses ~ulp(|v|) per member (|v| ~ 110 at the config-1 vortex against
// gradient noise ~0.01), which moved the Red Sea chain's P maps by ~1e-4;
// with the pair the gradient is c * ((H.hi - L.hi) + (H.lo - L.lo)) and the
// chain meets the fp32 probability bar against the fp64 oracle.
//   s = u^2 + v^2 with its exact rounding errors (two FMA products, Fast2Sum),
//   hi = s * rsqrt(s), lo2 = 2 * lo = (s + err - hi^2) / hi  (kept doubled:
//   one multiply fewer; grad_diff_pair halves the difference exactly).
// A non-finite u or v makes lo2 NaN (fma(u, u, -u*u) is NaN for u = inf, and
// the error terms keep a NaN that fmax / fmin would drop).
__device__ __forceinline__ void mag_pair(float u, float v, float& hi, float& lo2) {
  const float p1 = __fmul_rn(u, u), p2 = __fmul_rn(v, v);
  const float e1 = fmaf(u, u, -p1), e2 = fmaf(v, v, -p2);
  const float a = fmaxf(p1, p2), b = fminf(p1, p2);
  const float s = __fadd_rn(a, b);
  const float es = __fsub_rn(b, __fsub_rn(s, a));   // Fast2Sum (a >= b >= 0): exact
  const float rs = rsqrt_approx(fmaxf(s, 1.17549435e-38f));
  hi = __fmul_rn(s, rs);
  const float E = __fadd_rn(fmaf(-hi, hi, s), __fadd_rn(es, __fadd_rn(e1, e2)));
  lo2 = __fmul_rn(E, rs);
}
// c * ((h_hi - l_hi) + (h_lo2 - l_lo2) / 2): the half is exact, one rounding
__device__ __forceinline__ float grad_diff_pair(float h_hi, float l_hi, float h_lo2, float l_lo2, float c) {
  return __fmul_rn(c, fmaf(0.5f, __fsub_rn(h_lo2, l_lo2), __fsub_rn(h_hi, l_hi)));
}

// one gradient component, stencils.py:87-96.  fp64: f[hi]*c - f[lo]*c with
// each product rounded (the reference's order, bitwise).  fp32 (1e-5 bar):
// c*(f[hi] - f[lo]), one rounding fewer and one instruction fewer.
__device__ __forceinline__ double grad_diff(double hi, double lo, double c) {
  return __dsub_rn(__dmul_rn(hi, c), __dmul_rn(lo, c));
}
__device__ __forceinline__ float grad_diff(float hi, float lo, float c) {
  return __fmul_rn(c, __fsub_rn(hi, lo));
}

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
// A CTA of 32 x 8 threads owns a 64 x 16 tile (2 x 2 points per thread) and
// walks several members of it: every index (the clamped tile + one-point halo
// load offsets, the output offsets, coefficients and neighbour slots) is
// member-invariant and computed once, so the member loop is loads, one
// magnitude per loaded point into shared memory (halo re-reads, 16 %, hit
// L2), then the one-axis differences and two stores per point.
// planes: `members` blocks of (u[, v]) with stride in_mstride; outputs
// (gx, gy) per member.
constexpr int kGrTX = 64, kGrTY = 16, kGrBX = 32, kGrBY = 8;
constexpr int kGrV = (kGrTX + 2) * (kGrTY + 2);
constexpr int kGrNQ = (kGrV + kGrBX * kGrBY - 1) / (kGrBX * kGrBY);
constexpr int kGrPY = kGrTY / kGrBY, kGrPX = kGrTX / kGrBX;   // points per thread
constexpr int64_t kGrMembersPerCta = 8;   // members a CTA walks (sweep: 1 2 4 8 20 -> 171 155 146 142 155 us)

template <typename T, bool MAG>
__global__ void __launch_bounds__(kGrBX * kGrBY, 3)
gradient2d_kernel(const T* __restrict__ in, int64_t members, int64_t in_mstride, int64_t nx,
                  int64_t ny, T cx_in, T cx_bd, T cy_in, T cy_bd, T* __restrict__ out,
                  int64_t out_mstride, int* err) {
  constexpr bool PAIR = MAG && sizeof(T) == 4;   // fp32 magnitudes as (hi, lo) pairs
  __shared__ T f[kGrTY + 2][kGrTX + 2];
  __shared__ T flo_[PAIR ? kGrTY + 2 : 1][PAIR ? kGrTX + 2 : 1];
  T* const fl = &f[0][0];
  T* const flo = &flo_[0][0];
  const int64_t n = nx * ny;
  const int tid = threadIdx.y * kGrBX + threadIdx.x;
  const int64_t i0 = int64_t(blockIdx.x) * kGrTX, j0 = int64_t(blockIdx.y) * kGrTY;
  // (tile + halo) load slots with clamped coordinates: a clamped slot is only
  // read as the one-sided boundary neighbour, which IS the clamped point
  int64_t ld_off[kGrNQ];
  bool ld_st[kGrNQ];
#pragma unroll
  for (int k = 0; k < kGrNQ; ++k) {
    const int q = min(tid + k * kGrBX * kGrBY, kGrV - 1);
    const int qy = q / (kGrTX + 2), qx = q - qy * (kGrTX + 2);
    const int64_t gi = min(max(i0 + qx - 1, int64_t(0)), nx - 1);
    const int64_t gj = min(max(j0 + qy - 1, int64_t(0)), ny - 1);
    ld_off[k] = gj * nx + gi;
    ld_st[k] = tid + k * kGrBX * kGrBY < kGrV;
  }
  // this thread's points: output offset (-1: outside), coefficients, slots
  int64_t o_off[kGrPY * kGrPX];
  T o_cx[kGrPY * kGrPX], o_cy[kGrPY * kGrPX];
  int o_xh[kGrPY * kGrPX], o_xl[kGrPY * kGrPX], o_yh[kGrPY * kGrPX], o_yl[kGrPY * kGrPX];
#pragma unroll
  for (int py = 0; py < kGrPY; ++py)
#pragma unroll
    for (int px = 0; px < kGrPX; ++px) {
      const int e = py * kGrPX + px;
      const int64_t i = i0 + threadIdx.x + px * kGrBX, j = j0 + threadIdx.y + py * kGrBY;
      const int x = threadIdx.x + px * kGrBX + 1, y = threadIdx.y + py * kGrBY + 1;
      const bool bx = i == 0 || i == nx - 1, by = j == 0 || j == ny - 1;
      o_off[e] = (i < nx && j < ny) ? j * nx + i : -1;
      o_cx[e] = bx ? cx_bd : cx_in;
      o_cy[e] = by ? cy_bd : cy_in;
      const int w = kGrTX + 2;
      o_xh[e] = y * w + (i < nx - 1 ? x + 1 : x);
      o_xl[e] = y * w + (i > 0 ? x - 1 : x);
      o_yh[e] = (j < ny - 1 ? y + 1 : y) * w + x;
      o_yl[e] = (j > 0 ? y - 1 : y) * w + x;
    }
  int errbits = 0;
  for (int64_t m = blockIdx.z; m < members; m += gridDim.z) {
    const T* src = in + m * in_mstride;
    T a[kGrNQ], b[kGrNQ];
#pragma unroll
    for (int k = 0; k < kGrNQ; ++k) {   // all of a thread's loads in flight at once
      a[k] = src[ld_off[k]];
      if constexpr (MAG) b[k] = src[n + ld_off[k]];
    }
#pragma unroll
    for (int k = 0; k < kGrNQ; ++k) {
      if (ld_st[k]) {
        if constexpr (PAIR) {
          float h, l;
          mag_pair(a[k], b[k], h, l);
          fl[tid + k * kGrBX * kGrBY] = h;
          flo[tid + k * kGrBX * kGrBY] = l;
        } else {
          fl[tid + k * kGrBX * kGrBY] = MAG ? hypot_(a[k], b[k]) : a[k];
        }
      }
      errbits |= check_value(a[k]);
      if constexpr (MAG) errbits |= check_value(b[k]);
    }
    __syncthreads();
    T* dst = out + m * out_mstride;
#pragma unroll
    for (int e = 0; e < kGrPY * kGrPX; ++e) {
      if (o_off[e] < 0) continue;
      if constexpr (PAIR) {
        dst[o_off[e]] = grad_diff_pair(fl[o_xh[e]], fl[o_xl[e]], flo[o_xh[e]], flo[o_xl[e]], o_cx[e]);
        dst[n + o_off[e]] = grad_diff_pair(fl[o_yh[e]], fl[o_yl[e]], flo[o_yh[e]], flo[o_yl[e]], o_cy[e]);
      } else {
        dst[o_off[e]] = grad_diff(fl[o_xh[e]], fl[o_xl[e]], o_cx[e]);
        dst[n + o_off[e]] = grad_diff(fl[o_yh[e]], fl[o_yl[e]], o_cy[e]);
      }
    }
    __syncthreads();
  }
  flush_error(err, errbits);
}

// gradient_ensemble, TMA-staged (nx * sizeof(T) % 16 == 0): a CTA owns a
// 64 x 16 tile and walks its members; each member's (u, v) region (x-halo of
// 16 bytes -- a TMA box must start on a 16-byte boundary -- and a 1-row
// y-halo) arrives by cp.async.bulk.tensor into one of S stages, so S members
// are in flight while the CTA differentiates the current one (the
// register-loaded kernel above only has a member's loads in flight during
// its load phase: 70 % of HBM).  Magnitudes go to a double-buffered tile,
// one barrier per member; same arithmetic as gradient2d_kernel.
template <typename T>
struct GrTma {
  static constexpr int HX = 16 / int(sizeof(T)), HY = 1;
  static constexpr int RW = kGrTX + 2 * HX, RH = kGrTY + 2 * HY, R = RW * RH;
  static constexpr int NL = (R + kGrBX * kGrBY - 1) / (kGrBX * kGrBY);
  static constexpr int S = 4;
  static constexpr uint32_t COMP = ((R * sizeof(T) + 127) / 128) * 128;
  static constexpr uint32_t STAGE = 2 * COMP;
  static constexpr uint32_t MAG = S * STAGE;
  static constexpr uint32_t LO = MAG + 2 * R * sizeof(T);      // fp32: the pairs' lo parts
  static constexpr uint32_t BAR = LO + (sizeof(T) == 4 ? 2 * R * sizeof(T) : 0);
  static constexpr uint32_t SMEM = BAR + S * 8;
  static constexpr int MINB = sizeof(T) == 8 ? 2 : 4;
};

template <typename T>
__global__ void __launch_bounds__(kGrBX * kGrBY, GrTma<T>::MINB)
gradient_tma_kernel(const __grid_constant__ CUtensorMap map, int64_t members, int64_t nx, int64_t ny,
                    T cx_in, T cx_bd, T cy_in, T cy_bd, T* __restrict__ out, int64_t out_mstride,
                    int* err) {
  using G = GrTma<T>;
  extern __shared__ __align__(128) unsigned char gr_smem[];
  constexpr bool PAIR = sizeof(T) == 4;
  T* const mag = reinterpret_cast<T*>(gr_smem + G::MAG);
  T* const mlo = reinterpret_cast<T*>(gr_smem + G::LO);
  uint64_t* const full = reinterpret_cast<uint64_t*>(gr_smem + G::BAR);
  const int tid = threadIdx.y * kGrBX + threadIdx.x;
  const int64_t n = nx * ny;
  const int64_t i0 = int64_t(blockIdx.x) * kGrTX, j0 = int64_t(blockIdx.y) * kGrTY;
  // this CTA's members: blockIdx.z, blockIdx.z + gridDim.z, ...
  const int64_t cnt = blockIdx.z < members ? (members - blockIdx.z + gridDim.z - 1) / gridDim.z : 0;
  auto issue = [&](int64_t k, int st) {
    const int64_t m = blockIdx.z + k * gridDim.z;
    unsigned char* dst = gr_smem + st * G::STAGE;
    mbar_expect_tx(&full[st], 2 * G::R * sizeof(T));
    tma_load_3d(dst, &map, &full[st], int(i0) - G::HX, int(j0) - G::HY, int(2 * m));
    tma_load_3d(dst + G::COMP, &map, &full[st], int(i0) - G::HX, int(j0) - G::HY, int(2 * m + 1));
  };
  if (tid == 0) {
    for (int st = 0; st < G::S; ++st) mbar_init(&full[st], 1);
    mbar_fence_init();
    for (int st = 0; st < G::S && st < cnt; ++st) issue(st, st);
  }
  // this thread's points: output offset (-1: outside), coefficients, slots
  int64_t o_off[kGrPY * kGrPX];
  T o_cx[kGrPY * kGrPX], o_cy[kGrPY * kGrPX];
  int o_xh[kGrPY * kGrPX], o_xl[kGrPY * kGrPX], o_yh[kGrPY * kGrPX], o_yl[kGrPY * kGrPX];
#pragma unroll
  for (int e = 0; e < kGrPY * kGrPX; ++e) {
    const int py = e / kGrPX, px = e % kGrPX;
    const int64_t i = i0 + threadIdx.x + px * kGrBX, j = j0 + threadIdx.y + py * kGrBY;
    const int64_t gi = min(i, nx - 1), gj = min(j, ny - 1);
    const int x = int(gi - i0) + G::HX, y = int(gj - j0) + G::HY;
    o_off[e] = (i < nx && j < ny) ? j * nx + i : -1;
    o_cx[e] = (gi == 0 || gi == nx - 1) ? cx_bd : cx_in;
    o_cy[e] = (gj == 0 || gj == ny - 1) ? cy_bd : cy_in;
    o_xh[e] = y * G::RW + (gi < nx - 1 ? x + 1 : x);
    o_xl[e] = y * G::RW + (gi > 0 ? x - 1 : x);
    o_yh[e] = (gj < ny - 1 ? y + 1 : y) * G::RW + x;
    o_yl[e] = (gj > 0 ? y - 1 : y) * G::RW + x;
  }
  __syncthreads();
  int errbits = 0;
  for (int64_t k = 0; k < cnt; ++k) {
    const int st = int(k % G::S);
    mbar_wait(&full[st], uint32_t(k / G::S) & 1u);
    const T* su = reinterpret_cast<const T*>(gr_smem + st * G::STAGE);
    const T* sv = reinterpret_cast<const T*>(gr_smem + st * G::STAGE + G::COMP);
    T* const fl = mag + (k & 1) * G::R;
    T* const flo = mlo + (k & 1) * G::R;
#pragma unroll
    for (int q0 = 0; q0 < G::NL; ++q0) {
      const int q = tid + q0 * kGrBX * kGrBY;
      if (q0 < G::NL - 1 || q < G::R) {
        const T u = su[q], v = sv[q];
        errbits |= check_value(u) | check_value(v);
        if constexpr (PAIR) {
          float h, l;
          mag_pair(u, v, h, l);
          fl[q] = h;
          flo[q] = l;
        } else {
          fl[q] = hypot_(u, v);
        }
      }
    }
    __syncthreads();   // stage st consumed by every thread: refill it
    if (tid == 0 && k + G::S < cnt) issue(k + G::S, st);
    T* dst = out + (blockIdx.z + k * gridDim.z) * out_mstride;
#pragma unroll
    for (int e = 0; e < kGrPY * kGrPX; ++e) {
      if (o_off[e] < 0) continue;
      if constexpr (PAIR) {
        dst[o_off[e]] = grad_diff_pair(fl[o_xh[e]], fl[o_xl[e]], flo[o_xh[e]], flo[o_xl[e]], o_cx[e]);
        dst[n + o_off[e]] = grad_diff_pair(fl[o_yh[e]], fl[o_yl[e]], flo[o_yh[e]], flo[o_yl[e]], o_cy[e]);
      } else {
        dst[o_off[e]] = grad_diff(fl[o_xh[e]], fl[o_xl[e]], o_cx[e]);
        dst[n + o_off[e]] = grad_diff(fl[o_yh[e]], fl[o_yl[e]], o_cy[e]);
      }
    }
  }
  flush_error(err, errbits);
}

}  // namespace divuq
