// Fused Red Sea pipeline ("fusable into K3"):
//   members (u, v) -> |(u, v)|            velocity_magnitude  (gaussian.py:48-50)
//   -> gradient of the magnitude          gradient_ensemble   (gaussian.py:53-66,
//                                                              stencils.py:87-96)
//   -> ensemble moments of the gradient   fit_gaussian        (gaussian.py:35-45)
//   -> divergence mean and variance       propagate_divergence (divergence.py:48-70)
//   -> P(div > t), P(div < -t)            _tail_probs         (lcp.py:48-68)
// in ONE pass over the members.  The unfused chain writes the (M, 2, N)
// gradient ensemble and reads it back: 3x this kernel's HBM traffic.
//
// fp32 arithmetic identical, op for op, to gradient_ensemble2d_f32 followed
// by ensemble_divergence2d_f32 (hypot_<float>, the gradient's separately
// rounded products, shifted single-pass moments, StencilMath<float>,
// Tails<float>), so the fused result equals the composed one bit for bit.
//
// A CTA of 32 x 8 threads owns a 64 x 16 output tile and walks all members.
// Per member the (u, v) region with a 2-point halo (72 x 20) is staged in
// shared memory -- TMA (cp.async.bulk.tensor, S stages in flight, out-of-grid
// points zero-filled) when nx % 4 == 0, else plain loads of clamped
// coordinates one member ahead in registers -- turned into magnitudes in a
// double-buffered tile (one barrier per member), and every thread
// differentiates the gradient points it owns -- gx of its 4 outputs, gy of
// its 4 outputs, and one of the 160 halo points (gx one column left/right of
// the tile, gy one row above/below) -- into shifted moments.  After the last
// member the moments go to shared memory (aliasing the stages) and the
// divergence stencil + tails run on the tile.  Gradient points are evaluated
// at grid-clamped coordinates, so only in-grid region slots are ever read.
#pragma once

#include "common.cuh"
#include "gradient.cuh"
#include "tma.cuh"

#include <type_traits>

#ifndef DIVUQ_GF_MINB
#define DIVUQ_GF_MINB 4   // TMA variant (the register-staged one runs 2 CTAs / SM)
#endif
#ifndef DIVUQ_GF_MINB_LDG
#define DIVUQ_GF_MINB_LDG 2   // register-staged variant (nx % 4 != 0); 3 / 4 CTAs per SM measured equal / slower
#endif
#ifndef DIVUQ_GF_STAGES
#define DIVUQ_GF_STAGES 2   // 4 CTAs x 2 TMA stages: 8 members (92 KB) in flight per SM
#endif

namespace divuq {

#ifndef DIVUQ_GF_BY
#define DIVUQ_GF_BY 8
#endif
constexpr int kGfTX = 64, kGfBX = 32, kGfBY = DIVUQ_GF_BY, kGfTY = 2 * kGfBY, kGfThreads = kGfBX * kGfBY;
// staged region: 2-point halo, x extended to 4 left / 4 right so the TMA box
// starts on a 16-byte boundary (a start at x = i0 - 2 raises an illegal
// instruction on sm_100a: tools/gfprobe/tmabox.cu)
constexpr int kGfHX = 4, kGfHY = 2;
constexpr int kGfRW = kGfTX + 2 * kGfHX, kGfRH = kGfTY + 2 * kGfHY;
constexpr int kGfR = kGfRW * kGfRH;
constexpr int kGfNL = (kGfR + kGfThreads - 1) / kGfThreads;  // region slots per thread
constexpr int kGfHalo = 2 * kGfTY + 2 * kGfTX;               // halo gradient points
constexpr int kGfSlots = 9;                                  // 4 gx + 4 gy + 1 halo
constexpr int kGfS = DIVUQ_GF_STAGES;
constexpr uint32_t kGfCompBytes = ((kGfR * 4 + 127) / 128) * 128;   // one component, aligned
constexpr uint32_t kGfStageBytes = 2 * kGfCompBytes;
// the magnitude tile holds (hi, lo) pairs (mag_pair, gradient.cuh): one
// 8-byte load per differenced neighbour, double-buffered by member parity
// (a magnitude slot per thread and pass, kGfRP = kGfNL * threads >= kGfR: the
// region pass has no tail branch; the extra slots are never differenced)
constexpr int kGfRP = kGfNL * kGfThreads;
// the TMA path's last magnitude pass covers only the region's kGfR slots
// (warp-uniform: kGfR - (kGfNL-1) * threads is a multiple of 32), and only the
// first kGfHalo threads difference a halo slot -- no work on padding slots.
// (Skipping the region's two outer columns each side too -- they only pad the
// TMA box start to 16 bytes -- needs a per-thread slot table: 6 more
// registers, which spill at 64.)
static_assert((kGfR - (kGfNL - 1) * kGfThreads) % 32 == 0, "partial last pass is warp-uniform");
static_assert(kGfHalo % 32 == 0, "the halo gradient slot is warp-uniform");
constexpr uint32_t kGfMagOff = kGfS * kGfStageBytes;
constexpr uint32_t kGfMagBytes = 2 * kGfRP * 8;
constexpr uint32_t kGfBarOff = kGfMagOff + kGfMagBytes;
constexpr uint32_t kGfSmemTma = kGfBarOff + kGfS * 8;
constexpr uint32_t kGfMomBytes = 3 * (kGfTY * (kGfTX + 2) + (kGfTY + 2) * kGfTX) * 4;   // mu, sigma, r
static_assert(kGfMomBytes <= kGfS * kGfStageBytes + kGfMagBytes, "moments alias the stages + tile");
constexpr uint32_t kGfSmemLdg = kGfMagBytes > kGfMomBytes ? kGfMagBytes : kGfMomBytes;   // aliased

struct GfParams {
  const float* members;
  int64_t M, nx, ny;
  float cx_in, cx_bd, cy_in, cy_bd, theta;
  float *out_mu, *out_sigma, *out_psrc, *out_psnk, *out_mom_mu, *out_mom_sigma;
  int* err;
};

// gradient slot s of thread tid: axis and tile-local (row, column)
__device__ __forceinline__ void gf_slot(int s, int tid, bool& isx, int& r, int& c) {
  if (s < 8) {
    const int e = s & 3;
    isx = s < 4;
    r = (tid / kGfBX) + (e >> 1) * kGfBY;
    c = (tid % kGfBX) + (e & 1) * kGfBX;
  } else if (tid < 2 * kGfTY) {
    isx = true;
    r = tid % kGfTY;
    c = tid < kGfTY ? -1 : kGfTX;
  } else {
    const int h = min(tid, kGfHalo - 1) - 2 * kGfTY;
    isx = false;
    r = h < kGfTX ? -1 : kGfTY;
    c = h % kGfTX;
  }
}

template <bool TMA>
__global__ void __launch_bounds__(kGfThreads, TMA ? DIVUQ_GF_MINB : DIVUQ_GF_MINB_LDG)
gradfused_kernel(const __grid_constant__ CUtensorMap map, const GfParams p) {
  extern __shared__ __align__(128) unsigned char gf_smem[];
  const int64_t nx = p.nx, ny = p.ny, N = nx * ny;
  const int tid = threadIdx.y * kGfBX + threadIdx.x;
  const int64_t i0 = int64_t(blockIdx.x) * kGfTX, j0 = int64_t(blockIdx.y) * kGfTY;
  float2* mag = reinterpret_cast<float2*>(gf_smem + (TMA ? kGfMagOff : 0));
  float* mom = reinterpret_cast<float*>(gf_smem);   // after the last member: aliases stages / tile
  float* const mx_mu = mom;                                  // [kGfTY][kGfTX + 2]
  float* const mx_sg = mx_mu + kGfTY * (kGfTX + 2);
  float* const my_mu = mx_sg + kGfTY * (kGfTX + 2);          // [kGfTY + 2][kGfTX]
  float* const my_sg = my_mu + (kGfTY + 2) * kGfTX;
  float* const mx_r = my_sg + (kGfTY + 2) * kGfTX;            // the means' residuals
  float* const my_r = mx_r + kGfTY * (kGfTX + 2);
  uint64_t* full = reinterpret_cast<uint64_t*>(gf_smem + kGfBarOff);

  // the two differenced region slots and the coefficient of each gradient slot
  int g_hi[kGfSlots], g_lo[kGfSlots];
  float g_c[kGfSlots];
#pragma unroll
  for (int s = 0; s < kGfSlots; ++s) {
    bool isx;
    int r, c;
    gf_slot(s, tid, isx, r, c);
    const int64_t gi = min(max(i0 + c, int64_t(0)), nx - 1);
    const int64_t gj = min(max(j0 + r, int64_t(0)), ny - 1);
    const int rr = int(gj - j0) + kGfHY, rc = int(gi - i0) + kGfHX;
    if (isx) {
      g_hi[s] = rr * kGfRW + (gi < nx - 1 ? rc + 1 : rc);
      g_lo[s] = rr * kGfRW + (gi > 0 ? rc - 1 : rc);
      g_c[s] = (gi == 0 || gi == nx - 1) ? p.cx_bd : p.cx_in;
    } else {
      g_hi[s] = (gj < ny - 1 ? rr + 1 : rr) * kGfRW + rc;
      g_lo[s] = (gj > 0 ? rr - 1 : rr) * kGfRW + rc;
      g_c[s] = (gj == 0 || gj == ny - 1) ? p.cy_bd : p.cy_in;
    }
  }

  const int M = int(p.M);
  float a[kGfNL], b[kGfNL];
  int64_t ld_off[kGfNL];
  const bool last_pass = tid + (kGfNL - 1) * kGfThreads < kGfR;
  if constexpr (TMA) {
    if (tid == 0) {
      for (int s = 0; s < kGfS; ++s) mbar_init(&full[s], 1);
      mbar_fence_init();
      for (int s = 0; s < kGfS && s < M; ++s) {
        unsigned char* st = gf_smem + s * kGfStageBytes;
        mbar_expect_tx(&full[s], 2 * kGfR * 4);
        tma_load_3d(st, &map, &full[s], int(i0) - kGfHX, int(j0) - kGfHY, 2 * s);
        tma_load_3d(st + kGfCompBytes, &map, &full[s], int(i0) - kGfHX, int(j0) - kGfHY, 2 * s + 1);
      }
    }
    __syncthreads();
  } else {
#pragma unroll
    for (int k = 0; k < kGfNL; ++k) {
      const int q = min(tid + k * kGfThreads, kGfR - 1);
      const int qy = q / kGfRW, qx = q - qy * kGfRW;
      const int64_t gi = min(max(i0 + qx - kGfHX, int64_t(0)), nx - 1);
      const int64_t gj = min(max(j0 + qy - kGfHY, int64_t(0)), ny - 1);
      ld_off[k] = gj * nx + gi;
      a[k] = p.members[ld_off[k]];
      b[k] = p.members[N + ld_off[k]];
    }
  }

  ShiftedMoments<1> acc[kGfSlots];
  // non-finite input: u or v inf/NaN makes its magnitude pair NaN (mag_pair),
  // every gradient differencing it NaN, and so the divergence mean of some
  // in-grid output point (every grid point is a stencil neighbour of one) --
  // validated once per output instead of once per member and region point
  int errbits = 0;
  auto member = [&](int m, auto bufc, auto firstc) {
    constexpr int BUF = decltype(bufc)::value;
    constexpr bool FIRST = decltype(firstc)::value;
    float2* mg = mag + BUF * kGfRP;
    if constexpr (TMA) {
      const int st = m % kGfS;
      mbar_wait(&full[st], uint32_t(m / kGfS) & 1u);
      const float* su = reinterpret_cast<const float*>(gf_smem + st * kGfStageBytes);
      const float* sv = reinterpret_cast<const float*>(gf_smem + st * kGfStageBytes + kGfCompBytes);
#pragma unroll
      for (int k = 0; k < kGfNL; ++k) {
        if (k == kGfNL - 1 && !last_pass) break;
        const int q = tid + k * kGfThreads;
        float h, l;
        mag_pair(su[q], sv[q], h, l);
        mg[q] = make_float2(h, l);
      }
      __syncthreads();   // stage st consumed by every thread: refill it
      if (tid == 0 && m + kGfS < M) {
        unsigned char* sp = gf_smem + st * kGfStageBytes;
        mbar_expect_tx(&full[st], 2 * kGfR * 4);
        tma_load_3d(sp, &map, &full[st], int(i0) - kGfHX, int(j0) - kGfHY, 2 * (m + kGfS));
        tma_load_3d(sp + kGfCompBytes, &map, &full[st], int(i0) - kGfHX, int(j0) - kGfHY,
                    2 * (m + kGfS) + 1);
      }
    } else {
#pragma unroll
      for (int k = 0; k < kGfNL; ++k) {
        const int q = tid + k * kGfThreads;
        float h, l;
        mag_pair(a[k], b[k], h, l);
        mg[q] = make_float2(h, l);
      }
      if (m + 1 < M) {   // next member's loads in flight across the barrier and the math
        const float* src = p.members + int64_t(m + 1) * 2 * N;
#pragma unroll
        for (int k = 0; k < kGfNL; ++k) {
          a[k] = src[ld_off[k]];
          b[k] = src[N + ld_off[k]];
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int s = 0; s < kGfSlots; ++s) {
      if (s == kGfSlots - 1 && tid >= kGfHalo) break;   // halo slot: the first kGfHalo threads
      float hh, hl, lh, ll;   // (hi, lo) of the high and the low neighbour
      // plain shared loads (volatile asm measured the same: 61.9 vs 62.1 us);
      // BUF folds into the load's immediate offset
      const float2 ph = mg[g_hi[s]], pl = mg[g_lo[s]];
      hh = ph.x; hl = ph.y; lh = pl.x; ll = pl.y;
      const float g = grad_diff_pair(hh, lh, hl, ll, g_c[s]);   // stencils.py:87-96
      acc[s].add(FIRST ? 0 : 1, &g);   // member 0 sets the shift
    }
  };
  using B0 = std::integral_constant<int, 0>;
  using B1 = std::integral_constant<int, 1>;
  using NotFirst = std::false_type;
  member(0, B0{}, std::true_type{});
  int m = 1;
  for (; m + 1 < M; m += 2) {
    member(m, B1{}, NotFirst{});
    member(m + 1, B0{}, NotFirst{});
  }
  if (m < M) member(m, B1{}, NotFirst{});
  __syncthreads();   // the moments alias the stages and the magnitude tile
  float g_mu[kGfSlots], g_sg[kGfSlots];
#pragma unroll
  for (int s = 0; s < kGfSlots; ++s) {
    float g_r;
    acc[s].finish(M, &g_mu[s], &g_r, &g_sg[s]);
    bool isx;
    int r, c;
    gf_slot(s, tid, isx, r, c);
    if (s < 8 || tid < kGfHalo) {
      const int d = isx ? r * (kGfTX + 2) + c + 1 : (r + 1) * kGfTX + c;
      (isx ? mx_mu : my_mu)[d] = g_mu[s];
      (isx ? mx_sg : my_sg)[d] = g_sg[s];
      (isx ? mx_r : my_r)[d] = g_r;
    }
  }
  __syncthreads();
  using SM = StencilMath<float, true>;
  const bool t_zero = p.theta == 0.0f;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int r = threadIdx.y + (e >> 1) * kGfBY, c = threadIdx.x + (e & 1) * kGfBX;
    const int64_t i = i0 + c, j = j0 + r;
    if (i >= nx || j >= ny) continue;
    const int xh = r * (kGfTX + 2) + (i < nx - 1 ? c + 1 : c) + 1;
    const int xl = r * (kGfTX + 2) + (i > 0 ? c - 1 : c) + 1;
    const int yh = ((j < ny - 1 ? r + 1 : r) + 1) * kGfTX + c;
    const int yl = ((j > 0 ? r - 1 : r) + 1) * kGfTX + c;
    const float cxe = (i == 0 || i == nx - 1) ? p.cx_bd : p.cx_in;
    const float cye = (j == 0 || j == ny - 1) ? p.cy_bd : p.cy_in;
    const float mean = SM::mean_r(mx_mu[xh], mx_mu[xl], mx_r[xh], mx_r[xl], my_mu[yh], my_mu[yl],
                                  my_r[yh], my_r[yl], 0.0f, 0.0f, 0.0f, 0.0f, cxe, cye, 0.0f);
    const float var = SM::var(mx_sg[xh], mx_sg[xl], my_sg[yh], my_sg[yl], 0.0f, 0.0f, cxe, cye, 0.0f);
    errbits |= check_value(mean);
    float sg, ps, pk;
    Tails<float>::eval(mean, var, p.theta, t_zero, sg, ps, pk);
    const int64_t o = j * nx + i;
    if (p.out_mu) p.out_mu[o] = mean;
    if (p.out_sigma) p.out_sigma[o] = sg;
    if (p.out_psrc) p.out_psrc[o] = ps;
    if (p.out_psnk) p.out_psnk[o] = pk;
    if (p.out_mom_mu) {
      p.out_mom_mu[o] = g_mu[e];
      p.out_mom_mu[N + o] = g_mu[4 + e];
      p.out_mom_sigma[o] = g_sg[e];
      p.out_mom_sigma[N + o] = g_sg[4 + e];
    }
  }
  flush_error(p.err, errbits);
}

}  // namespace divuq
