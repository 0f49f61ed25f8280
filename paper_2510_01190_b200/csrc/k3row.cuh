// K3 for 2D ensembles as a ROW MARCH (BASELINE config 1).
//
// fit_gaussian (gaussian.py:35-45) -> propagate_divergence (divergence.py:
// 48-70) -> tails (lcp.py:48-68) on an (M, 2, ny*nx) fp32 member array, one
// pass over the members.  The tiled K3 (k3tma.cuh) treats a 2D grid as single
// planes: every tile is a short 10-item burst followed by an epilogue and a
// barrier, and it stays near 62 % of HBM.  Here a CTA owns a TX-column strip
// (TX = 32 * VEC = 64) and a run of rows and marches down the rows the way
// K2/K3 march z:
//
//   * the producer warp streams one ROW per stage: the M u-rows of the strip
//     WITH their 4-column x-halos (one 5D TMA box of TX + 8 columns) and the
//     M v-rows (box of TX columns); the run is padded by one halo row on each
//     side, so no halo boxes and no neighbour CTA timing are involved;
//   * NW consumer warps take rows round-robin in groups of NW: a warp folds
//     its row's members into single-pass shifted moments (ShiftedMoments, the
//     same routine as K1 / K3, so results are bitwise those of K1 + K2),
//     releases the stage at once and publishes (mu_u, r_u, s_u, mu_v, r_v,
//     s_v) of its TX points (+ the two x-halo points) in a shared ring of
//     2*NW + 2 rows (r = the mean's rounding residual, see ShiftedMoments);
//   * one named barrier per group; then each warp evaluates the stencil,
//     sigma and both tails for the row BEFORE its own (whose v neighbours
//     are now both in the ring) and streams the outputs;
//   * boundaries by operand substitution (the one-sided rule of
//     stencils.py:46-51 at the global edges only), no divergent slow path.
#pragma once

#include "common.cuh"
#include "tma.cuh"

namespace divuq {

// 2 CTAs x 8 consumer warps per SM: 37.6 us at config 1 vs 42.4 for 1 x 10
// (tools/sweep_c1.py over tools/variants builds; the small-problem floor of a
// perfect stream of the same bytes is 36.1 us, profiles/r01/bwbench.txt)
#ifndef DIVUQ_RM_NW
#define DIVUQ_RM_NW 8
#endif
#ifndef DIVUQ_RM_MINB
#define DIVUQ_RM_MINB 2
#endif
#ifndef DIVUQ_RM_VEC
#define DIVUQ_RM_VEC 2
#endif
struct RmCfg {
  static constexpr int VEC = DIVUQ_RM_VEC;       // points per lane
  static constexpr int TX = 32 * VEC, PAD = 4, TXP = TX + 2 * PAD;
  static constexpr int NW = DIVUQ_RM_NW;        // consumer warps
  static constexpr int THREADS = 32 * (NW + 1); // + producer warp
  static constexpr int R = 2 * NW + 2;          // moment ring rows
  static constexpr int SMAX = 16;               // stages (runtime S <= SMAX)
};

struct RmMaps {
  CUtensorMap u;   // box {TXP, 1, 1, 1, M} at (x0 - PAD, row, 0, comp u, 0)
  CUtensorMap v;   // box {TX, 1, 1, 1, M}  at (x0, row, 0, comp v, 0)
};

struct RmParams {
  int nx, ny, M, strips, seg_rows, S;
  uint32_t stage_bytes, stage_stride, v_off;   // TMA bytes per stage; smem layout
  float cx_in, cx_bd, cy_in, cy_bd, theta;
  float *out_mu, *out_sigma, *out_psrc, *out_psnk, *out_mom_mu, *out_mom_sigma;
  int* err;
};

// per ring row: mu_u, s_u, mu_v, s_v of the TX points, their residuals
// (r_u, r_v) packed as bf16x2 (keeps 2 CTAs x 8 stages per SM), then the
// x-halo points' (mu_u, s_u) left, right and their r_u
enum { kRmU = 0, kRmSU = 1, kRmV = 2, kRmSV = 3 };
struct RmRing {
  float m[RmCfg::R][4][RmCfg::TX];
  uint32_t r[RmCfg::R][RmCfg::TX];
  float h[RmCfg::R][6];
};

__global__ void __launch_bounds__(RmCfg::THREADS, DIVUQ_RM_MINB)
k3_rowmarch_kernel(const __grid_constant__ RmMaps tm, const RmParams p) {
  using C = RmCfg;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  RmRing& ring = *reinterpret_cast<RmRing*>(smem_raw);
  unsigned char* stages = smem_raw + ((sizeof(RmRing) + 1023) / 1024) * 1024;
  uint64_t* full = reinterpret_cast<uint64_t*>(stages + size_t(p.S) * p.stage_stride);
  uint64_t* empty = full + C::SMAX;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int strip = blockIdx.x % p.strips, seg = blockIdx.x / p.strips;
  const int x0 = strip * C::TX;
  const int y0 = seg * p.seg_rows, y1 = min(p.ny, y0 + p.seg_rows);
  const int nrows = (y1 - y0) + 2;   // + one halo row on each side (row index i -> y0 - 1 + i)

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);   // each stage is one row, consumed by one warp
    }
    mbar_fence_init();
  }
  if (warp == C::NW && lane < 2) tma_prefetch_desc(lane ? &tm.v : &tm.u);
  __syncthreads();

  if (warp == C::NW) {   // ------------------------------------------------ producer
    if (lane != 0) return;
    for (int i = 0; i < nrows; ++i) {
      const int s = i % p.S;
      const uint32_t ph = uint32_t(i / p.S) & 1u;
      mbar_wait_backoff<32>(&empty[s], ph ^ 1u);
      mbar_expect_tx(&full[s], p.stage_bytes);
      unsigned char* st = stages + size_t(s) * p.stage_stride;
      const int row = y0 - 1 + i;   // rows -1 and ny are zero-filled (never used)
      tma_load_5d(st, &tm.u, &full[s], x0 - C::PAD, row, 0, 0, 0);
      tma_load_5d(st + p.v_off, &tm.v, &full[s], x0, row, 0, 1, 0);
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int M = p.M;
  const int64_t N = int64_t(p.nx) * p.ny;
  const int cx0 = lane * C::VEC;
  const int xi = x0 + cx0;
  const bool act_x = xi < p.nx;
  const bool x_lo_edge = xi == 0, x_hi_edge = xi + C::VEC == p.nx;
  const float cx_first = x_lo_edge ? p.cx_bd : p.cx_in;
  const float cx_last = x_hi_edge ? p.cx_bd : p.cx_in;
  const bool t_zero = p.theta == 0.0f;
  const bool validate = p.err != nullptr;
  // every lane also folds one x-halo point (uniform work): lane 0 the left
  // one, the others the right one (published by lane 31)
  const int hcol = lane == 0 ? C::PAD - 1 : C::PAD + C::TX;
  int errbits = 0;
  const int groups = (nrows + C::NW - 1) / C::NW;
  for (int g = 0; g < groups; ++g) {
    const int i = g * C::NW + warp;   // this warp's row in the march
    if (i < nrows) {                  // phase A: moments of row i
      const int s = i % p.S;
      mbar_wait(&full[s], uint32_t(i / p.S) & 1u);
      const float* su = reinterpret_cast<const float*>(stages + size_t(s) * p.stage_stride);
      const float* sv = reinterpret_cast<const float*>(stages + size_t(s) * p.stage_stride + p.v_off);
      ShiftedMoments<C::VEC> au, av;
      ShiftedMoments<1> ah;
      const int row = y0 - 1 + i;
      const bool owned = i >= 1 && i <= nrows - 2;
      auto load = [&](int m, Vec<float, C::VEC>& xu, Vec<float, C::VEC>& xv, float& xh) {
        xu = *reinterpret_cast<const Vec<float, C::VEC>*>(su + m * C::TXP + C::PAD + cx0);
        xv = *reinterpret_cast<const Vec<float, C::VEC>*>(sv + m * C::TX + cx0);
        xh = su[m * C::TXP + hcol];
        if (validate && owned && act_x) {
#pragma unroll
          for (int e = 0; e < C::VEC; ++e) errbits |= check_value(xu.v[e]) | check_value(xv.v[e]);
        }
      };
      {  // member 0 sets the shift (peeled: no per-member branch)
        Vec<float, C::VEC> xu, xv;
        float xh;
        load(0, xu, xv, xh);
        au.first(xu.v);
        av.first(xv.v);
        ah.first(&xh);
      }
      for (int m = 1; m < M; ++m) {
        Vec<float, C::VEC> xu, xv;
        float xh;
        load(m, xu, xv, xh);
        au.next(xu.v);
        av.next(xv.v);
        ah.next(&xh);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);   // the stage can be refilled now
      Vec<float, C::VEC> mu_u, s_u, mu_v, s_v, r_u, r_v;
      au.finish(M, mu_u.v, r_u.v, s_u.v);
      av.finish(M, mu_v.v, r_v.v, s_v.v);
      float hmu, hsg, hr;
      ah.finish(M, &hmu, &hr, &hsg);
      const int q = i % C::R;
      *reinterpret_cast<Vec<float, C::VEC>*>(&ring.m[q][kRmU][cx0]) = mu_u;
      *reinterpret_cast<Vec<float, C::VEC>*>(&ring.m[q][kRmSU][cx0]) = s_u;
      *reinterpret_cast<Vec<float, C::VEC>*>(&ring.m[q][kRmV][cx0]) = mu_v;
      *reinterpret_cast<Vec<float, C::VEC>*>(&ring.m[q][kRmSV][cx0]) = s_v;
      {
        Vec<uint32_t, C::VEC> pr;
#pragma unroll
        for (int e = 0; e < C::VEC; ++e) pr.v[e] = pack_bf16x2(r_u.v[e], r_v.v[e]);
        *reinterpret_cast<Vec<uint32_t, C::VEC>*>(&ring.r[q][cx0]) = pr;
      }
      if (lane == 0) { ring.h[q][0] = hmu; ring.h[q][1] = hsg; ring.h[q][4] = hr; }
      if (lane == 31) { ring.h[q][2] = hmu; ring.h[q][3] = hsg; ring.h[q][5] = hr; }
      (void)row;
    }
    named_sync(1, 32 * C::NW);   // the group's rows are in the ring
    // phase B: the stencil of row j = i - 1 (its v neighbours i - 2, i are in)
    const int j = i - 1;
    if (j >= 1 && j <= nrows - 2 && act_x) {
      const int row = y0 - 1 + j;
      const int q = j % C::R, ql = (j - 1) % C::R, qh = (j + 1) % C::R;
      const bool jlo = row == 0, jhi = row == p.ny - 1;
      const float cy = (jlo || jhi) ? p.cy_bd : p.cy_in;
      using V = Vec<float, C::VEC>;
      const V mu_u = *reinterpret_cast<const V*>(&ring.m[q][kRmU][cx0]);
      const V s_u = *reinterpret_cast<const V*>(&ring.m[q][kRmSU][cx0]);
      using VU = Vec<uint32_t, C::VEC>;
      const VU pr = *reinterpret_cast<const VU*>(&ring.r[q][cx0]);
      // v rows below / above (the point itself at the global y faces)
      const int qlo = jlo ? q : ql, qhi = jhi ? q : qh;
      const V vl = *reinterpret_cast<const V*>(&ring.m[qlo][kRmV][cx0]);
      const V svl = *reinterpret_cast<const V*>(&ring.m[qlo][kRmSV][cx0]);
      const VU prl = *reinterpret_cast<const VU*>(&ring.r[qlo][cx0]);
      const V vh = *reinterpret_cast<const V*>(&ring.m[qhi][kRmV][cx0]);
      const V svh = *reinterpret_cast<const V*>(&ring.m[qhi][kRmSV][cx0]);
      const VU prh = *reinterpret_cast<const VU*>(&ring.r[qhi][cx0]);
      V r_u;
#pragma unroll
      for (int e = 0; e < C::VEC; ++e) r_u.v[e] = unpack_bf16_lo(pr.v[e]);
      // u x-neighbours of the lane's edge points: neighbour lanes or the halo points
      const int cr = cx0 + C::VEC < C::TX ? cx0 + C::VEC : cx0;
      float ul = lane == 0 ? ring.h[q][0] : ring.m[q][kRmU][cx0 - 1];
      float sl = lane == 0 ? ring.h[q][1] : ring.m[q][kRmSU][cx0 - 1];
      float rl = lane == 0 ? ring.h[q][4] : unpack_bf16_lo(ring.r[q][cx0 - 1]);
      float ur = lane == 31 ? ring.h[q][2] : ring.m[q][kRmU][cr];
      float sr = lane == 31 ? ring.h[q][3] : ring.m[q][kRmSU][cr];
      float rr = lane == 31 ? ring.h[q][5] : unpack_bf16_lo(ring.r[q][cr]);
      if (x_lo_edge) { ul = mu_u.v[0]; sl = s_u.v[0]; rl = r_u.v[0]; }
      if (x_hi_edge) { ur = mu_u.v[C::VEC - 1]; sr = s_u.v[C::VEC - 1]; rr = r_u.v[C::VEC - 1]; }
      Vec<float, C::VEC> omu, osg, ops, opk;
      // with VEC = 2 and nx = 2 one lane holds both x edges: cx_first/last cover it
      using SM = StencilMath<float, true>;
#pragma unroll
      for (int e = 0; e < C::VEC; ++e) {
        constexpr int L = C::VEC - 1;
        const float cxe = e == 0 ? cx_first : (e == L ? cx_last : p.cx_in);
        const float uL = e == 0 ? ul : mu_u.v[e == 0 ? 0 : e - 1];
        const float uH = e == L ? ur : mu_u.v[e == L ? 0 : e + 1];
        const float sL = e == 0 ? sl : s_u.v[e == 0 ? 0 : e - 1];
        const float sH = e == L ? sr : s_u.v[e == L ? 0 : e + 1];
        const float rL = e == 0 ? rl : r_u.v[e == 0 ? 0 : e - 1];
        const float rH = e == L ? rr : r_u.v[e == L ? 0 : e + 1];
        const float m = SM::mean_r(uH, uL, rH, rL, vh.v[e], vl.v[e], unpack_bf16_hi(prh.v[e]), unpack_bf16_hi(prl.v[e]), 0.0f, 0.0f,
                                   0.0f, 0.0f, cxe, cy, 0.0f);
        omu.v[e] = m;
        Tails<float>::eval(m, SM::var(sH, sL, svh.v[e], svl.v[e], 0.0f, 0.0f, cxe, cy, 0.0f),
                           p.theta, t_zero, osg.v[e], ops.v[e], opk.v[e]);
      }
      const int64_t o = int64_t(row) * p.nx + xi;
      if (p.out_mu) st_stream<float, C::VEC>(p.out_mu + o, omu);
      if (p.out_sigma) st_stream<float, C::VEC>(p.out_sigma + o, osg);
      if (p.out_psrc) st_stream<float, C::VEC>(p.out_psrc + o, ops);
      if (p.out_psnk) st_stream<float, C::VEC>(p.out_psnk + o, opk);
      if (p.out_mom_mu) {
        const V mu_v = *reinterpret_cast<const V*>(&ring.m[q][kRmV][cx0]);
        const V s_v = *reinterpret_cast<const V*>(&ring.m[q][kRmSV][cx0]);
        st_stream<float, C::VEC>(p.out_mom_mu + o, mu_u);
        st_stream<float, C::VEC>(p.out_mom_mu + N + o, mu_v);
        st_stream<float, C::VEC>(p.out_mom_sigma + o, s_u);
        st_stream<float, C::VEC>(p.out_mom_sigma + N + o, s_v);
      }
    }
  }
  if (validate) flush_error(p.err, errbits);
}

}  // namespace divuq
