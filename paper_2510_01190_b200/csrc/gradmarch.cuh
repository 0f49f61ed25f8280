// The Red Sea chain as a STRIP MARCH (K6m): the same arithmetic as the tiled
// K6 (gradfused.cuh) -- velocity magnitude pairs, the gradient of the
// magnitude, shifted moments over the members, the divergence of the
// gradient moments and both tails (gaussian.py:48-66, stencils.py:87-96,
// gaussian.py:35-45, divergence.py:48-70, lcp.py:48-68) -- with less
// recomputation:
//
//   * a CTA owns a 64-column strip and a segment of rows and marches down
//     it two rows per step; one TMA box per step carries the two rows of all
//     M members' (u, v) with 4-column x-halos ({72, 2, 2M} on the (x, y,
//     member*2 + component) view), S steps in flight;
//   * phase M: every magnitude pair of the two new rows (all members, 72
//     columns) is computed ONCE into a 4-row ring (the tile kernel computed
//     72 x 20 region magnitudes per 64 x 16 outputs: 1.41 per output and
//     member; here 1.125);
//   * phase G: one thread per gradient point of the two rows behind (66 gx
//     incl. the two x-halo columns, 64 gy per row: no y-halo gradients, the
//     neighbouring rows are the march's own), folding the members in order
//     into ShiftedMoments (member 0 peeled), the (mu, r, sigma) triples into
//     a 4-row moment ring;
//   * phase D: the divergence mean / variance of the two rows behind that
//     (the (mu, r) pairs differenced), sigma and both tails, streamed out.
// Two CTA barriers per step (after M: the stage is consumed, the ring rows
// are complete; after G: the moments are complete); the rings are four rows
// deep so a phase never overwrites rows the previous phase still reads.
// Output bits are those of gradient_ensemble2d_f32 + ensemble_divergence2d_f32
// (and of the tiled K6): same mag_pair, grad_diff_pair, ShiftedMoments,
// StencilMath<float>::mean_r / var and Tails<float>.
//
// Status: OPT-IN (DIVUQ_GRADMARCH=1).  It executes fewer magnitude pairs but
// measured 81 us against the tiled K6's 63 us at 1024^2 x M=20: 2 CTAs x 9
// warps per SM (the 4-row magnitude ring is 46 KB), two CTA barriers per step,
// every phase a per-thread dependent chain (members folded in order) -- 47 %
// issue-active, barrier-stalled.  Warp-specialised phases handing rows over
// mbarriers (magnitude warps one step ahead of gradient warps) would be the
// next step; not done.
#pragma once

#include "common.cuh"
#include "gradient.cuh"
#include "tma.cuh"

namespace divuq {

constexpr int kGmTX = 64, kGmPAD = 4, kGmW = kGmTX + 2 * kGmPAD;   // 72 staged columns
constexpr int kGmRows = 2;                                          // rows per step
constexpr int kGmRing = 4;                                          // ring depth (rows)
constexpr int kGmGx = kGmTX + 2, kGmGy = kGmTX;                     // gradient points per row
constexpr int kGmPts = kGmRows * (kGmGx + kGmGy);                   // 260 per step
constexpr int kGmThreads = 288;                                     // 9 warps
constexpr int kGmMaxStages = 8;

struct GmParams {
  int nx, ny, M, strips, seg_rows, S;
  uint32_t stage_bytes, stage_stride, mag_off, mom_off, bar_off;
  float cx_in, cx_bd, cy_in, cy_bd, theta;
  float *out_mu, *out_sigma, *out_psrc, *out_psnk, *out_mom_mu, *out_mom_sigma;
  int* err;
};

// one ring row of gradient moments: gx at columns -1..64, gy at 0..63
struct GmMomRow {
  float gx_mu[kGmGx], gx_r[kGmGx], gx_sg[kGmGx];
  float gy_mu[kGmGy], gy_r[kGmGy], gy_sg[kGmGy];
};

__global__ void __launch_bounds__(kGmThreads, 2)
gradmarch_kernel(const __grid_constant__ CUtensorMap map, const GmParams p) {
  extern __shared__ __align__(1024) unsigned char gm_smem[];
  const int tid = threadIdx.x;
  const int M = p.M;
  const int nx = p.nx, ny = p.ny;
  const int strip = blockIdx.x % p.strips, seg = blockIdx.x / p.strips;
  const int x0 = strip * kGmTX;
  const int y0 = seg * p.seg_rows, y1 = min(ny, y0 + p.seg_rows);
  const int mr0 = y0 - 2;                                   // first magnitude row
  const int steps = (y1 + 3 - y0) / 2 + 1;                  // until the last output row
  float2* const mag = reinterpret_cast<float2*>(gm_smem + p.mag_off);   // [ring][M][72]
  GmMomRow* const mom = reinterpret_cast<GmMomRow*>(gm_smem + p.mom_off);
  uint64_t* const full = reinterpret_cast<uint64_t*>(gm_smem + p.bar_off);
  auto stage_ptr = [&](int k) { return gm_smem + size_t(k % p.S) * p.stage_stride; };
  auto issue = [&](int k) {
    const int s = k % p.S;
    mbar_expect_tx(&full[s], p.stage_bytes);
    tma_load_3d(stage_ptr(k), &map, &full[s], x0 - kGmPAD, mr0 + 2 * k, 0);
  };
  if (tid == 0) {
    for (int s = 0; s < p.S; ++s) mbar_init(&full[s], 1);
    mbar_fence_init();
    for (int k = 0; k < p.S && k < steps; ++k) issue(k);
  }
  __syncthreads();

  // ---- phase M slot (fixed): column, row of the step, member parity
  // (72 columns x 2 rows x 2 parities = 288 threads: every thread busy)
  const bool m_act = tid < kGmW * kGmRows * 2;
  const int m_x = tid % kGmW, m_r = (tid / kGmW) % kGmRows, m_g0 = tid / (kGmW * kGmRows);
  // ---- phase G slot of this thread (fixed): step row 0/1, gx or gy, column
  const bool g_act = tid < kGmPts;
  const int g_row = tid / (kGmGx + kGmGy);                  // 0: row m-1, 1: row m
  const int g_q = tid - g_row * (kGmGx + kGmGy);
  const bool g_isx = g_q < kGmGx;
  const int g_col = g_isx ? g_q - 1 : g_q - kGmGx;          // strip-local column
  const int g_gi = min(max(x0 + g_col, 0), nx - 1);         // grid-clamped column
  const int g_sc = g_gi - x0 + kGmPAD;                      // its staged / ring column
  // x neighbours of a gx point (one-sided at the grid's x faces)
  const int g_xh = g_gi < nx - 1 ? g_sc + 1 : g_sc, g_xl = g_gi > 0 ? g_sc - 1 : g_sc;
  const float g_cx = (g_gi == 0 || g_gi == nx - 1) ? p.cx_bd : p.cx_in;
  // ---- phase D slot: row 0/1, column
  const bool d_act = tid < kGmRows * kGmTX;
  const int d_row = tid / kGmTX, d_col = tid - d_row * kGmTX;
  const int d_i = x0 + d_col;
  const bool t_zero = p.theta == 0.0f;
  int errbits = 0;

  for (int k = 0; k < steps; ++k) {
    const int mrow = mr0 + 2 * k;                           // magnitude rows mrow, mrow + 1
    // ---- phase M: magnitude pairs of the two new rows, all members
    mbar_wait(&full[k % p.S], uint32_t(k / p.S) & 1u);
    if (m_act) {
      // this thread: column m_x, row m_r, members m_g0, m_g0 + 2, ... (box
      // layout [plane = 2m + c][row][x]: constant strides, no index math)
      const float* su = reinterpret_cast<const float*>(stage_ptr(k)) + (2 * m_g0 * kGmRows + m_r) * kGmW + m_x;
      float2* dm = mag + ((((mrow + m_r) & (kGmRing - 1)) * M) + m_g0) * kGmW + m_x;
#pragma unroll 2
      for (int m = m_g0; m < M; m += 2) {
        float h, l;
        mag_pair(su[0], su[kGmRows * kGmW], h, l);   // u (plane 2m), v (plane 2m + 1)
        *dm = make_float2(h, l);
        su += 4 * kGmRows * kGmW;                    // plane 2(m + 2)
        dm += 2 * kGmW;
      }
    }
    __syncthreads();   // B1: stage consumed, magnitude rows complete
    if (tid == 0 && k + p.S < steps) issue(k + p.S);
    // ---- phase G: gradient moments of rows mrow - 1 (g_row 0) and mrow (g_row 1)
    const int grow = mrow - 1 + g_row;                      // global gradient row
    if (g_act && grow >= 0 && grow < ny) {
      const int gj = grow;
      const int rs = grow & (kGmRing - 1);
      const int hs = (gj < ny - 1 ? gj + 1 : gj) & (kGmRing - 1);   // gy neighbours
      const int ls = (gj > 0 ? gj - 1 : gj) & (kGmRing - 1);
      const float cy = (gj == 0 || gj == ny - 1) ? p.cy_bd : p.cy_in;
      const float c = g_isx ? g_cx : cy;
      const int hi_off = g_isx ? (rs * M) * kGmW + g_xh : (hs * M) * kGmW + g_sc;
      const int lo_off = g_isx ? (rs * M) * kGmW + g_xl : (ls * M) * kGmW + g_sc;
      ShiftedMoments<1> acc;
      {
        const float2 H = mag[hi_off], L = mag[lo_off];
        const float g = grad_diff_pair(H.x, L.x, H.y, L.y, c);
        acc.first(&g);
      }
#pragma unroll 4
      for (int m = 1; m < M; ++m) {
        const float2 H = mag[hi_off + m * kGmW], L = mag[lo_off + m * kGmW];
        const float g = grad_diff_pair(H.x, L.x, H.y, L.y, c);
        acc.next(&g);
      }
      float mu, r, sg;
      acc.finish(M, &mu, &r, &sg);
      GmMomRow& R = mom[rs];
      if (g_isx) { R.gx_mu[g_q] = mu; R.gx_r[g_q] = r; R.gx_sg[g_q] = sg; }
      else { const int c2 = g_q - kGmGx; R.gy_mu[c2] = mu; R.gy_r[c2] = r; R.gy_sg[c2] = sg; }
    }
    __syncthreads();   // B2: moments of the two gradient rows complete
    // ---- phase D: divergence of rows mrow - 2 (d_row 0) and mrow - 1 (d_row 1)
    const int drow = mrow - 2 + d_row;
    if (d_act && drow >= y0 && drow < y1 && d_i < nx) {
      using SM = StencilMath<float, true>;
      const int j = drow;
      const GmMomRow& R = mom[j & (kGmRing - 1)];
      const GmMomRow& RH = mom[(j < ny - 1 ? j + 1 : j) & (kGmRing - 1)];
      const GmMomRow& RL = mom[(j > 0 ? j - 1 : j) & (kGmRing - 1)];
      const int xc = d_col + 1;                              // gx index of this column
      const int xh = d_i < nx - 1 ? xc + 1 : xc, xl = d_i > 0 ? xc - 1 : xc;
      const float cxe = (d_i == 0 || d_i == nx - 1) ? p.cx_bd : p.cx_in;
      const float cye = (j == 0 || j == ny - 1) ? p.cy_bd : p.cy_in;
      const float mean = SM::mean_r(R.gx_mu[xh], R.gx_mu[xl], R.gx_r[xh], R.gx_r[xl], RH.gy_mu[d_col],
                                    RL.gy_mu[d_col], RH.gy_r[d_col], RL.gy_r[d_col], 0.0f, 0.0f, 0.0f,
                                    0.0f, cxe, cye, 0.0f);
      const float var = SM::var(R.gx_sg[xh], R.gx_sg[xl], RH.gy_sg[d_col], RL.gy_sg[d_col], 0.0f, 0.0f,
                                cxe, cye, 0.0f);
      errbits |= check_value(mean);   // a non-finite input reaches some output's mean (tiled K6)
      float sg, ps, pk;
      Tails<float>::eval(mean, var, p.theta, t_zero, sg, ps, pk);
      const int64_t o = int64_t(j) * nx + d_i;
      const int64_t N = int64_t(nx) * ny;
      if (p.out_mu) p.out_mu[o] = mean;
      if (p.out_sigma) p.out_sigma[o] = sg;
      if (p.out_psrc) p.out_psrc[o] = ps;
      if (p.out_psnk) p.out_psnk[o] = pk;
      if (p.out_mom_mu) {
        p.out_mom_mu[o] = R.gx_mu[xc];
        p.out_mom_mu[N + o] = R.gy_mu[d_col];
        p.out_mom_sigma[o] = R.gx_sg[xc];
        p.out_mom_sigma[N + o] = R.gy_sg[d_col];
      }
    }
    // the next phase M overwrites magnitude rows phase G of this step read --
    // every thread is past B2; the next phase G overwrites moment rows this
    // phase D reads -- every thread is past the next B1 first
  }
  flush_error(p.err, errbits);
}

}  // namespace divuq
