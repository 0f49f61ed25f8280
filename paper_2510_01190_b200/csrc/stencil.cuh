// K2 / K3: closed-form divergence mean, sigma and tail probabilities (sm_100a).
//
// K2 (Src = kMoments) replaces propagate_divergence (divergence.py:48-70) --
// divergence_kernel + divergence_variance_kernel (stencils.py:54-84) -- and the
// probability map _tail_probs (lcp.py:48-68).
// Src = kResidual is the same stencil on ShiftedMoments (mu, r, sigma)
// triples -- the fused-ensemble fallback for shapes the TMA kernels do not
// take (nx % 4 != 0, unaligned pointers): K1 writes the triples, this kernel
// differences the (mu, r) pairs exactly as k3row / k3tma / gradfused do, so
// every fused path agrees bit for bit.
// 2D is the nz == 1, no-w case; 3D restates the per-axis rule for z
// (SURVEY 8a a19).
//
// Design (HBM-bound; tensor cores irrelevant):
//   * persistent grid: one wave of CTAs walks (x-tile, y-tile, z-chunk) work
//     items round-robin; each item marches its z-chunk plane by plane
//     ("2.5D"), so every w value is loaded once and kept in registers
//     (w[k-1], w[k], w[k+1] rolling);
//   * a warp owns one row of TX = 32*VEC points (vector loads); the x
//     neighbours of u come from warp shuffles, the two row-end halos from
//     lanes 0 / 31; the y neighbours of v come from a double-buffered shared
//     tile with one halo row above and below (one __syncthreads per plane);
//   * the next plane's inputs are fetched before the current plane's math, so
//     two planes of traffic are in flight per warp;
//   * z-slab sharding: planes are slab-local; z0 / nzg give the global plane
//     for the one-sided boundary rule; the w planes just outside the slab come
//     from halo pointers filled by the caller's exchange.
#pragma once

#include "common.cuh"

namespace divuq {

enum Src { kMoments = 0, kResidual = 1 };

template <typename T>
struct StencilParams {
  // moment inputs (slab-local, plane-major (k, j, i)); kResidual adds r_*
  const T* mu_u; const T* mu_v; const T* mu_w;
  const T* s_u;  const T* s_v;  const T* s_w;
  const T* r_u;  const T* r_v;  const T* r_w;
  // fused-ensemble entry points: members[(m*C + c)*Nl + idx], C = 2 or 3
  const T* members;
  int64_t n_members, comp_stride, member_stride;
  // w (moments) at global planes z0-1 and z0+nzl; read only when those exist
  const T* halo_lo_mu_w; const T* halo_lo_s_w;
  const T* halo_hi_mu_w; const T* halo_hi_s_w;
  const T* halo_lo_r_w; const T* halo_hi_r_w;   // kResidual / K3 (null: 0)
  int64_t nx, ny, nzl;      // slab-local extents
  int64_t z0, nzg;          // global z of local plane 0, global depth
  int64_t kbeg, kend;       // local planes to compute
  int64_t zchunk;           // planes per work item
  int64_t tiles_x, tiles_y, n_items;
  T cx_in, cx_bd, cy_in, cy_bd, cz_in, cz_bd;   // 1/(2h), 1/h (rounded from fp64)
  T theta;
  T* out_mu; T* out_sigma; T* out_psrc; T* out_psnk;
  T* out_mom_mu; T* out_mom_sigma;   // fused ensembles only, optional: (C, Nl)
  int* err;
};

constexpr int kStencilTY = 8;  // warps (rows) per CTA

template <typename T, int VEC, bool HAS_W, bool HAS_SIGMA, int SRC>
struct StencilKernel {
  using V = Vec<T, VEC>;
  using A = Arith<T>;
  static constexpr int TX = 32 * VEC;
  static constexpr int TY = kStencilTY;
  static constexpr bool RES = (SRC == kResidual);   // (mu, r) pairs (fp32 fused fallback)
  static_assert(!RES || (sizeof(T) == 4 && HAS_SIGMA), "residual pairs: fp32 with sigma");

  struct Plane {            // one plane's worth of this thread's inputs
    V u, su, v, sv, ru, rv; // own points (moments; r only when RES)
    T uL, uR, suL, suR, ruL, ruR;   // x-halo (lane 0 / lane 31 only)
    V vH, svH, rvH;         // y-halo row (ty == 0 / ty == TY-1 only)
  };

  struct Smem {
    T v[2][TY + 2][TX];
    T sv[2][TY + 2][TX];
    T rv[RES ? 2 : 1][RES ? TY + 2 : 1][RES ? TX : 1];
  };

  static __device__ __forceinline__ V zero() {
    V r;
#pragma unroll
    for (int e = 0; e < VEC; ++e) r.v[e] = T(0);
    return r;
  }

  static __device__ __forceinline__ void load_plane(const StencilParams<T>& p, Plane& P, int64_t k,
                                                    int64_t x0, int64_t xi, int64_t j, int64_t j0,
                                                    bool vx, bool vy, int lane, int ty) {
    const int64_t plane = p.nx * p.ny;
    const int64_t row = k * plane + j * p.nx;
    const bool act = vx && vy;
    P.u = P.su = P.v = P.sv = P.ru = P.rv = zero();
    if (act) {
      P.u = ldg_vec<T, VEC>(p.mu_u + row + xi);
      P.v = ldg_vec<T, VEC>(p.mu_v + row + xi);
      if constexpr (HAS_SIGMA) {
        P.su = ldg_vec<T, VEC>(p.s_u + row + xi);
        P.sv = ldg_vec<T, VEC>(p.s_v + row + xi);
      }
      if constexpr (RES) {
        P.ru = ldg_vec<T, VEC>(p.r_u + row + xi);
        P.rv = ldg_vec<T, VEC>(p.r_v + row + xi);
      }
    }
    P.uL = P.uR = P.suL = P.suR = P.ruL = P.ruR = T(0);
    if (lane == 0 && vy && x0 > 0) {
      P.uL = p.mu_u[row + x0 - 1];
      if constexpr (HAS_SIGMA) P.suL = p.s_u[row + x0 - 1];
      if constexpr (RES) P.ruL = p.r_u[row + x0 - 1];
    }
    if (lane == 31 && vy && x0 + TX < p.nx) {
      P.uR = p.mu_u[row + x0 + TX];
      if constexpr (HAS_SIGMA) P.suR = p.s_u[row + x0 + TX];
      if constexpr (RES) P.ruR = p.r_u[row + x0 + TX];
    }
    P.vH = P.svH = P.rvH = zero();
    if (ty == 0 || ty == TY - 1) {
      const int64_t jh = (ty == 0) ? j0 - 1 : j0 + TY;
      if (vx && jh >= 0 && jh < p.ny) {
        const int64_t o = k * plane + jh * p.nx + xi;
        P.vH = ldg_vec<T, VEC>(p.mu_v + o);
        if constexpr (HAS_SIGMA) P.svH = ldg_vec<T, VEC>(p.s_v + o);
        if constexpr (RES) P.rvH = ldg_vec<T, VEC>(p.r_v + o);
      }
    }
  }

  // w (moments) of local plane kk at this thread's points; kk may be -1 or
  // nzl (halo planes).  Planes outside the global grid are never used by the
  // one-sided rule and read as zero.
  static __device__ __forceinline__ void load_w(const StencilParams<T>& p, int64_t kk, int64_t off2d,
                                                bool act, V& w, V& sw, V& rw) {
    w = zero(); sw = zero(); rw = zero();
    if (!act) return;
    if (kk >= 0 && kk < p.nzl) {
      const int64_t o = kk * p.nx * p.ny + off2d;
      w = ldg_vec<T, VEC>(p.mu_w + o);
      if constexpr (HAS_SIGMA) sw = ldg_vec<T, VEC>(p.s_w + o);
      if constexpr (RES) rw = ldg_vec<T, VEC>(p.r_w + o);
    } else if (kk == -1 && p.z0 > 0) {
      w = ldg_vec<T, VEC>(p.halo_lo_mu_w + off2d);
      if constexpr (HAS_SIGMA) sw = ldg_vec<T, VEC>(p.halo_lo_s_w + off2d);
      if constexpr (RES) if (p.halo_lo_r_w) rw = ldg_vec<T, VEC>(p.halo_lo_r_w + off2d);
    } else if (kk == p.nzl && p.z0 + p.nzl < p.nzg) {
      w = ldg_vec<T, VEC>(p.halo_hi_mu_w + off2d);
      if constexpr (HAS_SIGMA) sw = ldg_vec<T, VEC>(p.halo_hi_s_w + off2d);
      if constexpr (RES) if (p.halo_hi_r_w) rw = ldg_vec<T, VEC>(p.halo_hi_r_w + off2d);
    }
  }

  static __device__ void run(const StencilParams<T>& p, Smem& sm) {
    const int lane = threadIdx.x;
    const int ty = threadIdx.y;
    const int64_t plane = p.nx * p.ny;
    int errbits = 0;
    for (int64_t item = blockIdx.x; item < p.n_items; item += gridDim.x) {
      const int64_t tx_id = item % p.tiles_x;
      const int64_t rest = item / p.tiles_x;
      const int64_t ty_id = rest % p.tiles_y;
      const int64_t zc = rest / p.tiles_y;
      const int64_t x0 = tx_id * TX;
      const int64_t j0 = ty_id * TY;
      const int64_t xi = x0 + int64_t(lane) * VEC;
      const int64_t j = j0 + ty;
      const bool vx = xi < p.nx;
      const bool vy = j < p.ny;
      const bool act = vx && vy;
      const int64_t kb = p.kbeg + zc * p.zchunk;
      const int64_t ke = min(p.kend, kb + p.zchunk);
      const int64_t off2d = j * p.nx + xi;

      V wm = zero(), w0 = zero(), wp = zero(), swm = zero(), sw0 = zero(), swp = zero();
      V rwm = zero(), rw0 = zero(), rwp = zero();
      if constexpr (HAS_W) {
        load_w(p, kb - 1, off2d, act, wm, swm, rwm);
        load_w(p, kb, off2d, act, w0, sw0, rw0);
        load_w(p, kb + 1, off2d, act, wp, swp, rwp);
      }
      Plane cur, nxt;
      load_plane(p, cur, kb, x0, xi, j, j0, vx, vy, lane, ty);
      int buf = 0;
      for (int64_t k = kb; k < ke; ++k) {
        // stage v / s_v (/ r_v) rows (own + halo) for the y-neighbour exchange
        if (act) {
          *reinterpret_cast<V*>(&sm.v[buf][ty + 1][lane * VEC]) = cur.v;
          if constexpr (HAS_SIGMA) *reinterpret_cast<V*>(&sm.sv[buf][ty + 1][lane * VEC]) = cur.sv;
          if constexpr (RES) *reinterpret_cast<V*>(&sm.rv[buf][ty + 1][lane * VEC]) = cur.rv;
        }
        if (vx && (ty == 0 || ty == TY - 1)) {
          const int r = (ty == 0) ? 0 : TY + 1;
          *reinterpret_cast<V*>(&sm.v[buf][r][lane * VEC]) = cur.vH;
          if constexpr (HAS_SIGMA) *reinterpret_cast<V*>(&sm.sv[buf][r][lane * VEC]) = cur.svH;
          if constexpr (RES) *reinterpret_cast<V*>(&sm.rv[buf][r][lane * VEC]) = cur.rvH;
        }
        __syncthreads();
        // fetch the next plane before this plane's math
        V wn = zero(), swn = zero(), rwn = zero();
        if (k + 1 < ke) {
          load_plane(p, nxt, k + 1, x0, xi, j, j0, vx, vy, lane, ty);
          if constexpr (HAS_W) load_w(p, k + 2, off2d, act, wn, swn, rwn);
        }

        // x neighbours across the warp
        const T leftU = __shfl_up_sync(0xffffffffu, cur.u.v[VEC - 1], 1);
        const T rightU = __shfl_down_sync(0xffffffffu, cur.u.v[0], 1);
        T leftS = T(0), rightS = T(0), leftR = T(0), rightR = T(0);
        if constexpr (HAS_SIGMA) {
          leftS = __shfl_up_sync(0xffffffffu, cur.su.v[VEC - 1], 1);
          rightS = __shfl_down_sync(0xffffffffu, cur.su.v[0], 1);
        }
        if constexpr (RES) {
          leftR = __shfl_up_sync(0xffffffffu, cur.ru.v[VEC - 1], 1);
          rightR = __shfl_down_sync(0xffffffffu, cur.ru.v[0], 1);
        }
        const T uLeft = lane == 0 ? cur.uL : leftU;
        const T uRight = lane == 31 ? cur.uR : rightU;
        const T sLeft = lane == 0 ? cur.suL : leftS;
        const T sRight = lane == 31 ? cur.suR : rightS;
        const T rLeft = lane == 0 ? cur.ruL : leftR;
        const T rRight = lane == 31 ? cur.ruR : rightR;

        if (act) {
          const V vlo = *reinterpret_cast<const V*>(&sm.v[buf][ty][lane * VEC]);
          const V vhi = *reinterpret_cast<const V*>(&sm.v[buf][ty + 2][lane * VEC]);
          V svlo = zero(), svhi = zero(), rvlo = zero(), rvhi = zero();
          if constexpr (HAS_SIGMA) {
            svlo = *reinterpret_cast<const V*>(&sm.sv[buf][ty][lane * VEC]);
            svhi = *reinterpret_cast<const V*>(&sm.sv[buf][ty + 2][lane * VEC]);
          }
          if constexpr (RES) {
            rvlo = *reinterpret_cast<const V*>(&sm.rv[buf][ty][lane * VEC]);
            rvhi = *reinterpret_cast<const V*>(&sm.rv[buf][ty + 2][lane * VEC]);
          }
          const bool jlo = (j == 0), jhi = (j == p.ny - 1);
          const T cy = (jlo || jhi) ? p.cy_bd : p.cy_in;
          const int64_t kg = p.z0 + k;
          const bool klo = (kg == 0), khi = (kg == p.nzg - 1);
          const T cz = (klo || khi) ? p.cz_bd : p.cz_in;

          V omu, osg, ops, opk;
#pragma unroll
          for (int e = 0; e < VEC; ++e) {
            const int64_t i = xi + e;
            const bool ilo = (i == 0), ihi = (i == p.nx - 1);
            const T cx = (ilo || ihi) ? p.cx_bd : p.cx_in;
            const T own_u = cur.u.v[e];
            const T u_lo = ilo ? own_u : (e > 0 ? cur.u.v[e > 0 ? e - 1 : 0] : uLeft);
            const T u_hi = ihi ? own_u : (e < VEC - 1 ? cur.u.v[e < VEC - 1 ? e + 1 : 0] : uRight);
            const T v_lo = jlo ? cur.v.v[e] : vlo.v[e];
            const T v_hi = jhi ? cur.v.v[e] : vhi.v[e];
            const T w_lo = HAS_W ? (klo ? w0.v[e] : wm.v[e]) : T(0);
            const T w_hi = HAS_W ? (khi ? w0.v[e] : wp.v[e]) : T(0);
            using SM = StencilMath<T, HAS_W>;
            T m;
            if constexpr (RES) {
              const T own_r = cur.ru.v[e];
              const T ru_lo = ilo ? own_r : (e > 0 ? cur.ru.v[e > 0 ? e - 1 : 0] : rLeft);
              const T ru_hi = ihi ? own_r : (e < VEC - 1 ? cur.ru.v[e < VEC - 1 ? e + 1 : 0] : rRight);
              const T rv_lo = jlo ? cur.rv.v[e] : rvlo.v[e];
              const T rv_hi = jhi ? cur.rv.v[e] : rvhi.v[e];
              const T rw_lo = HAS_W ? (klo ? rw0.v[e] : rwm.v[e]) : T(0);
              const T rw_hi = HAS_W ? (khi ? rw0.v[e] : rwp.v[e]) : T(0);
              m = SM::mean_r(u_hi, u_lo, ru_hi, ru_lo, v_hi, v_lo, rv_hi, rv_lo, w_hi, w_lo, rw_hi,
                             rw_lo, cx, cy, cz);
            } else {
              m = SM::mean(u_hi, u_lo, v_hi, v_lo, w_hi, w_lo, cx, cy, cz);
            }
            omu.v[e] = m;
            errbits |= check_value(own_u) | check_value(cur.v.v[e]);
            if constexpr (HAS_W) errbits |= check_value(w0.v[e]);
            if constexpr (HAS_SIGMA) {
              const T own_s = cur.su.v[e];
              const T s_lo = ilo ? own_s : (e > 0 ? cur.su.v[e > 0 ? e - 1 : 0] : sLeft);
              const T s_hi = ihi ? own_s : (e < VEC - 1 ? cur.su.v[e < VEC - 1 ? e + 1 : 0] : sRight);
              const T sv_lo = jlo ? cur.sv.v[e] : svlo.v[e];
              const T sv_hi = jhi ? cur.sv.v[e] : svhi.v[e];
              const T sw_lo = HAS_W ? (klo ? sw0.v[e] : swm.v[e]) : T(0);
              const T sw_hi = HAS_W ? (khi ? sw0.v[e] : swp.v[e]) : T(0);
              if constexpr (HAS_W) errbits |= check_sigma(sw0.v[e]);
              const T var = SM::var(s_hi, s_lo, sv_hi, sv_lo, sw_hi, sw_lo, cx, cy, cz);
              Tails<T>::eval(m, var, p.theta, p.theta == T(0), osg.v[e], ops.v[e], opk.v[e]);
              errbits |= check_sigma(own_s) | check_sigma(cur.sv.v[e]);
            }
          }
          const int64_t o = k * plane + off2d;
          if (p.out_mu) st_stream<T, VEC>(p.out_mu + o, omu);
          if constexpr (HAS_SIGMA) {
            if (p.out_sigma) st_stream<T, VEC>(p.out_sigma + o, osg);
            if (p.out_psrc) st_stream<T, VEC>(p.out_psrc + o, ops);
            if (p.out_psnk) st_stream<T, VEC>(p.out_psnk + o, opk);
          }
        }
        cur = nxt;
        if constexpr (HAS_W) {
          wm = w0; w0 = wp; wp = wn; swm = sw0; sw0 = swp; swp = swn;
          rwm = rw0; rw0 = rwp; rwp = rwn;
        }
        buf ^= 1;
      }
      __syncthreads();  // shared tile reuse across work items
    }
    flush_error(p.err, errbits);
  }
};

// 2D (no w) as a plain gather: one thread per point, the four stencil
// neighbours (and the residuals' / sigmas' four) loaded straight from global
// memory -- the x neighbours hit L1, the y neighbours L2 (adjacent rows run
// in adjacent CTAs).  The z-marching kernel above degenerates in 2D (one
// plane per work item: a barrier and a prologue per 256 points; 24 % of HBM
// on the unaligned residual fallback).  Same StencilMath / Tails calls with
// the same operands as StencilKernel<T, *, false, ...>: bitwise equal.
template <typename T, bool HAS_SIGMA, int SRC>
__global__ void __launch_bounds__(256)
stencil2d_gather_kernel(const StencilParams<T> p) {
  using SM = StencilMath<T, false>;
  constexpr bool RES = (SRC == kResidual);
  const int64_t nx = p.nx, ny = p.ny;
  int errbits = 0;
  const int64_t i = int64_t(blockIdx.x) * 256 + threadIdx.x;
  if (i < nx) {
    const bool ilo = i == 0, ihi = i == nx - 1;
    const T cx = (ilo || ihi) ? p.cx_bd : p.cx_in;
    for (int64_t j = blockIdx.y; j < ny; j += gridDim.y) {
      const int64_t q = j * nx + i;
      const bool jlo = j == 0, jhi = j == ny - 1;
      const T cy = (jlo || jhi) ? p.cy_bd : p.cy_in;
      const int64_t xl = ilo ? q : q - 1, xh = ihi ? q : q + 1;
      const int64_t yl = jlo ? q : q - nx, yh = jhi ? q : q + nx;
      T m;
      if constexpr (RES) {
        m = SM::mean_r(__ldg(p.mu_u + xh), __ldg(p.mu_u + xl), __ldg(p.r_u + xh), __ldg(p.r_u + xl),
                       __ldg(p.mu_v + yh), __ldg(p.mu_v + yl), __ldg(p.r_v + yh), __ldg(p.r_v + yl),
                       T(0), T(0), T(0), T(0), cx, cy, T(0));
      } else {
        m = SM::mean(__ldg(p.mu_u + xh), __ldg(p.mu_u + xl), __ldg(p.mu_v + yh), __ldg(p.mu_v + yl),
                     T(0), T(0), cx, cy, T(0));
      }
      if (p.out_mu) p.out_mu[q] = m;
      if (p.err) errbits |= check_value(__ldg(p.mu_u + q)) | check_value(__ldg(p.mu_v + q));
      if constexpr (HAS_SIGMA) {
        const T var = SM::var(__ldg(p.s_u + xh), __ldg(p.s_u + xl), __ldg(p.s_v + yh), __ldg(p.s_v + yl),
                              T(0), T(0), cx, cy, T(0));
        T sg, ps, pk;
        Tails<T>::eval(m, var, p.theta, p.theta == T(0), sg, ps, pk);
        if (p.out_sigma) p.out_sigma[q] = sg;
        if (p.out_psrc) p.out_psrc[q] = ps;
        if (p.out_psnk) p.out_psnk[q] = pk;
        if (p.err) errbits |= check_sigma(__ldg(p.s_u + q)) | check_sigma(__ldg(p.s_v + q));
      }
    }
  }
  flush_error(p.err, errbits);
}

template <typename T, int VEC, bool HAS_W, bool HAS_SIGMA, int SRC>
__global__ void __launch_bounds__(32 * kStencilTY, 2)
stencil_kernel(const StencilParams<T> p) {
  using K = StencilKernel<T, VEC, HAS_W, HAS_SIGMA, SRC>;
  __shared__ typename K::Smem sm;
  K::run(p, sm);
}

}  // namespace divuq
