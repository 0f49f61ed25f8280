// K2 / K3: closed-form divergence mean, sigma and tail probabilities (sm_100a).
//
// K2 (Src = kMoments) replaces propagate_divergence (divergence.py:48-70) --
// divergence_kernel + divergence_variance_kernel (stencils.py:54-84) -- and the
// probability map _tail_probs (lcp.py:48-68).
// K3 (Src = kEnsemble) fuses fit_gaussian (gaussian.py:35-45) in front of K2:
// members are read once, moments live in registers / shared memory and never
// touch HBM unless the caller asks for them.
// 2D is the nz == 1, no-w case; 3D restates the per-axis rule for z
// (SURVEY 8a a19).
//
// Design (HBM-bound; tensor cores irrelevant):
//   * persistent grid: one wave of CTAs walks (x-tile, y-tile, z-chunk) work
//     items round-robin; each item marches its z-chunk plane by plane
//     ("2.5D"), so every w value (or w moment) is produced once and kept in
//     registers (w[k-1], w[k], w[k+1] rolling);
//   * a warp owns one row of TX = 32*VEC points (vector loads); the x
//     neighbours of u come from warp shuffles, the two row-end halos from
//     lanes 0 / 31; the y neighbours of v come from a double-buffered shared
//     tile with one halo row above and below (one __syncthreads per plane);
//   * the next plane's inputs are fetched before the current plane's math, so
//     two planes of traffic are in flight per warp;
//   * z-slab sharding: planes are slab-local; z0 / nzg give the global plane
//     for the one-sided boundary rule; the w planes just outside the slab come
//     from halo pointers filled by the caller's exchange (for K3 these are
//     reduced w moments, 2 planes instead of 2*M).
#pragma once

#include "common.cuh"

namespace divuq {

enum Src { kMoments = 0, kEnsemble = 1 };

template <typename T>
struct StencilParams {
  // kMoments inputs (slab-local, plane-major (k, j, i))
  const T* mu_u; const T* mu_v; const T* mu_w;
  const T* s_u;  const T* s_v;  const T* s_w;
  // kEnsemble inputs: members[(m*C + c)*Nl + idx], C = 2 (2D) or 3 (3D)
  const T* members;
  int64_t n_members, comp_stride, member_stride;
  // w (moments) at global planes z0-1 and z0+nzl; read only when those exist
  const T* halo_lo_mu_w; const T* halo_lo_s_w;
  const T* halo_hi_mu_w; const T* halo_hi_s_w;
  int64_t nx, ny, nzl;      // slab-local extents
  int64_t z0, nzg;          // global z of local plane 0, global depth
  int64_t kbeg, kend;       // local planes to compute
  int64_t zchunk;           // planes per work item
  int64_t tiles_x, tiles_y, n_items;
  T cx_in, cx_bd, cy_in, cy_bd, cz_in, cz_bd;   // 1/(2h), 1/h (rounded from fp64)
  T theta;
  T* out_mu; T* out_sigma; T* out_psrc; T* out_psnk;
  T* out_mom_mu; T* out_mom_sigma;   // K3 only, optional: (C, Nl)
  int* err;
};

constexpr int kStencilTY = 8;  // warps (rows) per CTA

// --- ensemble moments ------------------------------------------------------
// fp64: numpy's algorithm bit for bit (gaussian.py:41-44) -- sequential sum /
//   M, then the two-pass ddof=1 variance.  The MR member values stay in
//   registers between the passes (fully unrolled and predicated on k < M);
//   M > MR falls back to re-reading the members.
// fp32: single pass shifted by the first member (ShiftedMoments in
//   common.cuh), the formula every fp32 kernel (K1, the register K3 and the
//   TMA K3) shares, so fused == K1 + K2 and sharded == whole bit for bit.
template <typename T, int VEC, int MR>
__device__ __forceinline__ void member_moments_2pass(const T* base, int64_t mstride, int M,
                                                     Vec<T, VEC>& mu, Vec<T, VEC>& sg, int& err);

template <typename T, int VEC, int MR>
__device__ __forceinline__ void member_moments(const T* base, int64_t mstride, int M,
                                               Vec<T, VEC>& mu, Vec<T, VEC>& sg, int& err) {
  if constexpr (sizeof(T) == 4) {
    ShiftedMoments<VEC> acc;
    if (M <= MR) {   // all M loads in flight before the first use
      Vec<T, VEC> x[MR];
#pragma unroll
      for (int k = 0; k < MR; ++k)
        if (k < M) x[k] = ld_stream<T, VEC>(base + k * mstride);
#pragma unroll
      for (int k = 0; k < MR; ++k)
        if (k < M) {
#pragma unroll
          for (int e = 0; e < VEC; ++e) err |= check_value(x[k].v[e]);
          acc.add(k, x[k].v);
        }
    } else {
#pragma unroll 8
      for (int k = 0; k < M; ++k) {
        const Vec<T, VEC> x = ld_stream<T, VEC>(base + k * mstride);
#pragma unroll
        for (int e = 0; e < VEC; ++e) err |= check_value(x.v[e]);
        acc.add(k, x.v);
      }
    }
    acc.finish(M, mu.v, sg.v);
    return;
  }
  member_moments_2pass<T, VEC, MR>(base, mstride, M, mu, sg, err);
}

template <typename T, int VEC, int MR>
__device__ __forceinline__ void member_moments_2pass(const T* base, int64_t mstride, int M,
                                                     Vec<T, VEC>& mu, Vec<T, VEC>& sg, int& err) {
  using A = Arith<T>;
  using V = Vec<T, VEC>;
  V s, q;
  // keep one reduction's M loads in flight at a time: without the fence
  // nvcc hoists the loads of several reductions and spills
  asm volatile("" ::: "memory");
  if (M <= MR) {
    V x[MR];
#pragma unroll
    for (int k = 0; k < MR; ++k)
      if (k < M) x[k] = ld_stream<T, VEC>(base + k * mstride);
    s = x[0];
#pragma unroll
    for (int k = 1; k < MR; ++k)
      if (k < M) {
#pragma unroll
        for (int e = 0; e < VEC; ++e) s.v[e] = A::add(s.v[e], x[k].v[e]);
      }
#pragma unroll
    for (int e = 0; e < VEC; ++e) mu.v[e] = A::div(s.v[e], T(M));
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      const T d = A::sub(x[0].v[e], mu.v[e]);
      q.v[e] = A::mul(d, d);
      err |= check_value(x[0].v[e]);
    }
#pragma unroll
    for (int k = 1; k < MR; ++k)
      if (k < M) {
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          const T d = A::sub(x[k].v[e], mu.v[e]);
          q.v[e] = A::add(q.v[e], A::mul(d, d));
          err |= check_value(x[k].v[e]);
        }
      }
  } else {
    s = ldg_vec<T, VEC>(base);
    for (int k = 1; k < M; ++k) {
      const V x = ldg_vec<T, VEC>(base + k * mstride);
#pragma unroll
      for (int e = 0; e < VEC; ++e) s.v[e] = A::add(s.v[e], x.v[e]);
    }
#pragma unroll
    for (int e = 0; e < VEC; ++e) mu.v[e] = A::div(s.v[e], T(M));
    for (int k = 0; k < M; ++k) {
      const V x = ldg_vec<T, VEC>(base + k * mstride);
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        const T d = A::sub(x.v[e], mu.v[e]);
        q.v[e] = k == 0 ? A::mul(d, d) : A::add(q.v[e], A::mul(d, d));
        err |= check_value(x.v[e]);
      }
    }
  }
#pragma unroll
  for (int e = 0; e < VEC; ++e) sg.v[e] = A::sqrt_(A::div(q.v[e], T(M - 1)));
  asm volatile("" ::: "memory");
}

template <typename T, int VEC, bool HAS_W, bool HAS_SIGMA, int SRC, int MR>
struct StencilKernel {
  using V = Vec<T, VEC>;
  using A = Arith<T>;
  static constexpr int TX = 32 * VEC;
  static constexpr int TY = kStencilTY;
  static constexpr bool ENS = (SRC == kEnsemble);

  struct Plane {            // one plane's worth of this thread's inputs
    V u, su, v, sv;         // own points (values or moments)
    T uL, uR, suL, suR;     // x-halo (lane 0 / lane 31 only)
    V vH, svH;              // y-halo row (ty == 0 / ty == TY-1 only)
  };

  struct Smem {
    T v[2][TY + 2][TX];
    T sv[2][TY + 2][TX];
  };

  static __device__ __forceinline__ V zero() {
    V r;
#pragma unroll
    for (int e = 0; e < VEC; ++e) r.v[e] = T(0);
    return r;
  }

  // (value, sigma) of component c at flat slab offset `off`, VEC points
  template <int W>
  static __device__ __forceinline__ void fetch(const StencilParams<T>& p, int c, int64_t off,
                                               const T* mu_arr, const T* s_arr,
                                               Vec<T, W>& m, Vec<T, W>& s, int& err) {
    if constexpr (ENS) {
      member_moments<T, W, MR>(p.members + c * p.comp_stride + off, p.member_stride,
                               int(p.n_members), m, s, err);
    } else {
      m = ldg_vec<T, W>(mu_arr + off);
      if constexpr (HAS_SIGMA) s = ldg_vec<T, W>(s_arr + off);
    }
  }

  static __device__ __forceinline__ void load_plane(const StencilParams<T>& p, Plane& P, int64_t k,
                                                    int64_t x0, int64_t xi, int64_t j, int64_t j0,
                                                    bool vx, bool vy, int lane, int ty, int& err) {
    const int64_t plane = p.nx * p.ny;
    const int64_t row = k * plane + j * p.nx;
    const bool act = vx && vy;
    P.u = P.su = P.v = P.sv = zero();
    if (act) {
      fetch<VEC>(p, 0, row + xi, p.mu_u, p.s_u, P.u, P.su, err);
      fetch<VEC>(p, 1, row + xi, p.mu_v, p.s_v, P.v, P.sv, err);
    }
    P.uL = P.uR = P.suL = P.suR = T(0);
    if (lane == 0 && vy && x0 > 0) {
      Vec<T, 1> m, s; int e2 = 0;
      fetch<1>(p, 0, row + x0 - 1, p.mu_u, p.s_u, m, s, e2);
      P.uL = m.v[0]; if constexpr (HAS_SIGMA) P.suL = s.v[0];
    }
    if (lane == 31 && vy && x0 + TX < p.nx) {
      Vec<T, 1> m, s; int e2 = 0;
      fetch<1>(p, 0, row + x0 + TX, p.mu_u, p.s_u, m, s, e2);
      P.uR = m.v[0]; if constexpr (HAS_SIGMA) P.suR = s.v[0];
    }
    P.vH = P.svH = zero();
    if (ty == 0 || ty == TY - 1) {
      const int64_t jh = (ty == 0) ? j0 - 1 : j0 + TY;
      if (vx && jh >= 0 && jh < p.ny) {
        int e2 = 0;
        fetch<VEC>(p, 1, k * plane + jh * p.nx + xi, p.mu_v, p.s_v, P.vH, P.svH, e2);
      }
    }
  }

  // w (or w moments) of local plane kk at this thread's points; kk may be -1
  // or nzl (halo planes).  Planes outside the global grid are never used by
  // the one-sided rule and read as zero.
  static __device__ __forceinline__ void load_w(const StencilParams<T>& p, int64_t kk, int64_t off2d,
                                                bool act, V& w, V& sw, int& err) {
    w = zero(); sw = zero();
    if (!act) return;
    if (kk >= 0 && kk < p.nzl) {
      fetch<VEC>(p, 2, kk * p.nx * p.ny + off2d, p.mu_w, p.s_w, w, sw, err);
    } else if (kk == -1 && p.z0 > 0) {
      w = ldg_vec<T, VEC>(p.halo_lo_mu_w + off2d);
      if constexpr (HAS_SIGMA) sw = ldg_vec<T, VEC>(p.halo_lo_s_w + off2d);
    } else if (kk == p.nzl && p.z0 + p.nzl < p.nzg) {
      w = ldg_vec<T, VEC>(p.halo_hi_mu_w + off2d);
      if constexpr (HAS_SIGMA) sw = ldg_vec<T, VEC>(p.halo_hi_s_w + off2d);
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
      if constexpr (HAS_W) {
        int e2 = 0;  // planes outside [kb, ke) are validated by the item owning them
        load_w(p, kb - 1, off2d, act, wm, swm, e2);
        load_w(p, kb, off2d, act, w0, sw0, errbits);
        load_w(p, kb + 1, off2d, act, wp, swp, kb + 1 < ke ? errbits : e2);
      }
      Plane cur, nxt;
      if constexpr (!ENS) load_plane(p, cur, kb, x0, xi, j, j0, vx, vy, lane, ty, errbits);
      int buf = 0;
      for (int64_t k = kb; k < ke; ++k) {
        if constexpr (ENS) load_plane(p, cur, k, x0, xi, j, j0, vx, vy, lane, ty, errbits);
        // stage v / s_v rows (own + halo) for the y-neighbour exchange
        if (act) {
          *reinterpret_cast<V*>(&sm.v[buf][ty + 1][lane * VEC]) = cur.v;
          if constexpr (HAS_SIGMA) *reinterpret_cast<V*>(&sm.sv[buf][ty + 1][lane * VEC]) = cur.sv;
        }
        if (vx && (ty == 0 || ty == TY - 1)) {
          const int r = (ty == 0) ? 0 : TY + 1;
          *reinterpret_cast<V*>(&sm.v[buf][r][lane * VEC]) = cur.vH;
          if constexpr (HAS_SIGMA) *reinterpret_cast<V*>(&sm.sv[buf][r][lane * VEC]) = cur.svH;
        }
        __syncthreads();
        // K2: fetch the next plane before this plane's math
        V wn = zero(), swn = zero();
        if (!ENS && k + 1 < ke) {
          load_plane(p, nxt, k + 1, x0, xi, j, j0, vx, vy, lane, ty, errbits);
          if constexpr (HAS_W) {
            int e2 = 0;
            load_w(p, k + 2, off2d, act, wn, swn, k + 2 < ke ? errbits : e2);
          }
        }

        // x neighbours across the warp
        const T leftU = __shfl_up_sync(0xffffffffu, cur.u.v[VEC - 1], 1);
        const T rightU = __shfl_down_sync(0xffffffffu, cur.u.v[0], 1);
        T leftS = T(0), rightS = T(0);
        if constexpr (HAS_SIGMA) {
          leftS = __shfl_up_sync(0xffffffffu, cur.su.v[VEC - 1], 1);
          rightS = __shfl_down_sync(0xffffffffu, cur.su.v[0], 1);
        }
        const T uLeft = lane == 0 ? cur.uL : leftU;
        const T uRight = lane == 31 ? cur.uR : rightU;
        const T sLeft = lane == 0 ? cur.suL : leftS;
        const T sRight = lane == 31 ? cur.suR : rightS;

        if (act) {
          const V vlo = *reinterpret_cast<const V*>(&sm.v[buf][ty][lane * VEC]);
          const V vhi = *reinterpret_cast<const V*>(&sm.v[buf][ty + 2][lane * VEC]);
          V svlo = zero(), svhi = zero();
          if constexpr (HAS_SIGMA) {
            svlo = *reinterpret_cast<const V*>(&sm.sv[buf][ty][lane * VEC]);
            svhi = *reinterpret_cast<const V*>(&sm.sv[buf][ty + 2][lane * VEC]);
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
            const T m = SM::mean(u_hi, u_lo, v_hi, v_lo, w_hi, w_lo, cx, cy, cz);
            omu.v[e] = m;
            if constexpr (!ENS) {
              errbits |= check_value(own_u) | check_value(cur.v.v[e]);
              if constexpr (HAS_W) errbits |= check_value(w0.v[e]);
            }
            if constexpr (HAS_SIGMA) {
              const T own_s = cur.su.v[e];
              const T s_lo = ilo ? own_s : (e > 0 ? cur.su.v[e > 0 ? e - 1 : 0] : sLeft);
              const T s_hi = ihi ? own_s : (e < VEC - 1 ? cur.su.v[e < VEC - 1 ? e + 1 : 0] : sRight);
              const T sv_lo = jlo ? cur.sv.v[e] : svlo.v[e];
              const T sv_hi = jhi ? cur.sv.v[e] : svhi.v[e];
              const T sw_lo = HAS_W ? (klo ? sw0.v[e] : swm.v[e]) : T(0);
              const T sw_hi = HAS_W ? (khi ? sw0.v[e] : swp.v[e]) : T(0);
              if constexpr (HAS_W && !ENS) errbits |= check_sigma(sw0.v[e]);
              const T var = SM::var(s_hi, s_lo, sv_hi, sv_lo, sw_hi, sw_lo, cx, cy, cz);
              Tails<T>::eval(m, var, p.theta, p.theta == T(0), osg.v[e], ops.v[e], opk.v[e]);
              if constexpr (!ENS) errbits |= check_sigma(own_s) | check_sigma(cur.sv.v[e]);
            }
          }
          const int64_t o = k * plane + off2d;
          if (p.out_mu) st_stream<T, VEC>(p.out_mu + o, omu);
          if constexpr (HAS_SIGMA) {
            if (p.out_sigma) st_stream<T, VEC>(p.out_sigma + o, osg);
            if (p.out_psrc) st_stream<T, VEC>(p.out_psrc + o, ops);
            if (p.out_psnk) st_stream<T, VEC>(p.out_psnk + o, opk);
          }
          if constexpr (ENS) {
            if (p.out_mom_mu) {
              const int64_t nl = p.comp_stride;
              st_stream<T, VEC>(p.out_mom_mu + o, cur.u);
              st_stream<T, VEC>(p.out_mom_mu + nl + o, cur.v);
              st_stream<T, VEC>(p.out_mom_sigma + o, cur.su);
              st_stream<T, VEC>(p.out_mom_sigma + nl + o, cur.sv);
              if constexpr (HAS_W) {
                st_stream<T, VEC>(p.out_mom_mu + 2 * nl + o, w0);
                st_stream<T, VEC>(p.out_mom_sigma + 2 * nl + o, sw0);
              }
            }
          }
        }
        if constexpr (ENS) {
          if (HAS_W && k + 1 < ke) load_w(p, k + 2, off2d, act, wn, swn, errbits);
        } else {
          cur = nxt;
        }
        if constexpr (HAS_W) { wm = w0; w0 = wp; wp = wn; swm = sw0; sw0 = swp; swp = swn; }
        buf ^= 1;
      }
      __syncthreads();  // shared tile reuse across work items
    }
    flush_error(p.err, errbits);
  }
};

template <typename T, int VEC, bool HAS_W, bool HAS_SIGMA, int SRC, int MR>
__global__ void __launch_bounds__(32 * kStencilTY, 2)
stencil_kernel(const StencilParams<T> p) {
  using K = StencilKernel<T, VEC, HAS_W, HAS_SIGMA, SRC, MR>;
  __shared__ typename K::Smem sm;
  K::run(p, sm);
}

}  // namespace divuq
