// K2 (3D) for shapes a tiled tensor map cannot describe: a tiled map needs
// its row pitch to be a multiple of 16 bytes (fp32 nx % 4 == 0, fp64 nx
// even), so those shapes ran the register-pipelined generic kernel at ~43 %
// of HBM (tools/shape_probe.py).  Here the same warp-specialised persistent
// pipeline as k2tma.cuh runs on 1D tensor maps over the flat arrays: one box
// per tile row.  A box must START on a 16-byte boundary (an unaligned start
// raises an illegal instruction on sm_100a), so each row box begins at the
// row's offset rounded down to VEC elements and is VEC elements wider; the
// consumers read their row at that (warp-uniform) shift with scalar loads.
// The u / s_u x-halo columns sit inside the row box, the v / s_v halo rows
// are two more row boxes; parts outside [0, N) arrive zero-filled, parts
// that wrap into a neighbouring row are only ever read as the one-sided
// boundary rule's discarded operand.  Lanes own strided points (x0 + lane +
// 32 e), so the row reads at any shift are conflict-free and the scalar
// stores coalesced (output rows are not 16-byte aligned either).  Arithmetic:
// StencilMath / Tails exactly as k2tma.cuh, so results are bitwise equal.
#pragma once

#include "common.cuh"
#include "tma.cuh"

#ifndef DIVUQ_FLAT_NS
#define DIVUQ_FLAT_NS 256
#endif
#ifndef DIVUQ_FLAT_NP
#define DIVUQ_FLAT_NP 2
#endif

namespace divuq {

template <typename T>
struct FlatCfg {
  static constexpr int VEC = 16 / int(sizeof(T));   // points per lane (4 fp32, 2 fp64)
  static constexpr int TX = 32 * VEC;                // tile width (points)
  static constexpr int PADE = VEC;                   // x-halo elements each side (16 bytes)
  static constexpr int UW = TX + 2 * PADE + VEC;      // u / s_u row box (elements, + alignment slack)
  static constexpr int RWB = TX + VEC;               // v / s_v / w / s_w row box
  static constexpr int UP = int(((UW * sizeof(T) + 127) / 128) * 128 / sizeof(T));   // smem pitch
  // one thread issues a 1D tensor load every ~72 cycles (tools/tmarate), and
  // a plane takes 6 ty + 4 of them: NP producer warps split the rows
  static constexpr int NP = DIVUQ_FLAT_NP;           // producer warps
  static constexpr int TYMAX = 16 - NP;              // consumer warps (tile rows, max): 16 warps x 128 regs
  static constexpr int S = 4;                        // pipeline stages
  static constexpr int THREADS = 32 * (TYMAX + NP);
};

template <typename T>
struct alignas(128) FlatStage {
  using C = FlatCfg<T>;
  alignas(128) T u[C::TYMAX][C::UP];      // row box: x0 - PADE .. x0 + TX + PADE (+ shift)
  alignas(128) T su[C::TYMAX][C::UP];
  alignas(128) T v[C::TYMAX + 2][C::UP];  // rows y0 - 1 .. y0 + ty (halo rows included)
  alignas(128) T sv[C::TYMAX + 2][C::UP];
  alignas(128) T w[C::TYMAX][C::UP];      // plane k + 1 (the z-march's next w)
  alignas(128) T sw[C::TYMAX][C::UP];
};

enum FlatMap { kFlU, kFlSU, kFlV, kFlSV, kFlW, kFlSW, kNumFlatMaps };
struct FlatMaps {
  CUtensorMap m[kNumFlatMaps];
};

template <typename T>
struct FlatParams {
  const T* mu_w; const T* s_w;                       // z-march restarts (scalar loads)
  const T* halo_lo_mu_w; const T* halo_lo_s_w;
  const T* halo_hi_mu_w; const T* halo_hi_s_w;
  int64_t nzl, z0, nzg, kbeg, kend;
  int nx, ny, ty, tiles_x, n_tiles;
  int n_chunks;                                      // z-chunks per tile column (small planes: > 1)
  int64_t zchunk;
  uint32_t stage_bytes;
  T cx_in, cx_bd, cy_in, cy_bd, cz_in, cz_bd;
  T theta;
  T* out_mu; T* out_sigma; T* out_psrc; T* out_psnk;
  int* err;
};

template <typename T, bool HAS_SIGMA>
struct K2Flat {
  using C = FlatCfg<T>;
  using V = Vec<T, C::VEC>;
  using Stage = FlatStage<T>;
  static constexpr int VEC = C::VEC, TX = C::TX, PADE = C::PADE, S = C::S;

  // w / s_w of local plane kk at this lane's points x + 32 e (scalar loads:
  // rows are not 16-byte aligned); the planes just outside the slab come from
  // the exchange's halo pointers
  static __device__ __forceinline__ void load_w(const FlatParams<T>& p, int64_t kk, int64_t off2d,
                                                int x, bool row_act, V& w, V& sw) {
#pragma unroll
    for (int e = 0; e < VEC; ++e) { w.v[e] = T(0); sw.v[e] = T(0); }
    if (!row_act) return;
    const int64_t plane = int64_t(p.nx) * p.ny;
    const T* bw = nullptr; const T* bs = nullptr;
    if (kk >= 0 && kk < p.nzl) {
      bw = p.mu_w + kk * plane; bs = HAS_SIGMA ? p.s_w + kk * plane : nullptr;
    } else if (kk == -1 && p.z0 > 0) {
      bw = p.halo_lo_mu_w; bs = p.halo_lo_s_w;
    } else if (kk == p.nzl && p.z0 + p.nzl < p.nzg) {
      bw = p.halo_hi_mu_w; bs = p.halo_hi_s_w;
    }
    if (!bw) return;
#pragma unroll
    for (int e = 0; e < VEC; ++e)
      if (x + 32 * e < p.nx) {
        w.v[e] = bw[off2d + 32 * e];
        if constexpr (HAS_SIGMA) sw.v[e] = bs[off2d + 32 * e];
      }
  }

  // element offset r rounded down to a VEC multiple (a 16-byte box start),
  // and the shift r - align_down(r) in [0, VEC) at which the row sits
  static __device__ __forceinline__ int64_t align_down(int64_t r) {
    const int64_t m = ((r % VEC) + VEC) % VEC;
    return r - m;
  }
  static __device__ __forceinline__ int shift_of(int64_t r) { return int(((r % VEC) + VEC) % VEC); }

  // producer warp pw (its elected thread) loads rows r = pw, pw + NP, ... of
  // every box set and arrives on the stage's full barrier with their bytes
  static __device__ void produce(const FlatParams<T>& p, const FlatMaps& fm, Stage* st,
                                 uint64_t* full, uint64_t* empty, int pw) {
    const int64_t plane = int64_t(p.nx) * p.ny;
    constexpr uint32_t comps = HAS_SIGMA ? 2u : 1u;
    const uint32_t na = uint32_t(p.ty > pw ? (p.ty - 1 - pw) / C::NP + 1 : 0);
    const uint32_t nb = uint32_t((p.ty + 1 - pw) / C::NP + 1);
    const uint32_t my_bytes = (na * (C::UW + C::RWB) + nb * C::RWB) * uint32_t(sizeof(T)) * comps;
    int s = 0;
    uint32_t ph = 0;
    for (int item = blockIdx.x; item < p.n_tiles * p.n_chunks; item += gridDim.x) {
      const int tile = item % p.n_tiles, chunk = item / p.n_tiles;
      const int64_t kb = p.kbeg + chunk * p.zchunk, ke = min(p.kend, kb + p.zchunk);
      const int x0 = (tile % p.tiles_x) * TX;
      const int y0 = (tile / p.tiles_x) * p.ty;
      for (int64_t k = kb; k < ke; ++k) {
        mbar_wait_backoff<DIVUQ_FLAT_NS>(&empty[s], ph ^ 1u);
        mbar_expect_tx(&full[s], my_bytes);
        Stage& S_ = st[s];
        const int64_t bk = k * plane + x0, bk1 = (k + 1) * plane + x0;
        for (int r = pw; r < p.ty; r += C::NP) {
          const int64_t ro = int64_t(y0 + r) * p.nx;
          const int cu = int(align_down(bk + ro - PADE)), cw = int(align_down(bk1 + ro));
          tma_load_1d(&S_.u[r][0], &fm.m[kFlU], &full[s], cu);
          tma_load_1d(&S_.w[r][0], &fm.m[kFlW], &full[s], cw);
          if constexpr (HAS_SIGMA) {
            tma_load_1d(&S_.su[r][0], &fm.m[kFlSU], &full[s], cu);
            tma_load_1d(&S_.sw[r][0], &fm.m[kFlSW], &full[s], cw);
          }
        }
        for (int r = pw; r < p.ty + 2; r += C::NP) {
          const int cv = int(align_down(bk + int64_t(y0 - 1 + r) * p.nx));
          tma_load_1d(&S_.v[r][0], &fm.m[kFlV], &full[s], cv);
          if constexpr (HAS_SIGMA) tma_load_1d(&S_.sv[r][0], &fm.m[kFlSV], &full[s], cv);
        }
        if (++s == S) { s = 0; ph ^= 1u; }
      }
    }
  }

  // Consumers: warp ty owns tile row y0 + ty; lane l owns the points
  // x0 + l + 32 e (e < VEC) -- strided, so every shared-memory read (own
  // value and both x neighbours straight from the row box) and every global
  // store is 32 consecutive elements: conflict-free and coalesced.
  static __device__ void consume(const FlatParams<T>& p, Stage* st, uint64_t* full, uint64_t* empty) {
    const int ty = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t plane = int64_t(p.nx) * p.ny;
    const bool validate = p.err != nullptr;
    const bool t_zero = (p.theta == T(0));
    int nonfinite = 0, negative = 0;
    int s = 0;
    uint32_t ph = 0;
    for (int item = blockIdx.x; item < p.n_tiles * p.n_chunks; item += gridDim.x) {
      const int tile = item % p.n_tiles, chunk = item / p.n_tiles;
      const int64_t kb = p.kbeg + chunk * p.zchunk, ke = min(p.kend, kb + p.zchunk);
      const int x0 = (tile % p.tiles_x) * TX;
      const int j = (tile / p.tiles_x) * p.ty + ty;
      const bool row_act = j < p.ny;
      const int64_t off2d = int64_t(j) * p.nx + x0 + lane;   // element e at + 32 e
      const bool jlo = j == 0, jhi = j == p.ny - 1;
      const T cy = (jlo || jhi) ? p.cy_bd : p.cy_in;
      V wm, w0, swm, sw0;
      load_w(p, kb - 1, off2d, x0 + lane, row_act, wm, swm);
      load_w(p, kb, off2d, x0 + lane, row_act, w0, sw0);
      int64_t o = kb * plane + off2d;
      for (int64_t k = kb; k < ke; ++k, o += plane) {
        mbar_wait(&full[s], ph);
        const Stage& S_ = st[s];
        // warp-uniform shifts of this warp's rows inside their boxes
        const int64_t rk = k * plane + int64_t(j) * p.nx;
        const int sh_u = shift_of(rk), sh_lo = shift_of(rk - p.nx), sh_hi = shift_of(rk + p.nx);
        const int sh_w = shift_of(rk + plane);
        const T* ur = &S_.u[ty][sh_u + PADE + lane];
        const T* vlr = &S_.v[ty][sh_lo + lane];
        const T* vor = &S_.v[ty + 1][sh_u + lane];
        const T* vhr = &S_.v[ty + 2][sh_hi + lane];
        const T* wr = &S_.w[ty][sh_w + lane];
        V u_own, u_lo, u_hi, v_lo, v_own, v_hi, wp;
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          u_own.v[e] = ur[32 * e]; u_lo.v[e] = ur[32 * e - 1]; u_hi.v[e] = ur[32 * e + 1];
          v_lo.v[e] = vlr[32 * e]; v_own.v[e] = vor[32 * e]; v_hi.v[e] = vhr[32 * e];
          wp.v[e] = wr[32 * e];
        }
        V su_own, su_lo, su_hi, sv_lo, sv_own, sv_hi, swp;
        if constexpr (HAS_SIGMA) {
          const T* sur = &S_.su[ty][sh_u + PADE + lane];
          const T* svl = &S_.sv[ty][sh_lo + lane];
          const T* svo = &S_.sv[ty + 1][sh_u + lane];
          const T* svh = &S_.sv[ty + 2][sh_hi + lane];
          const T* swr = &S_.sw[ty][sh_w + lane];
#pragma unroll
          for (int e = 0; e < VEC; ++e) {
            su_own.v[e] = sur[32 * e]; su_lo.v[e] = sur[32 * e - 1]; su_hi.v[e] = sur[32 * e + 1];
            sv_lo.v[e] = svl[32 * e]; sv_own.v[e] = svo[32 * e]; sv_hi.v[e] = svh[32 * e];
            swp.v[e] = swr[32 * e];
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);   // stage consumed: the producer may refill it
        if (++s == S) { s = 0; ph ^= 1u; }
        if (k + 1 == p.nzl) load_w(p, k + 1, off2d, x0 + lane, row_act, wp, swp);   // halo or none

        if (row_act) {
          const int64_t kg = p.z0 + k;
          const bool klo = kg == 0, khi = kg == p.nzg - 1;
          const T cz = (klo || khi) ? p.cz_bd : p.cz_in;
          const V& wl = klo ? w0 : wm;
          const V& wh = khi ? w0 : wp;
          const V& swl = klo ? sw0 : swm;
          const V& swh = khi ? sw0 : swp;
          using SM = StencilMath<T, true>;
#pragma unroll
          for (int e = 0; e < VEC; ++e) {
            const int i = x0 + lane + 32 * e;
            if (i >= p.nx) break;
            const bool ilo = i == 0, ihi = i == p.nx - 1;
            const T cx = (ilo || ihi) ? p.cx_bd : p.cx_in;
            const T own = u_own.v[e];
            const T ul = ilo ? own : u_lo.v[e];
            const T uh = ihi ? own : u_hi.v[e];
            const T vl = jlo ? v_own.v[e] : v_lo.v[e];
            const T vh = jhi ? v_own.v[e] : v_hi.v[e];
            const T m = SM::mean(uh, ul, vh, vl, wh.v[e], wl.v[e], cx, cy, cz);
            if (p.out_mu) __stcs(p.out_mu + o + 32 * e, m);
            if (validate)
              nonfinite |= int(!isfinite(own)) | int(!isfinite(v_own.v[e])) | int(!isfinite(w0.v[e]));
            if constexpr (HAS_SIGMA) {
              const T sown = su_own.v[e];
              const T sl = ilo ? sown : su_lo.v[e];
              const T sh = ihi ? sown : su_hi.v[e];
              const T svl = jlo ? sv_own.v[e] : sv_lo.v[e];
              const T svh = jhi ? sv_own.v[e] : sv_hi.v[e];
              T sg, ps, pk;
              Tails<T>::eval(m, SM::var(sh, sl, svh, svl, swh.v[e], swl.v[e], cx, cy, cz), p.theta,
                             t_zero, sg, ps, pk);
              if (p.out_sigma) __stcs(p.out_sigma + o + 32 * e, sg);
              if (p.out_psrc) __stcs(p.out_psrc + o + 32 * e, ps);
              if (p.out_psnk) __stcs(p.out_psnk + o + 32 * e, pk);
              if (validate) {
                nonfinite |= int(!isfinite(sown)) | int(!isfinite(sv_own.v[e])) | int(!isfinite(sw0.v[e]));
                negative |= int(sown < T(0)) | int(sv_own.v[e] < T(0)) | int(sw0.v[e] < T(0));
              }
            }
          }
        }
        wm = w0; w0 = wp;
        if constexpr (HAS_SIGMA) { swm = sw0; sw0 = swp; }
      }
    }
    if (validate) flush_error(p.err, (nonfinite ? kErrNonFinite : 0) | (negative ? kErrNegativeSigma : 0));
  }
};

template <typename T, bool HAS_SIGMA>
__global__ void __launch_bounds__(FlatCfg<T>::THREADS, 1)
k2_flat_kernel(const __grid_constant__ FlatMaps fm, const FlatParams<T> p) {
  using C = FlatCfg<T>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  auto* st = reinterpret_cast<FlatStage<T>*>(smem_raw);
  auto* bars = reinterpret_cast<uint64_t*>(smem_raw + sizeof(FlatStage<T>) * C::S);
  uint64_t* full = bars;
  uint64_t* empty = bars + C::S;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::S; ++s) {
      mbar_init(&full[s], C::NP);   // one expect_tx arrival per producer warp
      mbar_init(&empty[s], uint32_t(p.ty));
    }
    mbar_fence_init();
  }
  if (warp == C::TYMAX && (threadIdx.x & 31) < kNumFlatMaps) tma_prefetch_desc(&fm.m[threadIdx.x & 31]);
  __syncthreads();
  if (warp >= C::TYMAX) {
    if ((threadIdx.x & 31) == 0) K2Flat<T, HAS_SIGMA>::produce(p, fm, st, full, empty, warp - C::TYMAX);
  } else if (warp < p.ty) {
    K2Flat<T, HAS_SIGMA>::consume(p, st, full, empty);
  }
}

}  // namespace divuq
