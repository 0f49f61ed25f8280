// K2 (3D, TMA pipeline): the HBM-bound hot kernel of BASELINE config 3.
//
// Same arithmetic as stencil.cuh (StencilMath / Tails in common.cuh: the
// reference's op order in fp64, stencils.py:54-84, tails lcp.py:48-68) with
// Blackwell-native data movement:
//
//   * warp-specialised persistent CTA (one per SM): TY consumer warps, one
//     producer warp and one pacer warp; an S-stage shared-memory ring guarded
//     by mbarriers;
//   * per plane the producer issues 3D TMA box loads (cp.async.bulk.tensor):
//       main boxes  u, v, w(k+1) [and s_u, s_v, s_w]: the tile's own TX x TY
//                   points, 512-byte aligned rows;
//       halo boxes  u / s_u: 4 columns left and right of the tile;
//                   v / s_v: the row above and the row below.
//     Out-of-grid box parts are zero-filled by the TMA unit, so the producer
//     never branches on borders;
//   * the halo boxes of plane k are issued hdelay (2) stages after its main
//     boxes, and the pacer keeps every CTA within W planes of its four
//     neighbour tiles (consumer warp 0 publishes "planes consumed"; bounded
//     wait, never a correctness dependency).  So the neighbour has just pulled
//     the halo bytes into L2 with its own main box: halos cost L2 bandwidth,
//     not HBM bandwidth (without the pacer CTAs drift tens of planes apart
//     over a long march and every halo byte came from DRAM, +10 % reads);
//   * consumers (one grid row per warp, VEC points per lane) take their
//     operands from the stage (x neighbours by warp shuffle), keep w[k-1],
//     w[k] in registers (z-march), evaluate mean, sigma and both tails on ONE
//     branch-free path (boundary points by operand substitution) and stream
//     the four outputs to HBM;
//   * scheduling: a CTA owns whole tile COLUMNS (all planes of a tile) and
//     the host picks the tile height TY so #tiles is (close to) a multiple of
//     the SM count.
//
// Slab sharding: planes are slab-local; w at local planes -1 / nzl comes from
// the halo pointers (a neighbour's edge plane: exchanged, or read in place
// through a peer mapping), read with plain loads.
#pragma once

#include "common.cuh"
#include "tma.cuh"

#ifndef DIVUQ_K2_TYMAX
#define DIVUQ_K2_TYMAX 15
#endif
// fp64: 14 consumer rows keep the CTA at 16 warps, where the register
// allocation allows 128 per thread (17 warps: 96, and the fp64 consumers
// spilled); config 3's tile height is 14 either way.  fp64 config 3:
// 2.03 -> 1.91 ms.  (fp32 keeps 15: measured no better at 14.)
#ifndef DIVUQ_K2_TYMAX_F64
#define DIVUQ_K2_TYMAX_F64 14
#endif

namespace divuq {

template <typename T>
struct TmaCfg {
  static constexpr int VEC = 16 / int(sizeof(T));  // 4 x fp32 or 2 x fp64 per lane
  static constexpr int TX = 32 * VEC;               // tile width (points)
  static constexpr int PAD = VEC;                    // x-halo box width (16 bytes)
  static constexpr int TYMAX = sizeof(T) == 8 ? DIVUQ_K2_TYMAX_F64 : DIVUQ_K2_TYMAX;   // consumer warps
  static constexpr int S = 4;                        // pipeline stages
  static constexpr int D = 3;                        // max stages the halo boxes may trail (runtime hdelay)
  static constexpr int THREADS = 32 * (TYMAX + 2);  // + producer warp + pacer warp
};

template <typename T>
struct alignas(128) TmaStage {
  using C = TmaCfg<T>;
  // every TMA destination must be 128-byte aligned
  // main boxes (rows of TX, dense)
  alignas(128) T u[C::TYMAX][C::TX];
  alignas(128) T v[C::TYMAX][C::TX];
  alignas(128) T w[C::TYMAX][C::TX];
  alignas(128) T su[C::TYMAX][C::TX];
  alignas(128) T sv[C::TYMAX][C::TX];
  alignas(128) T sw[C::TYMAX][C::TX];
  // halo boxes
  alignas(128) T v_top[C::TX];
  alignas(128) T v_bot[C::TX];
  alignas(128) T sv_top[C::TX];
  alignas(128) T sv_bot[C::TX];
  alignas(128) T u_l[C::TYMAX][C::PAD];
  alignas(128) T u_r[C::TYMAX][C::PAD];
  alignas(128) T su_l[C::TYMAX][C::PAD];
  alignas(128) T su_r[C::TYMAX][C::PAD];
};

// tensor maps, one per (array, box shape)
enum TmaMap { kMapU, kMapV, kMapW, kMapSU, kMapSV, kMapSW, kMapUH, kMapVH, kMapSUH, kMapSVH, kNumMaps };

struct TmaMaps {
  CUtensorMap m[kNumMaps];
};

template <typename T>
struct TmaParams {
  const T* mu_w; const T* s_w;                      // for the z-march restarts
  const T* halo_lo_mu_w; const T* halo_lo_s_w;
  const T* halo_hi_mu_w; const T* halo_hi_s_w;
  int64_t nzl, z0, nzg, kbeg, kend;
  int nx, ny, ty, tiles_x, n_tiles;
  int n_chunks;                                      // z-chunks per tile column (small planes: > 1)
  int64_t zchunk;                                    // planes per chunk
  uint32_t stage_bytes;                              // TMA bytes per stage (depends on ty)
  int hdelay;                                        // halo boxes trail the main boxes by this many stages (<= D)
  int halo_off;                                      // diagnostics only: skip halo boxes (wrong edges; traffic attribution)
  unsigned long long* progress;                      // per-tile progress flags (nullptr: no lockstep)
  unsigned long long epoch;                          // launch tag in the flags' high word
  int sync_w;                                        // max planes ahead of a neighbour tile
  int sync_spin;                                     // bounded wait: polls before giving up
  int sync_sleep;                                    // ns between polls
  int pf_dist;                                       // L2 prefetch distance in planes (0: off)
  int diag_null;                                     // diagnostics only: skip the math
  T cx_in, cx_bd, cy_in, cy_bd, cz_in, cz_bd;
  T theta;
  T* out_mu; T* out_sigma; T* out_psrc; T* out_psnk;
  int* err;
};

template <typename T, bool HAS_SIGMA, bool HAS_W = true>
struct K2Tma {
  using C = TmaCfg<T>;
  using V = Vec<T, C::VEC>;
  using A = Arith<T>;
  using Stage = TmaStage<T>;
  static constexpr int VEC = C::VEC, TX = C::TX, S = C::S, PAD = C::PAD, D = C::D;

  static __device__ __forceinline__ V zero() {
    V r;
#pragma unroll
    for (int e = 0; e < VEC; ++e) r.v[e] = T(0);
    return r;
  }
  static __device__ __forceinline__ V lds(const T* p) { return *reinterpret_cast<const V*>(p); }

  // w / s_w of local plane kk at this lane's points by plain loads
  static __device__ __forceinline__ void load_w(const TmaParams<T>& p, int64_t kk, int64_t off2d,
                                                bool act, V& w, V& sw) {
    w = zero(); sw = zero();
    if (!act) return;
    const int64_t plane = int64_t(p.nx) * p.ny;
    const T* bw = nullptr; const T* bs = nullptr;
    if (kk >= 0 && kk < p.nzl) {
      bw = p.mu_w + kk * plane; bs = HAS_SIGMA ? p.s_w + kk * plane : nullptr;
    } else if (kk == -1 && p.z0 > 0) {
      bw = p.halo_lo_mu_w; bs = p.halo_lo_s_w;
    } else if (kk == p.nzl && p.z0 + p.nzl < p.nzg) {
      bw = p.halo_hi_mu_w; bs = p.halo_hi_s_w;
    }
    if (bw) {
      w = ldg_vec<T, VEC>(bw + off2d);
      if constexpr (HAS_SIGMA) sw = ldg_vec<T, VEC>(bs + off2d);
    }
  }

  template <bool B>
  static __device__ __forceinline__ void point(const TmaParams<T>& p, T ul, T uh, T vl, T vh, T wl,
                                               T wh, T sl, T sh, T svl, T svh, T swl, T swh,
                                               T cx, T cy, T cz, bool t_zero, T& m, T& sg, T& ps,
                                               T& pk) {
    using SM = StencilMath<T, HAS_W>;   // 2D (HAS_W false): the reference's 2D order
    m = SM::mean(uh, ul, vh, vl, wh, wl, cx, cy, cz);
    if constexpr (HAS_SIGMA)
      Tails<T>::eval(m, SM::var(sh, sl, svh, svl, swh, swl, cx, cy, cz), p.theta, t_zero, sg, ps, pk);
  }

  struct Pending { int x0, y0, k, s; };

  static __device__ __forceinline__ void issue_main(const TmaMaps& tm, Stage& st, uint64_t* bar,
                                                    int x0, int y0, int k) {
    tma_load_3d(&st.u[0][0], &tm.m[kMapU], bar, x0, y0, k);
    tma_load_3d(&st.v[0][0], &tm.m[kMapV], bar, x0, y0, k);
    if constexpr (HAS_W) tma_load_3d(&st.w[0][0], &tm.m[kMapW], bar, x0, y0, k + 1);
    if constexpr (HAS_SIGMA) {
      tma_load_3d(&st.su[0][0], &tm.m[kMapSU], bar, x0, y0, k);
      tma_load_3d(&st.sv[0][0], &tm.m[kMapSV], bar, x0, y0, k);
      if constexpr (HAS_W) tma_load_3d(&st.sw[0][0], &tm.m[kMapSW], bar, x0, y0, k + 1);
    }
  }

  static __device__ __forceinline__ void prefetch_main(const TmaMaps& tm, int x0, int y0, int k) {
    tma_prefetch_l2_3d(&tm.m[kMapU], x0, y0, k);
    tma_prefetch_l2_3d(&tm.m[kMapV], x0, y0, k);
    if constexpr (HAS_W) tma_prefetch_l2_3d(&tm.m[kMapW], x0, y0, k + 1);
    if constexpr (HAS_SIGMA) {
      tma_prefetch_l2_3d(&tm.m[kMapSU], x0, y0, k);
      tma_prefetch_l2_3d(&tm.m[kMapSV], x0, y0, k);
      if constexpr (HAS_W) tma_prefetch_l2_3d(&tm.m[kMapSW], x0, y0, k + 1);
    }
  }

  static __device__ __forceinline__ void issue_halo(const TmaMaps& tm, Stage& st, uint64_t* bar,
                                                    int x0, int y0, int k, int ty) {
    tma_load_3d(&st.u_l[0][0], &tm.m[kMapUH], bar, x0 - PAD, y0, k);
    tma_load_3d(&st.u_r[0][0], &tm.m[kMapUH], bar, x0 + TX, y0, k);
    tma_load_3d(&st.v_top[0], &tm.m[kMapVH], bar, x0, y0 - 1, k);
    tma_load_3d(&st.v_bot[0], &tm.m[kMapVH], bar, x0, y0 + ty, k);
    if constexpr (HAS_SIGMA) {
      tma_load_3d(&st.su_l[0][0], &tm.m[kMapSUH], bar, x0 - PAD, y0, k);
      tma_load_3d(&st.su_r[0][0], &tm.m[kMapSUH], bar, x0 + TX, y0, k);
      tma_load_3d(&st.sv_top[0], &tm.m[kMapSVH], bar, x0, y0 - 1, k);
      tma_load_3d(&st.sv_bot[0], &tm.m[kMapSVH], bar, x0, y0 + ty, k);
    }
  }

  static __device__ void produce(const TmaParams<T>& p, const TmaMaps& tm, Stage* st,
                                 uint64_t* full, uint64_t* empty, volatile int* permit) {
    Pending pend[D + 1];
    int n_pend = 0, head = 0;
    int s = 0;
    uint32_t ph = 0;
    const int hd = p.hdelay;
    // loose lockstep: only when every tile has its own resident CTA
    const bool sync = p.progress != nullptr && p.n_tiles <= int(gridDim.x) && p.n_chunks == 1;
    for (int item = blockIdx.x; item < p.n_tiles * p.n_chunks; item += gridDim.x) {
      const int tile = item % p.n_tiles, chunk = item / p.n_tiles;
      const int x0 = (tile % p.tiles_x) * TX;
      const int y0 = (tile / p.tiles_x) * p.ty;
      const int kb = int(p.kbeg + chunk * p.zchunk);
      const int ke = int(min(p.kend, p.kbeg + (chunk + 1) * p.zchunk));
      for (int k = kb; k < ke; ++k) {
        if (sync)   // the pacer warp grants planes (neighbour-progress window)
          while (int(k - p.kbeg) >= *permit) __nanosleep(32);
        if (p.pf_dist > 0) {   // keep pf_dist planes of this tile on their way into L2
          if (k == kb)
            for (int q = 1; q < p.pf_dist && k + q < ke; ++q) prefetch_main(tm, x0, y0, k + q);
          if (k + p.pf_dist < ke) prefetch_main(tm, x0, y0, k + p.pf_dist);
        }
        mbar_wait_backoff(&empty[s], ph ^ 1u);
        mbar_expect_tx(&full[s], p.stage_bytes);
        issue_main(tm, st[s], &full[s], x0, y0, k);
        pend[(head + n_pend) % (D + 1)] = Pending{x0, y0, k, s};
        ++n_pend;
        if (n_pend > hd) {  // the oldest pending stage gets its halos now (hd stages late)
          const Pending q = pend[head];
          if (!p.halo_off) issue_halo(tm, st[q.s], &full[q.s], q.x0, q.y0, q.k, p.ty);
          head = (head + 1) % (D + 1);
          --n_pend;
        }
        if (++s == S) { s = 0; ph ^= 1u; }
      }
    }
    for (int i = 0; i < n_pend; ++i) {
      const Pending q = pend[(head + i) % (D + 1)];
      if (!p.halo_off) issue_halo(tm, st[q.s], &full[q.s], q.x0, q.y0, q.k, p.ty);
    }
  }

  // Pacer warp (lane 0): polls the neighbour tiles' progress flags (planes
  // their consumers have finished; published by consumer warp 0 -- a store
  // from the producer thread would queue behind its bulk copies) and grants
  // the producer planes up to (slowest neighbour + W).  Kept off the producer
  // thread: a global load there would wait behind its outstanding bulk copies.
  // Bounded: after sync_spin polls without a change it grants everything.
  static __device__ void pace(const TmaParams<T>& p, volatile int* permit) {
    const int tile = blockIdx.x;
    const int nplanes = int(p.kend - p.kbeg);
    const int tcol = tile % p.tiles_x;
    int nb[4], n_nb = 0;
    if (tcol > 0) nb[n_nb++] = tile - 1;
    if (tcol + 1 < p.tiles_x && tile + 1 < p.n_tiles) nb[n_nb++] = tile + 1;
    if (tile >= p.tiles_x) nb[n_nb++] = tile - p.tiles_x;
    if (tile + p.tiles_x < p.n_tiles) nb[n_nb++] = tile + p.tiles_x;
    int granted = p.sync_w + 1, idle = 0;
    *permit = granted;
    while (granted < nplanes) {
      unsigned long long f[4];
      // weak L2-only loads (ld.global.cg): a .gpu-scope strong load here measurably
      // stalls the SM's memory pipeline (sweep in DESIGN.md); L2 is the coherence point
      for (int q = 0; q < 4; ++q) f[q] = q < n_nb ? __ldcg(p.progress + size_t(nb[q]) * kFlagStride) : 0ull;
      int lo = nplanes;
      for (int q = 0; q < n_nb; ++q) {
        const int c = (f[q] >> 32) == (p.epoch & 0xffffffffull) ? int(f[q] & 0xffffffffull) : 0;
        lo = min(lo, c);
      }
      const int g = min(nplanes, lo + p.sync_w + 1);
      if (g > granted) { granted = g; *permit = granted; idle = 0; }
      else if (++idle >= p.sync_spin) { granted = nplanes; *permit = granted; }
      __nanosleep(p.sync_sleep);
    }
  }

  static __device__ void consume(const TmaParams<T>& p, Stage* st, uint64_t* full,
                                 uint64_t* empty) {
    const int ty = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cx0 = lane * VEC;
    const int64_t plane = int64_t(p.nx) * p.ny;
    const bool validate = p.err != nullptr;
    const bool t_zero = (p.theta == T(0));
    const bool top = ty == 0, bot = ty == p.ty - 1;
    const bool sync = p.progress != nullptr && p.n_tiles <= int(gridDim.x) && p.n_chunks == 1;
    int errbits = 0;
    int s = 0;
    uint32_t ph = 0;
    for (int item = blockIdx.x; item < p.n_tiles * p.n_chunks; item += gridDim.x) {
      const int tile = item % p.n_tiles, chunk = item / p.n_tiles;
      const int64_t kb = p.kbeg + chunk * p.zchunk, ke = min(p.kend, kb + p.zchunk);
      const int x0 = (tile % p.tiles_x) * TX;
      const int j = (tile / p.tiles_x) * p.ty + ty;
      const int xi = x0 + cx0;
      const bool act = xi < p.nx && j < p.ny;
      const int64_t off2d = int64_t(j) * p.nx + xi;
      // Boundary handling is folded into ONE branch-free path (no divergent
      // slow path): the one-sided rule of stencils.py:46-51 is "lo or hi is the
      // point itself, c = 1/h".  With nx % VEC == 0 only element 0 of the lane
      // holding x = 0 and element VEC-1 of the lane holding x = nx-1 can be x
      // boundaries: they get their own coefficient and the shuffled neighbour
      // is replaced by the point itself.  Row / plane boundaries are
      // warp- / plane-uniform: the neighbour row / plane is replaced the same way.
      const bool x_lo_edge = xi == 0, x_hi_edge = xi + VEC == p.nx;
      const T cx_first = x_lo_edge ? p.cx_bd : p.cx_in;
      const T cx_last = x_hi_edge ? p.cx_bd : p.cx_in;
      const bool jlo = j == 0, jhi = j == p.ny - 1;
      const T cy = (jlo || jhi) ? p.cy_bd : p.cy_in;
      // byte offsets (within a stage) of this lane's v / s_v rows below and above
      const char* const sb0 = reinterpret_cast<const char*>(&st[0]);
      const uint32_t off_own = uint32_t(reinterpret_cast<const char*>(&st[0].v[ty][cx0]) - sb0);
      const uint32_t off_vlo = jlo ? off_own
                               : top ? uint32_t(reinterpret_cast<const char*>(&st[0].v_top[cx0]) - sb0)
                                     : off_own - uint32_t(sizeof(T) * TX);
      const uint32_t off_vhi = jhi ? off_own
                               : bot ? uint32_t(reinterpret_cast<const char*>(&st[0].v_bot[cx0]) - sb0)
                                     : off_own + uint32_t(sizeof(T) * TX);
      const uint32_t d_sv = uint32_t(reinterpret_cast<const char*>(&st[0].sv[0][0]) -
                                     reinterpret_cast<const char*>(&st[0].v[0][0]));
      const uint32_t d_svhalo = uint32_t(reinterpret_cast<const char*>(&st[0].sv_top[0]) -
                                         reinterpret_cast<const char*>(&st[0].v_top[0]));
      const uint32_t off_svlo = (!jlo && top) ? off_vlo + d_svhalo : off_vlo + d_sv;
      const uint32_t off_svhi = (!jhi && bot) ? off_vhi + d_svhalo : off_vhi + d_sv;
      V wm = zero(), w0 = zero(), swm = zero(), sw0 = zero();
      if constexpr (HAS_W) {
        load_w(p, kb - 1, off2d, act, wm, swm);
        load_w(p, kb, off2d, act, w0, sw0);
      }
      int64_t o = kb * plane + off2d;
      for (int64_t k = kb; k < ke; ++k, o += plane) {
        mbar_wait(&full[s], ph);
        const Stage& S_ = st[s];
        const char* sb = reinterpret_cast<const char*>(&S_);
        const V u_own = lds(&S_.u[ty][cx0]);
        const V v_own = validate ? lds(&S_.v[ty][cx0]) : zero();   // validation only
        const V v_lo = lds(reinterpret_cast<const T*>(sb + off_vlo));
        const V v_hi = lds(reinterpret_cast<const T*>(sb + off_vhi));
        V wp = HAS_W ? lds(&S_.w[ty][cx0]) : zero();
        T u_l = __shfl_up_sync(0xffffffffu, u_own.v[VEC - 1], 1);
        T u_r = __shfl_down_sync(0xffffffffu, u_own.v[0], 1);
        if (lane == 0) u_l = S_.u_l[ty][PAD - 1];
        if (lane == 31) u_r = S_.u_r[ty][0];
        V su_own = zero(), sv_own = zero(), sv_lo = zero(), sv_hi = zero(), swp = zero();
        T s_l = T(0), s_r = T(0);
        if constexpr (HAS_SIGMA) {
          su_own = lds(&S_.su[ty][cx0]);
          if (validate) sv_own = lds(&S_.sv[ty][cx0]);
          sv_lo = lds(reinterpret_cast<const T*>(sb + off_svlo));
          sv_hi = lds(reinterpret_cast<const T*>(sb + off_svhi));
          if constexpr (HAS_W) swp = lds(&S_.sw[ty][cx0]);
          s_l = __shfl_up_sync(0xffffffffu, su_own.v[VEC - 1], 1);
          s_r = __shfl_down_sync(0xffffffffu, su_own.v[0], 1);
          if (lane == 0) s_l = S_.su_l[ty][PAD - 1];
          if (lane == 31) s_r = S_.su_r[ty][0];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);   // stage consumed: the producer may refill it
        if (ty == 0 && lane == 0 && sync)        // publish progress (planes consumed) for the pacers
          st_relaxed_u64(p.progress + size_t(tile) * kFlagStride,
                         ((p.epoch & 0xffffffffull) << 32) | (unsigned long long)(k - p.kbeg + 1));
        if (++s == S) { s = 0; ph ^= 1u; }
        if (HAS_W && k + 1 == p.nzl) load_w(p, k + 1, off2d, act, wp, swp);  // past the slab: halo or none

        if (act && p.diag_null) {   // diagnostics: pipeline + stores only, no math
          V z;
#pragma unroll
          for (int e = 0; e < VEC; ++e) z.v[e] = u_own.v[e] + v_lo.v[e] + wp.v[e] + su_own.v[e];
          st_stream<T, VEC>(p.out_mu + o, z);
          st_stream<T, VEC>(p.out_sigma + o, z);
          st_stream<T, VEC>(p.out_psrc + o, z);
          st_stream<T, VEC>(p.out_psnk + o, z);
        } else if (act) {
          const int64_t kg = p.z0 + k;
          const bool klo = kg == 0, khi = kg == p.nzg - 1;
          const T cz = (klo || khi) ? p.cz_bd : p.cz_in;
          // one-sided substitutions (lane / plane uniform)
          if (x_lo_edge) { u_l = u_own.v[0]; s_l = su_own.v[0]; }
          if (x_hi_edge) { u_r = u_own.v[VEC - 1]; s_r = su_own.v[VEC - 1]; }
          const V& wl = klo ? w0 : wm;
          const V& wh = khi ? w0 : wp;
          const V& swl = klo ? sw0 : swm;
          const V& swh = khi ? sw0 : swp;
          V omu, osg, ops, opk;
#pragma unroll
          for (int e = 0; e < VEC; ++e) {
            const T cx = e == 0 ? cx_first : (e == VEC - 1 ? cx_last : p.cx_in);
            const T ul = e == 0 ? u_l : u_own.v[e == 0 ? 0 : e - 1];
            const T uh = e == VEC - 1 ? u_r : u_own.v[e == VEC - 1 ? 0 : e + 1];
            const T sl = e == 0 ? s_l : su_own.v[e == 0 ? 0 : e - 1];
            const T sh = e == VEC - 1 ? s_r : su_own.v[e == VEC - 1 ? 0 : e + 1];
            point<false>(p, ul, uh, v_lo.v[e], v_hi.v[e], wl.v[e], wh.v[e], sl, sh, sv_lo.v[e],
                         sv_hi.v[e], swl.v[e], swh.v[e], cx, cy, cz, t_zero, omu.v[e], osg.v[e],
                         ops.v[e], opk.v[e]);
          }
          if (validate) {
#pragma unroll
            for (int e = 0; e < VEC; ++e) {
              errbits |= check_value(u_own.v[e]) | check_value(v_own.v[e]) | check_value(w0.v[e]);
              if constexpr (HAS_SIGMA)
                errbits |= check_sigma(su_own.v[e]) | check_sigma(sv_own.v[e]) | check_sigma(sw0.v[e]);
              // (2D: w0 / sw0 are zeros, so their checks never fire)
            }
          }
          if (p.out_mu) st_stream<T, VEC>(p.out_mu + o, omu);
          if constexpr (HAS_SIGMA) {
            if (p.out_sigma) st_stream<T, VEC>(p.out_sigma + o, osg);
            if (p.out_psrc) st_stream<T, VEC>(p.out_psrc + o, ops);
            if (p.out_psnk) st_stream<T, VEC>(p.out_psnk + o, opk);
          }
        }
        wm = w0; w0 = wp;
        if constexpr (HAS_SIGMA) { swm = sw0; sw0 = swp; }
      }
    }
    if (validate) flush_error(p.err, errbits);
  }
};

template <typename T, bool HAS_SIGMA, bool HAS_W = true>
__global__ void __launch_bounds__(TmaCfg<T>::THREADS, 1)
k2_tma_kernel(const __grid_constant__ TmaMaps tm, const TmaParams<T> p) {
  using C = TmaCfg<T>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  auto* st = reinterpret_cast<TmaStage<T>*>(smem_raw);
  auto* bars = reinterpret_cast<uint64_t*>(smem_raw + sizeof(TmaStage<T>) * C::S);
  uint64_t* full = bars;
  uint64_t* empty = bars + C::S;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], uint32_t(p.ty));
    }
    mbar_fence_init();
  }
  if (warp == C::TYMAX && (threadIdx.x & 31) < kNumMaps) tma_prefetch_desc(&tm.m[threadIdx.x & 31]);
  __syncthreads();
  __shared__ int permit;
  const bool sync = p.progress != nullptr && p.n_tiles <= int(gridDim.x) && p.n_chunks == 1;
  if (threadIdx.x == 0) permit = sync ? 0 : 0x7fffffff;
  __syncthreads();
  if (warp == C::TYMAX) {
    if ((threadIdx.x & 31) == 0) K2Tma<T, HAS_SIGMA, HAS_W>::produce(p, tm, st, full, empty, &permit);
    return;
  }
  if (warp == C::TYMAX + 1) {
    if ((threadIdx.x & 31) == 0 && sync) K2Tma<T, HAS_SIGMA, HAS_W>::pace(p, &permit);
    return;
  }
  if (warp >= p.ty) return;  // tile shorter than TYMAX: spare warps sit out
  K2Tma<T, HAS_SIGMA, HAS_W>::consume(p, st, full, empty);
}

}  // namespace divuq
