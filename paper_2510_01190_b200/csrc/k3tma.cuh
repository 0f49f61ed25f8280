// K3 (3D fused ensemble, TMA member stream): BASELINE config 4's hot kernel.
//
// fit_gaussian (gaussian.py:35-45) -> propagate_divergence (divergence.py:
// 48-70) -> tails (lcp.py:48-68) in one pass over the (M, 3, N) member slab.
// Bytes per point: 3*M*4 in (192 at M = 16) + 16 out; the members are read
// once and the moments never touch HBM (unless the caller asks for them).
//
//   * warp-specialised persistent CTA, 16 warps: TY consumer warps (one tile
//     row each), one halo warp, one producer warp; an S-stage ring where every
//     stage carries ONE member's box of ONE component of one plane (TX x TY
//     fp32 + halos, ~8 KB), ~150 KB of member data in flight per SM;
//   * per plane the producer streams u(k) x M, v(k) x M, w(k+1) x M boxes
//     (5D TMA on the (x, y, plane, component, member) view); the u boxes'
//     4-column x-halos and the v boxes' halo rows are separate small boxes
//     issued with their main box (hdelay 0: a trailing halo would delay the
//     stage it completes, and the ring depth is worth more -- measured; the
//     delay and a K2-style lockstep pacer remain as knobs);
//   * consumers fold each member into per-point shifted single-pass moment
//     accumulators (ShiftedMoments, common.cuh) and release the stage at
//     once; the halo warp does the same for the tile's halo points (2*TY
//     x-halo columns, 2 halo rows) and publishes their moments in shared
//     memory; u moments' x-neighbours come by warp shuffle, v moments' rows
//     through a small double-buffered shared tile, w moments roll in
//     registers along z;
//   * then the same StencilMath / Tails as K2 (common.cuh) per point.
//
// Slab sharding: the w moments of the planes just outside the slab come from
// the halo pointers (the neighbour reduces its edge plane with K1 -- same
// ShiftedMoments -- and sends 2 planes instead of 2*M).
#pragma once

#include "common.cuh"
#include "tma.cuh"

namespace divuq {

struct K3Cfg {
  static constexpr int VEC = 4;
  static constexpr int TX = 128;
  static constexpr int PAD = 4;
  static constexpr int TYMAX = 14;   // consumer warps; + halo warp + producer = 16 -> 128 regs
  static constexpr int HALO_WARP = TYMAX;
  static constexpr int PROD_WARP = TYMAX + 1;
#ifndef DIVUQ_K3_MB
#define DIVUQ_K3_MB 4
#endif
#ifndef DIVUQ_K3_S
#define DIVUQ_K3_S 5
#endif
  static constexpr int MB = DIVUQ_K3_MB;   // members per stage (one 5D TMA box)
  static constexpr int S = DIVUQ_K3_S;     // stages of MB member boxes
  static constexpr int D = 3;        // halo boxes trail their main box by D stages
  static constexpr int THREADS = 32 * (TYMAX + 2);
};

// One stage = MB members of one component of one plane.  A 5D box
// {TX, TY, 1, 1, MB} lands densely as [MB][TY][TX] (TY = the runtime tile
// height), so member mb, row r starts at (mb*TY + r)*TX.
struct alignas(128) K3Stage {  // every TMA destination 128-byte aligned
  alignas(128) float main[K3Cfg::MB * K3Cfg::TYMAX * K3Cfg::TX];
  alignas(128) float hl[K3Cfg::MB * K3Cfg::TYMAX * K3Cfg::PAD];
  alignas(128) float hr[K3Cfg::MB * K3Cfg::TYMAX * K3Cfg::PAD];
  alignas(128) float top[K3Cfg::MB * K3Cfg::TX];
  alignas(128) float bot[K3Cfg::MB * K3Cfg::TX];
};

struct K3Pending { int idx, x0, y0, k, m0, s, comp, pad; };

struct K3Xchg {
  // v moments of the tile rows (1..TY) + the halo rows (0, TY+1)
  float mu[2][K3Cfg::TYMAX + 2][K3Cfg::TX];
  float sg[2][K3Cfg::TYMAX + 2][K3Cfg::TX];
  // u moments at the x-halo columns: [buf][left/right][row]
  float uh_mu[2][2][K3Cfg::TYMAX];
  float uh_sg[2][2][K3Cfg::TYMAX];
  K3Pending pend[K3Cfg::D + 1];  // producer-private halo queue
  // each consumer lane's w moments of plane k-1 (kept out of registers)
  Vec<float, 4> wm[K3Cfg::TYMAX][2][32];
};

enum K3Map { kK3Main, kK3HaloX, kK3HaloY, kK3NumMaps };
struct K3Maps {
  CUtensorMap m[kK3NumMaps];
};

struct K3Params {
  const float* halo_lo_mu_w; const float* halo_lo_s_w;   // reduced w moments
  const float* halo_hi_mu_w; const float* halo_hi_s_w;
  int64_t nzl, z0, nzg, kbeg, kend;
  int64_t comp_stride;                                   // Nl = nx*ny*nzl
  int nx, ny, ty, tiles_x, n_tiles, M;
  int has_w;                                             // 0: 2D ensemble (u, v only)
  int hdelay;                                            // halo boxes trail by this many items (<= D)
  unsigned long long* progress;                          // per-tile progress flags (nullptr: no lockstep)
  unsigned long long epoch;                              // launch tag in the flags' high word
  int sync_w, sync_spin, sync_sleep;                     // window (planes), bounded polls, ns per poll
  uint32_t bytes_u, bytes_v, bytes_w;
  float cx_in, cx_bd, cy_in, cy_bd, cz_in, cz_bd;
  float theta;
  float* out_mu; float* out_sigma; float* out_psrc; float* out_psnk;
  float* out_mom_mu; float* out_mom_sigma;               // (3, Nl) or null
  int* err;
};

enum K3Comp { kU = 0, kV = 1, kW = 2 };

struct K3 {
  using C = K3Cfg;
  using V4 = Vec<float, 4>;
  static constexpr int TX = C::TX, PAD = C::PAD, S = C::S, D = C::D;

  static constexpr int MB = C::MB;

  // The item sequence of one tile -- mirrored exactly by producer, consumers
  // and halo warp (an item = a block of MB members, NB = ceil(M/MB) blocks):
  // [w(kb-1) x NB if kb > 0] [w(kb) x NB] then per plane k:
  // u(k) x NB, v(k) x NB, [w(k+1) x NB if k+1 < nzl].
  static __device__ __forceinline__ int n_blocks(const K3Params& p) { return (p.M + MB - 1) / MB; }

  // ---------------------------------------------------------------- producer
  static __device__ void produce(const K3Params& p, const K3Maps& tm, K3Stage* st, uint64_t* full,
                                 uint64_t* empty, K3Pending* q) {
    int qh = 0, qn = 0, s = 0, idx = 0;
    uint32_t ph = 0;
    auto halo = [&](const K3Pending& e) {
      K3Stage& t = st[e.s];
      if (e.comp == kU) {
        tma_load_5d(&t.hl[0], &tm.m[kK3HaloX], &full[e.s], e.x0 - PAD, e.y0, e.k, kU, e.m0);
        tma_load_5d(&t.hr[0], &tm.m[kK3HaloX], &full[e.s], e.x0 + TX, e.y0, e.k, kU, e.m0);
      } else {
        tma_load_5d(&t.top[0], &tm.m[kK3HaloY], &full[e.s], e.x0, e.y0 - 1, e.k, kV, e.m0);
        tma_load_5d(&t.bot[0], &tm.m[kK3HaloY], &full[e.s], e.x0, e.y0 + p.ty, e.k, kV, e.m0);
      }
    };
    auto item = [&](int comp, int x0, int y0, int k, int b) {
      mbar_wait_backoff<32>(&empty[s], ph ^ 1u);
      mbar_expect_tx(&full[s], comp == kU ? p.bytes_u : comp == kV ? p.bytes_v : p.bytes_w);
      const int m0 = b * MB;
      tma_load_5d(&st[s].main[0], &tm.m[kK3Main], &full[s], x0, y0, k, comp, m0);
      if (comp != kW) {
        const int slot = (qh + qn) % (D + 1);
        q[slot] = K3Pending{idx, x0, y0, k, m0, s, comp, 0};
        ++qn;
      }
      while (qn > 0 && q[qh].idx <= idx - p.hdelay) {  // halos of the item hdelay stages back
        halo(q[qh]);
        qh = qh + 1 == D + 1 ? 0 : qh + 1;
        --qn;
      }
      ++idx;
      if (++s == S) { s = 0; ph ^= 1u; }
    };
    for (int tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
      const int x0 = (tile % p.tiles_x) * TX;
      const int y0 = (tile / p.tiles_x) * p.ty;
      const int kb = int(p.kbeg);
      const int nb = n_blocks(p);
      if (p.has_w) {
        if (kb - 1 >= 0)
          for (int b = 0; b < nb; ++b) item(kW, x0, y0, kb - 1, b);
        for (int b = 0; b < nb; ++b) item(kW, x0, y0, kb, b);
      }
      // loose inter-CTA lockstep (as K2): before plane k, wait (bounded) until
      // every neighbour tile has consumed plane k - W, so the delayed halo
      // boxes find the neighbour's bytes in L2
      const bool sync = p.progress != nullptr && p.n_tiles <= int(gridDim.x);
      const int tcol = tile % p.tiles_x;
      int nbr[4], n_nbr = 0;
      if (tcol > 0) nbr[n_nbr++] = tile - 1;
      if (tcol + 1 < p.tiles_x && tile + 1 < p.n_tiles) nbr[n_nbr++] = tile + 1;
      if (tile >= p.tiles_x) nbr[n_nbr++] = tile - p.tiles_x;
      if (tile + p.tiles_x < p.n_tiles) nbr[n_nbr++] = tile + p.tiles_x;
      int seen = -1;   // min consumed planes over the neighbours, as last observed
      for (int k = kb; k < int(p.kend); ++k) {
        const int need = (k - kb) - p.sync_w;
        for (int spin = 0; sync && seen < need && spin < p.sync_spin; ++spin) {
          unsigned long long f[4];
          for (int q = 0; q < 4; ++q)
            f[q] = q < n_nbr ? __ldcg(p.progress + size_t(nbr[q]) * kFlagStride) : 0ull;
          int lo = 1 << 30;
          for (int q = 0; q < n_nbr; ++q)
            lo = min(lo, (f[q] >> 32) == (p.epoch & 0xffffffffull) ? int(f[q] & 0xffffffffull) : 0);
          seen = lo;
          if (seen < need) __nanosleep(p.sync_sleep);
        }
        if (seen < need) seen = need;   // gave up (bounded): never a correctness dependency
        for (int b = 0; b < nb; ++b) item(kU, x0, y0, k, b);
        for (int b = 0; b < nb; ++b) item(kV, x0, y0, k, b);
        if (p.has_w && k + 1 < p.nzl)
          for (int b = 0; b < nb; ++b) item(kW, x0, y0, k + 1, b);
      }
    }
    while (qn > 0) {
      halo(q[qh]);
      qh = qh + 1 == D + 1 ? 0 : qh + 1;
      --qn;
    }
  }

  // ------------------------------------------------------- stage ring access
  struct Ring {
    K3Stage* st;
    uint64_t* full;
    uint64_t* empty;
    int s;
    uint32_t ph;
    __device__ __forceinline__ const K3Stage& wait() {
      mbar_wait(&full[s], ph);
      return st[s];
    }
    __device__ __forceinline__ void release(int lane) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == S) { s = 0; ph ^= 1u; }
    }
    __device__ __forceinline__ void skip(int n, int lane) {  // wait + release n items
#pragma unroll 1
      for (int i = 0; i < n; ++i) { wait(); release(lane); }
    }
  };

  static __device__ __forceinline__ int check4(const V4& x) {
    return check_value(x.v[0]) | check_value(x.v[1]) | check_value(x.v[2]) | check_value(x.v[3]);
  }

  // fold M member boxes into (mu, sigma) of this lane's 4 points of row `ty`
  static __device__ __forceinline__ void row_moments(const K3Params& p, Ring& r, int ty, int cx0,
                                                     int lane, bool validate, int& err, V4& mu,
                                                     V4& sg) {
    ShiftedMoments<4> acc;
    const int nb = n_blocks(p);
#pragma unroll 1
    for (int b = 0; b < nb; ++b) {
      const K3Stage& t = r.wait();
      V4 x[MB];
#pragma unroll
      for (int mb = 0; mb < MB; ++mb)
        x[mb] = *reinterpret_cast<const V4*>(&t.main[(mb * p.ty + ty) * TX + cx0]);
      r.release(lane);
#pragma unroll
      for (int mb = 0; mb < MB; ++mb) {
        const int m = b * MB + mb;
        if (m < p.M) {
          if (validate) err |= check4(x[mb]);
          acc.add(m, x[mb].v);
        }
      }
    }
    acc.finish(p.M, mu.v, sg.v);
  }

  static __device__ __forceinline__ void halo_w(const K3Params& p, int64_t kk, int64_t off2d,
                                                bool act, V4& mu, V4& sg) {
    mu = V4{{0.f, 0.f, 0.f, 0.f}};
    sg = mu;
    if (!act) return;
    if (kk == -1 && p.z0 > 0) {
      mu = ldg_vec<float, 4>(p.halo_lo_mu_w + off2d);
      sg = ldg_vec<float, 4>(p.halo_lo_s_w + off2d);
    } else if (kk == p.nzl && p.z0 + p.nzl < p.nzg) {
      mu = ldg_vec<float, 4>(p.halo_hi_mu_w + off2d);
      sg = ldg_vec<float, 4>(p.halo_hi_s_w + off2d);
    }
  }

  // ------------------------------------------------------------- halo warp
  static __device__ void halo_warp(const K3Params& p, K3Stage* st, uint64_t* full, uint64_t* empty,
                                   K3Xchg& xb) {
    const int lane = threadIdx.x & 31;
    const int cx0 = lane * 4;
    Ring r{st, full, empty, 0, 0u};
    int xbuf = 0;
    // x-halo point handled by this lane (lanes >= 2*ty idle): side, row
    const int side = lane / p.ty, row = lane % p.ty;
    const bool has_x = lane < 2 * p.ty;
    const int nb = n_blocks(p);
    for (int tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
      const int kb = int(p.kbeg);
      if (p.has_w) r.skip((kb - 1 >= 0 ? nb : 0) + nb, lane);
      for (int k = kb; k < int(p.kend); ++k) {
        {  // u: the 2*TY x-halo points
          ShiftedMoments<1> acc;
#pragma unroll 1
          for (int b = 0; b < nb; ++b) {
            const K3Stage& t = r.wait();
            float h[MB];
#pragma unroll
            for (int mb = 0; mb < MB; ++mb)
              h[mb] = side == 0 ? t.hl[(mb * p.ty + row) * PAD + PAD - 1] : t.hr[(mb * p.ty + row) * PAD];
            r.release(lane);
#pragma unroll
            for (int mb = 0; mb < MB; ++mb)
              if (b * MB + mb < p.M) acc.add(b * MB + mb, &h[mb]);
          }
          float mu, sg;
          acc.finish(p.M, &mu, &sg);
          if (has_x) {
            xb.uh_mu[xbuf][side][row] = mu;
            xb.uh_sg[xbuf][side][row] = sg;
          }
        }
        {  // v: the row above and the row below the tile
          ShiftedMoments<4> at, ab;
#pragma unroll 1
          for (int b = 0; b < nb; ++b) {
            const K3Stage& t = r.wait();
            // accumulate straight from the stage (holding MB rows in registers
            // on top of two accumulator sets spills); release afterwards
#pragma unroll
            for (int mb = 0; mb < MB; ++mb)
              if (b * MB + mb < p.M) {
                const V4 a = *reinterpret_cast<const V4*>(&t.top[mb * TX + cx0]);
                const V4 c = *reinterpret_cast<const V4*>(&t.bot[mb * TX + cx0]);
                at.add(b * MB + mb, a.v);
                ab.add(b * MB + mb, c.v);
              }
            r.release(lane);
          }
          V4 mu, sg;
          at.finish(p.M, mu.v, sg.v);
          *reinterpret_cast<V4*>(&xb.mu[xbuf][0][cx0]) = mu;
          *reinterpret_cast<V4*>(&xb.sg[xbuf][0][cx0]) = sg;
          ab.finish(p.M, mu.v, sg.v);
          *reinterpret_cast<V4*>(&xb.mu[xbuf][p.ty + 1][cx0]) = mu;
          *reinterpret_cast<V4*>(&xb.sg[xbuf][p.ty + 1][cx0]) = sg;
        }
        if (p.has_w && k + 1 < p.nzl) r.skip(nb, lane);
        named_sync(1, 32 * (p.ty + 1));
        xbuf ^= 1;
      }
    }
  }

  // ------------------------------------------------------------- consumers
  static __device__ void consume(const K3Params& p, K3Stage* st, uint64_t* full, uint64_t* empty,
                                 K3Xchg& xb) {
    const int ty = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cx0 = lane * 4;
    const int64_t plane = int64_t(p.nx) * p.ny;
    const bool validate = p.err != nullptr;
    const bool t_zero = p.theta == 0.0f;
    int err = 0;
    Ring r{st, full, empty, 0, 0u};
    int xbuf = 0;
    for (int tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
      const int x0 = (tile % p.tiles_x) * TX;
      const int j = (tile / p.tiles_x) * p.ty + ty;
      const int xi = x0 + cx0;
      const bool act = xi < p.nx && j < p.ny;
      const int64_t off2d = int64_t(j) * p.nx + xi;
      const bool xin = xi > 0 && xi + 4 < p.nx;
      const bool yin = j > 0 && j < p.ny - 1;
      const bool jlo = j == 0, jhi = j == p.ny - 1;
      const float cy = (jlo || jhi) ? p.cy_bd : p.cy_in;
      const int kb = int(p.kbeg);
      V4 w0_mu = V4{{0.f, 0.f, 0.f, 0.f}}, w0_sg = w0_mu;
      {
        V4 wm_mu = w0_mu, wm_sg = w0_mu;
        if (p.has_w) {
          if (kb - 1 >= 0) row_moments(p, r, ty, cx0, lane, false, err, wm_mu, wm_sg);
          else halo_w(p, -1, off2d, act, wm_mu, wm_sg);
        }
        xb.wm[ty][0][lane] = wm_mu;
        xb.wm[ty][1][lane] = wm_sg;
      }
      if (p.has_w) row_moments(p, r, ty, cx0, lane, validate, err, w0_mu, w0_sg);
      int64_t o = int64_t(kb) * plane + off2d;
      for (int k = kb; k < int(p.kend); ++k, o += plane) {
        V4 u_mu, u_sg, v_mu, v_sg, wp_mu, wp_sg;
        row_moments(p, r, ty, cx0, lane, validate, err, u_mu, u_sg);
        row_moments(p, r, ty, cx0, lane, validate, err, v_mu, v_sg);
        *reinterpret_cast<V4*>(&xb.mu[xbuf][ty + 1][cx0]) = v_mu;
        *reinterpret_cast<V4*>(&xb.sg[xbuf][ty + 1][cx0]) = v_sg;
        if (!p.has_w) wp_mu = wp_sg = V4{{0.f, 0.f, 0.f, 0.f}};
        else if (k + 1 < p.nzl) row_moments(p, r, ty, cx0, lane, validate && k + 1 < p.kend, err, wp_mu, wp_sg);
        else halo_w(p, k + 1, off2d, act, wp_mu, wp_sg);

        named_sync(1, 32 * (p.ty + 1));  // every row's v moments + the halo moments visible
        // v neighbours are read per point from shared memory below (holding
        // four more float4 here pushes the epilogue into local memory)
        const float* vlo_mu = &xb.mu[xbuf][ty][cx0];
        const float* vlo_sg = &xb.sg[xbuf][ty][cx0];
        const float* vhi_mu = &xb.mu[xbuf][ty + 2][cx0];
        const float* vhi_sg = &xb.sg[xbuf][ty + 2][cx0];
        float ul_mu = __shfl_up_sync(0xffffffffu, u_mu.v[3], 1);
        float ul_sg = __shfl_up_sync(0xffffffffu, u_sg.v[3], 1);
        float ur_mu = __shfl_down_sync(0xffffffffu, u_mu.v[0], 1);
        float ur_sg = __shfl_down_sync(0xffffffffu, u_sg.v[0], 1);
        if (lane == 0) { ul_mu = xb.uh_mu[xbuf][0][ty]; ul_sg = xb.uh_sg[xbuf][0][ty]; }
        if (lane == 31) { ur_mu = xb.uh_mu[xbuf][1][ty]; ur_sg = xb.uh_sg[xbuf][1][ty]; }
        xbuf ^= 1;

        if (act) {
          const int64_t kg = p.z0 + k;
          // 2D: no z terms (w moments are zero, so c*(0-0) adds exactly 0)
          const bool klo = p.has_w && kg == 0, khi = p.has_w && kg == p.nzg - 1;
          const bool interior = xin && yin && !klo && !khi;
          const float cz = (klo || khi) ? p.cz_bd : p.cz_in;
          V4 omu, osg, ops, opk;
          using SM = StencilMath<float, true>;
          const float* wm_mu = xb.wm[ty][0][lane].v;
          const float* wm_sg = xb.wm[ty][1][lane].v;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int i = xi + e;
            const bool ilo = !interior && i == 0, ihi = !interior && i == p.nx - 1;
            const float cx = (ilo || ihi) ? p.cx_bd : p.cx_in;
            const float uo = u_mu.v[e], so = u_sg.v[e];
            const float ul = ilo ? uo : (e == 0 ? ul_mu : u_mu.v[e == 0 ? 0 : e - 1]);
            const float uh = ihi ? uo : (e == 3 ? ur_mu : u_mu.v[e == 3 ? 0 : e + 1]);
            const float sl = ilo ? so : (e == 0 ? ul_sg : u_sg.v[e == 0 ? 0 : e - 1]);
            const float sh = ihi ? so : (e == 3 ? ur_sg : u_sg.v[e == 3 ? 0 : e + 1]);
            const float vl = jlo ? v_mu.v[e] : vlo_mu[e];
            const float vh = jhi ? v_mu.v[e] : vhi_mu[e];
            const float svl = jlo ? v_sg.v[e] : vlo_sg[e];
            const float svh = jhi ? v_sg.v[e] : vhi_sg[e];
            const float wl = klo ? w0_mu.v[e] : wm_mu[e];
            const float wh = khi ? w0_mu.v[e] : wp_mu.v[e];
            const float swl = klo ? w0_sg.v[e] : wm_sg[e];
            const float swh = khi ? w0_sg.v[e] : wp_sg.v[e];
            const float m = SM::mean(uh, ul, vh, vl, wh, wl, cx, cy, cz);
            omu.v[e] = m;
            Tails<float>::eval(m, SM::var(sh, sl, svh, svl, swh, swl, cx, cy, cz), p.theta,
                               t_zero, osg.v[e], ops.v[e], opk.v[e]);
          }
          if (p.out_mu) st_stream<float, 4>(p.out_mu + o, omu);
          if (p.out_sigma) st_stream<float, 4>(p.out_sigma + o, osg);
          if (p.out_psrc) st_stream<float, 4>(p.out_psrc + o, ops);
          if (p.out_psnk) st_stream<float, 4>(p.out_psnk + o, opk);
          if (p.out_mom_mu) {
            const int64_t nl = p.comp_stride;
            st_stream<float, 4>(p.out_mom_mu + o, u_mu);
            st_stream<float, 4>(p.out_mom_mu + nl + o, v_mu);
            if (p.has_w) st_stream<float, 4>(p.out_mom_mu + 2 * nl + o, w0_mu);
            st_stream<float, 4>(p.out_mom_sigma + o, u_sg);
            st_stream<float, 4>(p.out_mom_sigma + nl + o, v_sg);
            if (p.has_w) st_stream<float, 4>(p.out_mom_sigma + 2 * nl + o, w0_sg);
          }
        }
        if (ty == 0 && lane == 0 && p.progress != nullptr && p.n_tiles <= int(gridDim.x))
          st_relaxed_u64(p.progress + size_t(tile) * kFlagStride,   // planes consumed, for the pacing
                         ((p.epoch & 0xffffffffull) << 32) | (unsigned long long)(k - kb + 1));
        xb.wm[ty][0][lane] = w0_mu;  // plane k becomes k-1 (own slot: no sync needed)
        xb.wm[ty][1][lane] = w0_sg;
        w0_mu = wp_mu; w0_sg = wp_sg;
      }
    }
    if (validate) flush_error(p.err, err);
  }
};

__global__ void __launch_bounds__(K3Cfg::THREADS, 1)
k3_tma_kernel(const __grid_constant__ K3Maps tm, const K3Params p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  auto* st = reinterpret_cast<K3Stage*>(smem_raw);
  auto* xb = reinterpret_cast<K3Xchg*>(smem_raw + sizeof(K3Stage) * K3Cfg::S);
  auto* bars = reinterpret_cast<uint64_t*>(smem_raw + sizeof(K3Stage) * K3Cfg::S + sizeof(K3Xchg));
  uint64_t* full = bars;
  uint64_t* empty = bars + K3Cfg::S;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < K3Cfg::S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], uint32_t(p.ty + 1));  // consumer warps + halo warp
    }
    mbar_fence_init();
  }
  if (warp == K3Cfg::PROD_WARP && (threadIdx.x & 31) < kK3NumMaps)
    tma_prefetch_desc(&tm.m[threadIdx.x & 31]);
  __syncthreads();
  if (warp == K3Cfg::PROD_WARP) {
    if ((threadIdx.x & 31) == 0) K3::produce(p, tm, st, full, empty, xb->pend);
    return;
  }
  if (warp == K3Cfg::HALO_WARP) {
    K3::halo_warp(p, st, full, empty, *xb);
    return;
  }
  if (warp >= p.ty) return;
  K3::consume(p, st, full, empty, *xb);
}

}  // namespace divuq
