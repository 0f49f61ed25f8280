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
//     issued with their main box (a trailing halo would delay the stage it
//     completes, and the ring depth is worth more -- measured; a K2-style
//     lockstep pacer remains as a knob);
//   * consumers fold each member into per-point shifted single-pass moment
//     accumulators (ShiftedMoments, common.cuh) and release the stage at
//     once; the halo warp does the same for the tile's halo points (2*TY
//     x-halo columns, 2 halo rows) and publishes their moments in shared
//     memory; u moments' x-neighbours come by warp shuffle, v moments' rows
//     through a small double-buffered shared tile, w moments roll in
//     registers along z;
//   * then the same StencilMath / Tails as K2 (common.cuh) per point, the
//     mean differenced on (mu, r) pairs (ShiftedMoments: r is the mean's
//     rounding residual, bf16, packed two per word where it is stored).
//
// Slab sharding: the w moments of the planes just outside the slab come from
// the halo pointers (the neighbour reduces its edge plane with K1 -- same
// ShiftedMoments -- and sends 3 planes (mu, r, sigma) instead of 2*M).
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


struct K3Xchg {
  // v moments of the tile rows (1..TY) + the halo rows (0, TY+1)
  float mu[2][K3Cfg::TYMAX + 2][K3Cfg::TX];
  float sg[2][K3Cfg::TYMAX + 2][K3Cfg::TX];
  uint2 mr[2][K3Cfg::TYMAX + 2][K3Cfg::TX / 4];   // their residuals, 4 x bf16 per lane
  // u moments at the x-halo columns: [buf][left/right][row]
  float uh_mu[2][2][K3Cfg::TYMAX];
  float uh_sg[2][2][K3Cfg::TYMAX];
  float uh_r[2][2][K3Cfg::TYMAX];
  // each consumer lane's w moments of plane k-1 (kept out of registers)
  Vec<float, 4> wm[K3Cfg::TYMAX][2][32];
  uint2 wr[K3Cfg::TYMAX][32];
};
// 5 stages + exchange + barriers must fit the 227 KB opt-in limit
static_assert(sizeof(K3Stage) * K3Cfg::S + sizeof(K3Xchg) + 2 * K3Cfg::S * 8 <= 232448,
              "K3 shared memory");

enum K3Map { kK3Main, kK3HaloX, kK3HaloY, kK3NumMaps };
struct K3Maps {
  CUtensorMap m[kK3NumMaps];
};

struct K3Params {
  const float* halo_lo_mu_w; const float* halo_lo_s_w;   // reduced w moments
  const float* halo_hi_mu_w; const float* halo_hi_s_w;
  const float* halo_lo_r_w; const float* halo_hi_r_w;    // their residuals (null: 0)
  int64_t nzl, z0, nzg, kbeg, kend;
  int64_t comp_stride;                                   // Nl = nx*ny*nzl
  int nx, ny, ty, tiles_x, n_tiles, M;
  int n_chunks;                                      // z-chunks per tile column (small planes: > 1)
  int64_t zchunk;
  int has_w;                                             // 0: 2D ensemble (u, v only)
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
  static constexpr int TX = C::TX, PAD = C::PAD, S = C::S;

  static constexpr int MB = C::MB;

  // The item sequence of one tile -- mirrored exactly by producer, consumers
  // and halo warp (an item = a block of MB members, NB = ceil(M/MB) blocks):
  // [w(kb-1) x NB if kb > 0] [w(kb) x NB] then per plane k:
  // u(k) x NB, v(k) x NB, [w(k+1) x NB if k+1 < nzl].
  static __device__ __forceinline__ int n_blocks(const K3Params& p) { return (p.M + MB - 1) / MB; }

  // ---------------------------------------------------------------- producer
  static __device__ void produce(const K3Params& p, const K3Maps& tm, K3Stage* st, uint64_t* full,
                                 uint64_t* empty) {
    int s = 0;
    uint32_t ph = 0;
    // a stage = the main box + (u, v) its halo boxes, all on the stage's
    // barrier: the halos go out with their main box (a trailing halo would
    // delay the stage it completes; the ring depth is worth more -- measured)
    auto item = [&](int comp, int x0, int y0, int k, int b) {
      mbar_wait_backoff<32>(&empty[s], ph ^ 1u);
      mbar_expect_tx(&full[s], comp == kU ? p.bytes_u : comp == kV ? p.bytes_v : p.bytes_w);
      const int m0 = b * MB;
      K3Stage& t = st[s];
      tma_load_5d(&t.main[0], &tm.m[kK3Main], &full[s], x0, y0, k, comp, m0);
      if (comp == kU) {
        tma_load_5d(&t.hl[0], &tm.m[kK3HaloX], &full[s], x0 - PAD, y0, k, kU, m0);
        tma_load_5d(&t.hr[0], &tm.m[kK3HaloX], &full[s], x0 + TX, y0, k, kU, m0);
      } else if (comp == kV) {
        tma_load_5d(&t.top[0], &tm.m[kK3HaloY], &full[s], x0, y0 - 1, k, kV, m0);
        tma_load_5d(&t.bot[0], &tm.m[kK3HaloY], &full[s], x0, y0 + p.ty, k, kV, m0);
      }
      if (++s == S) { s = 0; ph ^= 1u; }
    };
    for (int wi = blockIdx.x; wi < p.n_tiles * p.n_chunks; wi += gridDim.x) {
      const int tile = wi % p.n_tiles, chunk = wi / p.n_tiles;
      const int ke = int(min(p.kend, p.kbeg + (chunk + 1) * p.zchunk));
      const int x0 = (tile % p.tiles_x) * TX;
      const int y0 = (tile / p.tiles_x) * p.ty;
      const int kb = int(p.kbeg + chunk * p.zchunk);
      const int nb = n_blocks(p);
      if (p.has_w) {
        if (kb - 1 >= 0)
          for (int b = 0; b < nb; ++b) item(kW, x0, y0, kb - 1, b);
        for (int b = 0; b < nb; ++b) item(kW, x0, y0, kb, b);
      }
      // loose inter-CTA lockstep (as K2): before plane k, wait (bounded) until
      // every neighbour tile has consumed plane k - W, so the delayed halo
      // boxes find the neighbour's bytes in L2
      const bool sync = p.progress != nullptr && p.n_tiles <= int(gridDim.x) && p.n_chunks == 1;
      const int tcol = tile % p.tiles_x;
      int nbr[4], n_nbr = 0;
      if (tcol > 0) nbr[n_nbr++] = tile - 1;
      if (tcol + 1 < p.tiles_x && tile + 1 < p.n_tiles) nbr[n_nbr++] = tile + 1;
      if (tile >= p.tiles_x) nbr[n_nbr++] = tile - p.tiles_x;
      if (tile + p.tiles_x < p.n_tiles) nbr[n_nbr++] = tile + p.tiles_x;
      int seen = -1;   // min consumed planes over the neighbours, as last observed
      for (int k = kb; k < ke; ++k) {
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

  static __device__ __forceinline__ uint2 pack4(const float* r) {
    return make_uint2(pack_bf16x2(r[0], r[1]), pack_bf16x2(r[2], r[3]));
  }
  static __device__ __forceinline__ float unpack4(uint2 w, int e) {
    const uint32_t h = (e < 2) ? w.x : w.y;
    return (e & 1) ? unpack_bf16_hi(h) : unpack_bf16_lo(h);
  }

  // fold M member boxes into (mu, r, sigma) of this lane's 4 points of row `ty`
  static __device__ __forceinline__ void row_moments(const K3Params& p, Ring& r, int ty, int cx0,
                                                     int lane, bool validate, int& err, V4& mu,
                                                     uint2& mr, V4& sg) {
    ShiftedMoments<4> acc;
    const int nb = n_blocks(p);
    const bool full_blocks = (p.M % MB) == 0;
    {  // block 0: member 0 sets the shift (peeled: no per-member branch)
      const K3Stage& t = r.wait();
      V4 x[MB];
#pragma unroll
      for (int mb = 0; mb < MB; ++mb)
        x[mb] = *reinterpret_cast<const V4*>(&t.main[(mb * p.ty + ty) * TX + cx0]);
      r.release(lane);
      if (validate) err |= check4(x[0]);
      acc.first(x[0].v);
#pragma unroll
      for (int mb = 1; mb < MB; ++mb)
        if (full_blocks || mb < p.M) {
          if (validate) err |= check4(x[mb]);
          acc.next(x[mb].v);
        }
    }
#pragma unroll 1
    for (int b = 1; b < nb; ++b) {
      const K3Stage& t = r.wait();
      V4 x[MB];
#pragma unroll
      for (int mb = 0; mb < MB; ++mb)
        x[mb] = *reinterpret_cast<const V4*>(&t.main[(mb * p.ty + ty) * TX + cx0]);
      r.release(lane);
#pragma unroll
      for (int mb = 0; mb < MB; ++mb)
        if (full_blocks || b * MB + mb < p.M) {
          if (validate) err |= check4(x[mb]);
          acc.next(x[mb].v);
        }
    }
    V4 rr;
    acc.finish(p.M, mu.v, rr.v, sg.v);
    mr = pack4(rr.v);
  }

  static __device__ __forceinline__ void halo_w(const K3Params& p, int64_t kk, int64_t off2d,
                                                bool act, V4& mu, uint2& mr, V4& sg) {
    mu = V4{{0.f, 0.f, 0.f, 0.f}};
    sg = mu;
    V4 rr = mu;
    if (act) {
      if (kk == -1 && p.z0 > 0) {
        mu = ldg_vec<float, 4>(p.halo_lo_mu_w + off2d);
        sg = ldg_vec<float, 4>(p.halo_lo_s_w + off2d);
        if (p.halo_lo_r_w) rr = ldg_vec<float, 4>(p.halo_lo_r_w + off2d);
      } else if (kk == p.nzl && p.z0 + p.nzl < p.nzg) {
        mu = ldg_vec<float, 4>(p.halo_hi_mu_w + off2d);
        sg = ldg_vec<float, 4>(p.halo_hi_s_w + off2d);
        if (p.halo_hi_r_w) rr = ldg_vec<float, 4>(p.halo_hi_r_w + off2d);
      }
    }
    mr = pack4(rr.v);
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
    for (int wi = blockIdx.x; wi < p.n_tiles * p.n_chunks; wi += gridDim.x) {
      const int tile = wi % p.n_tiles, chunk = wi / p.n_tiles;
      const int ke = int(min(p.kend, p.kbeg + (chunk + 1) * p.zchunk));
      const int kb = int(p.kbeg + chunk * p.zchunk);
      if (p.has_w) r.skip((kb - 1 >= 0 ? nb : 0) + nb, lane);
      for (int k = kb; k < ke; ++k) {
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
          float mu, sg, rr;
          acc.finish(p.M, &mu, &rr, &sg);
          if (has_x) {
            xb.uh_mu[xbuf][side][row] = mu;
            xb.uh_sg[xbuf][side][row] = sg;
            xb.uh_r[xbuf][side][row] = rr;
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
          V4 mu, sg, rr;
          at.finish(p.M, mu.v, rr.v, sg.v);
          *reinterpret_cast<V4*>(&xb.mu[xbuf][0][cx0]) = mu;
          *reinterpret_cast<V4*>(&xb.sg[xbuf][0][cx0]) = sg;
          xb.mr[xbuf][0][lane] = pack4(rr.v);
          ab.finish(p.M, mu.v, rr.v, sg.v);
          *reinterpret_cast<V4*>(&xb.mu[xbuf][p.ty + 1][cx0]) = mu;
          *reinterpret_cast<V4*>(&xb.sg[xbuf][p.ty + 1][cx0]) = sg;
          xb.mr[xbuf][p.ty + 1][lane] = pack4(rr.v);
        }
        if (p.has_w && k + 1 < p.nzl) r.skip(nb, lane);
        named_sync(1, 32 * (p.ty + 1));
        xbuf ^= 1;
      }
    }
  }

  // ------------------------------------------------------------- consumers
  // Per plane: u(k) moments -> the x terms (warp shuffles); v(k) moments ->
  // shared tile; w(k+1) moments -> the z terms of the stencil (w(k) rolls to
  // the shared k-1 slot); barrier; the y terms from the shared tile; sigma
  // and tails.  Each axis' terms are formed as soon as their operands exist
  // (the same values StencilMath<float>::mean_r / var compute, factored per
  // axis), so at most one component's moments are live at a time -- the
  // consumer fits 128 registers without local-memory spills, which on a
  // full-smem SM (28 KB of L1 left) thrash L1 and come back from DRAM.
  static __device__ void consume(const K3Params& p, K3Stage* st, uint64_t* full, uint64_t* empty,
                                 K3Xchg& xb) {
    using SM = StencilMath<float, true>;
    const int ty = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cx0 = lane * 4;
    const int64_t plane = int64_t(p.nx) * p.ny;
    const bool validate = p.err != nullptr;
    const bool t_zero = p.theta == 0.0f;
    int err = 0;
    Ring r{st, full, empty, 0, 0u};
    int xbuf = 0;
    const uint2 zr = make_uint2(0u, 0u);
    for (int wi = blockIdx.x; wi < p.n_tiles * p.n_chunks; wi += gridDim.x) {
      const int tile = wi % p.n_tiles, chunk = wi / p.n_tiles;
      const int ke = int(min(p.kend, p.kbeg + (chunk + 1) * p.zchunk));
      const int x0 = (tile % p.tiles_x) * TX;
      const int j = (tile / p.tiles_x) * p.ty + ty;
      const int xi = x0 + cx0;
      const bool act = xi < p.nx && j < p.ny;
      const int64_t off2d = int64_t(j) * p.nx + xi;
      const bool jlo = j == 0, jhi = j == p.ny - 1;
      const float cy = (jlo || jhi) ? p.cy_bd : p.cy_in;
      const int kb = int(p.kbeg + chunk * p.zchunk);
      V4 w0_mu = V4{{0.f, 0.f, 0.f, 0.f}}, w0_sg = w0_mu;
      uint2 w0_r = zr;
      {
        V4 wm_mu = w0_mu, wm_sg = w0_mu;
        uint2 wm_r = zr;
        if (p.has_w) {
          if (kb - 1 >= 0) row_moments(p, r, ty, cx0, lane, false, err, wm_mu, wm_r, wm_sg);
          else halo_w(p, -1, off2d, act, wm_mu, wm_r, wm_sg);
        }
        xb.wm[ty][0][lane] = wm_mu;
        xb.wm[ty][1][lane] = wm_sg;
        xb.wr[ty][lane] = wm_r;
      }
      if (p.has_w) row_moments(p, r, ty, cx0, lane, validate, err, w0_mu, w0_r, w0_sg);
      int64_t o = int64_t(kb) * plane + off2d;
      for (int k = kb; k < ke; ++k, o += plane) {
        const int64_t kg = p.z0 + k;
        // 2D: no z terms (w moments are zero, so c*(0-0) adds exactly 0)
        const bool klo = p.has_w && kg == 0, khi = p.has_w && kg == p.nzg - 1;
        const float cz = (klo || khi) ? p.cz_bd : p.cz_in;
        float dx_m[4], dx_v[4];   // x terms
        float keep_mu, keep_sg, keep_r;
        {
          V4 u_mu, u_sg;
          uint2 u_r;
          row_moments(p, r, ty, cx0, lane, validate, err, u_mu, u_r, u_sg);
          if (act && p.out_mom_mu) {
            st_stream<float, 4>(p.out_mom_mu + o, u_mu);
            st_stream<float, 4>(p.out_mom_sigma + o, u_sg);
          }
          float ul_mu = __shfl_up_sync(0xffffffffu, u_mu.v[3], 1);
          float ul_sg = __shfl_up_sync(0xffffffffu, u_sg.v[3], 1);
          const uint32_t ul_rw = __shfl_up_sync(0xffffffffu, u_r.y, 1);
          float ur_mu = __shfl_down_sync(0xffffffffu, u_mu.v[0], 1);
          float ur_sg = __shfl_down_sync(0xffffffffu, u_sg.v[0], 1);
          const uint32_t ur_rw = __shfl_down_sync(0xffffffffu, u_r.x, 1);
          const float ul_r = unpack_bf16_hi(ul_rw), ur_r = unpack_bf16_lo(ur_rw);
          // lanes 0 / 31: the tile's x-halo points come from the halo warp
          // after the barrier; keep the in-lane neighbour of the edge point
          keep_mu = lane == 0 ? u_mu.v[1] : u_mu.v[2];
          keep_sg = lane == 0 ? u_sg.v[1] : u_sg.v[2];
          keep_r = unpack4(u_r, lane == 0 ? 1 : 2);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int i = xi + e;
            const bool ilo = i == 0, ihi = i == p.nx - 1;
            const float uo = u_mu.v[e], so = u_sg.v[e], ro = unpack4(u_r, e);
            const float ul = ilo ? uo : (e == 0 ? ul_mu : u_mu.v[e == 0 ? 0 : e - 1]);
            const float uh = ihi ? uo : (e == 3 ? ur_mu : u_mu.v[e == 3 ? 0 : e + 1]);
            const float sl = ilo ? so : (e == 0 ? ul_sg : u_sg.v[e == 0 ? 0 : e - 1]);
            const float sh = ihi ? so : (e == 3 ? ur_sg : u_sg.v[e == 3 ? 0 : e + 1]);
            const float rl = ilo ? ro : (e == 0 ? ul_r : unpack4(u_r, e == 0 ? 0 : e - 1));
            const float rh = ihi ? ro : (e == 3 ? ur_r : unpack4(u_r, e == 3 ? 0 : e + 1));
            dx_m[e] = SM::dpair(uh, ul, rh, rl);
            dx_v[e] = fmaf(sh, sh, sl * sl);
          }
        }

        {  // v(k): straight to the shared tile
          V4 v_mu, v_sg;
          uint2 v_r;
          row_moments(p, r, ty, cx0, lane, validate, err, v_mu, v_r, v_sg);
          *reinterpret_cast<V4*>(&xb.mu[xbuf][ty + 1][cx0]) = v_mu;
          *reinterpret_cast<V4*>(&xb.sg[xbuf][ty + 1][cx0]) = v_sg;
          xb.mr[xbuf][ty + 1][lane] = v_r;
        }
        float dz_m[4], dz_v[4];   // z terms: (w_hi - w_lo) as a pair difference, s_hi^2 + s_lo^2
        {
          V4 wp_mu, wp_sg;
          uint2 wp_r;
          if (!p.has_w) { wp_mu = wp_sg = V4{{0.f, 0.f, 0.f, 0.f}}; wp_r = zr; }
          else if (k + 1 < p.nzl) row_moments(p, r, ty, cx0, lane, validate && k + 1 < p.kend, err, wp_mu, wp_r, wp_sg);
          else halo_w(p, k + 1, off2d, act, wp_mu, wp_r, wp_sg);
          const V4 wm_mu = xb.wm[ty][0][lane], wm_sg = xb.wm[ty][1][lane];
          const uint2 wm_r = xb.wr[ty][lane];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float wl = klo ? w0_mu.v[e] : wm_mu.v[e];
            const float wh = khi ? w0_mu.v[e] : wp_mu.v[e];
            const float rwl = unpack4(klo ? w0_r : wm_r, e);
            const float rwh = unpack4(khi ? w0_r : wp_r, e);
            const float swl = klo ? w0_sg.v[e] : wm_sg.v[e];
            const float swh = khi ? w0_sg.v[e] : wp_sg.v[e];
            dz_m[e] = SM::dpair(wh, wl, rwh, rwl);
            dz_v[e] = fmaf(swh, swh, swl * swl);
          }
          if (act && p.out_mom_mu && p.has_w) {
            st_stream<float, 4>(p.out_mom_mu + 2 * p.comp_stride + o, w0_mu);
            st_stream<float, 4>(p.out_mom_sigma + 2 * p.comp_stride + o, w0_sg);
          }
          xb.wm[ty][0][lane] = w0_mu;  // plane k becomes k-1 (own slot: no sync needed)
          xb.wm[ty][1][lane] = w0_sg;
          xb.wr[ty][lane] = w0_r;
          w0_mu = wp_mu; w0_sg = wp_sg; w0_r = wp_r;
        }
        named_sync(1, 32 * (p.ty + 1));  // every row's v moments + the halo moments visible
        // v rows below / above (the point itself at the global y faces: the one-sided rule)
        const int rlo = jlo ? ty + 1 : ty, rhi = jhi ? ty + 1 : ty + 2;
        const V4 vl = *reinterpret_cast<const V4*>(&xb.mu[xbuf][rlo][cx0]);
        const V4 vh = *reinterpret_cast<const V4*>(&xb.mu[xbuf][rhi][cx0]);
        const V4 svl = *reinterpret_cast<const V4*>(&xb.sg[xbuf][rlo][cx0]);
        const V4 svh = *reinterpret_cast<const V4*>(&xb.sg[xbuf][rhi][cx0]);
        const uint2 vlo_r = xb.mr[xbuf][rlo][lane];
        const uint2 vhi_r = xb.mr[xbuf][rhi][lane];
        if (lane == 0 && xi > 0) {            // left x-halo point of the tile
          const float hm = xb.uh_mu[xbuf][0][ty], hs = xb.uh_sg[xbuf][0][ty], hr = xb.uh_r[xbuf][0][ty];
          dx_m[0] = SM::dpair(keep_mu, hm, keep_r, hr);   // (nx % 4 == 0: point 0 is never the last)
          dx_v[0] = fmaf(keep_sg, keep_sg, hs * hs);
        }
        if (lane == 31 && xi + 4 < p.nx) {     // right x-halo point
          const float hm = xb.uh_mu[xbuf][1][ty], hs = xb.uh_sg[xbuf][1][ty], hr = xb.uh_r[xbuf][1][ty];
          dx_m[3] = SM::dpair(hm, keep_mu, hr, keep_r);
          dx_v[3] = fmaf(hs, hs, keep_sg * keep_sg);
        }
        if (act && p.out_mom_mu) {
          st_stream<float, 4>(p.out_mom_mu + p.comp_stride + o,
                              *reinterpret_cast<const V4*>(&xb.mu[xbuf][ty + 1][cx0]));
          st_stream<float, 4>(p.out_mom_sigma + p.comp_stride + o,
                              *reinterpret_cast<const V4*>(&xb.sg[xbuf][ty + 1][cx0]));
        }
        xbuf ^= 1;

        if (act) {
          V4 omu, osg, ops, opk;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int i = xi + e;
            const float cx = (i == 0 || i == p.nx - 1) ? p.cx_bd : p.cx_in;
            const float dy_m = SM::dpair(vh.v[e], vl.v[e], unpack4(vhi_r, e), unpack4(vlo_r, e));
            const float dy_v = fmaf(svh.v[e], svh.v[e], svl.v[e] * svl.v[e]);
            // = SM::mean_r / SM::var of the same operands, bit for bit
            const float m = fmaf(cx, dx_m[e], fmaf(cy, dy_m, __fmul_rn(cz, dz_m[e])));
            const float var = fmaf(cx * cx, dx_v[e], fmaf(cy * cy, dy_v, (cz * cz) * dz_v[e]));
            omu.v[e] = m;
            Tails<float>::eval(m, var, p.theta, t_zero, osg.v[e], ops.v[e], opk.v[e]);
          }
          if (p.out_mu) st_stream<float, 4>(p.out_mu + o, omu);
          if (p.out_sigma) st_stream<float, 4>(p.out_sigma + o, osg);
          if (p.out_psrc) st_stream<float, 4>(p.out_psrc + o, ops);
          if (p.out_psnk) st_stream<float, 4>(p.out_psnk + o, opk);
        }
        if (ty == 0 && lane == 0 && p.progress != nullptr && p.n_tiles <= int(gridDim.x) && p.n_chunks == 1)
          st_relaxed_u64(p.progress + size_t(tile) * kFlagStride,   // planes consumed, for the pacing
                         ((p.epoch & 0xffffffffull) << 32) | (unsigned long long)(k - kb + 1));
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
    if ((threadIdx.x & 31) == 0) K3::produce(p, tm, st, full, empty);
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
