// K5: seeded on-device generation of the BASELINE.json synthetic inputs.
//
// The paper's wind / Red Sea ensembles are not available;
// BASELINE.json configs 1, 3 and 4 define seeded synthetic stand-ins.  Their
// mean fields follow the reference's synthetic recipe (synthetic.py:30-52):
// Gaussian sources/sinks A*(x-c)*exp(-|x-c|^2/w^2), plus a vortex (2D) or a
// divergence-free shear flow (3D).  Bump parameters are drawn on the host
// (numpy default_rng(seed)) and passed in; per-point noise is counter-based
// (Philox keyed by the seed, counter = (point, member/component, domain)), so
// any slab of a huge grid can be generated independently on its own GPU.
// Bench-only: not part of the reference-facing API.
#pragma once

#include "common.cuh"
#include "mc.cuh"   // philox4x32_10

namespace divuq {

struct Bump { float cx, cy, cz, amp, inv_w2; };

struct GenParams {
  const Bump* bumps; int n_bumps;
  int64_t nx, ny, nzl, z0;     // slab [z0, z0+nzl) of the global grid (nzl = 1, 2D)
  float dx, dy, dz;
  int dims;                    // 2 or 3
  float vortex_amp, vortex_cx, vortex_cy, vortex_inv_r2;   // 2D extra term
  float shear_amp, shear_ly;                              // 3D extra term: u += A (y/Ly - 1/2)
  uint64_t seed;
  float sig_lo, sig_hi;        // sigma range
  int sigma_mode;              // 0: iid U[lo,hi] per point & component; 1: smooth field in [lo,hi]
  int64_t n_members;           // 0: write (mu, sigma) model; >0: write members (M, C, Nl)
  float* out[6];               // model: mu_u, mu_v, (mu_w), s_u, s_v, (s_w)
  float* members;
};

__device__ __forceinline__ float u24(uint32_t x) { return (float(x >> 8) + 0.5f) * 0x1p-24f; }

__global__ void gen_kernel(const GenParams p) {
  const int64_t plane = p.nx * p.ny;
  const int64_t nl = plane * p.nzl;
  const int C = p.dims;
  for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < nl;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t k = idx / plane, r = idx % plane;
    const int64_t j = r / p.nx, i = r % p.nx;
    const float x = float(i) * p.dx, y = float(j) * p.dy, z = float(p.z0 + k) * p.dz;
    float m[3] = {0.f, 0.f, 0.f};
    for (int b = 0; b < p.n_bumps; ++b) {
      const Bump bp = p.bumps[b];
      const float ddx = x - bp.cx, ddy = y - bp.cy, ddz = (p.dims == 3) ? z - bp.cz : 0.f;
      const float g = bp.amp * __expf(-(ddx * ddx + ddy * ddy + ddz * ddz) * bp.inv_w2);
      m[0] += ddx * g; m[1] += ddy * g; m[2] += ddz * g;
    }
    if (p.dims == 2) {
      const float ddx = x - p.vortex_cx, ddy = y - p.vortex_cy;
      const float g = p.vortex_amp * __expf(-(ddx * ddx + ddy * ddy) * p.vortex_inv_r2);
      m[0] += -ddy * g; m[1] += ddx * g;
    } else {
      m[0] += p.shear_amp * (y / p.shear_ly - 0.5f);
    }
    const uint64_t gidx = uint64_t(p.z0 * plane + idx);
    float sg[3];
    if (p.sigma_mode == 0) {
      const Philox4 q = philox4x32_10(Philox4{uint32_t(gidx), uint32_t(gidx >> 32), 0xFFFFFFFFu, 0u},
                                      uint32_t(p.seed), uint32_t(p.seed >> 32));
      sg[0] = p.sig_lo + (p.sig_hi - p.sig_lo) * u24(q.x);
      sg[1] = p.sig_lo + (p.sig_hi - p.sig_lo) * u24(q.y);
      sg[2] = p.sig_lo + (p.sig_hi - p.sig_lo) * u24(q.z);
    } else {
      const float lx = float(p.nx) * p.dx, ly = float(p.ny) * p.dy;
      const float s = 0.5f + 0.5f * __sinf(6.2831853f * x / lx) * __cosf(6.2831853f * y / ly) *
                                 (p.dims == 3 ? __cosf(0.7f * z) : 1.0f);
      sg[0] = sg[1] = sg[2] = p.sig_lo + (p.sig_hi - p.sig_lo) * s;
    }
    if (p.n_members == 0) {
      for (int c = 0; c < C; ++c) { p.out[c][idx] = m[c]; p.out[C + c][idx] = sg[c]; }
    } else {
      for (int64_t mb = 0; mb < p.n_members; ++mb) {
        const Philox4 q = philox4x32_10(Philox4{uint32_t(gidx), uint32_t(gidx >> 32), uint32_t(mb), 1u},
                                        uint32_t(p.seed), uint32_t(p.seed >> 32));
        const float r1 = sqrtf(-2.0f * __logf(u24(q.x))), r2 = sqrtf(-2.0f * __logf(u24(q.z)));
        float s1, c1, s2, c2;
        __sincosf(6.2831853f * u24(q.y), &s1, &c1);
        __sincosf(6.2831853f * u24(q.w), &s2, &c2);
        const float zz[3] = {r1 * c1, r1 * s1, r2 * c2};
        for (int c = 0; c < C; ++c)
          p.members[(mb * C + c) * nl + idx] = m[c] + sg[c] * zz[c];
      }
    }
  }
}

}  // namespace divuq
