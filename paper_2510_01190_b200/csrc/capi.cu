// C ABI of the divergence-uncertainty hot path: launchers + host pipelines.
// Declarations and reference citations: include/divuq_b200.h.
#include <cuda_runtime.h>
#include <emmintrin.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "../../include/divuq_b200.h"
#include "gen.cuh"
#include "k2tma.cuh"
#include "k2flat.cuh"
#include "k3tma.cuh"
#include "k3row.cuh"
#include "divuq1.cuh"
#include "gradient.cuh"
#include "gradfused.cuh"
#include "gradmarch.cuh"
#include "lcp.cuh"
#include "mc.cuh"
#include "stencil.cuh"

using namespace divuq;

namespace {

#define DIVUQ_CUDA(call)                         \
  do {                                           \
    const int e_ = int(call);                    \
    if (e_ != 0) return e_;                      \
  } while (0)

int sm_count() {
  static std::mutex mu;
  static std::unordered_map<int, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  cache[dev] = n > 0 ? n : 1;
  return cache[dev];
}

template <typename K>
int blocks_per_sm(K kernel, int threads, size_t smem) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> cache;
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(reinterpret_cast<const void*>(kernel));
  if (it != cache.end()) return it->second;
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, smem);
  cache[reinterpret_cast<const void*>(kernel)] = n > 0 ? n : 1;
  return cache[reinterpret_cast<const void*>(kernel)];
}

int64_t env_int(const char* name, int64_t dflt) {
  const char* s = std::getenv(name);
  return s ? std::atoll(s) : dflt;
}

bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

int grid_ok(int64_t nx, int64_t ny, double dx, double dy) {
  if (nx < 2 || ny < 2) return DIVUQ_EGRID;
  if (!(dx > 0.0) || !(dy > 0.0)) return DIVUQ_EGRID;
  return DIVUQ_OK;
}

template <typename T>
void set_coeffs(StencilParams<T>& p, double dx, double dy, double dz) {
  // stencils.py:48-50: interior 1/(2h), boundary 1/h, evaluated in fp64
  p.cx_in = T(1.0 / (2.0 * dx)); p.cx_bd = T(1.0 / dx);
  p.cy_in = T(1.0 / (2.0 * dy)); p.cy_bd = T(1.0 / dy);
  p.cz_in = T(1.0 / (2.0 * dz)); p.cz_bd = T(1.0 / dz);
}

template <typename T, int VEC, bool HAS_W, bool HAS_SIGMA, int SRC>
int launch_stencil_impl(StencilParams<T> p, cudaStream_t s) {
  using K = StencilKernel<T, VEC, HAS_W, HAS_SIGMA, SRC>;
  auto kern = stencil_kernel<T, VEC, HAS_W, HAS_SIGMA, SRC>;
  const int threads = 32 * kStencilTY;
  const int64_t nk = p.kend - p.kbeg;
  if (nk <= 0) return DIVUQ_OK;
  p.tiles_x = (p.nx + K::TX - 1) / K::TX;
  p.tiles_y = (p.ny + K::TY - 1) / K::TY;
  const int64_t tiles = p.tiles_x * p.tiles_y;
  const int64_t cap = int64_t(blocks_per_sm(kern, threads, 0)) * sm_count();
  int64_t zc = env_int("DIVUQ_ZCHUNK", 0);
  if (zc <= 0) {
    // ~16 items per resident CTA keeps the round-robin tail small; >= 8
    // planes per item amortises the 2-plane w prologue
    const int64_t target = cap * 16;
    zc = std::max<int64_t>(8, (nk * tiles + target - 1) / target);
  }
  p.zchunk = std::min<int64_t>(zc, nk);
  p.n_items = tiles * ((nk + p.zchunk - 1) / p.zchunk);
  const int64_t grid = std::min<int64_t>(p.n_items, cap);
  kern<<<dim3(unsigned(grid)), dim3(32, kStencilTY), 0, s>>>(p);
  return int(cudaGetLastError());
}

template <typename T, bool HAS_SIGMA, int SRC>
int launch_gather2d(const StencilParams<T>& p, cudaStream_t s) {
  const dim3 grid(unsigned((p.nx + 255) / 256), unsigned(std::min<int64_t>(p.ny, 65535)));
  stencil2d_gather_kernel<T, HAS_SIGMA, SRC><<<grid, 256, 0, s>>>(p);
  return int(cudaGetLastError());
}

template <typename T, int VEC, bool HAS_W, int SRC>
int dispatch_sigma(const StencilParams<T>& p, bool has_sigma, cudaStream_t s) {
  if constexpr (SRC == kResidual) {
    return launch_stencil_impl<T, VEC, HAS_W, true, SRC>(p, s);
  } else {
    if (has_sigma) return launch_stencil_impl<T, VEC, HAS_W, true, SRC>(p, s);
    return launch_stencil_impl<T, VEC, HAS_W, false, SRC>(p, s);
  }
}

template <typename T, bool HAS_W, int SRC>
int dispatch_vec(const StencilParams<T>& p, bool has_sigma, cudaStream_t s) {
  constexpr int VW = (sizeof(T) == 4) ? 4 : 2;
  bool vec = (p.nx % VW) == 0;
  const void* ptrs[] = {p.mu_u, p.mu_v, p.mu_w, p.s_u, p.s_v, p.s_w, p.r_u, p.r_v, p.r_w,
                        p.halo_lo_mu_w, p.halo_lo_s_w, p.halo_hi_mu_w, p.halo_hi_s_w,
                        p.halo_lo_r_w, p.halo_hi_r_w,
                        p.out_mu, p.out_sigma, p.out_psrc, p.out_psnk};
  for (const void* q : ptrs) vec = vec && aligned(q, 16);
  // latency-bound small grids (config 0: 128^2 fp64): one point per lane
  // doubles the CTAs and halves each lane's dependent erfc chain
  if (vec) {
    const int64_t tiles_vec = ((p.nx + 32 * VW - 1) / (32 * VW)) * ((p.ny + kStencilTY - 1) / kStencilTY);
    if (tiles_vec * (p.kend - p.kbeg) < sm_count()) vec = false;
  }
  if constexpr (!HAS_W) {   // 2D: the gather kernel where the vector kernel cannot run,
                            // and for fp64 from 512^2 up (tools/p2d_probe.py: 4096^2
                            // 377 -> 299 us; the vector kernel stays ahead below)
    const bool big64 = sizeof(T) == 8 && p.nx * p.ny >= (int64_t(1) << 18);
    if ((!vec || big64 || env_int("DIVUQ_GATHER2D", 0)) && !env_int("DIVUQ_NO_GATHER2D", 0) &&
        p.kbeg == 0 && p.kend == 1) {
      if (SRC == kResidual || has_sigma) return launch_gather2d<T, true, SRC>(p, s);
      return launch_gather2d<T, false, SRC>(p, s);
    }
  }
  if (vec) return dispatch_sigma<T, VW, HAS_W, SRC>(p, has_sigma, s);
  return dispatch_sigma<T, 1, HAS_W, SRC>(p, has_sigma, s);
}

template <typename T>
StencilParams<T> blank_params() {
  StencilParams<T> p;
  std::memset(&p, 0, sizeof(p));
  return p;
}

template <typename T, bool HAS_SIGMA, bool HAS_W = true>
int launch_k2_tma(const StencilParams<T>& sp, cudaStream_t s, bool* used);   // below

template <typename T>
int propagate2d(const T* mu_u, const T* mu_v, const T* s_u, const T* s_v, int64_t nx, int64_t ny,
                double dx, double dy, double t, T* out_mu, T* out_sigma, T* out_ps, T* out_pk,
                int32_t* err, void* stream) {
  if (int r = grid_ok(nx, ny, dx, dy)) return r;
  if (!mu_u || !mu_v) return DIVUQ_EINVAL;
  const bool has_sigma = out_sigma || out_ps || out_pk;
  if (has_sigma && (!s_u || !s_v)) return DIVUQ_EINVAL;
  StencilParams<T> p = blank_params<T>();
  p.mu_u = mu_u; p.mu_v = mu_v; p.s_u = s_u; p.s_v = s_v;
  p.nx = nx; p.ny = ny; p.nzl = 1; p.z0 = 0; p.nzg = 1; p.kbeg = 0; p.kend = 1;
  set_coeffs(p, dx, dy, 1.0);
  p.theta = T(t);
  p.out_mu = out_mu; p.out_sigma = out_sigma; p.out_psrc = out_ps; p.out_psnk = out_pk;
  p.err = err;
  // large 2D grids: the 3D TMA pipeline without w (one "plane", tiles as work
  // items); small ones stay on the register kernels (launch-latency bound)
  if (!env_int("DIVUQ_NO_TMA", 0) && !env_int("DIVUQ_NO_TMA2D", 0) && nx * ny >= (int64_t(1) << 18) &&
      nx % TmaCfg<T>::VEC == 0 && nx < (int64_t(1) << 31) && ny < (int64_t(1) << 31)) {
    bool ok = true;
    for (const void* q : {(const void*)mu_u, (const void*)mu_v, (const void*)s_u, (const void*)s_v,
                          (const void*)out_mu, (const void*)out_sigma, (const void*)out_ps, (const void*)out_pk})
      ok = ok && aligned(q, 16);
    if (ok) {
      bool used = false;
      const cudaStream_t cs = static_cast<cudaStream_t>(stream);
      const int r = has_sigma ? launch_k2_tma<T, true, false>(p, cs, &used)
                              : launch_k2_tma<T, false, false>(p, cs, &used);
      if (r || used) return r;
    }
  }
  return dispatch_vec<T, false, kMoments>(p, has_sigma, static_cast<cudaStream_t>(stream));
}

// ---- TMA path for 3D K2 -------------------------------------------------
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

template <typename T>
bool make_map3d(CUtensorMap* m, const T* base, int64_t nx, int64_t ny, int64_t nz, int bx, int by,
                int64_t promo) {
  EncodeTiledFn fn = encode_tiled();
  if (!fn || !base) return false;
  const cuuint64_t dims[3] = {cuuint64_t(nx), cuuint64_t(ny), cuuint64_t(nz)};
  const cuuint64_t strides[2] = {cuuint64_t(nx) * sizeof(T), cuuint64_t(nx * ny) * sizeof(T)};
  const cuuint32_t box[3] = {cuuint32_t(bx), cuuint32_t(by), 1};
  const cuuint32_t es[3] = {1, 1, 1};
  const CUtensorMapDataType dt = sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
  const CUtensorMapL2promotion l2 = promo >= 256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
                                    : promo >= 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                    : promo >= 64  ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                                   : CU_TENSOR_MAP_L2_PROMOTION_NONE;
  return fn(m, dt, 3, const_cast<T*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, l2, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Per-device progress flags for the loose inter-CTA lockstep of the TMA
// kernels (k2tma.cuh / k3tma.cuh): allocated once, never reset -- every launch
// gets a fresh epoch tag, so stale flags from earlier launches are ignored.
constexpr int kMaxFlagTiles = 4096;
cudaError_t progress_flags(unsigned long long** flags_out, unsigned long long* epoch_out) {
  static unsigned long long* flags[64] = {};
  static unsigned long long epoch = 0;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return e;
  if (dev >= 64) { *flags_out = nullptr; return cudaSuccess; }
  if (!flags[dev]) {
    const size_t bytes = size_t(kMaxFlagTiles) * kFlagStride * sizeof(unsigned long long);
    if (cudaError_t e = cudaMalloc(&flags[dev], bytes)) return e;
    if (cudaError_t e = cudaMemset(flags[dev], 0, bytes)) return e;
  }
  *flags_out = flags[dev];
  *epoch_out = ++epoch;
  return cudaSuccess;
}

// Work items for the persistent TMA kernels: whole tile columns, or -- when
// the columns do not spread evenly over the SMs (fewer columns than SMs, or
// a last wave mostly empty) -- columns cut into z-chunks.  Each chunk restarts
// the z-march (two w planes by plain loads, a pipeline fill: ~2 planes of
// cost) and runs without the neighbour lockstep, so chunking is taken only
// when it cuts the busiest SM's planes by more than 15 %.  Results are the
// same bits: every point's arithmetic is unchanged.
void z_chunks(int n_tiles, int64_t nk, int64_t sms, int* n_chunks, int64_t* zchunk) {
  int64_t best_n = 1;
  if (n_tiles > 0 && nk > 0 && !env_int("DIVUQ_NO_ZCHUNK", 0)) {
    auto cost = [&](int64_t nch) {
      const int64_t zc = (nk + nch - 1) / nch;
      return ((int64_t(n_tiles) * nch + sms - 1) / sms) * (zc + 2);
    };
    const int64_t c1 = cost(1);
    int64_t best = c1;
    for (int64_t nch = 2; nch <= nk / 16; ++nch) {
      const int64_t c = cost(nch);
      if (c < best) { best = c; best_n = nch; }
    }
    if (best * 100 > c1 * 85) best_n = 1;
  }
  const int64_t zc = std::max<int64_t>(1, (nk + best_n - 1) / best_n);
  *zchunk = zc;
  *n_chunks = int(std::max<int64_t>(1, (nk + zc - 1) / zc));
}

// Tile height for the persistent TMA kernels: minimise the rows x planes the
// busiest SM marches, counting z-chunks (z_chunks above) when the tile
// columns do not fill the GPU; ties go to the taller tile (more warps).
int pick_ty(int64_t tiles_x, int64_t ny, int64_t nk, int tymax, int64_t sms) {
  int ty = tymax;
  int64_t best = INT64_MAX;
  for (int cand = tymax; cand >= 8; --cand) {
    const int64_t tiles = tiles_x * ((ny + cand - 1) / cand);
    int nch = 1;
    int64_t zc = nk;
    z_chunks(int(std::min<int64_t>(tiles, INT32_MAX)), nk, sms, &nch, &zc);
    const int64_t items = tiles * nch;
    // a CTA with fewer than 12 consumer rows streams less than a full one:
    // count short tiles as 12 rows
    const int64_t cost = ((items + sms - 1) / sms) * std::max(cand, 12) * (nch > 1 ? zc + 2 : zc);
    if (cost < best) { best = cost; ty = cand; }
  }
  return ty;
}

template <typename T, bool HAS_SIGMA, bool HAS_W>
int launch_k2_tma(const StencilParams<T>& sp, cudaStream_t s, bool* used) {
  using C = TmaCfg<T>;
  *used = false;
  // tile height: all CTAs own whole tile columns and march the planes in
  // lockstep, so pick TY minimising (waves of tiles) x (rows per tile)
  const int64_t sms = sm_count();
  const int64_t tiles_x = (sp.nx + C::TX - 1) / C::TX;
  int ty = pick_ty(tiles_x, sp.ny, sp.kend - sp.kbeg, C::TYMAX, sms);
  if (const int64_t forced = env_int("DIVUQ_TMA_TY", 0)) ty = int(std::max<int64_t>(1, std::min<int64_t>(forced, C::TYMAX)));
  // main boxes: whole 512-byte rows, L2 fill promotion on; halo boxes: 16-byte
  // columns / single rows, no promotion (they are L2 hits by design)
  const int64_t promo = env_int("DIVUQ_TMA_PROMO", 256);
  TmaMaps tm;
  std::memset(&tm, 0, sizeof(tm));
  const T* arrs[6] = {sp.mu_u, sp.mu_v, sp.mu_w, sp.s_u, sp.s_v, sp.s_w};
  for (int a = 0; a < (HAS_SIGMA ? 6 : 3); ++a) {
    if (!HAS_W && (a == 2 || a == 5)) { tm.m[kMapU + a] = tm.m[kMapU + a - 2]; continue; }   // 2D: no w
    if (!make_map3d<T>(&tm.m[kMapU + a], arrs[a], sp.nx, sp.ny, sp.nzl, C::TX, ty, promo)) return DIVUQ_OK;
  }
  if (!make_map3d<T>(&tm.m[kMapUH], sp.mu_u, sp.nx, sp.ny, sp.nzl, C::PAD, ty, 0)) return DIVUQ_OK;
  if (!make_map3d<T>(&tm.m[kMapVH], sp.mu_v, sp.nx, sp.ny, sp.nzl, C::TX, 1, 0)) return DIVUQ_OK;
  if (HAS_SIGMA) {
    if (!make_map3d<T>(&tm.m[kMapSUH], sp.s_u, sp.nx, sp.ny, sp.nzl, C::PAD, ty, 0)) return DIVUQ_OK;
    if (!make_map3d<T>(&tm.m[kMapSVH], sp.s_v, sp.nx, sp.ny, sp.nzl, C::TX, 1, 0)) return DIVUQ_OK;
  } else {
    for (int a = kMapSU; a <= kMapSW; ++a) tm.m[a] = tm.m[a - kMapSU];
    tm.m[kMapSUH] = tm.m[kMapUH];
    tm.m[kMapSVH] = tm.m[kMapVH];
  }
  TmaParams<T> p;
  std::memset(&p, 0, sizeof(p));
  p.mu_w = sp.mu_w; p.s_w = sp.s_w;
  p.halo_lo_mu_w = sp.halo_lo_mu_w; p.halo_lo_s_w = sp.halo_lo_s_w;
  p.halo_hi_mu_w = sp.halo_hi_mu_w; p.halo_hi_s_w = sp.halo_hi_s_w;
  p.nx = int(sp.nx); p.ny = int(sp.ny); p.nzl = sp.nzl; p.z0 = sp.z0; p.nzg = sp.nzg;
  p.kbeg = sp.kbeg; p.kend = sp.kend;
  p.ty = ty;
  p.tiles_x = int(tiles_x);
  p.n_tiles = int(tiles_x * ((sp.ny + ty - 1) / ty));
  z_chunks(p.n_tiles, sp.kend - sp.kbeg, sms, &p.n_chunks, &p.zchunk);
  p.hdelay = int(std::max<int64_t>(0, std::min<int64_t>(C::D, env_int("DIVUQ_K2_HDELAY", 2))));
  p.halo_off = int(env_int("DIVUQ_K2_HALO_OFF", 0));   // diagnostics only (wrong edge points)
  p.sync_w = int(env_int("DIVUQ_K2_SYNC_W", 8));
  p.sync_spin = int(env_int("DIVUQ_K2_SYNC_SPIN", 256));
  p.sync_sleep = int(env_int("DIVUQ_K2_SYNC_SLEEP", 1000));
  p.pf_dist = int(env_int("DIVUQ_K2_PF", 0));
  p.diag_null = HAS_SIGMA && sp.out_mu && sp.out_sigma && sp.out_psrc && sp.out_psnk
                    ? int(env_int("DIVUQ_K2_NULL", 0)) : 0;   // diagnostics only
  p.progress = nullptr;
  // lockstep pays off only on long z-marches (drift grows with the march);
  // short launches -- e.g. the host pipeline's 32-plane chunks, two of which
  // run concurrently and so are never fully co-resident -- skip it
  const int64_t min_planes = env_int("DIVUQ_K2_SYNC_MIN_PLANES", 64);
  if (p.sync_w > 0 && p.n_tiles <= kMaxFlagTiles && sp.kend - sp.kbeg >= min_planes)
    DIVUQ_CUDA(progress_flags(&p.progress, &p.epoch));
  p.stage_bytes = uint32_t(((HAS_W ? 3 : 2) * ty * C::TX + (p.halo_off ? 0 : 2 * ty * C::PAD + 2 * C::TX)) *
                           sizeof(T)) * (HAS_SIGMA ? 2u : 1u);
  const int64_t n_work = int64_t(p.n_tiles) * (sp.kend - sp.kbeg);
  p.cx_in = sp.cx_in; p.cx_bd = sp.cx_bd; p.cy_in = sp.cy_in; p.cy_bd = sp.cy_bd;
  p.cz_in = sp.cz_in; p.cz_bd = sp.cz_bd; p.theta = sp.theta;
  p.out_mu = sp.out_mu; p.out_sigma = sp.out_sigma; p.out_psrc = sp.out_psrc; p.out_psnk = sp.out_psnk;
  p.err = sp.err;
  if (n_work <= 0) { *used = true; return DIVUQ_OK; }
  auto kern = k2_tma_kernel<T, HAS_SIGMA, HAS_W>;
  const size_t smem = sizeof(TmaStage<T>) * C::S + 2 * C::S * sizeof(uint64_t);
  // function attributes are per device context: set on every launch (cheap)
  DIVUQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  const int64_t grid = std::min<int64_t>(int64_t(p.n_tiles) * p.n_chunks, sms);
  kern<<<unsigned(grid), C::THREADS, smem, s>>>(tm, p);
  *used = true;
  return int(cudaGetLastError());
}

// ---- TMA path for the fused 3D ensemble kernel (K3) ---------------------
bool make_map5d_members(CUtensorMap* m, const float* base, int64_t nx, int64_t ny, int64_t nzl,
                        int64_t comps, int64_t members, int bx, int by, int bm, int64_t promo) {
  // view of the (M, 3, nzl, ny, nx) member slab as (x, y, plane, component, member)
  EncodeTiledFn fn = encode_tiled();
  if (!fn || !base) return false;
  const cuuint64_t nl = cuuint64_t(nx * ny * nzl);
  const cuuint64_t dims[5] = {cuuint64_t(nx), cuuint64_t(ny), cuuint64_t(nzl), cuuint64_t(comps),
                              cuuint64_t(members)};
  const cuuint64_t strides[4] = {cuuint64_t(nx) * 4, cuuint64_t(nx * ny) * 4, nl * 4,
                                 cuuint64_t(comps) * nl * 4};
  const cuuint32_t box[5] = {cuuint32_t(bx), cuuint32_t(by), 1, 1, cuuint32_t(bm)};
  const cuuint32_t es[5] = {1, 1, 1, 1, 1};
  const CUtensorMapL2promotion l2 = promo >= 256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
                                                 : CU_TENSOR_MAP_L2_PROMOTION_NONE;
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, l2,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int try_k3_tma(const StencilParams<float>& sp, int comps, cudaStream_t s, bool* used) {
  using C = K3Cfg;
  *used = false;
  if (env_int("DIVUQ_NO_TMA", 0)) return DIVUQ_OK;
  if (sp.nx % 4 || sp.n_members < 2) return DIVUQ_OK;
  const void* ptrs[] = {sp.members, sp.halo_lo_mu_w, sp.halo_lo_s_w, sp.halo_hi_mu_w, sp.halo_hi_s_w,
                        sp.halo_lo_r_w, sp.halo_hi_r_w, sp.out_mu, sp.out_sigma, sp.out_psrc, sp.out_psnk, sp.out_mom_mu, sp.out_mom_sigma};
  for (const void* q : ptrs)
    if (!aligned(q, 16)) return DIVUQ_OK;
  if (sp.nx > (int64_t(1) << 30) || sp.ny > (int64_t(1) << 30) || sp.nzl > (int64_t(1) << 30)) return DIVUQ_OK;
  const int64_t sms = sm_count();
  const int64_t tiles_x = (sp.nx + C::TX - 1) / C::TX;
  int ty = pick_ty(tiles_x, sp.ny, sp.kend - sp.kbeg, C::TYMAX, sms);
  if (const int64_t forced = env_int("DIVUQ_TMA_TY", 0)) ty = int(std::max<int64_t>(1, std::min<int64_t>(forced, C::TYMAX)));
  K3Maps tm;
  std::memset(&tm, 0, sizeof(tm));
  const int64_t promo = env_int("DIVUQ_TMA_PROMO", 256);
  const int64_t M = sp.n_members;
  if (!make_map5d_members(&tm.m[kK3Main], sp.members, sp.nx, sp.ny, sp.nzl, comps, M, C::TX, ty, C::MB, promo) ||
      !make_map5d_members(&tm.m[kK3HaloX], sp.members, sp.nx, sp.ny, sp.nzl, comps, M, C::PAD, ty, C::MB, 0) ||
      !make_map5d_members(&tm.m[kK3HaloY], sp.members, sp.nx, sp.ny, sp.nzl, comps, M, C::TX, 1, C::MB, 0))
    return DIVUQ_OK;
  K3Params p;
  std::memset(&p, 0, sizeof(p));
  p.halo_lo_mu_w = sp.halo_lo_mu_w; p.halo_lo_s_w = sp.halo_lo_s_w;
  p.halo_hi_mu_w = sp.halo_hi_mu_w; p.halo_hi_s_w = sp.halo_hi_s_w;
  p.halo_lo_r_w = sp.halo_lo_r_w; p.halo_hi_r_w = sp.halo_hi_r_w;
  p.nzl = sp.nzl; p.z0 = sp.z0; p.nzg = sp.nzg; p.kbeg = sp.kbeg; p.kend = sp.kend;
  p.comp_stride = sp.comp_stride;
  p.nx = int(sp.nx); p.ny = int(sp.ny); p.ty = ty; p.tiles_x = int(tiles_x);
  p.n_tiles = int(tiles_x * ((sp.ny + ty - 1) / ty));
  z_chunks(p.n_tiles, sp.kend - sp.kbeg, sms, &p.n_chunks, &p.zchunk);
  p.M = int(sp.n_members);
  p.has_w = comps == 3;
  p.sync_w = int(env_int("DIVUQ_K3_SYNC_W", 0));   // lockstep off: no gain measured for K3
  p.sync_spin = int(env_int("DIVUQ_K3_SYNC_SPIN", 256));
  p.sync_sleep = int(env_int("DIVUQ_K3_SYNC_SLEEP", 500));
  p.progress = nullptr;
  if (p.sync_w > 0 && p.n_tiles <= kMaxFlagTiles && p.has_w)
    DIVUQ_CUDA(progress_flags(&p.progress, &p.epoch));
  p.bytes_u = uint32_t((C::TX * ty + 2 * C::PAD * ty) * 4 * C::MB);
  p.bytes_v = uint32_t((C::TX * ty + 2 * C::TX) * 4 * C::MB);
  p.bytes_w = uint32_t(C::TX * ty * 4 * C::MB);
  p.cx_in = sp.cx_in; p.cx_bd = sp.cx_bd; p.cy_in = sp.cy_in; p.cy_bd = sp.cy_bd;
  p.cz_in = sp.cz_in; p.cz_bd = sp.cz_bd; p.theta = sp.theta;
  p.out_mu = sp.out_mu; p.out_sigma = sp.out_sigma; p.out_psrc = sp.out_psrc; p.out_psnk = sp.out_psnk;
  p.out_mom_mu = sp.out_mom_mu; p.out_mom_sigma = sp.out_mom_sigma;
  p.err = sp.err;
  *used = true;
  if (sp.kend <= sp.kbeg) return DIVUQ_OK;
  const size_t smem = sizeof(K3Stage) * C::S + sizeof(K3Xchg) + 2 * C::S * sizeof(uint64_t);
  // function attributes are per device context: set on every launch (cheap)
  DIVUQ_CUDA(cudaFuncSetAttribute(k3_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  const int64_t grid = std::min<int64_t>(int64_t(p.n_tiles) * p.n_chunks, sms);
  k3_tma_kernel<<<unsigned(grid), C::THREADS, smem, s>>>(tm, p);
  return int(cudaGetLastError());
}

// ---- K2 on 1D tensor maps (k2flat.cuh): shapes whose row pitch a tiled map
// cannot take (fp32 nx % 4 != 0, fp64 nx odd) ---------------------------
template <typename T>
bool make_map1d(CUtensorMap* m, const T* base, int64_t n, int box) {
  EncodeTiledFn fn = encode_tiled();
  if (!fn || !base) return false;
  const cuuint64_t dims[1] = {cuuint64_t(n)};
  const cuuint64_t strides[1] = {0};
  const cuuint32_t bx[1] = {cuuint32_t(box)};
  const cuuint32_t es[1] = {1};
  const CUtensorMapDataType dt = sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
  return fn(m, dt, 1, const_cast<T*>(base), dims, strides, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <typename T, bool HAS_SIGMA>
int launch_k2_flat(const StencilParams<T>& sp, cudaStream_t s, bool* used) {
  using C = FlatCfg<T>;
  *used = false;
  const int64_t n = sp.nx * sp.ny * sp.nzl;
  const int64_t plane = sp.nx * sp.ny;
  // element coordinates are int32: the furthest box (plane nzl, row ny) must fit
  if (n + 2 * plane + C::UW >= (int64_t(1) << 31)) return DIVUQ_OK;
  const int64_t sms = sm_count();
  const int64_t tiles_x = (sp.nx + C::TX - 1) / C::TX;
  int ty = pick_ty(tiles_x, sp.ny, sp.kend - sp.kbeg, C::TYMAX, sms);
  FlatMaps fm;
  std::memset(&fm, 0, sizeof(fm));
  const T* arrs[6] = {sp.mu_u, sp.s_u, sp.mu_v, sp.s_v, sp.mu_w, sp.s_w};
  for (int a = 0; a < 6; ++a) {
    if (!HAS_SIGMA && (a & 1)) { fm.m[a] = fm.m[a - 1]; continue; }
    if (!make_map1d<T>(&fm.m[a], arrs[a], n, a < 2 ? C::UW : C::RWB)) return DIVUQ_OK;
  }
  FlatParams<T> p;
  std::memset(&p, 0, sizeof(p));
  p.mu_w = sp.mu_w; p.s_w = sp.s_w;
  p.halo_lo_mu_w = sp.halo_lo_mu_w; p.halo_lo_s_w = sp.halo_lo_s_w;
  p.halo_hi_mu_w = sp.halo_hi_mu_w; p.halo_hi_s_w = sp.halo_hi_s_w;
  p.nzl = sp.nzl; p.z0 = sp.z0; p.nzg = sp.nzg; p.kbeg = sp.kbeg; p.kend = sp.kend;
  p.nx = int(sp.nx); p.ny = int(sp.ny); p.ty = ty;
  p.tiles_x = int(tiles_x);
  p.n_tiles = int(tiles_x * ((sp.ny + ty - 1) / ty));
  z_chunks(p.n_tiles, sp.kend - sp.kbeg, sms, &p.n_chunks, &p.zchunk);
  const uint32_t comps = HAS_SIGMA ? 2u : 1u;
  p.stage_bytes = uint32_t((ty * (C::UW + C::RWB) + (ty + 2) * C::RWB) * sizeof(T)) * comps;
  p.cx_in = sp.cx_in; p.cx_bd = sp.cx_bd; p.cy_in = sp.cy_in; p.cy_bd = sp.cy_bd;
  p.cz_in = sp.cz_in; p.cz_bd = sp.cz_bd; p.theta = sp.theta;
  p.out_mu = sp.out_mu; p.out_sigma = sp.out_sigma; p.out_psrc = sp.out_psrc; p.out_psnk = sp.out_psnk;
  p.err = sp.err;
  *used = true;
  if (sp.kend <= sp.kbeg) return DIVUQ_OK;
  auto kern = k2_flat_kernel<T, HAS_SIGMA>;
  const size_t smem = sizeof(FlatStage<T>) * C::S + 2 * C::S * sizeof(uint64_t);
  DIVUQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  const int64_t grid = std::min<int64_t>(int64_t(p.n_tiles) * p.n_chunks, sms);
  kern<<<unsigned(grid), C::THREADS, smem, s>>>(fm, p);
  return int(cudaGetLastError());
}

template <typename T>
int try_k2_flat(const StencilParams<T>& p, bool has_sigma, cudaStream_t s, bool* used) {
  *used = false;
  if (env_int("DIVUQ_NO_FLAT", 0)) return DIVUQ_OK;
  const void* ptrs[] = {p.mu_u, p.mu_v, p.mu_w, p.s_u, p.s_v, p.s_w};   // tensor-map bases
  for (int a = 0; a < 6; ++a)
    if ((has_sigma || a < 3) && !aligned(ptrs[a], 16)) return DIVUQ_OK;
  return has_sigma ? launch_k2_flat<T, true>(p, s, used) : launch_k2_flat<T, false>(p, s, used);
}

template <typename T>
int try_k2_tma(const StencilParams<T>& p, bool has_sigma, cudaStream_t s, bool* used) {
  *used = false;
  if (env_int("DIVUQ_NO_TMA", 0)) return DIVUQ_OK;
  constexpr int VW = TmaCfg<T>::VEC;
  if (p.nx % VW) return try_k2_flat<T>(p, has_sigma, s, used);
  const void* ptrs[] = {p.mu_u, p.mu_v, p.mu_w, p.s_u, p.s_v, p.s_w, p.halo_lo_mu_w, p.halo_lo_s_w,
                        p.halo_hi_mu_w, p.halo_hi_s_w, p.out_mu, p.out_sigma, p.out_psrc, p.out_psnk};
  for (const void* q : ptrs)
    if (!aligned(q, 16)) return try_k2_flat<T>(p, has_sigma, s, used);   // vector accesses need 16 B
  if (p.nx > (int64_t(1) << 31) || p.ny > (int64_t(1) << 31) || p.nzl > (int64_t(1) << 31)) return DIVUQ_OK;
  return has_sigma ? launch_k2_tma<T, true>(p, s, used) : launch_k2_tma<T, false>(p, s, used);
}

template <typename T>
int propagate3d(const T* mu_u, const T* mu_v, const T* mu_w, const T* s_u, const T* s_v, const T* s_w,
                const T* hl_mu, const T* hl_s, const T* hh_mu, const T* hh_s, int64_t nx, int64_t ny,
                int64_t nzl, int64_t z0, int64_t nzg, int64_t kb, int64_t ke, double dx, double dy,
                double dz, double t, T* out_mu, T* out_sigma, T* out_ps, T* out_pk, int32_t* err,
                void* stream) {
  if (int r = grid_ok(nx, ny, dx, dy)) return r;
  if (nzg < 2 || !(dz > 0.0)) return DIVUQ_EGRID;
  if (nzl < 1 || z0 < 0 || z0 + nzl > nzg || kb < 0 || ke > nzl || kb > ke) return DIVUQ_EINVAL;
  if (!mu_u || !mu_v || !mu_w) return DIVUQ_EINVAL;
  const bool has_sigma = out_sigma || out_ps || out_pk;
  if (has_sigma && (!s_u || !s_v || !s_w)) return DIVUQ_EINVAL;
  if (z0 > 0 && (!hl_mu || (has_sigma && !hl_s))) return DIVUQ_EINVAL;
  if (z0 + nzl < nzg && (!hh_mu || (has_sigma && !hh_s))) return DIVUQ_EINVAL;
  StencilParams<T> p = blank_params<T>();
  p.mu_u = mu_u; p.mu_v = mu_v; p.mu_w = mu_w; p.s_u = s_u; p.s_v = s_v; p.s_w = s_w;
  p.halo_lo_mu_w = hl_mu; p.halo_lo_s_w = hl_s; p.halo_hi_mu_w = hh_mu; p.halo_hi_s_w = hh_s;
  p.nx = nx; p.ny = ny; p.nzl = nzl; p.z0 = z0; p.nzg = nzg; p.kbeg = kb; p.kend = ke;
  set_coeffs(p, dx, dy, dz);
  p.theta = T(t);
  p.out_mu = out_mu; p.out_sigma = out_sigma; p.out_psrc = out_ps; p.out_psnk = out_pk;
  p.err = err;
  bool used = false;
  if (int r = try_k2_tma<T>(p, has_sigma, static_cast<cudaStream_t>(stream), &used)) return r;
  if (used) return DIVUQ_OK;
  return dispatch_vec<T, true, kMoments>(p, has_sigma, static_cast<cudaStream_t>(stream));
}

// ---- K1: per-point moments over members, all components ----------------
// K1 streaming form: one thread per (component, VEC points), a handful of
// registers, U member loads (16 B each) in flight per thread and every SM full
// of threads.  fp64 keeps numpy's two-pass algorithm bit for bit (sequential
// sum / M, then the sequential sum of squared deviations, gaussian.py:41-44)
// by re-reading the members for the second pass -- the first pass just
// pulled them into L2, so HBM sees each member once.  fp32: ShiftedMoments,
// one pass.
template <typename T, int VEC, int U, int MINB, bool REREAD>
__global__ void __launch_bounds__(256, MINB) fit_stream_kernel(const T* __restrict__ members, int64_t M,
                                                            int64_t C, int64_t N, int64_t mstride,
                                                            T* __restrict__ out_mu,
                                                            T* __restrict__ out_sigma,
                                                            T* __restrict__ out_r, int* err) {
  using A = Arith<T>;
  using V = Vec<T, VEC>;
  int errbits = 0;
  const int64_t groups = N / VEC, total = C * groups;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t c = i / groups;
    const int64_t off = c * N + (i - c * groups) * VEC;
    const T* base = members + off;
    V mu, sg;
    if constexpr (sizeof(T) == 8) {
      V s, q;
      if constexpr (!REREAD) {   // requires M <= U
        // all M values of the point in registers (running pointer: one live
        // address), both passes from registers
        V x[U];
        const T* pm = base;
#pragma unroll
        for (int j = 0; j < U; ++j) {
          if (j < M) x[j] = ld_stream<T, VEC>(pm);
          pm += mstride;
        }
#pragma unroll
        for (int e = 0; e < VEC; ++e) s.v[e] = x[0].v[e];
#pragma unroll
        for (int j = 1; j < U; ++j)
          if (j < M) {
#pragma unroll
            for (int e = 0; e < VEC; ++e) s.v[e] = A::add(s.v[e], x[j].v[e]);
          }
#pragma unroll
        for (int e = 0; e < VEC; ++e) mu.v[e] = A::div(s.v[e], T(M));
#pragma unroll
        for (int j = 0; j < U; ++j)
          if (j < M) {
#pragma unroll
            for (int e = 0; e < VEC; ++e) {
              errbits |= check_value(x[j].v[e]);
              const T d = A::sub(x[j].v[e], mu.v[e]);
              q.v[e] = j == 0 ? A::mul(d, d) : A::add(q.v[e], A::mul(d, d));
            }
          }
      } else {
        for (int64_t k0 = 0; k0 < M; k0 += U) {   // pass 1: sum in member order
          V x[U];
#pragma unroll
          for (int j = 0; j < U; ++j)   // plain loads: the lines must stay in L2 for pass 2
            if (k0 + j < M) x[j] = ldg_vec<T, VEC>(base + (k0 + j) * mstride);
#pragma unroll
          for (int j = 0; j < U; ++j)
            if (k0 + j < M) {
#pragma unroll
              for (int e = 0; e < VEC; ++e) {
                errbits |= check_value(x[j].v[e]);
                s.v[e] = (k0 + j == 0) ? x[j].v[e] : A::add(s.v[e], x[j].v[e]);
              }
            }
        }
#pragma unroll
        for (int e = 0; e < VEC; ++e) mu.v[e] = A::div(s.v[e], T(M));
        for (int64_t k0 = 0; k0 < M; k0 += U) {   // pass 2: L2-resident re-read
          V x[U];
#pragma unroll
          for (int j = 0; j < U; ++j)
            if (k0 + j < M) x[j] = ld_stream<T, VEC>(base + (k0 + j) * mstride);
#pragma unroll
          for (int j = 0; j < U; ++j)
            if (k0 + j < M) {
#pragma unroll
              for (int e = 0; e < VEC; ++e) {
                const T d = A::sub(x[j].v[e], mu.v[e]);
                q.v[e] = (k0 + j == 0) ? A::mul(d, d) : A::add(q.v[e], A::mul(d, d));
              }
            }
        }
      }
#pragma unroll
      for (int e = 0; e < VEC; ++e) sg.v[e] = A::sqrt_(A::div(q.v[e], T(M - 1)));
    } else {
      ShiftedMoments<VEC> acc;
      for (int64_t k0 = 0; k0 < M; k0 += U) {
        V x[U];
#pragma unroll
        for (int j = 0; j < U; ++j)
          if (k0 + j < M) x[j] = ld_stream<T, VEC>(base + (k0 + j) * mstride);
#pragma unroll
        for (int j = 0; j < U; ++j)
          if (k0 + j < M) {
#pragma unroll
            for (int e = 0; e < VEC; ++e) errbits |= check_value(x[j].v[e]);
            acc.add(int(k0 + j), x[j].v);
          }
      }
      V rr;
      acc.finish(int(M), mu.v, rr.v, sg.v);
      if (out_r != nullptr) st_stream<T, VEC>(out_r + off, rr);
    }
    st_stream<T, VEC>(out_mu + off, mu);
    st_stream<T, VEC>(out_sigma + off, sg);
  }
  flush_error(err, errbits);
}

// fp64 K1 with the members parked in shared memory between the two passes
// (slot [m][thread]: consecutive threads, conflict-free): HBM is read once
// and the second pass never leaves the SM.  256 threads x M doubles per CTA.
template <int U>
__global__ void __launch_bounds__(256) fit_smem_kernel(const double* __restrict__ members, int64_t M,
                                                       int64_t C, int64_t N, int64_t mstride,
                                                       double* __restrict__ out_mu,
                                                       double* __restrict__ out_sigma, int* err) {
  using A = Arith<double>;
  extern __shared__ double park[];   // [M][256]
  int errbits = 0;
  const int64_t total = C * N;
  for (int64_t i0 = int64_t(blockIdx.x) * 256; i0 < total; i0 += int64_t(gridDim.x) * 256) {
    const int64_t i = i0 + threadIdx.x;
    const bool act = i < total;
    const int64_t c = act ? i / N : 0;
    const double* base = members + (act ? c * N + (i - c * N) : 0);
    double s = 0.0;
    for (int64_t k0 = 0; k0 < M; k0 += U) {   // pass 1: sum in member order, park the values
      double x[U];
#pragma unroll
      for (int j = 0; j < U; ++j)
        if (act && k0 + j < M) x[j] = __ldcs(base + (k0 + j) * mstride);
#pragma unroll
      for (int j = 0; j < U; ++j)
        if (act && k0 + j < M) {
          errbits |= check_value(x[j]);
          s = (k0 + j == 0) ? x[j] : A::add(s, x[j]);
          park[(k0 + j) * 256 + threadIdx.x] = x[j];
        }
    }
    if (act) {
      const double mu = A::div(s, double(M));
      double q = 0.0;
      for (int64_t k = 0; k < M; ++k) {   // pass 2 from the thread's own parked slots
        const double d = A::sub(park[k * 256 + threadIdx.x], mu);
        q = (k == 0) ? A::mul(d, d) : A::add(q, A::mul(d, d));
      }
      __stcs(out_mu + i, mu);
      __stcs(out_sigma + i, A::sqrt_(A::div(q, double(M - 1))));
    }
  }
  flush_error(err, errbits);
}

// fp64 K1, bulk-staged: a CTA streams tiles of 256 points; for each tile one
// warp issues M 1D bulk copies (one 2 KB member row each) into a stage of
// S per CTA, completion on one mbarrier, so a whole tile's members are in
// flight at once (the register-loaded fit_smem_kernel keeps 8 loads per
// thread in flight and was latency-bound: ncu long-scoreboard 7.9 per
// issue).  Both passes then read the stage: thread j owns point j, sums in
// member order (bitwise numpy, gaussian.py:41-44) and writes mu / sigma.
constexpr int kFbTile = 256;
__global__ void __launch_bounds__(kFbTile, 2) fit_bulk_kernel(const double* __restrict__ members, int M,
                                                              int64_t C, int64_t N, int64_t mstride,
                                                              int S, double* __restrict__ out_mu,
                                                              double* __restrict__ out_sigma, int* err) {
  using A = Arith<double>;
  extern __shared__ __align__(128) unsigned char fb_smem[];
  const size_t stage_bytes = size_t(M) * kFbTile * sizeof(double);
  uint64_t* full = reinterpret_cast<uint64_t*>(fb_smem + size_t(S) * stage_bytes);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t tpc = (N + kFbTile - 1) / kFbTile, ntiles = C * tpc;
  auto issue = [&](int64_t t, int s) {   // warp 0
    const int64_t c = t / tpc, n0 = (t - c * tpc) * kFbTile;
    const uint32_t bytes = uint32_t(min(int64_t(kFbTile), N - n0) * sizeof(double));
    double* dst = reinterpret_cast<double*>(fb_smem + size_t(s) * stage_bytes);
    if (lane == 0) mbar_expect_tx(&full[s], uint32_t(M) * bytes);
    __syncwarp();
    for (int m = lane; m < M; m += 32)
      bulk_load(dst + m * kFbTile, members + m * mstride + c * N + n0, bytes, &full[s]);
  };
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (warp == 0)
    for (int s = 0; s < S; ++s)
      if (blockIdx.x + int64_t(s) * gridDim.x < ntiles) issue(blockIdx.x + int64_t(s) * gridDim.x, s);
  int errbits = 0;
  for (int64_t k = 0;; ++k) {
    const int64_t t = blockIdx.x + k * gridDim.x;
    if (t >= ntiles) break;
    const int s = int(k % S);
    mbar_wait(&full[s], uint32_t(k / S) & 1u);
    const double* x = reinterpret_cast<const double*>(fb_smem + size_t(s) * stage_bytes);
    const int64_t c = t / tpc, n0 = (t - c * tpc) * kFbTile;
    if (n0 + tid < N) {
      double sum = x[tid];
      errbits |= check_value(sum);
      for (int m = 1; m < M; ++m) {   // pass 1: member order
        const double v = x[m * kFbTile + tid];
        errbits |= check_value(v);
        sum = A::add(sum, v);
      }
      const double mu = A::div(sum, double(M));
      double d = A::sub(x[tid], mu);
      double q = A::mul(d, d);
      for (int m = 1; m < M; ++m) {   // pass 2 from the stage
        d = A::sub(x[m * kFbTile + tid], mu);
        q = A::add(q, A::mul(d, d));
      }
      __stcs(out_mu + c * N + n0 + tid, mu);
      __stcs(out_sigma + c * N + n0 + tid, A::sqrt_(A::div(q, double(M - 1))));
    }
    __syncthreads();   // stage s consumed: refill it
    const int64_t tn = t + int64_t(S) * gridDim.x;
    if (warp == 0 && tn < ntiles) issue(tn, s);
  }
  flush_error(err, errbits);
}

template <typename T, int VEC, int U, int MINB, bool REREAD = true>
int launch_fit_stream(const T* m, int64_t M, int64_t C, int64_t N, int64_t ms, T* mu, T* sg,
                      T* r, int32_t* err, cudaStream_t s) {
  auto kern = fit_stream_kernel<T, VEC, U, MINB, REREAD>;
  const int64_t cap = int64_t(blocks_per_sm(kern, 256, 0)) * sm_count();
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((C * (N / VEC) + 255) / 256, cap));
  kern<<<unsigned(grid), 256, 0, s>>>(m, M, C, N, ms, mu, sg, r, err);
  return int(cudaGetLastError());
}

// measured on B200 (tools/fit_probe.py, M=20, C=2, 1024^2): fp32 float4 lanes,
// 4 loads in flight, 4 CTAs/SM: 33 us (86 % of HBM, was 113 us); fp64 one
// point per lane, 8 loads in flight, second pass re-read from L2: 113 us
// (50 %, was 194 us) -- the two passes serialise per thread
template <typename T>
int fit_stream(const T* m, int64_t M, int64_t C, int64_t N, int64_t ms, T* mu, T* sg, T* r,
               int32_t* err, cudaStream_t s) {
  const bool v16 = (N % (16 / int(sizeof(T)))) == 0 && (ms % (16 / int(sizeof(T)))) == 0 &&
                   aligned(m, 16) && aligned(mu, 16) && aligned(sg, 16) && aligned(r, 16);
  if constexpr (sizeof(T) == 4) {
    if (v16) return launch_fit_stream<T, 4, 4, 4>(m, M, C, N, ms, mu, sg, r, err, s);
    return launch_fit_stream<T, 1, 8, 4>(m, M, C, N, ms, mu, sg, r, err, s);
  } else {
    // holding all M doubles for both passes spills at these register caps;
    // parking them in shared memory keeps HBM at one read (measured faster
    // than the L2 re-read below, which remains for very large M)
    const size_t stage = size_t(M) * kFbTile * sizeof(double);
    if (!env_int("DIVUQ_FIT_NOBULK", 0) && N % 2 == 0 && ms % 2 == 0 && aligned(m, 16) &&
        2 * stage <= 200 * 1024) {
      // 2 CTAs / SM x S stages (S = 4 for M <= 12 .. 1 for M <= 50), <= ~200 KB per SM
      const int S = int(std::max<size_t>(1, std::min<size_t>(4, (100 * 1024) / stage)));
      const size_t smem = size_t(S) * stage + size_t(S) * sizeof(uint64_t);
      DIVUQ_CUDA(cudaFuncSetAttribute(fit_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      int per_sm = 0;
      DIVUQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fit_bulk_kernel, kFbTile, smem));
      const int64_t tiles = C * ((N + kFbTile - 1) / kFbTile);
      const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(tiles, int64_t(std::max(1, per_sm)) * sm_count()));
      fit_bulk_kernel<<<unsigned(grid), kFbTile, smem, s>>>(m, int(M), C, N, ms, S, mu, sg, err);
      return int(cudaGetLastError());
    }
    const size_t park = size_t(M) * 256 * sizeof(double);
    if (M <= 64 && !env_int("DIVUQ_FIT_REREAD", 0)) {
      auto kern = fit_smem_kernel<8>;
      DIVUQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(park)));
      int per_sm = 0;
      DIVUQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, park));
      const int64_t cap = std::max<int64_t>(1, int64_t(per_sm)) * sm_count();
      const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((C * N + 255) / 256, cap));
      kern<<<unsigned(grid), 256, park, s>>>(m, M, C, N, ms, mu, sg, err);
      return int(cudaGetLastError());
    }
    return launch_fit_stream<T, 1, 8, 4, true>(m, M, C, N, ms, mu, sg, nullptr, err, s);
  }
}

// out_r (fp32 only, optional): the means' rounding residuals (ShiftedMoments)
template <typename T>
int fit_gaussian(const T* members, int64_t M, int64_t C, int64_t N, T* out_mu, T* out_sigma,
                 int32_t* err, void* stream, int64_t mstride = -1, T* out_r = nullptr) {
  if (!members || !out_mu || !out_sigma || C < 1 || N < 1) return DIVUQ_EINVAL;
  if (M < 2) return DIVUQ_EMEMBERS;
  if (mstride < 0) mstride = C * N;
  if (mstride < C * N) return DIVUQ_EINVAL;
  if (sizeof(T) == 8 && out_r) return DIVUQ_EINVAL;
  return fit_stream<T>(members, M, C, N, mstride, out_mu, out_sigma, out_r, err,
                       static_cast<cudaStream_t>(stream));
}

// ---- probability map on an existing Gaussian scalar field (lcp.py:48-68)
template <typename T>
__global__ void tail_probs_kernel(const T* __restrict__ mu, const T* __restrict__ sigma, int64_t n,
                                  T theta, T* __restrict__ below, T* __restrict__ above, int* err) {
  int errbits = 0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const T m = mu[i], s = sigma[i];
    errbits |= check_value(m) | check_sigma(s);
    T b, a;
    tail_pair(m, s, theta, b, a);
    if (below) below[i] = b;
    if (above) above[i] = a;
  }
  flush_error(err, errbits);
}

template <typename T>
int tail_probs(const T* mu, const T* sigma, int64_t n, double theta, T* below, T* above, int32_t* err,
               void* stream) {
  if (!mu || !sigma || n < 0) return DIVUQ_EINVAL;
  if (n == 0 || (!below && !above)) return DIVUQ_OK;
  const int64_t grid = std::min<int64_t>((n + 255) / 256, int64_t(sm_count()) * 8);
  tail_probs_kernel<T><<<unsigned(grid), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      mu, sigma, n, T(theta), below, above, err);
  return int(cudaGetLastError());
}

int check_err_word(const int32_t* d_err, cudaStream_t s, int* status) {
  int32_t h = 0;
  DIVUQ_CUDA(cudaMemcpyAsync(&h, d_err, sizeof(h), cudaMemcpyDeviceToHost, s));
  DIVUQ_CUDA(cudaStreamSynchronize(s));
  *status = (h & DIVUQ_ERRBIT_NONFINITE) ? DIVUQ_ENONFINITE
            : (h & DIVUQ_ERRBIT_NEGSIGMA) ? DIVUQ_ENEGSIGMA : DIVUQ_OK;
  return 0;
}

// The host entry points stage through a stream-ordered pool.  With a release
// threshold of 0 every call handed its scratch back to the driver and the
// next call re-mapped it: ~40 ms per 180 MB call on B200, more than the
// copies themselves.  The library keeps its OWN pool per device (the
// process-wide default pool -- and so any other user of it -- is left
// alone), and caps what that pool keeps cached between calls at
// DIVUQ_POOL_KEEP_MB (default 4096 MB): larger peaks (the 3D pipelines,
// MC scratch) go back to the driver at the next synchronisation.
cudaError_t library_pool(cudaMemPool_t* out) {
  static cudaMemPool_t pools[64] = {};
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return e;
  if (dev >= 64) return cudaErrorInvalidDevice;
  if (!pools[dev]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    if (cudaError_t e = cudaMemPoolCreate(&pools[dev], &props)) return e;
    uint64_t keep = uint64_t(std::max<int64_t>(0, env_int("DIVUQ_POOL_KEEP_MB", 4096))) << 20;
    if (cudaError_t e = cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &keep))
      return e;
  }
  *out = pools[dev];
  return cudaSuccess;
}

// RAII device scratch from the library pool.  alloc(): released with a
// synchronising cudaFree, so no stream of the call can still be using it
// (the multi-stream 3D pipelines).  alloc_on(): every use is on stream st, so
// the release is stream-ordered there (cudaFreeAsync: no device-wide sync --
// ~5 us of a small drop-in call, and a hidden sync in device-API fallbacks).
struct DevBuf {
  void* p = nullptr;
  cudaStream_t only = nullptr;
  bool one_stream = false;
  cudaError_t alloc(size_t bytes, cudaStream_t st) {
    cudaMemPool_t pool;
    if (cudaError_t e = library_pool(&pool)) return e;
    return cudaMallocFromPoolAsync(&p, bytes ? bytes : 1, pool, st);
  }
  cudaError_t alloc_on(size_t bytes, cudaStream_t st) {
    only = st;
    one_stream = true;
    return alloc(bytes, st);
  }
  ~DevBuf() {
    if (!p) return;
    if (one_stream) cudaFreeAsync(p, only);
    else cudaFree(p);
  }
  template <typename T> T* as() const { return static_cast<T*>(p); }
};

// Pageable host memory (plain numpy arrays through the drop-in API) moves at a
// fraction of PCIe speed.  Large pageable copies go through the pinned staging
// ring instead: all host cores memcpy a chunk into a pinned buffer while the
// previous chunk's DMA runs.  Pinned / registered memory and small copies go
// straight to cudaMemcpyAsync.  Both helpers leave the stream drained.
// below these the driver's own pageable path wins (measured on B200 with the
// drop-in probe, tools/dropin_probe.py): pageable D2H is the slower direction
constexpr size_t kStageMinH2D = size_t(64) << 20, kStageMinD2H = size_t(12) << 20;

// Host copies of the staged paths.  Every staged byte is read by the host
// copy, written to the staging buffer and read again by the DMA, so these
// paths are bound by host DRAM bandwidth (tools/host_membw_probe.py, ~45 GB/s
// on the B200 boxes).  Streaming (non-temporal) stores drop the
// read-for-ownership of each destination line: one DRAM pass fewer per byte.
static void copy_lines(char* dst, const char* src, size_t n) {
  static const bool streaming = env_int("DIVUQ_NT_COPY", 1) != 0;
  if (!streaming || n < (size_t(64) << 10)) { std::memcpy(dst, src, n); return; }
  const size_t head = std::min(n, (16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & size_t(15));
  std::memcpy(dst, src, head);
  dst += head; src += head; n -= head;
  const size_t v = n / 64;
  for (size_t i = 0; i < v; ++i, src += 64, dst += 64) {
    const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src));
    const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + 16));
    const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + 32));
    const __m128i d = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + 48));
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst), a);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + 16), b);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + 32), c);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + 48), d);
  }
  std::memcpy(dst, src, n - v * 64);
  _mm_sfence();   // the streamed lines are globally visible before the DMA / the caller reads them
}
static int copy_threads() {
  static const int v = int(std::max<int64_t>(1, std::min<int64_t>(16, env_int("DIVUQ_COPY_THREADS", 16))));
  return v;
}

static void memcpy_parallel(char* dst, const char* src, int64_t len) {
  const int64_t kSlice = int64_t(2) << 20;
  const int64_t hw = std::max(1u, std::thread::hardware_concurrency());
  const int nt = int(std::min<int64_t>(std::min<int64_t>(copy_threads(), hw), (len + kSlice - 1) / kSlice));
  if (nt <= 1) { copy_lines(dst, src, size_t(len)); return; }
  const int64_t per = (len + nt - 1) / nt;
  io::HostPool::get().run(nt, [&](int t) {
    const int64_t a = t * per, n = std::min(per, len - a);
    if (n > 0) copy_lines(dst + a, src + a, size_t(n));
  });
}

static bool pageable(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return true; }
  return a.type == cudaMemoryTypeUnregistered;
}

int h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes < kStageMinH2D || !pageable(src))
    return int(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
  io::Staging& st = io::staging();
  std::lock_guard<std::mutex> lock(st.mu);
  if (int r = st.ensure()) return r;
  cudaEvent_t done[io::Staging::kBuffers] = {};
  int status = 0;
  for (auto& e : done)
    if (!status) status = int(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  const char* in = static_cast<const char*>(src);
  char* out = static_cast<char*>(dst);
  int b = 0;
  for (size_t off = 0; !status && off < bytes; off += io::Staging::kChunk, b = (b + 1) % io::Staging::kBuffers) {
    const int64_t len = int64_t(std::min<size_t>(io::Staging::kChunk, bytes - off));
    if ((status = int(cudaEventSynchronize(done[b])))) break;   // buffer b's last DMA finished
    memcpy_parallel(st.buf[b], in + off, len);
    if ((status = int(cudaMemcpyAsync(out + off, st.buf[b], size_t(len), cudaMemcpyHostToDevice, s)))) break;
    status = int(cudaEventRecord(done[b], s));
  }
  if (!status) status = int(cudaStreamSynchronize(s));   // the staging ring is released below
  for (auto& e : done)
    if (e) cudaEventDestroy(e);
  return status;
}

int d2h(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes < kStageMinD2H || !pageable(dst))
    return int(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
  io::Staging& st = io::staging();
  std::lock_guard<std::mutex> lock(st.mu);
  if (int r = st.ensure()) return r;
  const char* in = static_cast<const char*>(src);
  char* out = static_cast<char*>(dst);
  const int nb = io::Staging::kBuffers;
  cudaEvent_t done[io::Staging::kBuffers] = {};
  int status = 0;
  for (auto& e : done)
    if (!status) status = int(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  const size_t chunks = (bytes + io::Staging::kChunk - 1) / io::Staging::kChunk;
  // DMA chunk c into buffer c % nb; the host drains chunk c - (nb - 1) meanwhile
  for (size_t c = 0; !status && c < chunks + nb - 1; ++c) {
    if (c < chunks) {
      const size_t off = c * io::Staging::kChunk, len = std::min<size_t>(io::Staging::kChunk, bytes - off);
      if ((status = int(cudaMemcpyAsync(st.buf[c % nb], in + off, len, cudaMemcpyDeviceToHost, s)))) break;
      if ((status = int(cudaEventRecord(done[c % nb], s)))) break;
    }
    if (c + 1 >= size_t(nb)) {
      const size_t d = c + 1 - nb;
      if (d < chunks) {
        if ((status = int(cudaEventSynchronize(done[d % nb])))) break;
        const size_t off = d * io::Staging::kChunk, len = std::min<size_t>(io::Staging::kChunk, bytes - off);
        memcpy_parallel(out + off, st.buf[d % nb], int64_t(len));
      }
    }
  }
  for (auto& e : done)
    if (e) cudaEventDestroy(e);
  return status;
}

// Several arrays of one call as ONE staged stream: the per-array decision
// above sends an 8 MB fp64 map through the driver's pageable path, so a 1024^2
// propagate_divergence paid 4 + 2 such copies back to back.  Here the spans'
// chunks share the ring, so span k's host copy overlaps span k-1's DMA; used
// when the pageable bytes of the call reach kStageManyH2D / kStageManyD2H.  Non-pageable spans
// and small totals go straight to cudaMemcpyAsync.  Leaves the stream drained.
struct Span { void* dev; const void* host; size_t bytes; };
// same-box A/B (tools/dropin_probe.py): 2 x 8 MB in was slower staged, 4 x 8 MB
// faster; pageable D2H is the slow direction and gains from 12 MB up
constexpr size_t kStageManyH2D = size_t(32) << 20, kStageManyD2H = size_t(12) << 20;

int h2d_many(const Span* sp, int n, cudaStream_t s) {
  size_t paged = 0;
  for (int i = 0; i < n; ++i)
    if (sp[i].host && sp[i].bytes && pageable(sp[i].host)) paged += sp[i].bytes;
  if (paged < kStageManyH2D || env_int("DIVUQ_NO_STAGE_MANY", 0)) {
    for (int i = 0; i < n; ++i)
      if (sp[i].host && sp[i].bytes)
        if (int r = h2d(sp[i].dev, sp[i].host, sp[i].bytes, s)) return r;
    return 0;
  }
  io::Staging& st = io::staging();
  std::lock_guard<std::mutex> lock(st.mu);
  if (int r = st.ensure()) return r;
  cudaEvent_t done[io::Staging::kBuffers] = {};
  int status = 0;
  for (auto& e : done)
    if (!status) status = int(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  int b = 0;
  for (int i = 0; i < n && !status; ++i) {
    if (!sp[i].host || !sp[i].bytes) continue;
    if (!pageable(sp[i].host)) {
      status = int(cudaMemcpyAsync(sp[i].dev, sp[i].host, sp[i].bytes, cudaMemcpyHostToDevice, s));
      continue;
    }
    const char* in = static_cast<const char*>(sp[i].host);
    char* out = static_cast<char*>(sp[i].dev);
    for (size_t off = 0; !status && off < sp[i].bytes; off += io::Staging::kChunk, b = (b + 1) % io::Staging::kBuffers) {
      const int64_t len = int64_t(std::min<size_t>(io::Staging::kChunk, sp[i].bytes - off));
      if ((status = int(cudaEventSynchronize(done[b])))) break;
      memcpy_parallel(st.buf[b], in + off, len);
      if ((status = int(cudaMemcpyAsync(out + off, st.buf[b], size_t(len), cudaMemcpyHostToDevice, s)))) break;
      status = int(cudaEventRecord(done[b], s));
    }
  }
  if (!status) status = int(cudaStreamSynchronize(s));
  for (auto& e : done)
    if (e) cudaEventDestroy(e);
  return status;
}

// device -> host for several arrays; `host` is the destination here
int d2h_many(const Span* sp, int n, cudaStream_t s) {
  size_t paged = 0;
  for (int i = 0; i < n; ++i)
    if (sp[i].host && sp[i].bytes && pageable(sp[i].host)) paged += sp[i].bytes;
  if (paged < kStageManyD2H || env_int("DIVUQ_NO_STAGE_MANY", 0)) {
    for (int i = 0; i < n; ++i)
      if (sp[i].host && sp[i].bytes)
        if (int r = d2h(const_cast<void*>(sp[i].host), sp[i].dev, sp[i].bytes, s)) return r;
    return 0;
  }
  io::Staging& st = io::staging();
  std::lock_guard<std::mutex> lock(st.mu);
  if (int r = st.ensure()) return r;
  struct Chunk { char* dst; const char* src; size_t len; };
  std::vector<Chunk> chunks;
  for (int i = 0; i < n; ++i) {
    if (!sp[i].host || !sp[i].bytes) continue;
    if (!pageable(sp[i].host)) {
      if (int r = int(cudaMemcpyAsync(const_cast<void*>(sp[i].host), sp[i].dev, sp[i].bytes,
                                      cudaMemcpyDeviceToHost, s)))
        return r;
      continue;
    }
    for (size_t off = 0; off < sp[i].bytes; off += io::Staging::kChunk)
      chunks.push_back({static_cast<char*>(const_cast<void*>(sp[i].host)) + off,
                        static_cast<const char*>(sp[i].dev) + off,
                        std::min<size_t>(io::Staging::kChunk, sp[i].bytes - off)});
  }
  const int nb = io::Staging::kBuffers;
  cudaEvent_t done[io::Staging::kBuffers] = {};
  int status = 0;
  for (auto& e : done)
    if (!status) status = int(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  const size_t nc = chunks.size();
  for (size_t c = 0; !status && c < nc + nb - 1; ++c) {
    if (c < nc) {
      if ((status = int(cudaMemcpyAsync(st.buf[c % nb], chunks[c].src, chunks[c].len, cudaMemcpyDeviceToHost, s)))) break;
      if ((status = int(cudaEventRecord(done[c % nb], s)))) break;
    }
    if (c + 1 >= size_t(nb)) {
      const size_t d = c + 1 - nb;
      if (d < nc) {
        if ((status = int(cudaEventSynchronize(done[d % nb])))) break;
        memcpy_parallel(chunks[d].dst, st.buf[d % nb], int64_t(chunks[d].len));
      }
    }
  }
  if (!status) status = int(cudaStreamSynchronize(s));
  for (auto& e : done)
    if (e) cudaEventDestroy(e);
  return status;
}

// Small calls (the paper's own grids: 68^2 wind, 500^2 Red Sea) are latency
// bound: every pageable cudaMemcpyAsync is a synchronous driver copy, and a
// 68^2 propagate_divergence paid four of them in, two out, one for the
// validation word and a stream sync per output (~100 us of a 170 us call).
// Here a call's pageable inputs are packed into ONE per-thread pinned arena
// and go down as async DMAs (adjacent device spans merged into one copy);
// its outputs and the validation word come back into the arena, ONE stream
// sync, then memcpy out.  The arena is append-only until a sync on its
// stream (d2h side) or until it fills (then the stream is drained), so no
// bytes are overwritten while a DMA may still read them.
struct Bounce {
  char* buf = nullptr;
  char* dbuf = nullptr;   // the arena as the device sees it (mapped pinned memory)
  size_t cap = 0, cur = 0;
  cudaStream_t stream = nullptr;
};
static Bounce& bounce() {
  thread_local Bounce b;
  return b;
}
static size_t bounce_max() {
  static const size_t v = size_t(std::max<int64_t>(0, env_int("DIVUQ_BOUNCE_MAX_KB", 32832))) << 10;
  return v;
}
// room for `bytes` more on stream s; returns the arena offset or -1 (use the
// regular path)
static int64_t bounce_reserve(size_t bytes, cudaStream_t s, int* status) {
  Bounce& b = bounce();
  const size_t need = (bytes + 255) & ~size_t(255);
  if (need > bounce_max()) return -1;
  if (b.stream != s || b.cur + need > b.cap) {   // drain what may still use the arena
    if (b.stream && b.cur)
      if ((*status = int(cudaStreamSynchronize(b.stream)))) return -1;
    b.cur = 0;
    b.stream = s;
  }
  if (need > b.cap) {
    if (b.buf) cudaFreeHost(b.buf);
    b.buf = nullptr;
    b.cap = 0;
    size_t cap = size_t(1) << 20;
    while (cap < need) cap <<= 1;
    cap = std::min(cap, bounce_max());
    if (cudaHostAlloc(reinterpret_cast<void**>(&b.buf), cap, cudaHostAllocPortable | cudaHostAllocMapped) !=
        cudaSuccess) {   // no pinned arena (limit reached): the regular paths, not an error
      cudaGetLastError();
      b.buf = nullptr;
      return -1;
    }
    if (cudaHostGetDevicePointer(reinterpret_cast<void**>(&b.dbuf), b.buf, 0) != cudaSuccess) {
      cudaGetLastError();
      b.dbuf = nullptr;   // no zero-copy: the DMA paths still work
    }
    b.cap = cap;
  }
  const int64_t off = int64_t(b.cur);
  b.cur += need;
  return off;
}

// several (dst, src, len) copies as one job: from 512 KB on the bytes are
// split evenly over the host workers (a 500^2 call moves 8 MB in and 4 MB out:
// one thread per array ran at memcpy speed, ~1 ms)
struct Seg { char* dst; const char* src; size_t len; };
static void memcpy_segs(const Seg* sg, int n) {
  size_t total = 0;
  for (int i = 0; i < n; ++i) total += sg[i].len;
  const int64_t hw = std::max(1u, std::thread::hardware_concurrency());
  const int nt = total < (size_t(512) << 10) ? 1
                 : int(std::min<int64_t>({int64_t(copy_threads()), hw, int64_t(total / (size_t(256) << 10))}));
  if (nt <= 1) {
    for (int i = 0; i < n; ++i) copy_lines(sg[i].dst, sg[i].src, sg[i].len);
    return;
  }
  const size_t per = (total + nt - 1) / nt;
  io::HostPool::get().run(nt, [&](int t) {
    size_t a = size_t(t) * per, b = std::min(total, a + per), base = 0;
    for (int i = 0; i < n && a < b; ++i) {
      const size_t e = base + sg[i].len;
      if (a < e) {
        const size_t lo = a - base, hi = std::min(b, e) - base;
        copy_lines(sg[i].dst + lo, sg[i].src + lo, hi - lo);
        a = base + hi;
      }
      base = e;
    }
  });
}

// Small calls: ONE copy kernel instead of one DMA per span.  A DMA of
// <= 128 KB costs ~5 us of copy-engine time (config 0's e2e call was nine of
// them around a 2.8 us kernel, tools/host_entry_trace.py); a grid of CTAs
// reading mapped pinned memory (the arena, or the caller's pinned buffers)
// keeps ~100 KB of PCIe reads in flight, so a whole call's inputs -- or its
// outputs plus the validation word -- move in one launch.  Host-side sources
// are read with ld.global.cv (never served from a cache line of an earlier
// call); writes to host memory are visible after the stream sync.
constexpr int kCopyMax = 10;
struct CopyList {
  const char* src[kCopyMax];
  char* dst[kCopyMax];
  int64_t bytes[kCopyMax];
  int n;
};
template <typename V>
__device__ __forceinline__ void copy_run(const char* a, char* b, int64_t nb, int64_t tid, int64_t nt) {
  const int64_t nv = nb / int64_t(sizeof(V));
  const V* av = reinterpret_cast<const V*>(a);
  V* bv = reinterpret_cast<V*>(b);
  for (int64_t i = tid; i < nv; i += nt) bv[i] = __ldcv(av + i);
  for (int64_t i = nv * int64_t(sizeof(V)) + tid; i < nb; i += nt) b[i] = __ldcv(a + i);
}
__global__ void __launch_bounds__(256) copy_spans_kernel(const CopyList L) {
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nt = int64_t(gridDim.x) * blockDim.x;
  for (int s = 0; s < L.n; ++s) {
    const uintptr_t al = reinterpret_cast<uintptr_t>(L.src[s]) | reinterpret_cast<uintptr_t>(L.dst[s]);
    if ((al & 15) == 0) copy_run<int4>(L.src[s], L.dst[s], L.bytes[s], tid, nt);
    else if ((al & 7) == 0) copy_run<long long>(L.src[s], L.dst[s], L.bytes[s], tid, nt);
    else if ((al & 3) == 0) copy_run<int>(L.src[s], L.dst[s], L.bytes[s], tid, nt);
    else copy_run<char>(L.src[s], L.dst[s], L.bytes[s], tid, nt);
  }
}
static size_t zc_max() {
  static const size_t v = size_t(std::max<int64_t>(0, env_int("DIVUQ_ZC_MAX_KB", 4096))) << 10;
  return v;
}
static int launch_copy(const CopyList& L, size_t total, cudaStream_t s) {
  if (L.n == 0) return 0;
  const int64_t vecs = int64_t((total + 15) / 16);
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((vecs + 255) / 256, 2 * int64_t(sm_count())));
  copy_spans_kernel<<<unsigned(grid), 256, 0, s>>>(L);
  return int(cudaGetLastError());
}

// A call's spans through the arena (async): pageable ones are packed (one
// parallel job); then either ONE copy kernel moves every span (small calls,
// zc_max()) or DMAs do -- from the arena, a run of spans adjacent in device
// memory as one copy, and pinned spans straight from the caller's buffer.
// `hdev[i]`: span i's host buffer as the device sees it when it is pinned,
// nullptr when pageable.  false: not taken (too large for the arena).
static bool bounce_h2d(const Span* sp, const char* const* hdev, int n, cudaStream_t s, int* status) {
  size_t total = 0, all = 0;
  for (int i = 0; i < n; ++i) {
    if (!sp[i].host || !sp[i].bytes) continue;
    all += sp[i].bytes;
    if (!hdev[i]) total += (sp[i].bytes + 255) & ~size_t(255);
  }
  char* arena = nullptr;
  const char* darena = nullptr;
  if (total) {
    const int64_t base = bounce_reserve(total, s, status);
    if (base < 0) return false;
    arena = bounce().buf + base;
    darena = bounce().dbuf ? bounce().dbuf + base : nullptr;
    std::vector<Seg> segs;
    size_t o = 0;
    for (int i = 0; i < n; ++i) {
      if (!sp[i].host || !sp[i].bytes || hdev[i]) continue;
      segs.push_back({arena + o, static_cast<const char*>(sp[i].host), sp[i].bytes});
      o += (sp[i].bytes + 255) & ~size_t(255);
    }
    memcpy_segs(segs.data(), int(segs.size()));
  }
  if (all <= zc_max() && n <= kCopyMax && (darena || !total)) {
    CopyList L{};
    size_t off = 0;
    for (int i = 0; i < n; ++i) {
      if (!sp[i].host || !sp[i].bytes) continue;
      L.src[L.n] = hdev[i] ? hdev[i] : darena + off;
      L.dst[L.n] = static_cast<char*>(sp[i].dev);
      L.bytes[L.n++] = int64_t(sp[i].bytes);
      if (!hdev[i]) off += (sp[i].bytes + 255) & ~size_t(255);
    }
    *status = launch_copy(L, all, s);
    return true;
  }
  size_t off = 0;
  const char* run_dev = nullptr;   // a run of arena spans adjacent in device memory -> one DMA
  const char* run_host = nullptr;
  size_t run_len = 0;
  auto flush = [&]() {
    if (run_len && !*status)
      *status = int(cudaMemcpyAsync(const_cast<char*>(run_dev), run_host, run_len, cudaMemcpyHostToDevice, s));
    run_len = 0;
  };
  for (int i = 0; i < n && !*status; ++i) {
    if (!sp[i].host || !sp[i].bytes) continue;
    if (hdev[i]) {
      *status = int(cudaMemcpyAsync(sp[i].dev, sp[i].host, sp[i].bytes, cudaMemcpyHostToDevice, s));
      continue;
    }
    const char* dev = static_cast<const char*>(sp[i].dev);
    if (run_len && run_dev + run_len == dev && run_host + run_len == arena + off) {
      run_len += sp[i].bytes;
    } else {
      flush();
      run_dev = dev;
      run_host = arena + off;
      run_len = sp[i].bytes;
    }
    off += (sp[i].bytes + 255) & ~size_t(255);
  }
  flush();
  return true;
}

// outputs (host = destination) and the validation word, ONE stream sync:
// pinned destinations are written directly, pageable ones (and the word)
// land in the arena and are copied out after the sync; small calls move
// everything with one copy kernel
static bool bounce_d2h(const Span* sp, const char* const* hdev, int n, const int32_t* derr,
                       cudaStream_t s, int* code, int* status) {
  size_t total = derr ? 256 : 0, all = derr ? sizeof(int32_t) : 0;
  for (int i = 0; i < n; ++i) {
    if (!sp[i].host || !sp[i].bytes) continue;
    all += sp[i].bytes;
    if (!hdev[i]) total += (sp[i].bytes + 255) & ~size_t(255);
  }
  char* arena = nullptr;
  char* darena = nullptr;
  if (total) {
    const int64_t base = bounce_reserve(total, s, status);
    if (base < 0) return false;
    arena = bounce().buf + base;
    darena = bounce().dbuf ? bounce().dbuf + base : nullptr;
  }
  if (all <= zc_max() && n + 1 <= kCopyMax && (darena || !total)) {
    CopyList L{};
    if (derr) {
      L.src[L.n] = reinterpret_cast<const char*>(derr);
      L.dst[L.n] = darena;
      L.bytes[L.n++] = sizeof(int32_t);
    }
    size_t off = derr ? 256 : 0;
    for (int i = 0; i < n; ++i) {
      if (!sp[i].host || !sp[i].bytes) continue;
      L.src[L.n] = static_cast<const char*>(sp[i].dev);
      L.dst[L.n] = hdev[i] ? const_cast<char*>(hdev[i]) : darena + off;
      L.bytes[L.n++] = int64_t(sp[i].bytes);
      if (!hdev[i]) off += (sp[i].bytes + 255) & ~size_t(255);
    }
    *status = launch_copy(L, all, s);
  } else {
    size_t off = derr ? 256 : 0;
    if (derr && !*status)
      *status = int(cudaMemcpyAsync(arena, derr, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    for (int i = 0; i < n && !*status; ++i) {
      if (!sp[i].host || !sp[i].bytes) continue;
      if (hdev[i]) {
        *status = int(cudaMemcpyAsync(const_cast<void*>(sp[i].host), sp[i].dev, sp[i].bytes,
                                      cudaMemcpyDeviceToHost, s));
        continue;
      }
      *status = int(cudaMemcpyAsync(arena + off, sp[i].dev, sp[i].bytes, cudaMemcpyDeviceToHost, s));
      off += (sp[i].bytes + 255) & ~size_t(255);
    }
  }
  if (!*status) *status = int(cudaStreamSynchronize(s));
  if (*status) return true;
  if (total) bounce().cur = 0;   // the stream is drained: the whole arena is free
  size_t off = derr ? 256 : 0;
  std::vector<Seg> segs;
  for (int i = 0; i < n; ++i) {
    if (!sp[i].host || !sp[i].bytes || hdev[i]) continue;
    segs.push_back({static_cast<char*>(const_cast<void*>(sp[i].host)), arena + off, sp[i].bytes});
    off += (sp[i].bytes + 255) & ~size_t(255);
  }
  memcpy_segs(segs.data(), int(segs.size()));
  if (derr) {
    int32_t h;
    std::memcpy(&h, arena, sizeof(h));
    *code = (h & DIVUQ_ERRBIT_NONFINITE) ? DIVUQ_ENONFINITE
            : (h & DIVUQ_ERRBIT_NEGSIGMA) ? DIVUQ_ENEGSIGMA : DIVUQ_OK;
  }
  return true;
}

constexpr int kMaxSpans = 8;
// hdev[i]: the device view of span i's host buffer when it is pinned (or
// registered) host memory, nullptr when it is pageable or empty
static void classify(const Span* sp, int n, const char** hdev) {
  for (int i = 0; i < n; ++i) {
    hdev[i] = nullptr;
    if (!sp[i].host || !sp[i].bytes) continue;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, sp[i].host) != cudaSuccess) { cudaGetLastError(); continue; }
    if (a.type == cudaMemoryTypeUnregistered) continue;
    // device memory passed as a "host" span: let the DMA path handle it
    hdev[i] = a.type == cudaMemoryTypeHost && a.devicePointer ? static_cast<const char*>(a.devicePointer)
                                                              : nullptr;
    if (!hdev[i]) hdev[i] = static_cast<const char*>(sp[i].host);   // pinned but unmapped: DMA only
  }
}

// inputs of a call: through the arena / one copy kernel when small, else
// h2d_many (the staged ring for large pageable totals)
int h2d_in(const Span* sp, int n, cudaStream_t s) {
  if (n <= kMaxSpans) {
    const char* hdev[kMaxSpans];
    classify(sp, n, hdev);
    int status = 0;
    if (bounce_h2d(sp, hdev, n, s, &status)) return status;
    if (status) return status;
  }
  return h2d_many(sp, n, s);
}

// outputs of a call + the validation word -> *code (DIVUQ_OK / ENONFINITE /
// ENEGSIGMA); returns a CUDA status.  Leaves the stream drained.
int d2h_out(const Span* sp, int n, const int32_t* derr, cudaStream_t s, int* code) {
  *code = DIVUQ_OK;
  if (n <= kMaxSpans) {
    const char* hdev[kMaxSpans];
    classify(sp, n, hdev);
    int status = 0;
    if (bounce_d2h(sp, hdev, n, derr, s, code, &status)) return status;
    if (status) return status;
  }
  if (int r = d2h_many(sp, n, s)) return r;
  return derr ? check_err_word(derr, s, code) : 0;
}

// The host entry points run on a per-(thread, device) pair of non-blocking
// streams created once: creating and destroying a stream per call cost more
// than a small call's copies and kernel.  The guard only drains the stream.
cudaError_t cached_stream(int slot, cudaStream_t* out) {
  thread_local cudaStream_t streams[64][3] = {};
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return e;
  if (dev >= 64 || slot < 0 || slot > 2) return cudaStreamCreateWithFlags(out, cudaStreamNonBlocking);
  if (!streams[dev][slot])
    if (cudaError_t e = cudaStreamCreateWithFlags(&streams[dev][slot], cudaStreamNonBlocking)) return e;
  *out = streams[dev][slot];
  return cudaSuccess;
}

struct StreamGuard {
  cudaStream_t s = nullptr;
  ~StreamGuard() { if (s) cudaStreamSynchronize(s); }
};

// ---- velocity-magnitude-gradient prologue ----------
template <typename T>
int launch_gradient(const T* in, int64_t members, int64_t in_mstride, int64_t nx, int64_t ny,
                    double dx, double dy, T* out, int64_t out_mstride, bool mag, int32_t* err,
                    void* stream) {
  if (int r = grid_ok(nx, ny, dx, dy)) return r;
  if (!in || !out || members < 1) return DIVUQ_EINVAL;
  const dim3 grid(unsigned((nx + kGrTX - 1) / kGrTX), unsigned((ny + kGrTY - 1) / kGrTY),
                  unsigned(std::max<int64_t>(1, std::min<int64_t>(
                      (members + env_int("DIVUQ_GR_MPC", kGrMembersPerCta) - 1) /
                          std::max<int64_t>(1, env_int("DIVUQ_GR_MPC", kGrMembersPerCta)), 65535))));
  if ((nx + kGrTX - 1) / kGrTX > INT32_MAX || (ny + kGrTY - 1) / kGrTY > 65535) return DIVUQ_EGRID;
  const T cxi = T(1.0 / (2.0 * dx)), cxb = T(1.0 / dx), cyi = T(1.0 / (2.0 * dy)), cyb = T(1.0 / dy);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CUtensorMap map{};
  if (mag && in_mstride == 2 * nx * ny && out_mstride == 2 * nx * ny && !env_int("DIVUQ_NO_TMA", 0) &&
      (nx * int64_t(sizeof(T))) % 16 == 0 && aligned(in, 16) && nx < (int64_t(1) << 31) &&
      ny < (int64_t(1) << 31) && 2 * members < (int64_t(1) << 31) &&
      make_map3d<T>(&map, in, nx, ny, 2 * members, GrTma<T>::RW, GrTma<T>::RH, 256)) {
    // one CTA per tile walks all members (DIVUQ_GR_MPC splits them)
    const int64_t mpc = std::max<int64_t>(1, env_int("DIVUQ_GR_MPC", members));
    const dim3 g3{grid.x, grid.y, unsigned(std::min<int64_t>((members + mpc - 1) / mpc, 65535))};
    DIVUQ_CUDA(cudaFuncSetAttribute(gradient_tma_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(GrTma<T>::SMEM)));
    gradient_tma_kernel<T><<<g3, dim3(kGrBX, kGrBY), GrTma<T>::SMEM, s>>>(map, members, nx, ny, cxi, cxb,
                                                                          cyi, cyb, out, out_mstride, err);
    return int(cudaGetLastError());
  }
  if (mag)
    gradient2d_kernel<T, true><<<grid, dim3(kGrBX, kGrBY), 0, s>>>(in, members, in_mstride, nx, ny, cxi, cxb,
                                                              cyi, cyb, out, out_mstride, err);
  else
    gradient2d_kernel<T, false><<<grid, dim3(kGrBX, kGrBY), 0, s>>>(in, members, in_mstride, nx, ny, cxi, cxb,
                                                               cyi, cyb, out, out_mstride, err);
  return int(cudaGetLastError());
}

}  // namespace (reopened below)

extern "C" {

int divuq_velocity_magnitude_f64(const double* u, const double* v, int64_t n, double* out,
                                 int32_t* err, void* stream) {
  if (n < 0 || (n && (!u || !v || !out))) return DIVUQ_EINVAL;
  if (n == 0) return DIVUQ_OK;
  const int64_t grid = std::min<int64_t>((n + 255) / 256, int64_t(sm_count()) * 8);
  vmag_kernel<double><<<unsigned(grid), 256, 0, static_cast<cudaStream_t>(stream)>>>(u, v, n, out, err);
  return int(cudaGetLastError());
}

int divuq_gradient2d_f64(const double* values, int64_t nx, int64_t ny, double dx, double dy,
                         double* out_gx_gy, int32_t* err, void* stream) {
  return launch_gradient<double>(values, 1, 0, nx, ny, dx, dy, out_gx_gy, 0, false, err, stream);
}

int divuq_gradient_ensemble2d_f64(const double* members, int64_t n_members, int64_t nx, int64_t ny,
                                  double dx, double dy, double* out_members, int32_t* err,
                                  void* stream) {
  if (n_members < 1) return DIVUQ_EMEMBERS;
  return launch_gradient<double>(members, n_members, 2 * nx * ny, nx, ny, dx, dy, out_members,
                                 2 * nx * ny, true, err, stream);
}

int divuq_gradient_ensemble2d_f32(const float* members, int64_t n_members, int64_t nx, int64_t ny,
                                  double dx, double dy, float* out_members, int32_t* err,
                                  void* stream) {
  if (n_members < 1) return DIVUQ_EMEMBERS;
  return launch_gradient<float>(members, n_members, 2 * nx * ny, nx, ny, dx, dy, out_members,
                                2 * nx * ny, true, err, stream);
}

// host-buffer variants: kind 0 = velocity magnitude (n = nx*ny), 1 = gradient
// of a scalar field, 2 = gradient_ensemble of (M, 2, nx*ny) members
static int host_gradient_common(int kind, const double* a, const double* b, int64_t M, int64_t nx,
                                int64_t ny, double dx, double dy, double* out, int device) {
  DIVUQ_CUDA(cudaSetDevice(device));
  StreamGuard sg;
  DIVUQ_CUDA(cached_stream(0, &sg.s));
  const int64_t n = nx * ny;
  const int64_t in_elems = kind == 0 ? 2 * n : kind == 1 ? n : 2 * M * n;
  const int64_t out_elems = kind == 0 ? n : kind == 1 ? 2 * n : 2 * M * n;
  DevBuf d;
  DIVUQ_CUDA(d.alloc_on(size_t(in_elems + out_elems) * sizeof(double) + 256, sg.s));
  double* din = d.as<double>();
  double* dout = din + in_elems;
  int32_t* derr = reinterpret_cast<int32_t*>(dout + out_elems);
  DIVUQ_CUDA(cudaMemsetAsync(derr, 0, sizeof(int32_t), sg.s));
  if (kind == 0) {
    const Span ins[2] = {{din, a, size_t(n) * 8}, {din + n, b, size_t(n) * 8}};
    DIVUQ_CUDA(h2d_in(ins, 2, sg.s));
    if (int r = divuq_velocity_magnitude_f64(din, din + n, n, dout, derr, sg.s)) return r;
  } else {
    const Span ins[1] = {{din, a, size_t(in_elems) * 8}};
    DIVUQ_CUDA(h2d_in(ins, 1, sg.s));
    const int r = kind == 1 ? divuq_gradient2d_f64(din, nx, ny, dx, dy, dout, derr, sg.s)
                            : divuq_gradient_ensemble2d_f64(din, M, nx, ny, dx, dy, dout, derr, sg.s);
    if (r) return r;
  }
  const Span res1[1] = {{dout, out, size_t(out_elems) * 8}};
  int status = 0;
  DIVUQ_CUDA(d2h_out(res1, 1, derr, sg.s, &status));
  return status;
}

int divuq_host_velocity_magnitude_f64(const double* u, const double* v, int64_t n, double* out,
                                      int device) {
  if (n < 0 || (n && (!u || !v || !out))) return DIVUQ_EINVAL;
  if (n == 0) return DIVUQ_OK;
  return host_gradient_common(0, u, v, 1, n, 1, 1.0, 1.0, out, device);
}

int divuq_host_gradient2d_f64(const double* values, int64_t nx, int64_t ny, double dx, double dy,
                              double* out_gx_gy, int device) {
  if (int r = grid_ok(nx, ny, dx, dy)) return r;
  if (!values || !out_gx_gy) return DIVUQ_EINVAL;
  return host_gradient_common(1, values, nullptr, 1, nx, ny, dx, dy, out_gx_gy, device);
}

int divuq_host_gradient_ensemble2d_f64(const double* members, int64_t n_members, int64_t nx,
                                       int64_t ny, double dx, double dy, double* out_members,
                                       int device) {
  if (int r = grid_ok(nx, ny, dx, dy)) return r;
  if (!members || !out_members) return DIVUQ_EINVAL;
  if (n_members < 1) return DIVUQ_EMEMBERS;
  return host_gradient_common(2, members, nullptr, n_members, nx, ny, dx, dy, out_members, device);
}

}  // extern "C"

namespace {


}  // namespace

// =====================================================================
extern "C" {

int divuq_abi_version(void) { return DIVUQ_ABI_VERSION; }

const char* divuq_status_string(int status) {
  switch (status) {
    case DIVUQ_OK: return "ok";
    case DIVUQ_EINVAL: return "invalid argument (null pointer or bad size)";
    case DIVUQ_EGRID: return "grid must be at least 2 per axis with positive spacing";
    case DIVUQ_EMEMBERS: return "ensemble needs at least 2 members";
    case DIVUQ_ESAMPLES: return "mc_divergence needs n_samples >= 2";
    case DIVUQ_ENONFINITE: return "non-finite values are not allowed";
    case DIVUQ_ENEGSIGMA: return "sigma must be non-negative";
    case DIVUQ_EFORMAT: return "not a DIVUQ1 file or malformed header";
    case DIVUQ_ELENGTH: return "payload length differs from what the header promises";
    case DIVUQ_EOS: return "cannot read or write the file";
    case DIVUQ_EDATA: return "payload contains non-finite values";
    default: return status > 0 ? cudaGetErrorString(cudaError_t(status)) : "unknown status";
  }
}

int divuq_propagate2d_f64(const double* mu_u, const double* mu_v, const double* s_u, const double* s_v,
                          int64_t nx, int64_t ny, double dx, double dy, double t, double* out_mu,
                          double* out_sigma, double* out_p_src, double* out_p_snk, int32_t* err,
                          void* stream) {
  return propagate2d<double>(mu_u, mu_v, s_u, s_v, nx, ny, dx, dy, t, out_mu, out_sigma, out_p_src,
                             out_p_snk, err, stream);
}

int divuq_propagate2d_f32(const float* mu_u, const float* mu_v, const float* s_u, const float* s_v,
                          int64_t nx, int64_t ny, double dx, double dy, double t, float* out_mu,
                          float* out_sigma, float* out_p_src, float* out_p_snk, int32_t* err,
                          void* stream) {
  return propagate2d<float>(mu_u, mu_v, s_u, s_v, nx, ny, dx, dy, t, out_mu, out_sigma, out_p_src,
                            out_p_snk, err, stream);
}

int divuq_propagate3d_f32(const float* mu_u, const float* mu_v, const float* mu_w, const float* s_u,
                          const float* s_v, const float* s_w, const float* hl_mu, const float* hl_s,
                          const float* hh_mu, const float* hh_s, int64_t nx, int64_t ny, int64_t nzl,
                          int64_t z0, int64_t nzg, int64_t kb, int64_t ke, double dx, double dy,
                          double dz, double t, float* out_mu, float* out_sigma, float* out_p_src,
                          float* out_p_snk, int32_t* err, void* stream) {
  return propagate3d<float>(mu_u, mu_v, mu_w, s_u, s_v, s_w, hl_mu, hl_s, hh_mu, hh_s, nx, ny, nzl, z0,
                            nzg, kb, ke, dx, dy, dz, t, out_mu, out_sigma, out_p_src, out_p_snk, err,
                            stream);
}

int divuq_propagate3d_f64(const double* mu_u, const double* mu_v, const double* mu_w, const double* s_u,
                          const double* s_v, const double* s_w, const double* hl_mu, const double* hl_s,
                          const double* hh_mu, const double* hh_s, int64_t nx, int64_t ny, int64_t nzl,
                          int64_t z0, int64_t nzg, int64_t kb, int64_t ke, double dx, double dy,
                          double dz, double t, double* out_mu, double* out_sigma, double* out_p_src,
                          double* out_p_snk, int32_t* err, void* stream) {
  return propagate3d<double>(mu_u, mu_v, mu_w, s_u, s_v, s_w, hl_mu, hl_s, hh_mu, hh_s, nx, ny, nzl,
                             z0, nzg, kb, ke, dx, dy, dz, t, out_mu, out_sigma, out_p_src, out_p_snk,
                             err, stream);
}

int divuq_fit_gaussian_f64(const double* members, int64_t M, int64_t C, int64_t N, double* out_mu,
                           double* out_sigma, int32_t* err, void* stream) {
  return fit_gaussian<double>(members, M, C, N, out_mu, out_sigma, err, stream);
}

int divuq_fit_gaussian_f32(const float* members, int64_t M, int64_t C, int64_t N, float* out_mu,
                           float* out_sigma, int32_t* err, void* stream) {
  return fit_gaussian<float>(members, M, C, N, out_mu, out_sigma, err, stream);
}

int divuq_fit_gaussian_strided_f32(const float* members, int64_t M, int64_t member_stride,
                                   int64_t N, float* out_mu, float* out_sigma, float* out_r,
                                   int32_t* err, void* stream) {
  return fit_gaussian<float>(members, M, 1, N, out_mu, out_sigma, err, stream, member_stride, out_r);
}

// ---- page-locking caller-owned host memory (the drop-in output pool) -----
// api.py keeps its large results in a small pool of host blocks pinned once
// (portable, mapped): the host entries then DMA (or copy-kernel) straight
// into the returned arrays -- no staging copy, no page faults on fresh
// output pages (fit_gaussian 1024^2 x 20: 8.7 ms in the C entry, 17 ms with
// fresh numpy outputs, tools/fit_trace.py).
// a refusal (no device, the pinned-memory limit) is reported and cleared, so
// it never surfaces later as a launch's cudaGetLastError
int divuq_host_register(void* ptr, int64_t bytes) {
  if (!ptr || bytes <= 0) return DIVUQ_EINVAL;
  const cudaError_t e = cudaHostRegister(ptr, size_t(bytes), cudaHostRegisterPortable | cudaHostRegisterMapped);
  if (e != cudaSuccess) cudaGetLastError();
  return int(e);
}
int divuq_host_unregister(void* ptr) {
  if (!ptr) return DIVUQ_EINVAL;
  const cudaError_t e = cudaHostUnregister(ptr);
  if (e != cudaSuccess) cudaGetLastError();
  return int(e);
}

// ---- peer memory (CUDA IPC) for the z-slab exchange over NVLink ----------
// A rank exports the allocation holding a tensor (handle + the tensor's offset
// in it); a neighbour imports it and its kernels read the halo planes straight
// from the owner's HBM -- no separate exchange step.
using GetAddressRangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);

int divuq_ipc_export(const void* ptr, void* handle_out, int64_t* offset_out) {
  if (!ptr || !handle_out || !offset_out) return DIVUQ_EINVAL;
  static GetAddressRangeFn range = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<GetAddressRangeFn>(p);
  }();
  if (!range) return int(cudaErrorNotSupported);
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS) return int(cudaErrorInvalidValue);
  cudaIpcMemHandle_t h;
  DIVUQ_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  std::memcpy(handle_out, &h, sizeof(h));
  *offset_out = int64_t(reinterpret_cast<CUdeviceptr>(ptr) - base);
  return DIVUQ_OK;
}

int divuq_ipc_import(const void* handle, int64_t offset, void** base_out, void** ptr_out) {
  if (!handle || !base_out || !ptr_out || offset < 0) return DIVUQ_EINVAL;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  void* base = nullptr;
  DIVUQ_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  *base_out = base;
  *ptr_out = static_cast<char*>(base) + offset;
  return DIVUQ_OK;
}

int divuq_ipc_close(void* base) {
  if (!base) return DIVUQ_EINVAL;
  return int(cudaIpcCloseMemHandle(base));
}

int64_t divuq_ipc_handle_bytes(void) { return int64_t(sizeof(cudaIpcMemHandle_t)); }

// 2D fused ensemble as a row march (k3row.cuh); *used = false when not eligible
int try_k3_rowmarch(const StencilParams<float>& sp, cudaStream_t s, bool* used) {
  using C = RmCfg;
  *used = false;
  if (env_int("DIVUQ_NO_TMA", 0) || env_int("DIVUQ_NO_ROWMARCH", 0)) return DIVUQ_OK;
  if (sp.nx % 4 || sp.n_members < 2 || sp.n_members > 256) return DIVUQ_OK;   // TMA rows: 16 B units
  const void* ptrs[] = {sp.members, sp.out_mu, sp.out_sigma, sp.out_psrc, sp.out_psnk,
                        sp.out_mom_mu, sp.out_mom_sigma};
  for (const void* q : ptrs)
    if (!aligned(q, 16)) return DIVUQ_OK;
  if (sp.nx > (int64_t(1) << 30) || sp.ny > (int64_t(1) << 30)) return DIVUQ_OK;
  const int64_t M = sp.n_members;
  RmParams p;
  std::memset(&p, 0, sizeof(p));
  const uint32_t u_bytes = uint32_t(M * C::TXP * 4), v_bytes = uint32_t(M * C::TX * 4);
  p.v_off = (u_bytes + 127) / 128 * 128;
  p.stage_stride = (p.v_off + v_bytes + 127) / 128 * 128;
  p.stage_bytes = u_bytes + v_bytes;
  const size_t ring = (sizeof(RmRing) + 1023) / 1024 * 1024;
  // CTAs per SM: DIVUQ_RM_MINB (2) when its share of shared memory holds
  // S >= NW stages, else 1.  Every consumer warp of a group waits on its own
  // stage: S >= NW, or two rows one phase apart would share a stage (parity
  // aliasing).
  int64_t cps = std::max<int64_t>(1, std::min<int64_t>(4, env_int("DIVUQ_RM_CPS", DIVUQ_RM_MINB)));
  for (;; --cps) {
    const size_t budget = 227 * 1024 / size_t(cps) - ring - 2 * C::SMAX * sizeof(uint64_t) - 1024;
    p.S = int(std::min<size_t>(C::SMAX, budget / p.stage_stride));
    if (p.S >= C::NW) break;
    if (cps == 1) return DIVUQ_OK;
  }
  RmMaps tm;
  std::memset(&tm, 0, sizeof(tm));
  if (!make_map5d_members(&tm.u, sp.members, sp.nx, sp.ny, 1, 2, M, C::TXP, 1, int(M), 256) ||
      !make_map5d_members(&tm.v, sp.members, sp.nx, sp.ny, 1, 2, M, C::TX, 1, int(M), 256))
    return DIVUQ_OK;
  p.nx = int(sp.nx); p.ny = int(sp.ny); p.M = int(M);
  p.strips = int((sp.nx + C::TX - 1) / C::TX);
  const int64_t sms = sm_count();
  const int64_t segs_wanted = std::max<int64_t>(1, cps * sms / p.strips);
  p.seg_rows = int(std::max<int64_t>(C::NW, (sp.ny + segs_wanted - 1) / segs_wanted));
  const int64_t segs = (sp.ny + p.seg_rows - 1) / p.seg_rows;
  p.cx_in = sp.cx_in; p.cx_bd = sp.cx_bd; p.cy_in = sp.cy_in; p.cy_bd = sp.cy_bd; p.theta = sp.theta;
  p.out_mu = sp.out_mu; p.out_sigma = sp.out_sigma; p.out_psrc = sp.out_psrc; p.out_psnk = sp.out_psnk;
  p.out_mom_mu = sp.out_mom_mu; p.out_mom_sigma = sp.out_mom_sigma;
  p.err = sp.err;
  const size_t smem = ring + size_t(p.S) * p.stage_stride + 2 * C::SMAX * sizeof(uint64_t);
  DIVUQ_CUDA(cudaFuncSetAttribute(k3_rowmarch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(smem)));
  k3_rowmarch_kernel<<<unsigned(int64_t(p.strips) * segs), C::THREADS, smem, s>>>(tm, p);
  *used = true;
  return int(cudaGetLastError());
}

// Fused-ensemble fallback for the shapes the TMA kernels do not take
// (nx % 4 != 0, unaligned pointers): K1 writes the ShiftedMoments triples
// (mu, r, sigma), the kResidual stencil differences the (mu, r) pairs exactly
// as the fused kernels do, so every path agrees bit for bit.  Scratch comes
// from the stream-ordered pool (the moments go straight to out_mom_* when the
// caller asked for them).
static int ensemble_fallback(StencilParams<float> p, int comps, cudaStream_t s) {
  const int64_t nl = p.comp_stride;
  const bool own = p.out_mom_mu != nullptr;
  DevBuf scratch;
  DIVUQ_CUDA(scratch.alloc_on(size_t(comps) * nl * (own ? 1 : 3) * sizeof(float), s));
  float* r = scratch.as<float>();
  float* mu = own ? p.out_mom_mu : r + comps * nl;
  float* sg = own ? p.out_mom_sigma : r + 2 * comps * nl;
  if (int e = fit_gaussian<float>(p.members, p.n_members, comps, nl, mu, sg, p.err, s, p.member_stride, r))
    return e;
  p.mu_u = mu; p.mu_v = mu + nl; p.mu_w = comps == 3 ? mu + 2 * nl : nullptr;
  p.s_u = sg; p.s_v = sg + nl; p.s_w = comps == 3 ? sg + 2 * nl : nullptr;
  p.r_u = r; p.r_v = r + nl; p.r_w = comps == 3 ? r + 2 * nl : nullptr;
  if (comps == 3) return dispatch_vec<float, true, kResidual>(p, true, s);
  return dispatch_vec<float, false, kResidual>(p, true, s);
}

int divuq_ensemble_divergence2d_f32(const float* members, int64_t M, int64_t nx, int64_t ny, double dx,
                                    double dy, double t, float* out_mu, float* out_sigma,
                                    float* out_p_src, float* out_p_snk, float* out_mom_mu,
                                    float* out_mom_sigma, int32_t* err, void* stream) {
  if (int r = grid_ok(nx, ny, dx, dy)) return r;
  if (!members) return DIVUQ_EINVAL;
  if (M < 2) return DIVUQ_EMEMBERS;
  if ((out_mom_mu == nullptr) != (out_mom_sigma == nullptr)) return DIVUQ_EINVAL;
  StencilParams<float> p = blank_params<float>();
  p.members = members; p.n_members = M; p.comp_stride = nx * ny; p.member_stride = 2 * nx * ny;
  p.nx = nx; p.ny = ny; p.nzl = 1; p.z0 = 0; p.nzg = 1; p.kbeg = 0; p.kend = 1;
  set_coeffs(p, dx, dy, 1.0);
  p.theta = float(t);
  p.out_mu = out_mu; p.out_sigma = out_sigma; p.out_psrc = out_p_src; p.out_psnk = out_p_snk;
  p.out_mom_mu = out_mom_mu; p.out_mom_sigma = out_mom_sigma;
  p.err = err;
  bool used = false;
  if (int r = try_k3_rowmarch(p, static_cast<cudaStream_t>(stream), &used)) return r;
  if (used) return DIVUQ_OK;
  if (int r = try_k3_tma(p, 2, static_cast<cudaStream_t>(stream), &used)) return r;
  if (used) return DIVUQ_OK;
  return ensemble_fallback(p, 2, static_cast<cudaStream_t>(stream));
}

// K6 as a strip march (gradmarch.cuh; DIVUQ_GRADMARCH=1) when TMA applies and the rings fit:
// returns -1 when launched, 0 when not eligible, >0 on a CUDA error
static int try_gradmarch(const GfParams& g, cudaStream_t s) {
  // opt-in: measured 81 us against the tiled K6's 63 us at 1024^2 x 20 (18 warps
  // per SM with two CTA barriers per two-row step: latency-bound, 47 % issue)
  if (env_int("DIVUQ_NO_TMA", 0) || !env_int("DIVUQ_GRADMARCH", 0)) return 0;
  const int64_t nx = g.nx, ny = g.ny, M = g.M;
  if (nx % 4 || !aligned(g.members, 16) || 2 * M > 256 || nx >= (int64_t(1) << 31) ||
      ny >= (int64_t(1) << 30))
    return 0;
  GmParams p{};
  p.nx = int(nx); p.ny = int(ny); p.M = int(M);
  p.stage_bytes = uint32_t(kGmW * kGmRows * 2 * M * 4);
  p.stage_stride = (p.stage_bytes + 127) / 128 * 128;
  const uint32_t mag_bytes = uint32_t(kGmRing * M * kGmW * 8);
  const uint32_t mom_bytes = uint32_t(kGmRing * sizeof(GmMomRow));
  // 2 CTAs / SM with >= 2 stages, else 1 CTA / SM, else not eligible
  const size_t limit = 227 * 1024;
  int cps = 2, S = 0;
  for (; cps >= 1; --cps) {
    const size_t budget = limit / size_t(cps) - (cps > 1 ? 1024 : 0);
    const size_t fixed = size_t(mag_bytes) + mom_bytes + kGmMaxStages * 8 + 256;
    if (budget <= fixed) continue;
    S = int(std::min<size_t>(kGmMaxStages, (budget - fixed) / p.stage_stride));
    if (S >= 2) break;
  }
  if (S < 2) return 0;
  p.S = S;
  p.mag_off = uint32_t(S) * p.stage_stride;
  p.mom_off = (p.mag_off + mag_bytes + 127) / 128 * 128;
  p.bar_off = (p.mom_off + mom_bytes + 15) / 16 * 16;
  const size_t smem = p.bar_off + kGmMaxStages * 8;
  CUtensorMap map{};
  if (!make_map3d<float>(&map, g.members, nx, ny, 2 * M, kGmW, kGmRows, 256)) return 0;
  // the TMA box holds all 2M planes: make_map3d's box z is 1 -- re-encode
  {
    EncodeTiledFn fn = encode_tiled();
    const cuuint64_t dims[3] = {cuuint64_t(nx), cuuint64_t(ny), cuuint64_t(2 * M)};
    const cuuint64_t strides[2] = {cuuint64_t(nx) * 4, cuuint64_t(nx * ny) * 4};
    const cuuint32_t box[3] = {cuuint32_t(kGmW), cuuint32_t(kGmRows), cuuint32_t(2 * M)};
    const cuuint32_t es[3] = {1, 1, 1};
    if (fn(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(g.members), dims, strides, box, es,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return 0;
  }
  p.strips = int((nx + kGmTX - 1) / kGmTX);
  const int64_t want = std::max<int64_t>(1, int64_t(cps) * sm_count() / p.strips);
  p.seg_rows = int(std::max<int64_t>(8, (ny + want - 1) / want));
  p.seg_rows += p.seg_rows & 1;
  const int64_t segs = (ny + p.seg_rows - 1) / p.seg_rows;
  p.cx_in = g.cx_in; p.cx_bd = g.cx_bd; p.cy_in = g.cy_in; p.cy_bd = g.cy_bd; p.theta = g.theta;
  p.out_mu = g.out_mu; p.out_sigma = g.out_sigma; p.out_psrc = g.out_psrc; p.out_psnk = g.out_psnk;
  p.out_mom_mu = g.out_mom_mu; p.out_mom_sigma = g.out_mom_sigma;
  p.err = g.err;
  DIVUQ_CUDA(cudaFuncSetAttribute(gradmarch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  gradmarch_kernel<<<unsigned(int64_t(p.strips) * segs), kGmThreads, smem, s>>>(map, p);
  if (int e = int(cudaGetLastError())) return e;
  return -1;
}

int divuq_gradient_ensemble_divergence2d_f32(const float* members, int64_t M, int64_t nx,
                                             int64_t ny, double dx, double dy, double t,
                                             float* out_mu, float* out_sigma, float* out_p_src,
                                             float* out_p_snk, float* out_mom_mu,
                                             float* out_mom_sigma, int32_t* err, void* stream) {
  if (int r = grid_ok(nx, ny, dx, dy)) return r;
  if (!members) return DIVUQ_EINVAL;
  if (M < 2) return DIVUQ_EMEMBERS;
  if ((out_mom_mu == nullptr) != (out_mom_sigma == nullptr)) return DIVUQ_EINVAL;
  const int64_t tx = (nx + kGfTX - 1) / kGfTX, ty = (ny + kGfTY - 1) / kGfTY;
  if (tx > INT32_MAX || ty > 65535) return DIVUQ_EGRID;
  GfParams p{};
  p.members = members; p.M = M; p.nx = nx; p.ny = ny;
  p.cx_in = float(1.0 / (2.0 * dx)); p.cx_bd = float(1.0 / dx);   // stencils.py:48-50
  p.cy_in = float(1.0 / (2.0 * dy)); p.cy_bd = float(1.0 / dy);
  p.theta = float(t);
  p.out_mu = out_mu; p.out_sigma = out_sigma; p.out_psrc = out_p_src; p.out_psnk = out_p_snk;
  p.out_mom_mu = out_mom_mu; p.out_mom_sigma = out_mom_sigma;
  p.err = err;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (int r = try_gradmarch(p, s)) return r < 0 ? 0 : r;   // -1: launched
  const dim3 grid{unsigned(tx), unsigned(ty)}, block{kGfBX, kGfBY};
  CUtensorMap map{};
  const bool tma = !env_int("DIVUQ_NO_TMA", 0) && nx % 4 == 0 && aligned(members, 16) &&
                   nx < (int64_t(1) << 31) && ny < (int64_t(1) << 31) && 2 * M < (int64_t(1) << 31) &&
                   make_map3d<float>(&map, members, nx, ny, 2 * M, kGfRW, kGfRH, 256);
  if (tma) {
    DIVUQ_CUDA(cudaFuncSetAttribute(gradfused_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(kGfSmemTma)));
    gradfused_kernel<true><<<grid, block, kGfSmemTma, s>>>(map, p);
  } else {
    gradfused_kernel<false><<<grid, block, kGfSmemLdg, s>>>(map, p);
  }
  return int(cudaGetLastError());
}

int divuq_ensemble_divergence3d_f32(const float* members, int64_t M, const float* hl_mu,
                                    const float* hl_s, const float* hl_r, const float* hh_mu,
                                    const float* hh_s, const float* hh_r,
                                    int64_t nx, int64_t ny, int64_t nzl, int64_t z0, int64_t nzg,
                                    int64_t kb, int64_t ke, double dx, double dy, double dz, double t,
                                    float* out_mu, float* out_sigma, float* out_p_src,
                                    float* out_p_snk, float* out_mom_mu, float* out_mom_sigma,
                                    int32_t* err, void* stream) {
  if (int r = grid_ok(nx, ny, dx, dy)) return r;
  if (nzg < 2 || !(dz > 0.0)) return DIVUQ_EGRID;
  if (nzl < 1 || z0 < 0 || z0 + nzl > nzg || kb < 0 || ke > nzl || kb > ke) return DIVUQ_EINVAL;
  if (!members) return DIVUQ_EINVAL;
  if (M < 2) return DIVUQ_EMEMBERS;
  if (z0 > 0 && (!hl_mu || !hl_s)) return DIVUQ_EINVAL;
  if (z0 + nzl < nzg && (!hh_mu || !hh_s)) return DIVUQ_EINVAL;
  if ((out_mom_mu == nullptr) != (out_mom_sigma == nullptr)) return DIVUQ_EINVAL;
  StencilParams<float> p = blank_params<float>();
  const int64_t nl = nx * ny * nzl;
  p.members = members; p.n_members = M; p.comp_stride = nl; p.member_stride = 3 * nl;
  p.halo_lo_mu_w = hl_mu; p.halo_lo_s_w = hl_s; p.halo_hi_mu_w = hh_mu; p.halo_hi_s_w = hh_s;
  p.halo_lo_r_w = hl_r; p.halo_hi_r_w = hh_r;
  p.nx = nx; p.ny = ny; p.nzl = nzl; p.z0 = z0; p.nzg = nzg; p.kbeg = kb; p.kend = ke;
  set_coeffs(p, dx, dy, dz);
  p.theta = float(t);
  p.out_mu = out_mu; p.out_sigma = out_sigma; p.out_psrc = out_p_src; p.out_psnk = out_p_snk;
  p.out_mom_mu = out_mom_mu; p.out_mom_sigma = out_mom_sigma;
  p.err = err;
  bool used = false;
  if (int r = try_k3_tma(p, 3, static_cast<cudaStream_t>(stream), &used)) return r;
  if (used) return DIVUQ_OK;
  return ensemble_fallback(p, 3, static_cast<cudaStream_t>(stream));
}

int divuq_tail_probs_f64(const double* mu, const double* sigma, int64_t n, double theta,
                         double* out_below, double* out_above, int32_t* err, void* stream) {
  return tail_probs<double>(mu, sigma, n, theta, out_below, out_above, err, stream);
}

int divuq_tail_probs_f32(const float* mu, const float* sigma, int64_t n, double theta,
                         float* out_below, float* out_above, int32_t* err, void* stream) {
  return tail_probs<float>(mu, sigma, n, theta, out_below, out_above, err, stream);
}

int divuq_lcp2d_f64(const double* mu, const double* sigma, int64_t nx, int64_t ny, double isovalue,
                    double* out, int32_t* err, void* stream) {
  if (nx < 2 || ny < 2) return DIVUQ_EGRID;
  if (!mu || !sigma || !out) return DIVUQ_EINVAL;
  dim3 grid(unsigned((nx - 1 + kLcpTX - 1) / kLcpTX), unsigned((ny - 1 + kLcpTY - 1) / kLcpTY));
  CUtensorMap mm{}, ms{};
  if (!env_int("DIVUQ_NO_TMA", 0) && nx % 2 == 0 && aligned(mu, 16) && aligned(sigma, 16) &&
      nx < (int64_t(1) << 31) && ny < (int64_t(1) << 31) &&
      make_map3d<double>(&mm, mu, nx, ny, 1, LcpTma<double>::W, LcpTma<double>::H, 0) &&
      make_map3d<double>(&ms, sigma, nx, ny, 1, LcpTma<double>::W, LcpTma<double>::H, 0)) {
    const dim3 gt(grid.x, unsigned((ny - 1 + kLcpTYT - 1) / kLcpTYT));
    lcp2d_tma_kernel<double><<<gt, dim3(kLcpBX, kLcpBY), 0, static_cast<cudaStream_t>(stream)>>>(
        mm, ms, nx, ny, isovalue, out, err);
    return int(cudaGetLastError());
  }
  // odd nx: row boxes on 1D tensor maps (lcp2d_flat_kernel)
  if (!env_int("DIVUQ_NO_TMA", 0) && !env_int("DIVUQ_NO_FLAT", 0) && aligned(mu, 16) &&
      aligned(sigma, 16) && nx * ny + 2 * nx + LcpFlat::BOX < (int64_t(1) << 31) &&
      make_map1d<double>(&mm, mu, nx * ny, LcpFlat::BOX) && make_map1d<double>(&ms, sigma, nx * ny, LcpFlat::BOX)) {
    const dim3 gf(grid.x, unsigned((ny - 1 + kLcpFTY - 1) / kLcpFTY));
    lcp2d_flat_kernel<<<gf, dim3(kLcpBX, kLcpBY), 0, static_cast<cudaStream_t>(stream)>>>(
        mm, ms, nx, ny, isovalue, out, err);
    return int(cudaGetLastError());
  }
  lcp2d_kernel<double><<<grid, dim3(kLcpBX, kLcpBY), 0, static_cast<cudaStream_t>(stream)>>>(
      mu, sigma, nx, ny, isovalue, out, err);
  return int(cudaGetLastError());
}

// propagate_divergence -> lcp in one pass (lcp2d_fused_kernel); shapes the
// TMA boxes cannot take run K2 then the LCP kernel: the same bits either way
int divuq_propagate_lcp2d_f64(const double* mu_u, const double* mu_v, const double* s_u,
                              const double* s_v, int64_t nx, int64_t ny, double dx, double dy,
                              double isovalue, double* out_mu, double* out_sigma, double* out_lcp,
                              int32_t* err, void* stream) {
  if (int r = grid_ok(nx, ny, dx, dy)) return r;
  if (!mu_u || !mu_v || !s_u || !s_v || !out_lcp) return DIVUQ_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CUtensorMap m[4];
  const double* in[4] = {mu_u, s_u, mu_v, s_v};
  bool tma = !env_int("DIVUQ_NO_TMA", 0) && nx % 2 == 0 && nx < (int64_t(1) << 31) &&
             ny < (int64_t(1) << 31);
  for (int k = 0; k < 4 && tma; ++k)
    tma = aligned(in[k], 16) &&
          make_map3d<double>(&m[k], in[k], nx, ny, 1, k < 2 ? LcpFused::UW : LcpFused::VW,
                             k < 2 ? LcpFused::UH : LcpFused::VH, 0);
  if (!tma) {
    const int64_t n = nx * ny;
    DevBuf scratch;
    double* mu = out_mu;
    double* sg = out_sigma;
    if (!mu || !sg) {
      DIVUQ_CUDA(scratch.alloc_on(size_t(2 * n) * sizeof(double), s));
      if (!mu) mu = scratch.as<double>();
      if (!sg) sg = scratch.as<double>() + n;
    }
    if (int r = propagate2d<double>(mu_u, mu_v, s_u, s_v, nx, ny, dx, dy, 0.0, mu, sg, nullptr, nullptr,
                                    err, stream))
      return r;
    return divuq_lcp2d_f64(mu, sg, nx, ny, isovalue, out_lcp, err, stream);
  }
  LcpFusedParams p{};
  p.nx = nx; p.ny = ny;
  p.cx_in = 1.0 / (2.0 * dx); p.cx_bd = 1.0 / dx;   // stencils.py:48-50, fp64 on the host
  p.cy_in = 1.0 / (2.0 * dy); p.cy_bd = 1.0 / dy;
  p.theta = isovalue;
  p.out_mu = out_mu; p.out_sigma = out_sigma; p.out_lcp = out_lcp; p.err = err;
  const dim3 grid(unsigned((nx - 1 + kLcpTX - 1) / kLcpTX), unsigned((ny - 1 + kLcpFY - 1) / kLcpFY));
  if (grid.y > 65535) return DIVUQ_EGRID;
  DIVUQ_CUDA(cudaFuncSetAttribute(lcp2d_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(sizeof(LcpFusedSmem))));
  lcp2d_fused_kernel<<<grid, dim3(kLcpBX, kLcpBY), sizeof(LcpFusedSmem), s>>>(m[0], m[1], m[2], m[3], p);
  return int(cudaGetLastError());
}

int divuq_lcp2d_f32(const float* mu, const float* sigma, int64_t nx, int64_t ny, double isovalue,
                    float* out, int32_t* err, void* stream) {
  if (nx < 2 || ny < 2) return DIVUQ_EGRID;
  if (!mu || !sigma || !out) return DIVUQ_EINVAL;
  dim3 grid(unsigned((nx - 1 + kLcpTX - 1) / kLcpTX), unsigned((ny - 1 + kLcpTY - 1) / kLcpTY));
  lcp2d_kernel<float><<<grid, dim3(kLcpBX, kLcpBY), 0, static_cast<cudaStream_t>(stream)>>>(
      mu, sigma, nx, ny, float(isovalue), out, err);
  return int(cudaGetLastError());
}

int divuq_cell_crossing_f64(const double* mu4, const double* sigma4, int64_t n_cells, double isovalue,
                            double* out, int32_t* err, void* stream) {
  if (n_cells < 0 || (n_cells && (!mu4 || !sigma4 || !out))) return DIVUQ_EINVAL;
  if (n_cells == 0) return DIVUQ_OK;
  const int64_t grid = std::min<int64_t>((n_cells + 255) / 256, int64_t(sm_count()) * 8);
  cell_crossing_kernel<double><<<unsigned(grid), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      mu4, sigma4, n_cells, isovalue, out, err);
  return int(cudaGetLastError());
}

int64_t mc_slots(int64_t n_samples) {   // a function of n_samples only (launch-invariant)
  return std::min<int64_t>(32, (n_samples + kMcChunk - 1) / kMcChunk);
}

int64_t divuq_mc_scratch_bytes(int64_t nx, int64_t row_begin, int64_t row_end, int64_t n_samples) {
  if (nx < 1 || row_end <= row_begin || n_samples < 1) return 0;
  return 2 * mc_slots(n_samples) * (row_end - row_begin) * nx * int64_t(sizeof(double));
}

int divuq_mc_divergence2d_f64(const double* mu_u, const double* mu_v, const double* s_u,
                              const double* s_v, int64_t nx, int64_t ny, double dx, double dy,
                              int64_t n_samples, uint64_t seed, int64_t row_begin, int64_t row_end,
                              double* out_mean, double* out_std, void* scratch, int32_t* err,
                              void* stream) {
  if (int r = grid_ok(nx, ny, dx, dy)) return r;
  if (n_samples < 2) return DIVUQ_ESAMPLES;
  if (!mu_u || !mu_v || !s_u || !s_v || !out_mean || !out_std || !scratch) return DIVUQ_EINVAL;
  if (row_begin < 0 || row_end > ny || row_begin >= row_end) return DIVUQ_EINVAL;
  McParams p;
  std::memset(&p, 0, sizeof(p));
  p.mu_u = mu_u; p.mu_v = mu_v; p.s_u = s_u; p.s_v = s_v;
  p.nx = nx; p.ny = ny; p.row_begin = row_begin; p.row_end = row_end;
  p.n_samples = n_samples; p.n_chunks = (n_samples + kMcChunk - 1) / kMcChunk;
  p.n_slots = mc_slots(n_samples);
  p.seed = seed;
  for (int r = 0; r < 10; ++r) {  // Philox round keys: key + r * (W0, W1) mod 2^32
    p.k0[r] = uint32_t(seed) + uint32_t(r) * 0x9E3779B9u;
    p.k1[r] = uint32_t(seed >> 32) + uint32_t(r) * 0xBB67AE85u;
  }
  p.cx_in = 1.0 / (2.0 * dx); p.cx_bd = 1.0 / dx; p.cy_in = 1.0 / (2.0 * dy); p.cy_bd = 1.0 / dy;
  const int64_t nv = (row_end - row_begin) * nx;
  p.part_mean = static_cast<double*>(scratch);
  p.part_m2 = p.part_mean + p.n_slots * nv;
  p.out_mean = out_mean; p.out_std = out_std; p.err = err;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t gx = (nx + kMcTX - 1) / kMcTX, gy = (row_end - row_begin + kMcTY - 1) / kMcTY;
  if (gx > INT32_MAX || gy > 65535) return DIVUQ_EGRID;   // grid.z = slots <= 32
  dim3 grid(unsigned(gx), unsigned(gy), unsigned(p.n_slots));
  DIVUQ_CUDA(cudaFuncSetAttribute(mc_chunk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(sizeof(McSmem))));
  mc_chunk_kernel<<<grid, dim3(kMcTX, kMcTY), sizeof(McSmem), s>>>(p);
  DIVUQ_CUDA(cudaGetLastError());
  const int64_t threads = 256;
  mc_merge_kernel<<<unsigned((nv * 32 + threads - 1) / threads), unsigned(threads), 0, s>>>(p);
  return int(cudaGetLastError());
}

int divuq_mc_divergence2d_ref_f64(const double* mu_u, const double* mu_v, const double* s_u,
                                  const double* s_v, int64_t nx, int64_t ny, double dx, double dy,
                                  int64_t n_samples, uint64_t seed, int64_t row_begin,
                                  int64_t row_end, double* out_mean, double* out_std, int32_t* err,
                                  void* stream) {
  if (int r = grid_ok(nx, ny, dx, dy)) return r;
  if (n_samples < 2) return DIVUQ_ESAMPLES;
  if (!mu_u || !mu_v || !s_u || !s_v || !out_mean || !out_std) return DIVUQ_EINVAL;
  if (row_begin < 0 || row_end > ny || row_begin >= row_end) return DIVUQ_EINVAL;
  McRefParams p;
  p.mu_u = mu_u; p.mu_v = mu_v; p.s_u = s_u; p.s_v = s_v;
  p.nx = nx; p.ny = ny; p.row_begin = row_begin; p.row_end = row_end;
  p.n_samples = n_samples; p.seed = seed;
  p.cx_in = 1.0 / (2.0 * dx); p.cx_bd = 1.0 / dx; p.cy_in = 1.0 / (2.0 * dy); p.cy_bd = 1.0 / dy;
  p.out_mean = out_mean; p.out_std = out_std; p.err = err;
  dim3 grid(unsigned((nx + kMrTX - 1) / kMrTX), unsigned((row_end - row_begin + kMrTY - 1) / kMrTY));
  mc_ref_kernel<<<grid, dim3(kMrTX, kMrTY), 0, static_cast<cudaStream_t>(stream)>>>(p);
  return int(cudaGetLastError());
}

int divuq_sample_divergence1d_f64(const double* neighbors, double dx, double dy, int64_t n_samples,
                                  uint64_t seed, double* out, void* stream) {
  if (!neighbors || n_samples < 0 || (n_samples && !out)) return DIVUQ_EINVAL;
  for (int k = 1; k < 8; k += 2)
    if (neighbors[k] < 0.0) return DIVUQ_ENEGSIGMA;   // mc.py:147-149
  if (n_samples == 0) return DIVUQ_OK;
  const int64_t grid = std::min<int64_t>((n_samples + 255) / 256, int64_t(sm_count()) * 8);
  sample_1d_kernel<<<unsigned(grid), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      neighbors[0], neighbors[1], neighbors[2], neighbors[3], neighbors[4], neighbors[5],
      neighbors[6], neighbors[7], 2.0 * dx, 2.0 * dy, n_samples, seed, out);
  return int(cudaGetLastError());
}

int divuq_minmax_f64(const double* values, int64_t n, double* out_minmax, void* scratch16,
                     void* stream) {
  if (!values || n < 1 || !out_minmax || !scratch16) return DIVUQ_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const long long init[2] = {0x7fffffffffffffffll, (long long)0x8000000000000000ull};
  DIVUQ_CUDA(cudaMemcpyAsync(scratch16, init, sizeof(init), cudaMemcpyHostToDevice, s));
  const int64_t grid = std::min<int64_t>((n + 255) / 256, int64_t(sm_count()) * 8);
  minmax_kernel<<<unsigned(grid), 256, 0, s>>>(values, n, static_cast<long long*>(scratch16));
  DIVUQ_CUDA(cudaGetLastError());
  minmax_finish_kernel<<<1, 1, 0, s>>>(static_cast<long long*>(scratch16), out_minmax);
  return int(cudaGetLastError());
}

// np.linspace(lo, hi, nbins + 1) (numpy 2.3 function_base: step = (hi - lo) / nbins,
// edge_i = i * step + lo, last = hi) -- host arithmetic, no contraction
static void linspace_edges(double lo, double hi, int64_t nbins, double* edges) {
  volatile double step = (hi - lo) / double(nbins);
  for (int64_t i = 0; i <= nbins; ++i) {
    volatile double y = double(i) * step;
    edges[i] = y + lo;
  }
  edges[nbins] = hi;
}

int divuq_histogram_uniform_f64(const double* values, int64_t n, double lo, double hi,
                                int64_t n_bins, double* edges_dev, int64_t* counts_dev,
                                void* stream) {
  if (!values || n < 0 || n_bins < 1 || !edges_dev || !counts_dev || !(lo < hi)) return DIVUQ_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<double> e(size_t(n_bins) + 1);
  linspace_edges(lo, hi, n_bins, e.data());
  DIVUQ_CUDA(cudaMemcpyAsync(edges_dev, e.data(), e.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  DIVUQ_CUDA(cudaMemsetAsync(counts_dev, 0, size_t(n_bins) * sizeof(int64_t), s));
  if (n) {
    const int64_t grid = std::min<int64_t>((n + 255) / 256, int64_t(sm_count()) * 8);
    histogram_kernel<<<unsigned(grid), 256, 0, s>>>(values, n, edges_dev, n_bins,
                                                    reinterpret_cast<unsigned long long*>(counts_dev));
  }
  // the host edge vector must outlive the async copy
  DIVUQ_CUDA(cudaStreamSynchronize(s));
  return int(cudaGetLastError());
}

int divuq_gen_field_f32(const float* bumps, int n_bumps, int dims, int64_t nx, int64_t ny, int64_t nzl,
                        int64_t z0, double dx, double dy, double dz, double vortex_amp,
                        double vortex_cx, double vortex_cy, double vortex_r, double shear_amp,
                        uint64_t seed, double sig_lo, double sig_hi, int sigma_mode,
                        int64_t n_members, float* const* out, float* members, void* stream) {
  if ((dims != 2 && dims != 3) || nx < 1 || ny < 1 || nzl < 1) return DIVUQ_EINVAL;
  if (n_members == 0 && !out) return DIVUQ_EINVAL;
  if (n_members > 0 && !members) return DIVUQ_EINVAL;
  GenParams p;
  std::memset(&p, 0, sizeof(p));
  p.bumps = reinterpret_cast<const Bump*>(bumps); p.n_bumps = n_bumps;
  p.nx = nx; p.ny = ny; p.nzl = nzl; p.z0 = z0;
  p.dx = float(dx); p.dy = float(dy); p.dz = float(dz); p.dims = dims;
  p.vortex_amp = float(vortex_amp); p.vortex_cx = float(vortex_cx); p.vortex_cy = float(vortex_cy);
  p.vortex_inv_r2 = vortex_r > 0 ? float(1.0 / (vortex_r * vortex_r)) : 0.f;
  p.shear_amp = float(shear_amp); p.shear_ly = float(double(ny - 1) * dy);
  p.seed = seed; p.sig_lo = float(sig_lo); p.sig_hi = float(sig_hi); p.sigma_mode = sigma_mode;
  p.n_members = n_members;
  if (n_members == 0)
    for (int c = 0; c < 2 * dims; ++c) {
      if (!out[c]) return DIVUQ_EINVAL;
      p.out[c] = out[c];
    }
  p.members = members;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t nl = nx * ny * nzl;
  const int64_t grid = std::min<int64_t>((nl + 255) / 256, int64_t(sm_count()) * 16);
  gen_kernel<<<unsigned(grid), 256, 0, s>>>(p);
  return int(cudaGetLastError());
}

// ---------------------------------------------------------------------
// host-buffer entry points
// ---------------------------------------------------------------------

int divuq_host_propagate2d_f64(const double* mu_u, const double* mu_v, const double* s_u,
                               const double* s_v, int64_t nx, int64_t ny, double dx, double dy,
                               double t, double* out_mu, double* out_sigma, double* out_p_src,
                               double* out_p_snk, int device) {
  if (int r = grid_ok(nx, ny, dx, dy)) return r;
  if (!mu_u || !mu_v) return DIVUQ_EINVAL;
  const bool has_sigma = out_sigma || out_p_src || out_p_snk;
  if (has_sigma && (!s_u || !s_v)) return DIVUQ_EINVAL;
  DIVUQ_CUDA(cudaSetDevice(device));
  StreamGuard sg;
  DIVUQ_CUDA(cached_stream(0, &sg.s));
  const int64_t n = nx * ny;
  const size_t b = size_t(n) * sizeof(double);
  DevBuf d;
  DIVUQ_CUDA(d.alloc_on(8 * b + 256, sg.s));
  double* base = d.as<double>();
  double *dmu = base, *dmv = base + n, *dsu = base + 2 * n, *dsv = base + 3 * n;
  double* outs[4] = {base + 4 * n, base + 5 * n, base + 6 * n, base + 7 * n};
  int32_t* derr = reinterpret_cast<int32_t*>(base + 8 * n);
  DIVUQ_CUDA(cudaMemsetAsync(derr, 0, sizeof(int32_t), sg.s));
  const Span ins[4] = {{dmu, mu_u, b}, {dmv, mu_v, b}, {dsu, has_sigma ? s_u : nullptr, b},
                       {dsv, has_sigma ? s_v : nullptr, b}};
  DIVUQ_CUDA(h2d_in(ins, 4, sg.s));
  double* host_out[4] = {out_mu, out_sigma, out_p_src, out_p_snk};
  int r = propagate2d<double>(dmu, dmv, has_sigma ? dsu : nullptr, has_sigma ? dsv : nullptr, nx, ny,
                              dx, dy, t, out_mu ? outs[0] : nullptr, out_sigma ? outs[1] : nullptr,
                              out_p_src ? outs[2] : nullptr, out_p_snk ? outs[3] : nullptr, derr,
                              sg.s);
  if (r) return r;
  Span res[4];
  for (int q = 0; q < 4; ++q) res[q] = Span{outs[q], host_out[q], host_out[q] ? b : 0};
  int status = 0;
  DIVUQ_CUDA(d2h_out(res, 4, derr, sg.s, &status));
  return status;
}

int divuq_host_tail_probs_f64(const double* mu, const double* sigma, int64_t n, double theta,
                              double* out_below, double* out_above, int device) {
  if (!mu || !sigma || n < 0) return DIVUQ_EINVAL;
  if (n == 0) return DIVUQ_OK;
  DIVUQ_CUDA(cudaSetDevice(device));
  StreamGuard sg;
  DIVUQ_CUDA(cached_stream(0, &sg.s));
  const size_t b = size_t(n) * sizeof(double);
  DevBuf d;
  DIVUQ_CUDA(d.alloc_on(4 * b + 256, sg.s));
  double* base = d.as<double>();
  int32_t* derr = reinterpret_cast<int32_t*>(base + 4 * n);
  DIVUQ_CUDA(cudaMemsetAsync(derr, 0, sizeof(int32_t), sg.s));
  const Span ins[2] = {{base, mu, b}, {base + n, sigma, b}};
  DIVUQ_CUDA(h2d_in(ins, 2, sg.s));
  if (int r = tail_probs<double>(base, base + n, n, theta, out_below ? base + 2 * n : nullptr,
                                 out_above ? base + 3 * n : nullptr, derr, sg.s))
    return r;
  const Span res[2] = {{base + 2 * n, out_below, out_below ? b : 0}, {base + 3 * n, out_above, out_above ? b : 0}};
  int status = 0;
  DIVUQ_CUDA(d2h_out(res, 2, derr, sg.s, &status));
  return status;
}

int divuq_host_propagate_lcp2d_f64(const double* mu_u, const double* mu_v, const double* s_u,
                                   const double* s_v, int64_t nx, int64_t ny, double dx, double dy,
                                   double isovalue, double* out_mu, double* out_sigma,
                                   double* out_lcp, int device) {
  if (int r = grid_ok(nx, ny, dx, dy)) return r;
  if (!mu_u || !mu_v || !s_u || !s_v || !out_lcp) return DIVUQ_EINVAL;
  DIVUQ_CUDA(cudaSetDevice(device));
  StreamGuard sg;
  DIVUQ_CUDA(cached_stream(0, &sg.s));
  const int64_t n = nx * ny, nc = (nx - 1) * (ny - 1);
  DevBuf d;
  DIVUQ_CUDA(d.alloc_on(size_t(6 * n + nc) * sizeof(double) + 256, sg.s));
  double* din = d.as<double>();
  double* dmu = din + 4 * n;
  double* dsg = dmu + n;
  double* dout = dsg + n;
  int32_t* derr = reinterpret_cast<int32_t*>(dout + nc);
  DIVUQ_CUDA(cudaMemsetAsync(derr, 0, sizeof(int32_t), sg.s));
  const double* ins[4] = {mu_u, mu_v, s_u, s_v};
  Span spans[4];
  for (int k = 0; k < 4; ++k) spans[k] = Span{din + k * n, ins[k], size_t(n) * sizeof(double)};
  DIVUQ_CUDA(h2d_in(spans, 4, sg.s));
  if (int r = divuq_propagate_lcp2d_f64(din, din + n, din + 2 * n, din + 3 * n, nx, ny, dx, dy, isovalue,
                                        out_mu ? dmu : nullptr, out_sigma ? dsg : nullptr, dout, derr,
                                        sg.s))
    return r;
  const Span res[3] = {{dmu, out_mu, out_mu ? size_t(n) * sizeof(double) : 0},
                       {dsg, out_sigma, out_sigma ? size_t(n) * sizeof(double) : 0},
                       {dout, out_lcp, size_t(nc) * sizeof(double)}};
  int status = 0;
  DIVUQ_CUDA(d2h_out(res, 3, derr, sg.s, &status));
  return status;
}

int divuq_host_lcp2d_f64(const double* mu, const double* sigma, int64_t nx, int64_t ny,
                         double isovalue, double* out, int device) {
  if (nx < 2 || ny < 2) return DIVUQ_EGRID;
  if (!mu || !sigma || !out) return DIVUQ_EINVAL;
  DIVUQ_CUDA(cudaSetDevice(device));
  StreamGuard sg;
  DIVUQ_CUDA(cached_stream(0, &sg.s));
  const int64_t n = nx * ny, nc = (nx - 1) * (ny - 1);
  DevBuf d;
  DIVUQ_CUDA(d.alloc_on(size_t(2 * n + nc) * sizeof(double) + 256, sg.s));
  double* dmu = d.as<double>();
  double* dsg = dmu + n;
  double* dout = dsg + n;
  int32_t* derr = reinterpret_cast<int32_t*>(dout + nc);
  DIVUQ_CUDA(cudaMemsetAsync(derr, 0, sizeof(int32_t), sg.s));
  const Span ins[2] = {{dmu, mu, size_t(n) * sizeof(double)}, {dsg, sigma, size_t(n) * sizeof(double)}};
  DIVUQ_CUDA(h2d_in(ins, 2, sg.s));
  if (int r = divuq_lcp2d_f64(dmu, dsg, nx, ny, isovalue, dout, derr, sg.s)) return r;
  const Span res1[1] = {{dout, out, size_t(nc) * sizeof(double)}};
  int status = 0;
  DIVUQ_CUDA(d2h_out(res1, 1, derr, sg.s, &status));
  return status;
}

int divuq_host_cell_crossing_f64(const double* mu4, const double* sigma4, int64_t n_cells,
                                 double isovalue, double* out, int device) {
  if (n_cells < 0 || (n_cells && (!mu4 || !sigma4 || !out))) return DIVUQ_EINVAL;
  if (n_cells == 0) return DIVUQ_OK;
  DIVUQ_CUDA(cudaSetDevice(device));
  StreamGuard sg;
  DIVUQ_CUDA(cached_stream(0, &sg.s));
  DevBuf d;
  DIVUQ_CUDA(d.alloc_on(size_t(9 * n_cells) * sizeof(double) + 256, sg.s));
  double* dmu = d.as<double>();
  double* dsg = dmu + 4 * n_cells;
  double* dout = dsg + 4 * n_cells;
  int32_t* derr = reinterpret_cast<int32_t*>(dout + n_cells);
  DIVUQ_CUDA(cudaMemsetAsync(derr, 0, sizeof(int32_t), sg.s));
  const Span ins[2] = {{dmu, mu4, size_t(4 * n_cells) * sizeof(double)},
                       {dsg, sigma4, size_t(4 * n_cells) * sizeof(double)}};
  DIVUQ_CUDA(h2d_in(ins, 2, sg.s));
  if (int r = divuq_cell_crossing_f64(dmu, dsg, n_cells, isovalue, dout, derr, sg.s)) return r;
  const Span res1[1] = {{dout, out, size_t(n_cells) * sizeof(double)}};
  int status = 0;
  DIVUQ_CUDA(d2h_out(res1, 1, derr, sg.s, &status));
  return status;
}

int divuq_host_fit_gaussian_f64(const double* members, int64_t M, int64_t C, int64_t N, double* out_mu,
                                double* out_sigma, int device) {
  if (!members || !out_mu || !out_sigma || C < 1 || N < 1) return DIVUQ_EINVAL;
  if (M < 2) return DIVUQ_EMEMBERS;
  DIVUQ_CUDA(cudaSetDevice(device));
  StreamGuard sg;
  DIVUQ_CUDA(cached_stream(0, &sg.s));
  const size_t in_b = size_t(M * C * N) * sizeof(double), out_b = size_t(C * N) * sizeof(double);
  DevBuf d;
  DIVUQ_CUDA(d.alloc_on(in_b + 2 * out_b + 256, sg.s));
  double* dm = d.as<double>();
  double* dmu = dm + M * C * N;
  double* dsg = dmu + C * N;
  int32_t* derr = reinterpret_cast<int32_t*>(dsg + C * N);
  DIVUQ_CUDA(cudaMemsetAsync(derr, 0, sizeof(int32_t), sg.s));
  const Span ins[1] = {{dm, members, in_b}};
  DIVUQ_CUDA(h2d_in(ins, 1, sg.s));
  if (int r = fit_gaussian<double>(dm, M, C, N, dmu, dsg, derr, sg.s)) return r;
  const Span res[2] = {{dmu, out_mu, out_b}, {dsg, out_sigma, out_b}};
  int status = 0;
  DIVUQ_CUDA(d2h_out(res, 2, derr, sg.s, &status));
  return status;
}

int divuq_host_ensemble_divergence2d_f32(const float* members, int64_t M, int64_t nx, int64_t ny,
                                         double dx, double dy, double t, float* out_mu,
                                         float* out_sigma, float* out_p_src, float* out_p_snk,
                                         float* out_mom_mu, float* out_mom_sigma, int device) {
  if (int r = grid_ok(nx, ny, dx, dy)) return r;
  if (!members) return DIVUQ_EINVAL;
  if (M < 2) return DIVUQ_EMEMBERS;
  if ((out_mom_mu == nullptr) != (out_mom_sigma == nullptr)) return DIVUQ_EINVAL;
  DIVUQ_CUDA(cudaSetDevice(device));
  StreamGuard sg;
  DIVUQ_CUDA(cached_stream(0, &sg.s));
  const int64_t n = nx * ny;
  const size_t in_b = size_t(M * 2 * n) * sizeof(float), b = size_t(n) * sizeof(float);
  DevBuf d;
  DIVUQ_CUDA(d.alloc_on(in_b + 8 * b + 256, sg.s));
  float* dm = d.as<float>();
  float* o = dm + M * 2 * n;
  float* outs[4] = {o, o + n, o + 2 * n, o + 3 * n};
  float* mom_mu = o + 4 * n;      // (2, n)
  float* mom_sg = o + 6 * n;      // (2, n)
  int32_t* derr = reinterpret_cast<int32_t*>(o + 8 * n);
  DIVUQ_CUDA(cudaMemsetAsync(derr, 0, sizeof(int32_t), sg.s));
  const Span ins[1] = {{dm, members, in_b}};
  DIVUQ_CUDA(h2d_in(ins, 1, sg.s));
  float* host_out[4] = {out_mu, out_sigma, out_p_src, out_p_snk};
  int r = divuq_ensemble_divergence2d_f32(dm, M, nx, ny, dx, dy, t, out_mu ? outs[0] : nullptr,
                                          out_sigma ? outs[1] : nullptr, out_p_src ? outs[2] : nullptr,
                                          out_p_snk ? outs[3] : nullptr, out_mom_mu ? mom_mu : nullptr,
                                          out_mom_mu ? mom_sg : nullptr, derr, sg.s);
  if (r) return r;
  Span res[6];
  for (int q = 0; q < 4; ++q) res[q] = Span{outs[q], host_out[q], host_out[q] ? b : 0};
  res[4] = Span{mom_mu, out_mom_mu, out_mom_mu ? 2 * b : 0};
  res[5] = Span{mom_sg, out_mom_sigma, out_mom_mu ? 2 * b : 0};
  int status = 0;
  DIVUQ_CUDA(d2h_out(res, 6, derr, sg.s, &status));
  return status;
}

int divuq_host_gradient_ensemble_divergence2d_f32(const float* members, int64_t M, int64_t nx,
                                                  int64_t ny, double dx, double dy, double t,
                                                  float* out_mu, float* out_sigma, float* out_p_src,
                                                  float* out_p_snk, float* out_mom_mu,
                                                  float* out_mom_sigma, int device) {
  if (int r = grid_ok(nx, ny, dx, dy)) return r;
  if (!members) return DIVUQ_EINVAL;
  if (M < 2) return DIVUQ_EMEMBERS;
  if ((out_mom_mu == nullptr) != (out_mom_sigma == nullptr)) return DIVUQ_EINVAL;
  DIVUQ_CUDA(cudaSetDevice(device));
  StreamGuard sg;
  DIVUQ_CUDA(cached_stream(0, &sg.s));
  const int64_t n = nx * ny;
  const size_t in_b = size_t(M * 2 * n) * sizeof(float), b = size_t(n) * sizeof(float);
  DevBuf d;
  DIVUQ_CUDA(d.alloc_on(in_b + 8 * b + 256, sg.s));
  float* dm = d.as<float>();
  float* o = dm + M * 2 * n;
  float* outs[4] = {o, o + n, o + 2 * n, o + 3 * n};
  float* mom_mu = o + 4 * n;
  float* mom_sg = o + 6 * n;
  int32_t* derr = reinterpret_cast<int32_t*>(o + 8 * n);
  DIVUQ_CUDA(cudaMemsetAsync(derr, 0, sizeof(int32_t), sg.s));
  const Span ins[1] = {{dm, members, in_b}};
  DIVUQ_CUDA(h2d_in(ins, 1, sg.s));
  float* host_out[4] = {out_mu, out_sigma, out_p_src, out_p_snk};
  int r = divuq_gradient_ensemble_divergence2d_f32(
      dm, M, nx, ny, dx, dy, t, out_mu ? outs[0] : nullptr, out_sigma ? outs[1] : nullptr,
      out_p_src ? outs[2] : nullptr, out_p_snk ? outs[3] : nullptr, out_mom_mu ? mom_mu : nullptr,
      out_mom_mu ? mom_sg : nullptr, derr, sg.s);
  if (r) return r;
  Span res[6];
  for (int q = 0; q < 4; ++q) res[q] = Span{outs[q], host_out[q], host_out[q] ? b : 0};
  res[4] = Span{mom_mu, out_mom_mu, out_mom_mu ? 2 * b : 0};
  res[5] = Span{mom_sg, out_mom_sigma, out_mom_mu ? 2 * b : 0};
  int status = 0;
  DIVUQ_CUDA(d2h_out(res, 6, derr, sg.s, &status));
  return status;
}

int divuq_host_mc_divergence2d_f64(const double* mu_u, const double* mu_v, const double* s_u,
                                   const double* s_v, int64_t nx, int64_t ny, double dx, double dy,
                                   int64_t n_samples, uint64_t seed, double* out_mean,
                                   double* out_std, int device) {
  if (int r = grid_ok(nx, ny, dx, dy)) return r;
  if (n_samples < 2) return DIVUQ_ESAMPLES;
  if (!mu_u || !mu_v || !s_u || !s_v || !out_mean || !out_std) return DIVUQ_EINVAL;
  DIVUQ_CUDA(cudaSetDevice(device));
  StreamGuard sg;
  DIVUQ_CUDA(cached_stream(0, &sg.s));
  const int64_t n = nx * ny;
  const size_t b = size_t(n) * sizeof(double);
  const int64_t scratch = divuq_mc_scratch_bytes(nx, 0, ny, n_samples);
  DevBuf d;
  DIVUQ_CUDA(d.alloc_on(6 * b + size_t(scratch) + 256, sg.s));
  double* base = d.as<double>();
  double *dmu = base, *dmv = base + n, *dsu = base + 2 * n, *dsv = base + 3 * n;
  double *dmean = base + 4 * n, *dstd = base + 5 * n;
  int32_t* derr = reinterpret_cast<int32_t*>(base + 6 * n);
  void* dscr = reinterpret_cast<char*>(base + 6 * n) + 256;
  DIVUQ_CUDA(cudaMemsetAsync(derr, 0, sizeof(int32_t), sg.s));
  const Span ins[4] = {{dmu, mu_u, b}, {dmv, mu_v, b}, {dsu, s_u, b}, {dsv, s_v, b}};
  DIVUQ_CUDA(h2d_in(ins, 4, sg.s));
  int r = divuq_mc_divergence2d_f64(dmu, dmv, dsu, dsv, nx, ny, dx, dy, n_samples, seed, 0, ny, dmean,
                                    dstd, dscr, derr, sg.s);
  if (r) return r;
  const Span res[2] = {{dmean, out_mean, b}, {dstd, out_std, b}};
  int status = 0;
  DIVUQ_CUDA(d2h_out(res, 2, derr, sg.s, &status));
  return status;
}

// 3D host pipeline: z-chunks of `chunk_planes` planes; chunk c uses buffer
// set c % 2 and stream c % 2, so chunk c+1's host->device copies overlap
// chunk c's kernel and device->host copies (two copy engines + SMs busy).
int divuq_host_mc_divergence2d_ref_f64(const double* mu_u, const double* mu_v, const double* s_u,
                                       const double* s_v, int64_t nx, int64_t ny, double dx,
                                       double dy, int64_t n_samples, uint64_t seed,
                                       double* out_mean, double* out_std, int device) {
  if (int r = grid_ok(nx, ny, dx, dy)) return r;
  if (n_samples < 2) return DIVUQ_ESAMPLES;
  if (!mu_u || !mu_v || !s_u || !s_v || !out_mean || !out_std) return DIVUQ_EINVAL;
  DIVUQ_CUDA(cudaSetDevice(device));
  StreamGuard sg;
  DIVUQ_CUDA(cached_stream(0, &sg.s));
  const int64_t n = nx * ny;
  const size_t b = size_t(n) * sizeof(double);
  DevBuf d;
  DIVUQ_CUDA(d.alloc_on(6 * b + 256, sg.s));
  double* base = d.as<double>();
  int32_t* derr = reinterpret_cast<int32_t*>(base + 6 * n);
  DIVUQ_CUDA(cudaMemsetAsync(derr, 0, sizeof(int32_t), sg.s));
  const double* src[4] = {mu_u, mu_v, s_u, s_v};
  Span ins[4];
  for (int q = 0; q < 4; ++q) ins[q] = Span{base + q * n, src[q], b};
  DIVUQ_CUDA(h2d_in(ins, 4, sg.s));
  int r = divuq_mc_divergence2d_ref_f64(base, base + n, base + 2 * n, base + 3 * n, nx, ny, dx, dy,
                                        n_samples, seed, 0, ny, base + 4 * n, base + 5 * n, derr, sg.s);
  if (r) return r;
  const Span res[2] = {{base + 4 * n, out_mean, b}, {base + 5 * n, out_std, b}};
  int status = 0;
  DIVUQ_CUDA(d2h_out(res, 2, derr, sg.s, &status));
  return status;
}

// mc_histogram_1d (mc.py:120-139): samples, [min, max], then np.histogram's
// uniform bins; the all-identical case is the reference's one-bin histogram
// [lo - 0.5, hi + 0.5].  out_edges: n_bins + 1 doubles, out_counts: n_bins
// int64; *out_nbins receives the bin count actually used (1 when degenerate).
// out_values (nullable) receives the raw samples (sample_divergence_1d).
// error_metrics (mc.py:159-175), one launch; out3 = (e_m, e_sigma, sse) on the device
int divuq_error_metrics_f64(const double* est_mean, const double* est_std, const double* mu,
                            const double* sigma, int64_t n, double* out3, void* scratch,
                            void* stream) {
  if (!est_mean || !est_std || !mu || !sigma || !out3 || !scratch || n < 1) return DIVUQ_EINVAL;
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(kEmMaxBlocks, (n + 4 * kEmThreads - 1) /
                                                                             (4 * kEmThreads)));
  double* partials = static_cast<double*>(scratch);
  unsigned int* ticket = reinterpret_cast<unsigned int*>(partials + 4 * kEmMaxBlocks);
  error_metrics_kernel<<<unsigned(blocks), kEmThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      est_mean, est_std, mu, sigma, n, partials, ticket, out3);
  return int(cudaGetLastError());
}

int64_t divuq_error_metrics_scratch_bytes(void) {
  return int64_t(4 * kEmMaxBlocks * sizeof(double) + 256);   // partials + ticket (zeroed once)
}

int divuq_host_error_metrics_f64(const double* est_mean, const double* est_std, const double* mu,
                                 const double* sigma, int64_t n, double* out3, int device) {
  if (!est_mean || !est_std || !mu || !sigma || !out3 || n < 1) return DIVUQ_EINVAL;
  DIVUQ_CUDA(cudaSetDevice(device));
  StreamGuard sg;
  DIVUQ_CUDA(cached_stream(0, &sg.s));
  const size_t sb = size_t(divuq_error_metrics_scratch_bytes());
  DevBuf d;
  DIVUQ_CUDA(d.alloc_on(size_t(4 * n + 3) * sizeof(double) + sb, sg.s));
  double* din = d.as<double>();
  double* dout = din + 4 * n;
  void* scratch = dout + 3;
  DIVUQ_CUDA(cudaMemsetAsync(scratch, 0, sb, sg.s));
  const double* ins[4] = {est_mean, est_std, mu, sigma};
  Span sp[4];
  for (int k = 0; k < 4; ++k) sp[k] = Span{din + k * n, ins[k], size_t(n) * sizeof(double)};
  DIVUQ_CUDA(h2d_in(sp, 4, sg.s));
  if (int r = divuq_error_metrics_f64(din, din + n, din + 2 * n, din + 3 * n, n, dout, scratch, sg.s))
    return r;
  const Span res[1] = {{dout, out3, 3 * sizeof(double)}};
  int status = 0;
  DIVUQ_CUDA(d2h_out(res, 1, nullptr, sg.s, &status));
  return DIVUQ_OK;
}

int divuq_host_mc_histogram1d_f64(const double* neighbors, double dx, double dy,
                                  int64_t n_samples, uint64_t seed, int64_t n_bins,
                                  double* out_edges, int64_t* out_counts, int64_t* out_nbins,
                                  double* out_values, int device) {
  if (n_bins < 1) return DIVUQ_EINVAL;   // mc.py:131-132
  if (!neighbors || n_samples < 1 || !out_edges || !out_counts || !out_nbins) return DIVUQ_EINVAL;
  DIVUQ_CUDA(cudaSetDevice(device));
  StreamGuard sg;
  DIVUQ_CUDA(cached_stream(0, &sg.s));
  const size_t vb = size_t(n_samples) * sizeof(double);
  DevBuf d;
  DIVUQ_CUDA(d.alloc(vb + size_t(n_bins + 1) * 16 + 64, sg.s));
  double* vals = d.as<double>();
  double* edges = vals + n_samples;
  int64_t* counts = reinterpret_cast<int64_t*>(edges + n_bins + 1);
  double* mm = reinterpret_cast<double*>(counts + n_bins);
  void* scratch = mm + 2;
  if (int r = divuq_sample_divergence1d_f64(neighbors, dx, dy, n_samples, seed, vals, sg.s)) return r;
  if (int r = divuq_minmax_f64(vals, n_samples, mm, scratch, sg.s)) return r;
  double lohi[2];
  DIVUQ_CUDA(d2h(lohi, mm, sizeof(lohi), sg.s));
  DIVUQ_CUDA(cudaStreamSynchronize(sg.s));
  if (out_values) DIVUQ_CUDA(d2h(out_values, vals, vb, sg.s));
  if (lohi[0] == lohi[1]) {   // all draws identical: one-bin degenerate histogram (mc.py:135-137)
    out_edges[0] = lohi[0] - 0.5;
    out_edges[1] = lohi[1] + 0.5;
    out_counts[0] = n_samples;
    *out_nbins = 1;
    DIVUQ_CUDA(cudaStreamSynchronize(sg.s));
    return DIVUQ_OK;
  }
  if (int r = divuq_histogram_uniform_f64(vals, n_samples, lohi[0], lohi[1], n_bins, edges, counts, sg.s))
    return r;
  DIVUQ_CUDA(cudaMemcpyAsync(out_edges, edges, size_t(n_bins + 1) * sizeof(double),
                             cudaMemcpyDeviceToHost, sg.s));
  DIVUQ_CUDA(cudaMemcpyAsync(out_counts, counts, size_t(n_bins) * sizeof(int64_t),
                             cudaMemcpyDeviceToHost, sg.s));
  DIVUQ_CUDA(cudaStreamSynchronize(sg.s));
  *out_nbins = n_bins;
  return DIVUQ_OK;
}

// 3D analytic propagation from host buffers (the e2e leg of config 3): a
// z-chunk pipeline over three cached streams -- copy-in, compute, copy-out --
// and four buffer sets.  Chunk c's w halo planes are read in place from the
// neighbour chunks' sets already in HBM (no ghost-plane re-upload), so the
// copy-in stream only waits for a set to be released (compute of chunk c-3)
// and never for a device-to-host copy: both PCIe directions stay busy.
int divuq_host_propagate3d_f32(const float* mu_u, const float* mu_v, const float* mu_w,
                               const float* s_u, const float* s_v, const float* s_w, int64_t nx,
                               int64_t ny, int64_t nz, double dx, double dy, double dz, double t,
                               float* out_mu, float* out_sigma, float* out_p_src, float* out_p_snk,
                               int64_t chunk_planes, int device) {
  if (int r = grid_ok(nx, ny, dx, dy)) return r;
  if (nz < 2 || !(dz > 0.0)) return DIVUQ_EGRID;
  const float* in[6] = {mu_u, mu_v, mu_w, s_u, s_v, s_w};
  for (const float* q : in)
    if (!q) return DIVUQ_EINVAL;
  float* host_out[4] = {out_mu, out_sigma, out_p_src, out_p_snk};
  DIVUQ_CUDA(cudaSetDevice(device));
  const int64_t plane = nx * ny;
  const size_t plane_b = size_t(plane) * sizeof(float);
  const int64_t cz = std::max<int64_t>(1, std::min<int64_t>(chunk_planes > 0 ? chunk_planes : 32, nz));
  const int64_t nch = (nz + cz - 1) / cz;
  constexpr int kSets = 4;
  const int nsets = int(std::min<int64_t>(kSets, nch));
  const int64_t set_elems = 10 * cz * plane;   // 6 fields + 4 outputs, cz planes each
  StreamGuard cin, cmp, cout;
  DIVUQ_CUDA(cached_stream(0, &cin.s));
  DIVUQ_CUDA(cached_stream(1, &cmp.s));
  DIVUQ_CUDA(cached_stream(2, &cout.s));
  DevBuf d;
  DIVUQ_CUDA(d.alloc(size_t(nsets * set_elems) * sizeof(float) + 256, cin.s));
  int32_t* derr = reinterpret_cast<int32_t*>(d.as<float>() + nsets * set_elems);
  DIVUQ_CUDA(cudaMemsetAsync(derr, 0, sizeof(int32_t), cin.s));
  struct Events {
    cudaEvent_t up[kSets] = {}, comp[kSets] = {}, out[kSets] = {};
    ~Events() {
      for (int i = 0; i < kSets; ++i)
        for (cudaEvent_t e : {up[i], comp[i], out[i]})
          if (e) cudaEventDestroy(e);
    }
  } ev;
  for (int i = 0; i < kSets; ++i) {
    DIVUQ_CUDA(cudaEventCreateWithFlags(&ev.up[i], cudaEventDisableTiming));
    DIVUQ_CUDA(cudaEventCreateWithFlags(&ev.comp[i], cudaEventDisableTiming));
    DIVUQ_CUDA(cudaEventCreateWithFlags(&ev.out[i], cudaEventDisableTiming));
  }
  auto nzl = [&](int64_t c) { return std::min(cz, nz - c * cz); };
  auto field = [&](int64_t c, int a) { return d.as<float>() + (c % kSets) * set_elems + a * cz * plane; };
  auto upload = [&](int64_t c) -> int {
    if (c >= kSets) DIVUQ_CUDA(cudaStreamWaitEvent(cin.s, ev.comp[(c - 3) % kSets], 0));
    for (int a = 0; a < 6; ++a)
      DIVUQ_CUDA(cudaMemcpyAsync(field(c, a), in[a] + c * cz * plane, size_t(nzl(c)) * plane_b,
                                 cudaMemcpyHostToDevice, cin.s));
    DIVUQ_CUDA(cudaEventRecord(ev.up[c % kSets], cin.s));
    return 0;
  };
  auto compute = [&](int64_t c) -> int {
    DIVUQ_CUDA(cudaStreamWaitEvent(cmp.s, ev.up[(c + 1 < nch ? c + 1 : c) % kSets], 0));
    if (c >= kSets) DIVUQ_CUDA(cudaStreamWaitEvent(cmp.s, ev.out[c % kSets], 0));
    const float* hl_mu = c > 0 ? field(c - 1, 2) + (nzl(c - 1) - 1) * plane : nullptr;
    const float* hl_s = c > 0 ? field(c - 1, 5) + (nzl(c - 1) - 1) * plane : nullptr;
    const float* hh_mu = c + 1 < nch ? field(c + 1, 2) : nullptr;
    const float* hh_s = c + 1 < nch ? field(c + 1, 5) : nullptr;
    float* o[4];
    for (int q = 0; q < 4; ++q) o[q] = host_out[q] ? field(c, 6 + q) : nullptr;
    if (int r = propagate3d<float>(field(c, 0), field(c, 1), field(c, 2), field(c, 3), field(c, 4),
                                   field(c, 5), hl_mu, hl_s, hh_mu, hh_s, nx, ny, nzl(c), c * cz, nz, 0,
                                   nzl(c), dx, dy, dz, t, o[0], o[1], o[2], o[3], derr, cmp.s))
      return r;
    DIVUQ_CUDA(cudaEventRecord(ev.comp[c % kSets], cmp.s));
    DIVUQ_CUDA(cudaStreamWaitEvent(cout.s, ev.comp[c % kSets], 0));
    for (int q = 0; q < 4; ++q)
      if (host_out[q])
        DIVUQ_CUDA(cudaMemcpyAsync(host_out[q] + c * cz * plane, o[q], size_t(nzl(c)) * plane_b,
                                   cudaMemcpyDeviceToHost, cout.s));
    DIVUQ_CUDA(cudaEventRecord(ev.out[c % kSets], cout.s));
    return 0;
  };
  if (int r = upload(0)) return r;
  for (int64_t c = 1; c < nch; ++c) {
    if (int r = upload(c)) return r;
    if (int r = compute(c - 1)) return r;
  }
  if (int r = compute(nch - 1)) return r;
  DIVUQ_CUDA(cudaStreamSynchronize(cin.s));
  DIVUQ_CUDA(cudaStreamSynchronize(cmp.s));
  DIVUQ_CUDA(cudaStreamSynchronize(cout.s));
  int status = 0;
  DIVUQ_CUDA(check_err_word(derr, cmp.s, &status));
  return status;
}

// 3D fused ensemble from host buffers: the end-to-end form of config 4 (one
// rank's z-slab).  members: (M, 3, nx*ny*nz_local) host fp32; the slab covers
// global planes [z0, z0 + nz_local) of nz_global.  ghost_lo_w / ghost_hi_w:
// the w component of global planes z0-1 / z0+nz_local for member 0, member m
// at + m * ghost_member_stride floats (required when that neighbour exists).
// z-chunk pipeline over three cached streams -- copy-in, compute, copy-out --
// and four buffer sets.  A chunk's reduced w halos are fitted from the
// NEIGHBOUR chunks' edge planes already resident in HBM, so every member byte
// crosses PCIe exactly once; the compute stream only waits for the upload of
// chunk c+1 (its hi ghost), and the fourth set keeps the copy engine busy
// meanwhile.
int divuq_host_ensemble_divergence3d_f32(const float* members, int64_t M, int64_t nx, int64_t ny,
                                         int64_t nz_local, int64_t z0, int64_t nz_global,
                                         const float* ghost_lo_w, const float* ghost_hi_w,
                                         int64_t ghost_member_stride, double dx, double dy,
                                         double dz, double t, float* out_mu, float* out_sigma,
                                         float* out_p_src, float* out_p_snk, int64_t chunk_planes,
                                         int device) {
  if (int r = grid_ok(nx, ny, dx, dy)) return r;
  if (nz_global < 2 || !(dz > 0.0)) return DIVUQ_EGRID;
  if (!members || nz_local < 1 || z0 < 0 || z0 + nz_local > nz_global) return DIVUQ_EINVAL;
  if (M < 2) return DIVUQ_EMEMBERS;
  const int64_t plane = nx * ny;
  const bool has_lo = z0 > 0, has_hi = z0 + nz_local < nz_global;
  if ((has_lo && !ghost_lo_w) || (has_hi && !ghost_hi_w)) return DIVUQ_EINVAL;
  if ((has_lo || has_hi) && ghost_member_stride < plane) return DIVUQ_EINVAL;
  DIVUQ_CUDA(cudaSetDevice(device));
  const size_t plane_b = size_t(plane) * sizeof(float);
  constexpr int kSets = 4;
  constexpr int64_t kChunkTarget = int64_t(1) << 30;   // member bytes per chunk
  int64_t cz = chunk_planes > 0 ? chunk_planes
                                : std::max<int64_t>(1, kChunkTarget / int64_t(3 * M * plane_b));
  cz = std::min(cz, nz_local);
  const int64_t nch = (nz_local + cz - 1) / cz;
  float* host_out[4] = {out_mu, out_sigma, out_p_src, out_p_snk};
  // set: members (M, 3, cz planes) | halo mu_lo s_lo r_lo mu_hi s_hi r_hi | 4 outputs (cz planes)
  const int64_t set_elems = 3 * M * cz * plane + 6 * plane + 4 * cz * plane;
  const int64_t ghost_elems = (has_lo || has_hi) ? 2 * M * plane : 0;
  const int nsets = int(std::min<int64_t>(kSets, nch));
  StreamGuard cin, cmp, cout;
  DIVUQ_CUDA(cached_stream(0, &cin.s));
  DIVUQ_CUDA(cached_stream(1, &cmp.s));
  DIVUQ_CUDA(cached_stream(2, &cout.s));
  DevBuf d;
  DIVUQ_CUDA(d.alloc(size_t(nsets * set_elems + ghost_elems) * sizeof(float) + 256, cin.s));
  float* ghost = d.as<float>() + nsets * set_elems;
  int32_t* derr = reinterpret_cast<int32_t*>(ghost + ghost_elems);
  DIVUQ_CUDA(cudaMemsetAsync(derr, 0, sizeof(int32_t), cin.s));
  struct Events {
    cudaEvent_t up[kSets] = {}, comp[kSets] = {}, out[kSets] = {};
    ~Events() {
      for (int i = 0; i < kSets; ++i)
        for (cudaEvent_t e : {up[i], comp[i], out[i]})
          if (e) cudaEventDestroy(e);
    }
  } ev;
  for (int i = 0; i < kSets; ++i) {
    DIVUQ_CUDA(cudaEventCreateWithFlags(&ev.up[i], cudaEventDisableTiming));
    DIVUQ_CUDA(cudaEventCreateWithFlags(&ev.comp[i], cudaEventDisableTiming));
    DIVUQ_CUDA(cudaEventCreateWithFlags(&ev.out[i], cudaEventDisableTiming));
  }
  for (int side = 0; side < 2; ++side) {   // slab ghosts: the w member planes only
    const float* g = side ? ghost_hi_w : ghost_lo_w;
    if (!(side ? has_hi : has_lo)) continue;
    for (int64_t m = 0; m < M; ++m)
      DIVUQ_CUDA(cudaMemcpyAsync(ghost + (side * M + m) * plane, g + m * ghost_member_stride, plane_b,
                                 cudaMemcpyHostToDevice, cin.s));
  }
  auto zc = [&](int64_t c) { return c * cz; };
  auto nzl = [&](int64_t c) { return std::min(cz, nz_local - c * cz); };
  auto set = [&](int64_t c) { return d.as<float>() + (c % kSets) * set_elems; };
  auto upload = [&](int64_t c) -> int {
    if (c >= kSets) DIVUQ_CUDA(cudaStreamWaitEvent(cin.s, ev.comp[(c - 3) % kSets], 0));
    const size_t row_b = size_t(nzl(c)) * plane_b;
    for (int64_t r = 0; r < 3 * M; ++r)   // rows (member, component)
      DIVUQ_CUDA(cudaMemcpyAsync(set(c) + r * nzl(c) * plane, members + (r * nz_local + zc(c)) * plane,
                                 row_b, cudaMemcpyHostToDevice, cin.s));
    DIVUQ_CUDA(cudaEventRecord(ev.up[c % kSets], cin.s));
    return 0;
  };
  auto compute = [&](int64_t c) -> int {
    DIVUQ_CUDA(cudaStreamWaitEvent(cmp.s, ev.up[(c + 1 < nch ? c + 1 : c) % kSets], 0));
    if (c >= kSets) DIVUQ_CUDA(cudaStreamWaitEvent(cmp.s, ev.out[c % kSets], 0));
    float* s = set(c);
    float* halo = s + 3 * M * cz * plane;
    const float* lo = nullptr; int64_t lo_stride = plane;
    const float* hi = nullptr; int64_t hi_stride = plane;
    if (c > 0) {   // last plane of chunk c-1, component w
      lo = set(c - 1) + (2 * nzl(c - 1) + nzl(c - 1) - 1) * plane;
      lo_stride = 3 * nzl(c - 1) * plane;
    } else if (has_lo) {
      lo = ghost;
    }
    if (c + 1 < nch) {   // first plane of chunk c+1, component w
      hi = set(c + 1) + 2 * nzl(c + 1) * plane;
      hi_stride = 3 * nzl(c + 1) * plane;
    } else if (has_hi) {
      hi = ghost + M * plane;
    }
    float* hlo = halo;              // mu, s, r of the plane below the chunk
    float* hhi = halo + 3 * plane;  // ... and above
    if (lo)
      if (int r = fit_gaussian<float>(lo, M, 1, plane, hlo, hlo + plane, derr, cmp.s, lo_stride, hlo + 2 * plane))
        return r;
    if (hi)
      if (int r = fit_gaussian<float>(hi, M, 1, plane, hhi, hhi + plane, derr, cmp.s, hi_stride, hhi + 2 * plane))
        return r;
    float* outs = halo + 6 * plane;
    float* o[4];
    for (int q = 0; q < 4; ++q) o[q] = host_out[q] ? outs + q * cz * plane : nullptr;
    if (int r = divuq_ensemble_divergence3d_f32(
            s, M, lo ? hlo : nullptr, lo ? hlo + plane : nullptr, lo ? hlo + 2 * plane : nullptr,
            hi ? hhi : nullptr, hi ? hhi + plane : nullptr, hi ? hhi + 2 * plane : nullptr, nx, ny, nzl(c), z0 + zc(c), nz_global, 0, nzl(c), dx, dy, dz,
            t, o[0], o[1], o[2], o[3], nullptr, nullptr, derr, cmp.s))
      return r;
    DIVUQ_CUDA(cudaEventRecord(ev.comp[c % kSets], cmp.s));
    DIVUQ_CUDA(cudaStreamWaitEvent(cout.s, ev.comp[c % kSets], 0));
    for (int q = 0; q < 4; ++q)
      if (host_out[q])
        DIVUQ_CUDA(cudaMemcpyAsync(host_out[q] + zc(c) * plane, o[q], size_t(nzl(c)) * plane_b,
                                   cudaMemcpyDeviceToHost, cout.s));
    DIVUQ_CUDA(cudaEventRecord(ev.out[c % kSets], cout.s));
    return 0;
  };
  if (int r = upload(0)) return r;
  for (int64_t c = 1; c < nch; ++c) {
    if (int r = upload(c)) return r;
    if (int r = compute(c - 1)) return r;
  }
  if (int r = compute(nch - 1)) return r;
  DIVUQ_CUDA(cudaStreamSynchronize(cin.s));
  DIVUQ_CUDA(cudaStreamSynchronize(cmp.s));
  DIVUQ_CUDA(cudaStreamSynchronize(cout.s));
  int status = 0;
  DIVUQ_CUDA(check_err_word(derr, cmp.s, &status));
  return status;
}

// ---------------------------------------------------------------------
// DIVUQ1 container (io.py:43-134)
// ---------------------------------------------------------------------

int divuq_divuq1_read_header(const char* path, int64_t* nx, int64_t* ny, double* dx, double* dy,
                             int64_t* n_members) {
  if (!path || !nx || !ny || !dx || !dy || !n_members) return DIVUQ_EINVAL;
  io::Header h;
  if (int r = io::read_header(path, &h)) return r;
  *nx = h.nx; *ny = h.ny; *dx = h.dx; *dy = h.dy; *n_members = h.members;
  return DIVUQ_OK;
}

// payload -> host buffer (pinned or pageable); check_finite mirrors the
// reference's DataError (io.py:89-90)
int divuq_divuq1_read_f32(const char* path, float* out, int64_t count, int check_finite) {
  if (!path || !out || count < 0) return DIVUQ_EINVAL;
  io::Header h;
  if (int r = io::read_header(path, &h)) return r;
  if (count != h.members * 2 * h.nx * h.ny) return DIVUQ_EINVAL;
  const int fd = ::open(path, O_RDONLY);
  if (fd < 0) return io::kOsError;
  const bool ok = io::pread_parallel(fd, reinterpret_cast<char*>(out), count * int64_t(sizeof(float)),
                                     h.offset);
  ::close(fd);
  if (!ok) return io::kOsError;
  if (check_finite)
    for (int64_t i = 0; i < count; ++i)
      if (!std::isfinite(out[i])) return io::kDataError;
  return DIVUQ_OK;
}

// payload -> HBM (M, 2, N) fp32.  The file is read with parallel pread()s
// into a persistent ring of pinned staging buffers (allocated once per
// process: pinning 100+ MB costs more than the copy), and each filled buffer
// is sent to the device with an async H2D copy, so the reads of chunk i+1
// overlap the PCIe transfer of chunk i.  Bound: min(page-cache/disk read
// bandwidth, host->device link).
int divuq_divuq1_ingest_f32(const char* path, float* dev_out, int64_t count, int device) {
  if (!path || !dev_out || count < 0) return DIVUQ_EINVAL;
  io::Header h;
  if (int r = io::read_header(path, &h)) return r;
  if (count != h.members * 2 * h.nx * h.ny) return DIVUQ_EINVAL;
  if (count == 0) return DIVUQ_OK;
  DIVUQ_CUDA(cudaSetDevice(device));
  io::Staging& st = io::staging();
  std::lock_guard<std::mutex> lock(st.mu);
  if (int r = st.ensure()) return r;
  const int fd = ::open(path, O_RDONLY | O_CLOEXEC);
  if (fd < 0) return io::kOsError;
  ::posix_fadvise(fd, 0, 0, POSIX_FADV_SEQUENTIAL);
  StreamGuard sg;
  cudaEvent_t done[io::Staging::kBuffers] = {};
  int status = DIVUQ_OK;
  do {
    if ((status = int(cached_stream(0, &sg.s)))) break;
    for (auto& e : done)
      if ((status = int(cudaEventCreateWithFlags(&e, cudaEventDisableTiming)))) break;
    if (status) break;
    const int64_t total = count * int64_t(sizeof(float));
    int b = 0;
    for (int64_t off = 0; off < total; off += io::Staging::kChunk, b = (b + 1) % io::Staging::kBuffers) {
      const int64_t len = std::min<int64_t>(io::Staging::kChunk, total - off);
      if ((status = int(cudaEventSynchronize(done[b])))) break;  // buffer b's last copy finished
      if (!io::pread_parallel(fd, st.buf[b], len, h.offset + off)) { status = io::kOsError; break; }
      if ((status = int(cudaMemcpyAsync(reinterpret_cast<char*>(dev_out) + off, st.buf[b], size_t(len),
                                        cudaMemcpyHostToDevice, sg.s)))) break;
      if ((status = int(cudaEventRecord(done[b], sg.s)))) break;
    }
    if (!status) status = int(cudaStreamSynchronize(sg.s));
  } while (false);
  ::close(fd);
  if (sg.s) cudaStreamSynchronize(sg.s);
  for (auto& e : done)
    if (e) cudaEventDestroy(e);
  return status;
}

// byte-identical to the reference's write_members (io.py:43-55)
int divuq_divuq1_write_f32(const char* path, int64_t nx, int64_t ny, double dx, double dy,
                           int64_t n_members, const float* data) {
  if (!path || (!data && n_members > 0) || n_members < 0) return DIVUQ_EINVAL;
  const std::string header = "DIVUQ1 " + std::to_string(nx) + " " + std::to_string(ny) + " " +
                             io::py_repr(dx) + " " + io::py_repr(dy) + " " +
                             std::to_string(n_members) + "\n";
  FILE* f = std::fopen(path, "wb");
  if (!f) return io::kOsError;
  const size_t count = size_t(n_members * 2 * nx * ny);
  const bool ok = std::fwrite(header.data(), 1, header.size(), f) == header.size() &&
                  std::fwrite(data, sizeof(float), count, f) == count;
  return (std::fclose(f) == 0 && ok) ? DIVUQ_OK : io::kOsError;
}

// Python repr of a header real (exposed for the format tests)
int divuq_divuq1_format_real(double x, char* out, int64_t cap) {
  if (!out || cap < 2) return DIVUQ_EINVAL;
  const std::string s = io::py_repr(x);
  if (int64_t(s.size()) + 1 > cap) return DIVUQ_EINVAL;
  std::memcpy(out, s.c_str(), s.size() + 1);
  return DIVUQ_OK;
}

}  // extern "C"
