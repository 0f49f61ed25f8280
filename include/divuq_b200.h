/* divuq_b200.h -- C ABI of the B200-native divergence-uncertainty hot path.
 *
 * Drop-in boundary for the reference package `divuq`
 * (/root/reference/pkg/src/divuq).  The reference is pure Python and has no
 * FFI; its only pluggable seam is the per-index kernel run by
 * parallel_map (parallel.py:65-116) under the public functions re-exported by
 * __init__.py:9-96.  Each entry point below replaces one of those functions
 * (file:line cited) and is what a ctypes binding inside the reference would
 * call (INTEGRATION.md shows the stub).
 *
 * Conventions
 *   - plain pointers + sizes only; no torch or CUDA types in signatures
 *     (`stream` is a cudaStream_t passed as void*, NULL = legacy default);
 *   - `divuq_*`      : DEVICE pointers, asynchronous on `stream`, caller owns
 *                      every buffer, inputs are never modified;
 *   - `divuq_host_*` : HOST pointers (pinned or pageable), synchronous; the
 *                      library stages device memory itself and checks the
 *                      validation word before returning;
 *   - arrays are flat row-major, x fastest: 2D index j*nx+i (grid.py:3-8),
 *     3D index (k*ny+j)*nx+i; ensembles are member-major (M, C, N) like the
 *     DIVUQ1 container (io.py:51-53);
 *   - grids need >= 2 vertices per axis and positive spacing (grid.py:42-46);
 *   - `err_word` (device int32, may be NULL) receives DIVUQ_ERRBIT_* bits
 *     when an input is non-finite or a sigma is negative -- the reference's
 *     construction-time checks (grid.py:26-27, divergence.py:34-35,
 *     gaussian.py:28-29) folded into the kernels at zero extra HBM traffic;
 *   - return value: 0 ok, < 0 DIVUQ_E* argument/validation error, > 0 a
 *     cudaError_t.
 *   - optional outputs may be NULL (not computed / not written).
 *
 * Probability maps: the reference has no public name for them; they are its
 * private _tail_probs (lcp.py:48-68): p_src = P(div > t) = "above" at
 * theta = t, p_snk = P(div < -t) = "below" at theta = -t (P(div <= -t) on
 * the sigma == 0 tie, lcp.py:56-59).
 */
#ifndef DIVUQ_B200_H
#define DIVUQ_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DIVUQ_ABI_VERSION 2

#define DIVUQ_OK 0
#define DIVUQ_EINVAL (-1)          /* null pointer / bad size */
#define DIVUQ_EGRID (-2)           /* grid smaller than 2 per axis or spacing <= 0 */
#define DIVUQ_EMEMBERS (-3)        /* fewer than 2 ensemble members */
#define DIVUQ_ESAMPLES (-4)        /* fewer than 2 Monte Carlo samples */
#define DIVUQ_ENONFINITE (-10)     /* an input value is NaN / inf */
#define DIVUQ_ENEGSIGMA (-11)      /* a sigma input is negative */
#define DIVUQ_EFORMAT (-20)        /* DIVUQ1: bad magic / malformed header (io.FormatError) */
#define DIVUQ_ELENGTH (-21)        /* DIVUQ1: payload length mismatch (io.LengthError) */
#define DIVUQ_EOS (-22)            /* DIVUQ1: file cannot be read / written (OSError) */
#define DIVUQ_EDATA (-23)          /* DIVUQ1: non-finite payload (io.DataError) */

#define DIVUQ_ERRBIT_NONFINITE 1
#define DIVUQ_ERRBIT_NEGSIGMA 2

int divuq_abi_version(void);
const char* divuq_status_string(int status);

/* ---- K2: analytic propagation + probability map ----------------------
 * Replaces propagate_divergence (divergence.py:48-70; per-index body
 * stencils.py:54-84) and _tail_probs (lcp.py:48-68).  fp64 results are
 * bit-identical to the reference.  s_u/s_v may be NULL only when
 * out_sigma/out_p_src/out_p_snk are all NULL: that is
 * divergence_deterministic (divergence.py:41-45). */
int divuq_propagate2d_f64(const double* mu_u, const double* mu_v,
                          const double* s_u, const double* s_v,
                          int64_t nx, int64_t ny, double dx, double dy, double t,
                          double* out_mu, double* out_sigma,
                          double* out_p_src, double* out_p_snk,
                          int32_t* err_word, void* stream);
int divuq_propagate2d_f32(const float* mu_u, const float* mu_v,
                          const float* s_u, const float* s_v,
                          int64_t nx, int64_t ny, double dx, double dy, double t,
                          float* out_mu, float* out_sigma,
                          float* out_p_src, float* out_p_snk,
                          int32_t* err_word, void* stream);

/* 3D (no reference code; restates stencils.py:46-51 for z).  Arrays hold the
 * z-slab [z0, z0+nz_local) of a grid with nz_global planes.  halo_* are the
 * (mu_w, s_w) planes at global z0-1 / z0+nz_local, required only when those
 * planes exist (z0 > 0 / z0+nz_local < nz_global).  Only local planes
 * [k_begin, k_end) are computed (lets a caller overlap the halo exchange
 * with the interior). */
int divuq_propagate3d_f32(const float* mu_u, const float* mu_v, const float* mu_w,
                          const float* s_u, const float* s_v, const float* s_w,
                          const float* halo_lo_mu_w, const float* halo_lo_s_w,
                          const float* halo_hi_mu_w, const float* halo_hi_s_w,
                          int64_t nx, int64_t ny, int64_t nz_local,
                          int64_t z0, int64_t nz_global, int64_t k_begin, int64_t k_end,
                          double dx, double dy, double dz, double t,
                          float* out_mu, float* out_sigma,
                          float* out_p_src, float* out_p_snk,
                          int32_t* err_word, void* stream);
int divuq_propagate3d_f64(const double* mu_u, const double* mu_v, const double* mu_w,
                          const double* s_u, const double* s_v, const double* s_w,
                          const double* halo_lo_mu_w, const double* halo_lo_s_w,
                          const double* halo_hi_mu_w, const double* halo_hi_s_w,
                          int64_t nx, int64_t ny, int64_t nz_local,
                          int64_t z0, int64_t nz_global, int64_t k_begin, int64_t k_end,
                          double dx, double dy, double dz, double t,
                          double* out_mu, double* out_sigma,
                          double* out_p_src, double* out_p_snk,
                          int32_t* err_word, void* stream);

/* Probability map of an existing Gaussian scalar field: _tail_probs
 * (lcp.py:48-68) elementwise.  out_below = P(X <= theta), out_above =
 * P(X > theta); either may be NULL. */
int divuq_tail_probs_f64(const double* mu, const double* sigma, int64_t n, double theta,
                         double* out_below, double* out_above, int32_t* err_word, void* stream);
int divuq_tail_probs_f32(const float* mu, const float* sigma, int64_t n, double theta,
                         float* out_below, float* out_above, int32_t* err_word, void* stream);

/* ---- level-crossing probability ----------------------
 * Replaces lcp() / cell_crossing_probability (lcp.py:71-100).  lcp2d: one
 * value per cell, cell index cj*(nx-1)+ci, corners v00, v00+1, v00+nx,
 * v00+nx+1; LCP = clip(1 - (prod below + prod above), 0, 1) with the
 * _tail_probs tails (lcp.py:48-68).  cell_crossing: stacked (n, 4) corner
 * arrays, same formula. */
int divuq_lcp2d_f64(const double* mu, const double* sigma, int64_t nx, int64_t ny, double isovalue,
                    double* out_cells, int32_t* err_word, void* stream);
int divuq_lcp2d_f32(const float* mu, const float* sigma, int64_t nx, int64_t ny, double isovalue,
                    float* out_cells, int32_t* err_word, void* stream);
int divuq_cell_crossing_f64(const double* mu4, const double* sigma4, int64_t n_cells,
                            double isovalue, double* out, int32_t* err_word, void* stream);
/* propagate_divergence (divergence.py:48-70) followed by lcp (lcp.py:80-100)
 * in ONE pass: the crossing probability of `isovalue` per cell of the
 * divergence field of the Gaussian (u, v) model, without the (mu, sigma)
 * round trip through HBM.  out_mu / out_sigma (optional) receive the
 * divergence moments.  Bitwise equal to divuq_propagate2d_f64 followed by
 * divuq_lcp2d_f64 (same arithmetic, same corner order). */
int divuq_propagate_lcp2d_f64(const double* mu_u, const double* mu_v, const double* s_u,
                              const double* s_v, int64_t nx, int64_t ny, double dx, double dy,
                              double isovalue, double* out_mu, double* out_sigma, double* out_lcp,
                              int32_t* err_word, void* stream);

/* ---- velocity-magnitude-gradient prologue ---------------
 * velocity_magnitude (gaussian.py:48-50) = hypot(u, v); gradient
 * (gaussian.py:53-58, stencils.py:87-96) = (f[hi]*cx - f[lo]*cx,
 * f[hi]*cy - f[lo]*cy) with the divergence's one-sided boundary rule, output
 * (2, n); gradient_ensemble (gaussian.py:61-66): every member of (M, 2, n)
 * mapped through both, fused (magnitudes recomputed per neighbour, never
 * stored), output (M, 2, n). */
int divuq_velocity_magnitude_f64(const double* u, const double* v, int64_t n, double* out,
                                 int32_t* err_word, void* stream);
int divuq_gradient2d_f64(const double* values, int64_t nx, int64_t ny, double dx, double dy,
                         double* out_gx_gy, int32_t* err_word, void* stream);
int divuq_gradient_ensemble2d_f64(const double* members, int64_t n_members, int64_t nx, int64_t ny,
                                  double dx, double dy, double* out_members, int32_t* err_word,
                                  void* stream);
int divuq_gradient_ensemble2d_f32(const float* members, int64_t n_members, int64_t nx, int64_t ny,
                                  double dx, double dy, float* out_members, int32_t* err_word,
                                  void* stream);

/* ---- K1: ensemble moments ---------------------------------------------
 * Replaces fit_gaussian (gaussian.py:35-45): mean = sequential sum / M,
 * sigma = sqrt(two-pass sum of squared deviations / (M-1)); fp64 is
 * bit-identical to numpy's mean / std(ddof=1).  members: (M, C, n_points)
 * with member stride C*n_points; outputs (C, n_points). */
int divuq_fit_gaussian_f64(const double* members, int64_t n_members, int64_t n_components,
                           int64_t n_points, double* out_mu, double* out_sigma,
                           int32_t* err_word, void* stream);
int divuq_fit_gaussian_f32(const float* members, int64_t n_members, int64_t n_components,
                           int64_t n_points, float* out_mu, float* out_sigma,
                           int32_t* err_word, void* stream);

/* ---- K3: fused ensemble -> moments -> divergence -> probabilities --------
 * fit_gaussian followed by propagate_divergence and _tail_probs in one pass
 * over the members.  members: (M, 2, nx*ny) [2D] or (M, 3, nx*ny*nz_local)
 * [3D slab].  out_mom_mu/out_mom_sigma (optional, (C, N)) receive the
 * fitted moments.  3D halos are REDUCED w moments (mu_w, s_w, r_w) of the
 * neighbouring planes (compute them with divuq_fit_gaussian_strided_f32 on
 * the owner's edge plane; r_w -- the means' rounding residuals, see
 * ShiftedMoments in csrc/common.cuh -- may be NULL and then reads as 0, at
 * the cost of bitwise agreement with the unsharded run). */
int divuq_ensemble_divergence2d_f32(const float* members, int64_t n_members,
                                    int64_t nx, int64_t ny, double dx, double dy, double t,
                                    float* out_mu, float* out_sigma,
                                    float* out_p_src, float* out_p_snk,
                                    float* out_mom_mu, float* out_mom_sigma,
                                    int32_t* err_word, void* stream);
int divuq_ensemble_divergence3d_f32(const float* members, int64_t n_members,
                                    const float* halo_lo_mu_w, const float* halo_lo_s_w,
                                    const float* halo_lo_r_w,
                                    const float* halo_hi_mu_w, const float* halo_hi_s_w,
                                    const float* halo_hi_r_w,
                                    int64_t nx, int64_t ny, int64_t nz_local,
                                    int64_t z0, int64_t nz_global, int64_t k_begin, int64_t k_end,
                                    double dx, double dy, double dz, double t,
                                    float* out_mu, float* out_sigma,
                                    float* out_p_src, float* out_p_snk,
                                    float* out_mom_mu, float* out_mom_sigma,
                                    int32_t* err_word, void* stream);

/* ---- K6: fused Red Sea pipeline -----------------------------------------
 * velocity_magnitude -> gradient_ensemble (gaussian.py:48-66) -> fit_gaussian
 * (gaussian.py:35-45) -> propagate_divergence (divergence.py:48-70) -> tails
 * (lcp.py:48-68) in one pass over (M, 2, nx*ny) fp32 velocity members.
 * Equal bit for bit to divuq_gradient_ensemble2d_f32 followed by
 * divuq_ensemble_divergence2d_f32.  out_mom_* (optional, (2, N)) receive the
 * moments of the gradient ensemble. */
int divuq_gradient_ensemble_divergence2d_f32(const float* members, int64_t n_members,
                                             int64_t nx, int64_t ny, double dx, double dy,
                                             double t, float* out_mu, float* out_sigma,
                                             float* out_p_src, float* out_p_snk,
                                             float* out_mom_mu, float* out_mom_sigma,
                                             int32_t* err_word, void* stream);

/* ---- K4: Monte Carlo estimator ------------------------------------------
 * Replaces mc_divergence (mc.py:94-117) with a Philox4x32-10 + Box-Muller
 * stream (contract: oracle/philox.py).  Inputs: the full grid model (fp64).
 * Rows [row_begin, row_end) are estimated (vertex sharding needs no
 * communication: draws are keyed by global vertex).  Outputs hold
 * (row_end-row_begin)*nx values.  scratch: divuq_mc_scratch_bytes() bytes of
 * device memory. */
int64_t divuq_mc_scratch_bytes(int64_t nx, int64_t row_begin, int64_t row_end, int64_t n_samples);
int divuq_mc_divergence2d_f64(const double* mu_u, const double* mu_v,
                              const double* s_u, const double* s_v,
                              int64_t nx, int64_t ny, double dx, double dy,
                              int64_t n_samples, uint64_t seed,
                              int64_t row_begin, int64_t row_end,
                              double* out_mean, double* out_std, void* scratch,
                              int32_t* err_word, void* stream);

/* ---- K5: synthetic inputs (bench only; BASELINE.json configs) -----------
 * bumps: n_bumps x 5 floats (cx, cy, cz, amp, 1/width^2) in world units on
 * the device.  Writes the model (n_members == 0: mu_u, mu_v[, mu_w], s_u,
 * s_v[, s_w] into out[0..2C-1]) or the members (M, C, nx*ny*nz_local). */
int divuq_gen_field_f32(const float* bumps, int n_bumps, int dims,
                        int64_t nx, int64_t ny, int64_t nz_local, int64_t z0,
                        double dx, double dy, double dz,
                        double vortex_amp, double vortex_cx, double vortex_cy, double vortex_r,
                        double shear_amp, uint64_t seed, double sig_lo, double sig_hi,
                        int sigma_mode, int64_t n_members, float* const* out, float* members,
                        void* stream);

/* ---- DIVUQ1 container (io.py:43-134) ---------------------
 * Header "DIVUQ1 nx ny dx dy M\n" then M blocks of (u-plane, v-plane) LE fp32:
 * exactly the (M, 2, N) layout the ensemble kernels read.  ingest_f32 streams
 * the payload disk -> pinned staging (double-buffered) -> device memory;
 * write_f32 is byte-identical to the reference writer (Python-repr header
 * reals, io.py:38-55). */
int divuq_divuq1_read_header(const char* path, int64_t* nx, int64_t* ny, double* dx, double* dy,
                             int64_t* n_members);
int divuq_divuq1_read_f32(const char* path, float* out, int64_t count, int check_finite);
int divuq_divuq1_ingest_f32(const char* path, float* dev_out, int64_t count, int device);
int divuq_divuq1_write_f32(const char* path, int64_t nx, int64_t ny, double dx, double dy,
                           int64_t n_members, const float* data);
int divuq_divuq1_format_real(double x, char* out, int64_t cap);

/* ---- host-buffer entry points (the reference-facing path) ----------------
 * Same semantics as the device versions; synchronous; `device` = CUDA
 * ordinal.  Host buffers may be pinned (direct DMA) or pageable, mixed in
 * one call.  Pageable spans of a call up to DIVUQ_BOUNCE_MAX_KB (32 MB) are
 * packed into a per-thread pinned arena (adjacent device spans as one DMA;
 * each calling thread keeps its arena, sized to its largest such call, for
 * the life of the process -- set DIVUQ_BOUNCE_MAX_KB=0 to never allocate it);
 * outputs and the validation word come back with one stream sync; calls up
 * to DIVUQ_ZC_MAX_KB (4 MB) per direction move all their spans with one copy
 * kernel over mapped pinned memory instead of one DMA each; larger
 * pageable totals go through a staged ring of pinned buffers.  The 3D
 * variant pipelines z-chunks: host->device copies, the kernel and
 * device->host copies of consecutive chunks overlap on separate streams. */
int divuq_host_propagate2d_f64(const double* mu_u, const double* mu_v,
                               const double* s_u, const double* s_v,
                               int64_t nx, int64_t ny, double dx, double dy, double t,
                               double* out_mu, double* out_sigma,
                               double* out_p_src, double* out_p_snk, int device);
int divuq_host_propagate3d_f32(const float* mu_u, const float* mu_v, const float* mu_w,
                               const float* s_u, const float* s_v, const float* s_w,
                               int64_t nx, int64_t ny, int64_t nz,
                               double dx, double dy, double dz, double t,
                               float* out_mu, float* out_sigma,
                               float* out_p_src, float* out_p_snk,
                               int64_t chunk_planes, int device);
/* 3D fused ensemble (config 4) from host buffers, for one rank's z-slab:
 * members (M, 3, nx*ny*nz_local) covering global planes [z0, z0+nz_local) of
 * nz_global; ghost_lo_w / ghost_hi_w point at the w component of global plane
 * z0-1 / z0+nz_local for member 0 (member m at + m*ghost_member_stride
 * floats), required when that plane exists.  Three-stream z-chunk pipeline;
 * each member byte crosses PCIe once.  Host form of K3 3D: fit_gaussian
 * (gaussian.py:35-45) then the z-extended stencil (stencils.py:46-51, no
 * reference 3D code) and the tail probabilities, per slab. */
int divuq_host_ensemble_divergence3d_f32(const float* members, int64_t n_members,
                                         int64_t nx, int64_t ny, int64_t nz_local,
                                         int64_t z0, int64_t nz_global,
                                         const float* ghost_lo_w, const float* ghost_hi_w,
                                         int64_t ghost_member_stride,
                                         double dx, double dy, double dz, double t,
                                         float* out_mu, float* out_sigma,
                                         float* out_p_src, float* out_p_snk,
                                         int64_t chunk_planes, int device);
int divuq_host_gradient_ensemble_divergence2d_f32(const float* members, int64_t n_members,
                                                  int64_t nx, int64_t ny, double dx, double dy,
                                                  double t, float* out_mu, float* out_sigma,
                                                  float* out_p_src, float* out_p_snk,
                                                  float* out_mom_mu, float* out_mom_sigma,
                                                  int device);
int divuq_host_tail_probs_f64(const double* mu, const double* sigma, int64_t n, double theta,
                              double* out_below, double* out_above, int device);
int divuq_host_propagate_lcp2d_f64(const double* mu_u, const double* mu_v, const double* s_u,
                                   const double* s_v, int64_t nx, int64_t ny, double dx, double dy,
                                   double isovalue, double* out_mu, double* out_sigma,
                                   double* out_lcp, int device);
int divuq_host_lcp2d_f64(const double* mu, const double* sigma, int64_t nx, int64_t ny,
                         double isovalue, double* out_cells, int device);
int divuq_host_cell_crossing_f64(const double* mu4, const double* sigma4, int64_t n_cells,
                                 double isovalue, double* out, int device);
int divuq_host_velocity_magnitude_f64(const double* u, const double* v, int64_t n, double* out,
                                      int device);
int divuq_host_gradient2d_f64(const double* values, int64_t nx, int64_t ny, double dx, double dy,
                              double* out_gx_gy, int device);

/* ---- K4 parity mode: the reference's own stream ---------------------------
 * splitmix64 + AS241 (rng.py:23-92), counters (2s) n + v / (2s+1) n + v
 * (mc.py:80-91), one Welford pass per vertex in strict sample order with
 * mean += delta / count (mc.py:106-117): replaces mc_divergence draw for draw.
 * No scratch (no chunk split). */
int divuq_mc_divergence2d_ref_f64(const double* mu_u, const double* mu_v,
                                  const double* s_u, const double* s_v,
                                  int64_t nx, int64_t ny, double dx, double dy,
                                  int64_t n_samples, uint64_t seed,
                                  int64_t row_begin, int64_t row_end,
                                  double* out_mean, double* out_std,
                                  int32_t* err_word, void* stream);
/* sample_divergence_1d (mc.py:142-156): neighbors = host array of 8 doubles
 * (mu, sigma) x (u_{i-1}, u_{i+1}, v_{j-1}, v_{j+1}); out = device array. */
int divuq_sample_divergence1d_f64(const double* neighbors, double dx, double dy,
                                  int64_t n_samples, uint64_t seed, double* out, void* stream);
/* min / max of a device array -> out_minmax[2] (device); scratch16: 16 bytes. */
int divuq_minmax_f64(const double* values, int64_t n, double* out_minmax, void* scratch16,
                     void* stream);
/* np.histogram(values, bins=n_bins, range=(lo, hi)) (numpy's uniform-bin rule,
 * linspace edges): edges_dev n_bins+1 doubles, counts_dev n_bins int64.
 * Synchronises the stream (the edges are staged from the host). */
int divuq_histogram_uniform_f64(const double* values, int64_t n, double lo, double hi,
                                int64_t n_bins, double* edges_dev, int64_t* counts_dev,
                                void* stream);

int divuq_host_gradient_ensemble2d_f64(const double* members, int64_t n_members, int64_t nx,
                                       int64_t ny, double dx, double dy, double* out_members,
                                       int device);
int divuq_host_fit_gaussian_f64(const double* members, int64_t n_members, int64_t n_components,
                                int64_t n_points, double* out_mu, double* out_sigma, int device);
int divuq_host_ensemble_divergence2d_f32(const float* members, int64_t n_members,
                                         int64_t nx, int64_t ny, double dx, double dy, double t,
                                         float* out_mu, float* out_sigma,
                                         float* out_p_src, float* out_p_snk,
                                         float* out_mom_mu, float* out_mom_sigma, int device);
int divuq_host_mc_divergence2d_f64(const double* mu_u, const double* mu_v,
                                   const double* s_u, const double* s_v,
                                   int64_t nx, int64_t ny, double dx, double dy,
                                   int64_t n_samples, uint64_t seed,
                                   double* out_mean, double* out_std, int device);

/* K1 on a member-strided view: member m's N values start at members + m*member_stride
 * (e.g. the w plane of a z-slab: stride 3*n_local) -- the reduced halo a slab
 * neighbour needs, read in place (also through peer memory).  out_r
 * (optional): the means' rounding residuals the fused kernels difference. */
int divuq_fit_gaussian_strided_f32(const float* members, int64_t n_members, int64_t member_stride,
                                   int64_t n_points, float* out_mu, float* out_sigma,
                                   float* out_r, int32_t* err_word, void* stream);

/* Page-lock (portable, mapped) / release caller-owned host memory: the
 * drop-in layer pins its pooled output blocks once so host entries write
 * results straight into them (cudaHostRegister / cudaHostUnregister). */
int divuq_host_register(void* ptr, int64_t bytes);
int divuq_host_unregister(void* ptr);

/* Peer memory (CUDA IPC) for the z-slab exchange over NVLink: export the
 * allocation holding `ptr` (handle: divuq_ipc_handle_bytes() bytes, plus the
 * offset of ptr inside it); import maps a neighbour's export (peer access
 * enabled lazily) and returns the mapping base (for close) and the pointer. */
int64_t divuq_ipc_handle_bytes(void);
int divuq_ipc_export(const void* ptr, void* handle_out, int64_t* offset_out);
int divuq_ipc_import(const void* handle, int64_t offset, void** base_out, void** ptr_out);
int divuq_ipc_close(void* base);

/* host twins of the parity mode (mc.py:94-156) */
int divuq_host_mc_divergence2d_ref_f64(const double* mu_u, const double* mu_v,
                                       const double* s_u, const double* s_v,
                                       int64_t nx, int64_t ny, double dx, double dy,
                                       int64_t n_samples, uint64_t seed,
                                       double* out_mean, double* out_std, int device);
/* mc_histogram_1d (mc.py:120-139): out_edges n_bins+1, out_counts n_bins,
 * *out_nbins = bins used (1 for the all-identical degenerate case),
 * out_values (nullable) = the raw samples. */
/* error_metrics (mc.py:159-175): (e_m, e_sigma, sse) = (mean|est.mean - mu|,
 * mean|est.std - sigma|, sum (est.mean - mu)^2 + sum (est.std - sigma)^2)
 * in one launch (grid-stride partials, the last block folds them in block
 * order: deterministic).  Device: out3 is 3 device doubles; scratch is
 * divuq_error_metrics_scratch_bytes() bytes, zeroed once before first use. */
int divuq_error_metrics_f64(const double* est_mean, const double* est_std, const double* mu,
                            const double* sigma, int64_t n, double* out3, void* scratch,
                            void* stream);
int64_t divuq_error_metrics_scratch_bytes(void);
int divuq_host_error_metrics_f64(const double* est_mean, const double* est_std, const double* mu,
                                 const double* sigma, int64_t n, double* out3, int device);
int divuq_host_mc_histogram1d_f64(const double* neighbors, double dx, double dy,
                                  int64_t n_samples, uint64_t seed, int64_t n_bins,
                                  double* out_edges, int64_t* out_counts, int64_t* out_nbins,
                                  double* out_values, int device);

#ifdef __cplusplus
}
#endif

#endif /* DIVUQ_B200_H */
