// Level-crossing probability per grid cell.
//
// Replaces lcp() / cell_crossing_probability (lcp.py:71-100): for cell
// (ci, cj) with corners v00 = cj*nx + ci, v00+1, v00+nx, v00+nx+1 (that
// order, lcp.py:88-91), LCP = clip(1 - (prod_k below_k + prod_k above_k), 0, 1)
// with (below, above) = _tail_probs(mu, sigma, theta) per corner
// (lcp.py:48-68) and np.prod's sequential order ((c0*c1)*c2)*c3.
//
// Layout of the work: a CTA of 32 x 8 threads owns a 64 x 16 tile of cells
// (2 x 2 cells per thread).  It loads the tile's 65 x 17 corner vertices with
// all of a thread's loads in flight at once, evaluates each vertex's tail pair
// ONCE into shared memory (one erfc per vertex, 1.08 per cell -- the fp64 erfc
// is the kernel's bound, not HBM), then every thread forms its cells' products.
#pragma once

#include "common.cuh"
#include "tma.cuh"

namespace divuq {

// ---- branch-free fp64 erfc for the level-crossing kernels ----------------
// libdevice's erfc takes different code paths by range, so a warp whose
// vertices straddle the ranges runs several of them (ncu: the LCP kernel was
// issue-bound at ~330 instructions per cell).  Here: erfc(a) =
// exp(-a^2) * h(q) / (a + K), q = (a - K) / (a + K), K = 3, h a degree-16
// polynomial fitted offline against scipy's erfcx on [0, 6.2]
// (tools/fit_erfc.py: fit64(3.0, 16, amax=6.2); max error 1.3e-15 absolute,
// 2.9e-15 relative), one reciprocal (one Newton step), one branch-free exp,
// and the a*a rounding corrected by one FMA.  The LCP bar is ABSOLUTE
// (1e-12 on products of tail probabilities): past a = 6.2 erfc(a) < 1.9e-18,
// returned as 0 (also for a = inf, sigma -> 0+).  (The first version fitted
// degree 20 on [0, 26.5] to 3.8e-15 relative: 4 more FMAs per vertex.)
__constant__ double kErfcLcp[17] = {
    0x1.12f21ddd9f5e1p+0, -0x1.c44c471baa268p-1, 0x1.2e326945de38ap-1, -0x1.3deb21416ca90p-2,
    0x1.e995f11b16886p-4, -0x1.b78993b5e4be8p-6, -0x1.3dd3e5fc26ebfp-10, 0x1.8dae28f56a401p-9,
    -0x1.1f7943276e395p-11, -0x1.2234c8a90349bp-12, 0x1.c350cc2d97cf3p-14, 0x1.fd736047b47bdp-16,
    -0x1.28c763237c059p-16, -0x1.4c4280ee09a7ap-18, 0x1.9657f8bc02840p-19, 0x1.d4b67a91621acp-20,
    0x1.2479dd117d25fp-22};

// exp(t) for t in [-39, 0] (a <= 6.2): k = rint(t/ln2), r = t - k ln2
// (fdlibm's hi/lo split), e^r by its Taylor series to r^11 (|r| <= 0.347:
// truncation < 7e-15 relative), times 2^k built in the exponent bits.
// Coefficients come from constant memory (no UMOV-materialised literals), no
// range branches.
__constant__ double kExpTaylor[12] = {
    0x1.0000000000000p+0, 0x1.0000000000000p+0, 0x1.0000000000000p-1, 0x1.5555555555555p-3,
    0x1.5555555555555p-5, 0x1.1111111111111p-7, 0x1.6c16c16c16c17p-10, 0x1.a01a01a01a01ap-13,
    0x1.a01a01a01a01ap-16, 0x1.71de3a556c734p-19, 0x1.27e4fb7789f5cp-22, 0x1.ae64567f544e4p-26};

__device__ __forceinline__ double exp_neg_lcp(double t) {
  const double y = fma(t, 0x1.71547652b82fep+0, 0x1.8p52);   // 1.5*2^52 + rint(t*log2(e))
  const double kd = y - 0x1.8p52;
  const int ki = __double2loint(y);
  double r = fma(kd, -6.93147180369123816490e-01, t);
  r = fma(kd, -1.90821492927058770002e-10, r);
  double p = kExpTaylor[11];
#pragma unroll
  for (int k = 10; k >= 0; --k) p = fma(p, r, kExpTaylor[k]);
  return p * __hiloint2double((ki + 1023) << 20, 0);
}

// 1/d: rcp.approx (~2^-23) and one Newton step (~2^-46 relative) -- ample for
// the absolute 1e-12 LCP bar; lcp_div below adds a residual correction
__device__ __forceinline__ double rcp_lcp(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  return fma(r, fma(-d, r, 1.0), r);
}

__device__ __forceinline__ double erfc_abs_lcp(double x) {
  constexpr double K = 3.0;
  const double a = fabs(x);
  const double r = rcp_lcp(a + K);
  const double q = (a - K) * r;
  double p = kErfcLcp[16];
#pragma unroll
  for (int k = 15; k >= 0; --k) p = fma(p, q, kErfcLcp[k]);
  const double s = a * a;
  const double lo = fma(a, a, -s);   // a*a - s exactly
  double y = p * r * exp_neg_lcp(fmax(-s, -39.0));
  y = fma(y, -lo, y);                // * exp(-lo) ~ (1 - lo)
  // erfc(0) = 1 exactly, so a tail argument of exactly 0 gives 1/2 on both
  // sides like ndtr(0) -- the reference's exact negation symmetry of the
  // LCP (test_lcp.py:53-62) needs it (the fit is ~1e-15 off at 0)
  return a > 6.2 ? 0.0 : (a == 0.0 ? 1.0 : y);
}
__device__ __forceinline__ float erfc_abs_lcp(float x) { return erfc_abs(x); }

// erfc(a) / 2 for a = |x| >= 0: erfc_abs_lcp with the 1/2 folded into the
// coefficients (every Horner step, product and the FMA correction are the
// halved values exactly: bitwise 0.5 * erfc_abs_lcp(a)) and without the
// exponent clamp -- past a = 6.2 (and for a = inf) the exp's garbage is
// discarded by the final select, never propagated.
__constant__ double kErfcLcpHalf[17] = {
    0x1.12f21ddd9f5e1p-1, -0x1.c44c471baa268p-2, 0x1.2e326945de38ap-2, -0x1.3deb21416ca90p-3,
    0x1.e995f11b16886p-5, -0x1.b78993b5e4be8p-7, -0x1.3dd3e5fc26ebfp-11, 0x1.8dae28f56a401p-10,
    -0x1.1f7943276e395p-12, -0x1.2234c8a90349bp-13, 0x1.c350cc2d97cf3p-15, 0x1.fd736047b47bdp-17,
    -0x1.28c763237c059p-17, -0x1.4c4280ee09a7ap-19, 0x1.9657f8bc02840p-20, 0x1.d4b67a91621acp-21,
    0x1.2479dd117d25fp-23};
// Table-driven erfc(a)/2 (round 2, late): 100 intervals of width 1/16 on
// [0, 6.25), each a degree-9 Taylor polynomial in d = a - c_j about its
// centre (|d| <= 1/32; tools/fit_erfc_table.py: coefficients from mpmath,
// max abs error 5.55e-17, max rel error 1.56e-11 on [0, 6.2]).  One index, five 16-byte
// loads (L1-resident 8 KB) and 10 FMAs replace the reciprocal, the 16-FMA
// fit and the 13-FMA exp of half_erfc_fit below: the LCP kernels were bound
// by the fp64 pipe and issue (~67 fp64 instructions per vertex).
#ifndef DIVUQ_LCP_ERFC_TAB
#define DIVUQ_LCP_ERFC_TAB 1
#endif
// coefficient-pair-major: pair k of interval j at [k][j], so a warp's gathers for one
// pair fall in one 1.6 KB span (<= 13 lines) instead of one 80-byte row per lane
__device__ __align__(16) double kErfcTab[5][100][2] = {
    {{0x1.edf3a9ba22dadp-2, -0x1.209546ad13ccfp-1}, {0x1.c9fefdd6eaf19p-2, -0x1.1e565bca400d4p-1}, {0x1.a6757d08215d8p-2, -0x1.19e5e92b964abp-1}, {0x1.839bd55eaafc8p-2, -0x1.135e3075d076bp-1}, {0x1.61b2aba3da093p-2, -0x1.0ae54fa490723p-1}, {0x1.40f535d93160ep-2, -0x1.00abcf3e187a9p-1}, {0x1.219809edbd524p-2, -0x1.e9d5a8e4c934ep-2}, {0x1.03c82ab5eb831p-2, -0x1.cfc41e36c7df9p-2}, {0x1.cf54b4058455fp-3, -0x1.b3aafcc27502ep-2}, {0x1.9ab5668e4930ap-3, -0x1.96164fafd8de3p-2}, {0x1.69d91d8a595dap-3, -0x1.7791b886e7403p-2}, {0x1.3cd553f045d45p-3, -0x1.58a445da7c74cp-2}, {0x1.13af1e11be721p-3, -0x1.39ccc1b136d5ap-2}, {0x1.dcb8cae2d747fp-4, -0x1.1b7e98fe26217p-2}, {0x1.998af9b56a3aep-4, -0x1.fc3ee5d1524b0p-3}, {0x1.5d8debd20aacep-4, -0x1.c40b0729ed548p-3}, {0x1.286740c7a7dabp-4, -0x1.8eed36b886d93p-3}, {0x1.f35a715b2f3e1p-5, -0x1.5d4fd33729015p-3}, {0x1.a1d5a5c4edb96p-5, -0x1.2f7cc3fe6f423p-3}, {0x1.5b478318ff939p-5, -0x1.059f59af7a906p-3}, {0x1.1eb024fc75285p-5, -0x1.bf8e1b1ca2279p-4}, {0x1.d61dd57628999p-6, -0x1.7bd5c7df3fe9cp-4}, {0x1.7ed039b24c96bp-6, -0x1.3fda6bc016994p-4}, {0x1.3593328f6abbep-6, -0x1.0b3f52ce8c383p-4}, {0x1.f13a043742333p-7, -0x1.bb1c972f23e50p-5}, {0x1.8c87b7a37834fp-7, -0x1.6c7e64e7281cbp-5}, {0x1.3a02ffb1b7ceep-7, -0x1.297db960e4f63p-5}, {0x1.edd4d2aec5adbp-8, -0x1.e1d4cf1e2450ap-6}, {0x1.81915cb0e3323p-8, -0x1.83298d717210ep-6}, {0x1.2ae6f94510dd8p-8, -0x1.34ac36ad8dafep-6}, {0x1.cc218694238a2p-9, -0x1.e85c449e377f3p-7}, {0x1.5fa14942c3d54p-9, -0x1.7f5188610ddc8p-7}, {0x1.0ac8fce979b96p-9, -0x1.2a875b5ffab56p-7}, {0x1.91e8bd0830a74p-10, -0x1.cd5ec93c12432p-8}, {0x1.2c8c79e6f04a3p-10, -0x1.61beae53b72b7p-8}, {0x1.be3eb08ae7c20p-11, -0x1.0d1d69569b82dp-8}, {0x1.48e09b21414bfp-11, -0x1.9646f35a76624p-9}, {0x1.e139bb05eb49ep-12, -0x1.30499b503957fp-9}, {0x1.5d80693276a6dp-12, -0x1.c4412bf4b8f0bp-10}, {0x1.f7f3581a4dc2cp-13, -0x1.4d78bba8ca5fdp-10}, {0x1.68a8e4b2fc8c2p-13, -0x1.e7f232d9e2630p-11}, {0x1.003692548d98bp-13, -0x1.6235fbd7a4345p-11}, {0x1.695875fb574a0p-14, -0x1.fe41cd9bb4eeep-12}, {0x1.f9da9fde95755p-15, -0x1.6caa0d3582fe9p-12}, {0x1.5f7524a8e81a2p-15, -0x1.0295ef6591848p-12}, {0x1.e4c0b066a4970p-16, -0x1.6be02102b3520p-13}, {0x1.4bd1bfa2aba3dp-16, -0x1.fc0d55470cf51p-14}, {0x1.c2e43d417197bp-17, -0x1.5feada379d8b7p-14}, {0x1.3010aa198de78p-17, -0x1.e3bcf436a1a95p-15}, {0x1.970b05888fda2p-18, -0x1.49e17724f4d41p-15}, {0x1.0e69f27a37df3p-18, -0x1.be6abbb10a5aap-16}, {0x1.649b01d73110ap-19, -0x1.2bb5cc22e5db6p-16}, {0x1.d2bfc6210880ap-20, -0x1.8f4ccca7fc90dp-17}, {0x1.2f2aa92823e80p-20, -0x1.07ebd2a2d2844p-17}, {0x1.86e0050236315p-21, -0x1.5a2adfa0b4bc4p-18}, {0x1.f42c17ae0ebf6p-22, -0x1.c282cd3957edap-19}, {0x1.3d9be56279ee9p-22, -0x1.22df298214423p-19}, {0x1.90538b942ea7cp-23, -0x1.74adc8f4064d3p-20}, {0x1.f4c8c392fb944p-24, -0x1.d9c73698fb1dcp-21}, {0x1.36dcf18a6465cp-24, -0x1.2acee2f5ecdb8p-21}, {0x1.7f064a8ba8323p-25, -0x1.75fa8dbc84becp-22}, {0x1.d45f15b49b35ep-26, -0x1.d06ad6ecdf971p-23}, {0x1.1c33cd3c37addp-26, -0x1.1e1e857adc568p-23}, {0x1.564a91cd221f0p-27, -0x1.5dcd669f2cd34p-24}, {0x1.99218b8ac7f8ep-28, -0x1.a854ea14102a8p-25}, {0x1.e5510173b9a50p-29, -0x1.febc107d5efaap-26}, {0x1.1da9433aebbcfp-29, -0x1.30f93c3699078p-26}, {0x1.4dbb989001d84p-30, -0x1.6961b8d641d06p-27}, {0x1.82eedbe410407p-31, -0x1.a8e405e651ab6p-28}, {0x1.bd3474ec16ca5p-32, -0x1.efac5187b2863p-29}, {0x1.fc5b8748842b2p-33, -0x1.1edfa3c5f5ccap-29}, {0x1.2006aeb6bc768p-33, -0x1.4979ac8b28927p-30}, {0x1.43e56c3e340a7p-34, -0x1.77756ec9f78fap-31}, {0x1.697595326d7dcp-35, -0x1.a887bd2b4404dp-32}, {0x1.904e0b3aa82a3p-36, -0x1.dc479de0ef001p-33}, {0x1.b7f1f31b571b6p-37, -0x1.0916f04b6e18bp-33}, {0x1.dfd296adef82ap-38, -0x1.24caf2c32af14p-34}, {0x1.03a918225a966p-38, -0x1.40dfd87456f4cp-35}, {0x1.16e3ca3d4393fp-39, -0x1.5ce9ab1670dd2p-36}, {0x1.294150fb19119p-40, -0x1.7872d9fa10aadp-37}, {0x1.3a68a8c1234e1p-41, -0x1.92ff33023d5bdp-38}, {0x1.4a029a7ea7cd1p-42, -0x1.ac0f5f3229372p-39}, {0x1.57bc950253825p-43, -0x1.c324c20e337dcp-40}, {0x1.634b7f56b0a5cp-44, -0x1.d7c593130dd0bp-41}, {0x1.6c6e61e57bf9bp-45, -0x1.e9810295890ecp-42}, {0x1.72f0c4c8e9bffp-46, -0x1.f7f338086a86bp-43}, {0x1.76aca47764427p-47, -0x1.01647ba798745p-43}, {0x1.778be2bd9795bp-48, -0x1.04e15ecc7f3f6p-44}, {0x1.7589207e91ad1p-49, -0x1.065b9616170d4p-45}, {0x1.70aff489136ebp-50, -0x1.05ca50205d26ap-46}, {0x1.691c7c768becep-51, -0x1.0330f0fd69921p-47}, {0x1.5efa4d64f59f6p-52, -0x1.fd3de10d62855p-49}, {0x1.5282d2d5803fep-53, -0x1.f05e82aae2bb9p-50}, {0x1.43fb317b5dc37p-54, -0x1.e00e9148a1d25p-51}, {0x1.33b1c9d1576ecp-55, -0x1.ccaaea71ab0dfp-52}, {0x1.21fb7a81c5444p-56, -0x1.b69f10b0191b5p-53}, {0x1.0f30c4d0be5c0p-57, -0x1.9e614ecbf4af6p-54}, {0x1.f755ea760487dp-59, -0x1.846e9dda7a163p-55}, {0x1.cf82e0eb6196bp-60, -0x1.694680a9a3ee6p-56}, {0x1.a78e8252c204dp-61, -0x1.4d67050b31c2ap-57}},
    {{0x1.209546ad13ccfp-6, 0x1.8006a56251aebp-3}, {0x1.ad8189af6013dp-5, 0x1.7712743c42915p-3}, {0x1.605f63767bdd6p-4, 0x1.6582e9b69c9acp-3}, {0x1.e1e4d4ce2ccfbp-4, 0x1.4c04e66e0d59cp-3}, {0x1.2c41f99922807p-3, 0x1.2b900b640a202p-3}, {0x1.60ec3cf561a89p-3, 0x1.05599bafe4ecdp-3}, {0x1.8dfd9939e37afp-3, 0x1.b588d8dc5bb93p-4}, {0x1.b2c7dc535b619p-3, 0x1.5a9de93f9c0d1p-4}, {0x1.cee5ac8e9c531p-3, 0x1.fa02983c853cbp-5}, {0x1.e23a7ea0d187ep-3, 0x1.3f5ee1564be41p-5}, {0x1.ecef42310f844p-3, 0x1.15c3c5ce705cdp-6}, {0x1.ef6c246a12e7ep-3, -0x1.e83e0da030501p-9}, {0x1.ea4feea4e5addp-3, -0x1.715e595343362p-6}, {0x1.de65a22ce0587p-3, -0x1.40686a3f3dc32p-5}, {0x1.cc990045b293fp-3, -0x1.b37338e6ac819p-5}, {0x1.b5eaaef09de9dp-3, -0x1.0847c7dad86b1p-4}, {0x1.9b64a06e4b100p-3, -0x1.2bb6e2c74d4fep-4}, {0x1.7e0f4f0454d97p-3, -0x1.444bc66c35bc3p-4}, {0x1.5ee8429e30a49p-3, -0x1.52a8395f9626ep-4}, {0x1.3eda354ddd5ffp-3, -0x1.57b85ad436065p-4}, {0x1.1eb7095e57e16p-3, -0x1.549ea6f7a013cp-4}, {0x1.fe674493fde22p-4, -0x1.4a9feacf7e220p-4}, {0x1.c1cb27861fc79p-4, -0x1.3b1051230b980p-4}, {0x1.8885019f5df29p-4, -0x1.274275fc87eacp-4}, {0x1.5341e3c0177b6p-4, -0x1.107929f6e7527p-4}, {0x1.2274b86833f6ep-4, -0x1.efb890e5b6631p-5}, {0x1.ecb83b087b37bp-5, -0x1.bce18363bbbb7p-5}, {0x1.9e12e1fde7354p-5, -0x1.8a27806de834fp-5}, {0x1.58d101f909971p-5, -0x1.58f1456f7db5ep-5}, {0x1.1c8ec267fe9e2p-5, -0x1.2a52c5d83c051p-5}, {0x1.d177f166cce53p-6, -0x1.fe23b75845ce1p-6}, {0x1.7954423f89a51p-6, -0x1.af5baae337ae8p-6}, {0x1.2f3178cd7aa03p-6, -0x1.68d1c45b96f01p-6}, {0x1.e2ff3aaae31e4p-7, -0x1.2aa4e58242523p-6}, {0x1.7d6193f2417adp-7, -0x1.e947279e4a440p-7}, {0x1.2a8ca0dc14852p-7, -0x1.8cc071b719c47p-7}, {0x1.cf68ed932f081p-8, -0x1.3e8735b5b73b4p-7}, {0x1.6496420203331p-8, -0x1.fa73d7eb1b712p-8}, {0x1.100f34713740dp-8, -0x1.8ebda0768e8e9p-8}, {0x1.9ba107a459ce4p-9, -0x1.36f273fbd909cp-8}, {0x1.34c7442de142bp-9, -0x1.e066bed09942fp-9}, {0x1.cb5e029ba8f3dp-10, -0x1.6fa4c7ef470e7p-9}, {0x1.52d7b2896626ap-10, -0x1.16c192d8803d9p-9}, {0x1.efb729f4be121p-11, -0x1.a2da7cec0155dp-10}, {0x1.679880e93e5c4p-11, -0x1.37d38e3a705a8p-10}, {0x1.02b15777eb7c5p-11, -0x1.cc1d886874d4dp-11}, {0x1.7121aff59f6a1p-12, -0x1.506d6992fc8f3p-11}, {0x1.05304df546ed8p-12, -0x1.e79c081b79ea6p-12}, {0x1.6e95311166825p-13, -0x1.5e3edf674e2cap-12}, {0x1.fe48c44d2ab81p-14, -0x1.f2bd95d72a517p-13}, {0x1.60403819b22b8p-14, -0x1.5fff1dde5304ap-13}, {0x1.e258948829ed1p-15, -0x1.ec8a8e59d9d41p-14}, {0x1.478cffe1cd2edp-15, -0x1.559f04ad4de53p-14}, {0x1.b93e442837f52p-16, -0x1.d5cf1514977e4p-15}, {0x1.26c8826ed9e85p-16, -0x1.40473571d537fp-15}, {0x1.86ad6df7ba401p-17, -0x1.b0f313eeb65aep-16}, {0x1.00c902a4d5e27p-17, -0x1.22234eb745952p-16}, {0x1.4ed4228b3da96p-18, -0x1.81918baca19a6p-17}, {0x1.b11017e7d5893p-19, -0x1.fc0dfadc2c735p-18}, {0x1.15cc5700a2341p-19, -0x1.4be757b934876p-18}, {0x1.6186d9fc357c5p-20, -0x1.ae02322e088ccp-19}, {0x1.be46aa879edb2p-21, -0x1.143860c49d1bep-19}, {0x1.1769ce59fb2c8p-21, -0x1.5fe5d47560890p-20}, {0x1.5b11cbd1ee799p-22, -0x1.bc91a6b1c19d6p-21}, {0x1.aba593e8384aep-23, -0x1.167c252a457c1p-21}, {0x1.055a3c70279a4p-23, -0x1.59ff37766ebaap-22}, {0x1.3ce2f890bb01dp-24, -0x1.aa5010863cb4ep-23}, {0x1.7d2510f1f969dp-25, -0x1.0476b165acaa1p-23}, {0x1.c6c40e5083697p-26, -0x1.3ba47a1751665p-24}, {0x1.0d229044adeeep-26, -0x1.7b5bc9db481f1p-25}, {0x1.3c025a6810c37p-27, -0x1.c42f78a0990bep-26}, {0x1.7015eec377539p-28, -0x1.0b487791595c8p-26}, {0x1.a9530780ca70bp-29, -0x1.3962ecb10e64cp-27}, {0x1.e78be33fb01d8p-30, -0x1.6c6ef0b686c13p-28}, {0x1.1535aee3eb1b1p-30, -0x1.a4547ed26541fp-29}, {0x1.38b90f78fbe12p-31, -0x1.e0d7765327992p-30}, {0x1.5dfa962d49546p-32, -0x1.10ca1ff2b034ep-30}, {0x1.848f101ce14c6p-33, -0x1.32fed47f8ebc9p-31}, {0x1.abf69bd9866f4p-34, -0x1.56ae1e8abce90p-32}, {0x1.d39eaac4a0b43p-35, -0x1.7b67ab8af4bc5p-33}, {0x1.fae4fe28d12d7p-36, -0x1.a0a80964d8caep-34}, {0x1.108dc99cf03e2p-36, -0x1.c5db17016c62fp-35}, {0x1.22c6b11327301p-37, -0x1.ea5f66f89f9d5p-36}, {0x1.33c1e2f16e032p-38, -0x1.06c53fdc7635ep-36}, {0x1.43262ab4b77acp-39, -0x1.1756eae582bd3p-37}, {0x1.509f766d9f27fp-40, -0x1.268e278ee0a38p-38}, {0x1.5be1cf20840d3p-41, -0x1.3418096323cecp-39}, {0x1.64ac1f9b95f8ap-42, -0x1.3fa8302ae20aap-40}, {0x1.6acaa58a8be05p-43, -0x1.48fb92d09877ep-41}, {0x1.6e18ec0d42440p-44, -0x1.4fdb0511052bfp-42}, {0x1.6e8334c657489p-45, -0x1.541d56105d6abp-43}, {0x1.6c073be0916d5p-46, -0x1.55a8eab9e6eacp-44}, {0x1.66b44c6d7dd99p-47, -0x1.5474bd9d0d910p-45}, {0x1.5eaaa4200e34ap-48, -0x1.5088b65676d11p-46}, {0x1.541a2f15eb495p-49, -0x1.49fd53e8647ebp-47}, {0x1.4740ad7362bb6p-50, -0x1.40faaf0a489f7p-48}, {0x1.38675c67c3783p-51, -0x1.35b6e2bb8345bp-49}, {0x1.27e0423d6afeep-52, -0x1.2873f1a16f655p-50}, {0x1.160341028b267p-53, -0x1.197d455cd7bbap-51}, {0x1.032b14ebb3ae4p-54, -0x1.0924e9a1830bfp-52}},
    {{-0x1.20652dcbf6f44p-7, -0x1.cbee0f1e253f4p-5}, {-0x1.aafd4760d903cp-6, -0x1.ba14988b4bcffp-5}, {-0x1.5aa32b580e2eap-5, -0x1.97594c25a1706p-5}, {-0x1.d2855d59990c6p-5, -0x1.659a35f29f6ddp-5}, {-0x1.1c6c7eef8f2ebp-4, -0x1.277ad7822588ep-5}, {-0x1.451ef6280d21cp-4, -0x1.c06c6e435165cp-6}, {-0x1.62338788af9e4p-4, -0x1.26cf85bc62510p-6}, {-0x1.7317958d257edp-4, -0x1.133e02ab57e13p-7}, {-0x1.77cd75ec71e97p-4, 0x1.fa6f82fbb5d9fp-11}, {-0x1.70e469de059e7p-4, 0x1.3da6878b1601bp-7}, {-0x1.5f6890aff98fcp-4, 0x1.1da642fad787fp-6}, {-0x1.44cc65df8aba5p-4, 0x1.87d3c8dd7af2ep-6}, {-0x1.22cdbdb4cce39p-4, 0x1.da50ae5494465p-6}, {-0x1.f6b0cb6927bcfp-5, 0x1.09c7caecdcbd8p-5}, {-0x1.a0d11fe9bd454p-5, 0x1.19bb2ca3885ccp-5}, {-0x1.47de0a4f7b901p-5, 0x1.1d9de8b54e881p-5}, {-0x1.dee322c06360ap-6, 0x1.169960d5a948ap-5}, {-0x1.356dbb542cb81p-6, 0x1.0643de6e8a060p-5}, {-0x1.313759f197a47p-7, 0x1.dcf844d8f8d98p-6}, {-0x1.8e90c2a154b7fp-11, 0x1.a2893b28e9386p-6}, {0x1.b10f20d12a11bp-8, 0x1.61420b5b26b3ep-6}, {0x1.a0082c90a0f10p-7, 0x1.1cf0e7655281ap-6}, {0x1.1e645a2a663c1p-6, 0x1.b1f643b1359c6p-7}, {0x1.57f7386bfca8ep-6, 0x1.30769f4596ed0p-7}, {0x1.7e1b362eafc7fp-6, 0x1.73b61e485ae1cp-8}, {0x1.92c7dbb8800f6p-6, 0x1.45477088118d2p-9}, {0x1.985aaf9787740p-6, -0x1.cd95f2ac8c96dp-13}, {0x1.91674e13a24cdp-6, -0x1.3bc75e8fa20ecp-9}, {0x1.808d17b33c31fp-6, -0x1.0c1bdce6710d1p-8}, {0x1.68541b2c04ea9p-6, -0x1.5afe42214b417p-8}, {0x1.4b120f9dde3c0p-6, -0x1.8d9906d12ba63p-8}, {0x1.2ad77b77d2437p-6, -0x1.a7b8c4a8c6b64p-8}, {0x1.09648dd331c11p-6, -0x1.ad8b148079603p-8}, {0x1.d049824fc47cap-7, -0x1.a34eda0fb3216p-8}, {0x1.90603010923dbp-7, -0x1.8d14d4bd9c81ap-8}, {0x1.54a148886f143p-7, -0x1.6e91361de8e7ap-8}, {0x1.1e1611aabd28fp-7, -0x1.4afd8cd0f813fp-8}, {0x1.daa3005c2dc23p-8, -0x1.250942c315ddcp-8}, {0x1.850c68e8e66dep-8, -0x1.fdac8345ffa47p-9}, {0x1.3b38708f7b9b0p-8, -0x1.b3fdff1ddeb2bp-9}, {0x1.f914f2c60c37dp-9, -0x1.6f4662f6be647p-9}, {0x1.903a08305ea8cp-9, -0x1.30f12c8400179p-9}, {0x1.39bfce9b4ea0bp-9, -0x1.f376a554ed56fp-10}, {0x1.e6c27ad2b222fp-10, -0x1.93b1f34b2152bp-10}, {0x1.75b371a26483cp-10, -0x1.4231c3bfee1dep-10}, {0x1.1bff7066467a9p-10, -0x1.fc0f76c956e3dp-11}, {0x1.ab596015fc6e6p-11, -0x1.8bdd79a0a9af0p-11}, {0x1.3e5dc1062dff1p-11, -0x1.30eb20ccd1222p-11}, {0x1.d5be6d15ac109p-12, -0x1.d07da13e7c605p-12}, {0x1.57389188a72bbp-12, -0x1.5decc405a2204p-12}, {0x1.f0c93c73e7fc2p-13, -0x1.04cbf67b04634p-12}, {0x1.6425722b9f1f9p-13, -0x1.80a83a7115cc1p-13}, {0x1.f9e163b15c443p-14, -0x1.18bda8b8cc10cp-13}, {0x1.63f5eb46874f1p-14, -0x1.95a0411e7173ap-14}, {0x1.f057dbf3657c9p-15, -0x1.2217929ff05aep-14}, {0x1.56e457745d482p-15, -0x1.9ad1f65a72e01p-15}, {0x1.d57a2be01de03p-16, -0x1.200c2ffacaa99p-15}, {0x1.3e81c09c29629p-16, -0x1.9004afecfcd9cp-16}, {0x1.ac4e1aa49980ap-17, -0x1.131810ab0cea4p-16}, {0x1.1d6ab6f8cbfc3p-17, -0x1.76c5a3031abfap-17}, {0x1.79082befd4f56p-18, -0x1.f9c26e20a4046p-18}, {0x1.edabcbc3e60a1p-19, -0x1.52139c878146cp-18}, {0x1.405da04876021p-19, -0x1.bfc96a92d04ebp-19}, {0x1.9c2c5d12df900p-20, -0x1.25d1e3c672ee8p-19}, {0x1.06d78ca042594p-20, -0x1.7e0f59fc13c3cp-20}, {0x1.4c53adb9dcb0dp-21, -0x1.ec4924282f2bfp-21}, {0x1.a08ef1ca16292p-22, -0x1.3a4a6af2b777dp-21}, {0x1.02d3a3b9d1b6fp-22, -0x1.8db3567a51980p-22}, {0x1.3ee334beefa5dp-23, -0x1.f2bf9e69e1630p-23}, {0x1.8588212e67288p-24, -0x1.35f42dafddcf4p-23}, {0x1.d7c6c3583c86cp-25, -0x1.7dd6ccb35042bp-24}, {0x1.1b44b64c3cdc9p-25, -0x1.d23ff3ec1295fp-25}, {0x1.51494525df342p-26, -0x1.1a2961b6a4661p-25}, {0x1.8e36e9a44cc0ap-27, -0x1.5286ee3476028p-26}, {0x1.d2308d0deb9c8p-28, -0x1.929d46a52f04dp-27}, {0x1.0e9760d0ac874p-28, -0x1.daad91106f7a4p-28}, {0x1.377c7e98de3bbp-29, -0x1.156649dcc74b8p-28}, {0x1.638ff4a6981fdp-30, -0x1.416d25116bdd7p-29}, {0x1.927ca04d1b713p-31, -0x1.713d3b01418f3p-30}, {0x1.c3ced54e6aa51p-32, -0x1.a4875d81e79f8p-31}, {0x1.f6f47be47aa2ap-33, -0x1.dad968c324be0p-32}, {0x1.159f41ea08ab1p-33, -0x1.09ced3e32b2a9p-32}, {0x1.2ff1e0a81d3e6p-34, -0x1.270ddbd0d82c1p-33}, {0x1.4a029a8792fa3p-35, -0x1.44bd8619c5577p-34}, {0x1.6359d5b0d44e1p-36, -0x1.626391b1900aap-35}, {0x1.7b7b43e9a4237p-37, -0x1.7f7aad9d63600p-36}, {0x1.91e9beb94e3a4p-38, -0x1.9b762250ed191p-37}, {0x1.a62b70897acadp-39, -0x1.b5c6191326f37p-38}, {0x1.b7ce1a1ead01cp-40, -0x1.cddc55157d8dcp-39}, {0x1.c66b3f3fea78ap-41, -0x1.e33127fb0786ep-40}, {0x1.d1ac042ae075dp-42, -0x1.f54864a8e083bp-41}, {0x1.d94c87c1c2147p-43, -0x1.01db0808a2548p-41}, {0x1.dd1e8c33185d2p-44, -0x1.07114857a6607p-42}, {0x1.dd0b48e0fba89p-45, -0x1.0a271159d501ep-43}, {0x1.d9144beee5400p-46, -0x1.0b09b019fba1ep-44}, {0x1.d1535f4c89962p-47, -0x1.09b45cb7b2994p-45}, {0x1.c5f9735a691f6p-48, -0x1.0630644518e12p-46}, {0x1.b74c9f5960946p-49, -0x1.0094be7135e03p-47}, {0x1.a5a554b61e3a8p-50, -0x1.f20a2b19450a0p-49}, {0x1.916aed049ceaap-51, -0x1.df609ede6c895p-50}},
    {{0x1.8046ccf82fc25p-9, 0x1.b52bb52dae089p-7}, {0x1.1afcdb45106afp-7, 0x1.9d72effa6e9e9p-7}, {0x1.c69c625d3b6d6p-7, 0x1.6fa7f7f0703dcp-7}, {0x1.2cf626743c137p-6, 0x1.2ef4193d1c84ap-7}, {0x1.66c9b1f0773b7p-6, 0x1.bf7e7cb9d806fp-8}, {0x1.8e2d73338066ap-6, 0x1.0ea4a66be12c7p-8}, {0x1.a1bcaaadf9b4dp-6, 0x1.5b4a7759cb5eap-10}, {0x1.a155bbff2475ep-6, -0x1.7204a625822b1p-10}, {0x1.8e0db524c81dcp-6, -0x1.00bf7366f74adp-8}, {0x1.6a0d073ecb040p-6, -0x1.8cf08575fbdbfp-8}, {0x1.38599103c4a6dp-6, -0x1.fa4f3bca1aa94p-8}, {0x1.f9271a25f6a3dp-7, -0x1.2252368b2ae92p-7}, {0x1.75578f3e30674p-7, -0x1.35331b5e89cadp-7}, {0x1.da668fc2db935p-8, -0x1.364e735a3699bp-7}, {0x1.a0b7db1325892p-9, -0x1.274a5a689a95ap-7}, {-0x1.33252a6791a56p-11, -0x1.0ab3e3b3edd80p-7}, {-0x1.feab4a742cec1p-9, -0x1.c76eb949ab10cp-8}, {-0x1.b2e1f8689e99fp-8, -0x1.6ba6d94a3cf53p-8}, {-0x1.1e45f26b17623p-7, -0x1.091cb53598fa7p-8}, {-0x1.4d6af44a48e12p-7, -0x1.4ccee5911fdc8p-9}, {-0x1.677b7f2469de2p-7, -0x1.24f98c3fd74d6p-10}, {-0x1.6e3396e8cd5cfp-7, 0x1.3a2d69e6d7646p-13}, {-0x1.64297daf8bec0p-7, 0x1.3e36624a5589ap-10}, {-0x1.4c823166dce8cp-7, 0x1.0c2c9cc2c498dp-9}, {-0x1.2aa76417a1be6p-7, 0x1.59a38b686cba1p-9}, {-0x1.02047aa9ce18bp-7, 0x1.888356ea394e6p-9}, {-0x1.ab9d42e505531p-8, 0x1.9b93422908a7cp-9}, {-0x1.51b4d075ee6e4p-8, 0x1.96dc7ba236da7p-9}, {-0x1.f5ff1c3dc91a0p-9, 0x1.7f26b8534615cp-9}, {-0x1.56303be1c8a73p-9, 0x1.597eacbfefd2bp-9}, {-0x1.9201b7b454313p-10, 0x1.2aceabbfc291ep-9}, {-0x1.4593aebb99ad7p-11, 0x1.ef1cef1ad5ce0p-10}, {0x1.f00fa67ebe88ap-14, 0x1.871876029dbb9p-10}, {0x1.682d8cfac8335p-11, 0x1.239bf2d7c03e3p-10}, {0x1.1f795af53f4efp-10, 0x1.9222e9b7efe98p-11}, {0x1.65c02de45b821p-10, 0x1.e94b0474fcee9p-12}, {0x1.8c72003a09b22p-10, 0x1.c6a71752a9772p-13}, {0x1.997578c7d9ec2p-10, 0x1.3903ddc0ea04fp-16}, {0x1.929de6f287807p-10, -0x1.10c7146833c3bp-13}, {0x1.7d55d56a3ef1dp-10, -0x1.eae5e24d5bf4fp-13}, {0x1.5e664585b01aap-10, -0x1.3a1598ce4699fp-12}, {0x1.39d769ac96352p-10, -0x1.5d7942eed576cp-12}, {0x1.12e67cbb0835bp-10, -0x1.66d6e3486ab1ap-12}, {0x1.d8179ccc11a89p-11, -0x1.5cf51ca63ebecp-12}, {0x1.8e184d47ed800p-11, -0x1.45d5b433e7709p-12}, {0x1.4a222862f90aep-11, -0x1.2688860400a6bp-12}, {0x1.0d88da9a94441p-11, -0x1.031cdbc989ff4p-12}, {0x1.b1b06c1a9ab62p-12, -0x1.bd52f9ad1dc24p-13}, {0x1.58106cc48eb8ap-12, -0x1.76c83edb482d6p-13}, {0x1.0d559cf04d47bp-12, -0x1.35838ef55ffd2p-13}, {0x1.a0489350bd80dp-13, -0x1.f66b4fb65dcb5p-14}, {0x1.3dbb93752a497p-13, -0x1.913b2ed0e365ep-14}, {0x1.df381bd3e185bp-14, -0x1.3b94f4694e719p-14}, {0x1.652e5f2c75092p-14, -0x1.e950dcef974fcp-15}, {0x1.073240163609cp-14, -0x1.762758715b4c5p-15}, {0x1.7f92ad8659d0ep-15, -0x1.1a5578f060b5ep-15}, {0x1.147585d3742acp-15, -0x1.a4b07bc40554dp-16}, {0x1.8a40e183d930fp-16, -0x1.359243c3869dap-16}, {0x1.1629d94b96792p-16, -0x1.c22a7363543b3p-17}, {0x1.847332575e7e9p-17, -0x1.437f264b54207p-17}, {0x1.0c768236315eep-17, -0x1.cba71a8ed8f51p-18}, {0x1.6f567cd9e55d0p-18, -0x1.42ebd62151ae7p-18}, {0x1.f19ff5e45fc3cp-19, -0x1.c0c4db581ddadp-19}, {0x1.4dbe26c8d0a30p-19, -0x1.347bbd5d9a5b7p-19}, {0x1.bb4d483775aa6p-20, -0x1.a39f4316251b0p-20}, {0x1.23927ad6e706bp-20, -0x1.1a6e0ce5d038bp-20}, {0x1.7be1e8321e6cdp-21, -0x1.78477f9a1b7e9p-21}, {0x1.ea3ef4e1ecf36p-22, -0x1.f03b172701cd5p-22}, {0x1.395c08ab289a6p-22, -0x1.43ee563891805p-22}, {0x1.8cd98864b8351p-23, -0x1.a2b8684d082f0p-23}, {0x1.f1ec2f6866e11p-24, -0x1.0bf7ab9152a1ep-23}, {0x1.357d673b42871p-24, -0x1.53a573b7f0718p-24}, {0x1.7d35cd08f3156p-25, -0x1.aa5983b4abf1ep-25}, {0x1.d14639551744dp-26, -0x1.090911a5c938ap-25}, {0x1.195dbfd1ed94cp-26, -0x1.466323bb3bcdcp-26}, {0x1.513c51b62b55dp-27, -0x1.8e2816ccca1b4p-27}, {0x1.9092f4d6aeedbp-28, -0x1.e12a4da48415dp-28}, {0x1.d78fb229a6240p-29, -0x1.2009de1b81ee9p-28}, {0x1.1318f5d4273eep-29, -0x1.55abb3193e728p-29}, {0x1.3e213e6a5980dp-30, -0x1.91915d79cca1ap-30}, {0x1.6ca68a8578804p-31, -0x1.d3a7ce7658d89p-31}, {0x1.9e4dacd860232p-32, -0x1.0dd5fed637acep-31}, {0x1.d2992b5222d8bp-33, -0x1.3492fc37d4814p-32}, {0x1.0474ac344f72ap-33, -0x1.5db2d560438a6p-33}, {0x1.203efc65096edp-34, -0x1.88c0e6edfc52fp-34}, {0x1.3c3cc6a1aa18cp-35, -0x1.b52ca9d660407p-35}, {0x1.57f3209af6d1fp-36, -0x1.e24bc45fa28bfp-36}, {0x1.72de3204d30cap-37, -0x1.07aec04057e5bp-36}, {0x1.8c751cb2087a4p-38, -0x1.1dc7ce2e7245ep-37}, {0x1.a42e6952d695fp-39, -0x1.3302296771e2dp-38}, {0x1.b984c725f17cdp-40, -0x1.46ecb1c8cc3e3p-39}, {0x1.cbfbe4a9f1094p-41, -0x1.5917e72fe74ebp-40}, {0x1.db252298b3cc2p-42, -0x1.6919f20e59115p-41}, {0x1.e6a3e1bd51e07p-43, -0x1.7692a3260547bp-42}, {0x1.ee312fc55c626p-44, -0x1.812f347c3122cp-43}, {0x1.f19e9eea833b2p-45, -0x1.88ad97221859bp-44}, {0x1.f0d81fc2c0e05p-46, -0x1.8cdf1eaa9f699p-45}, {0x1.ebe4c2e111214p-47, -0x1.8daa63bd4ef98p-46}, {0x1.e2e6582c74059p-48, -0x1.8b0c4299667fbp-47}, {0x1.d617f2b9f57fcp-49, -0x1.8517e7b427d46p-48}},
    {{-0x1.8006b89f03431p-11, -0x1.535adf4340afep-9}, {-0x1.19525ddf3f4cdp-9, -0x1.3bb5e6ea92f0ep-9}, {-0x1.bf1cdc320d9e4p-9, -0x1.0e6e15a3efb70p-9}, {-0x1.231a416f74e60p-8, -0x1.9ea861a5d5a1ap-10}, {-0x1.52ff342577637p-8, -0x1.074d3ea39f81ep-10}, {-0x1.6c8dad9dfc8d3p-8, -0x1.8c6f86e3dd32fp-12}, {-0x1.6ee0d1c179205p-8, 0x1.03d1ee98bb736p-12}, {-0x1.5ae0108ee15dfp-8, 0x1.b0f56adafca62p-11}, {-0x1.3316e4cbda1d0p-8, 0x1.58b50ce93cab7p-10}, {-0x1.f6d13715c2f87p-9, 0x1.b96b2bac2cacap-10}, {-0x1.7152f8fa6e155p-9, 0x1.f5840c7474d81p-10}, {-0x1.c0a3b546bdb2ep-10, 0x1.05a259c9e4148p-9}, {-0x1.39c7ec725becep-11, 0x1.fc37138b356f3p-10}, {0x1.d40d5497244b0p-12, 0x1.ccc24c5c5bad5p-10}, {0x1.649ed3b0d13d9p-10, 0x1.838573c7ff370p-10}, {0x1.12d28b6e23ed9p-9, 0x1.288b662c0610ep-10}, {0x1.5842f0a2e142ap-9, 0x1.88e0a7329f2b3p-11}, {0x1.814017016f981p-9, 0x1.7e435ad5f2e17p-12}, {0x1.8ea51f67ebe98p-9, 0x1.56ce94486ac92p-18}, {0x1.83306d9f9abf5p-9, -0x1.41354f8648640p-12}, {0x1.630cad956fa78p-9, -0x1.226d647c07e0bp-11}, {0x1.334a5f89c0655p-9, -0x1.7e506026de7fbp-11}, {0x1.f2b1269ecdcb5p-10, -0x1.b36e890745711p-11}, {0x1.7512ff48292edp-10, -0x1.c41d52585e757p-11}, {0x1.eeb2576b68a22p-11, -0x1.b52a1bf3fd80cp-11}, {0x1.0310520a0991fp-11, -0x1.8d0a27c4654b5p-11}, {0x1.9b0d8d5c040e2p-14, -0x1.53067dbd42795p-11}, {-0x1.e17885adfabc3p-13, -0x1.0e794fd6e32aap-11}, {-0x1.f8692df59a132p-12, -0x1.8c59b56cc396bp-12}, {-0x1.57b3a452a3e64p-11, -0x1.ff9576cdb2d61p-13}, {-0x1.8d50166166d0fp-11, -0x1.0065f0686f1cap-13}, {-0x1.a19c43a3ee1acp-11, -0x1.3adc5e56ed709p-16}, {-0x1.9a7e67be0d4d0p-11, 0x1.0998ce97eff93p-14}, {-0x1.7e75974b08278p-11, 0x1.022f5fd15d054p-13}, {-0x1.53fad4664275bp-11, 0x1.52daef8a44c87p-13}, {-0x1.21062b0c0714cp-11, 0x1.7bbd36b872b6ep-13}, {-0x1.d575138f2cebap-12, 0x1.8392a82f5025fp-13}, {-0x1.6a6d7e0ecfeeap-12, 0x1.71ebbd0812e87p-13}, {-0x1.070dc03ed36e8p-12, 0x1.4e5c86e5ac2e0p-13}, {-0x1.5ebdd55388943p-13, 0x1.1fdf82d06ccf2p-13}, {-0x1.9657fa6defeecp-14, 0x1.d8db2c9ab88a8p-14}, {-0x1.5329371f5bcb6p-15, 0x1.718ea30e5a428p-14}, {0x1.54daddbec3b28p-19, 0x1.10cf51e84e26fp-14}, {0x1.16dab230dd345p-15, 0x1.7659280514d91p-15}, {0x1.bf8f1f20f6cfbp-15, 0x1.cc79b85fd7d65p-16}, {0x1.0fa2d34d24a2dp-14, 0x1.cb616af67580cp-17}, {0x1.22fcb12671bdbp-14, 0x1.b34b82ef58641p-19}, {0x1.214b603d05d95p-14, -0x1.1ac202c0bd766p-18}, {0x1.111dfd774cc68p-14, -0x1.31cf1258aef5fp-17}, {0x1.efd7ac18e5a0dp-15, -0x1.90a278f3be9f9p-17}, {0x1.b410db86974d5p-15, -0x1.b9ddb3017a23bp-17}, {0x1.75639c61776fep-15, -0x1.bc2b9a2742370p-17}, {0x1.385f307d640b4p-15, -0x1.a42dedad77fe8p-17}, {0x1.ffeb7215e383cp-16, -0x1.7c30c85f11c24p-17}, {0x1.9ba2396973759p-16, -0x1.4c28c3e7798f9p-17}, {0x1.4548ced07818cp-16, -0x1.19e319a9fc26fp-17}, {0x1.f9d09587b5d75p-17, -0x1.d2a535156b055p-18}, {0x1.834b95af66852p-17, -0x1.79d1a17c85b68p-18}, {0x1.24444bc61cca3p-17, -0x1.2bde78ed15236p-18}, {0x1.b305e7ea0c7f4p-18, -0x1.d3634fbd93391p-19}, {0x1.3f75bf4cf3ef0p-18, -0x1.661dc8f0e2042p-19}, {0x1.cf2f0a061465bp-19, -0x1.0e0e3e2d91a86p-19}, {0x1.4b9df739f8a25p-19, -0x1.9133e9b099612p-20}, {0x1.d51d3201f72c3p-20, -0x1.25c44b59c6da8p-20}, {0x1.47e83b474a779p-20, -0x1.a8505e571e19fp-21}, {0x1.c523a00a4c55bp-21, -0x1.2e659c938d5b8p-21}, {0x1.3593068b63311p-21, -0x1.a9858fcca8fb3p-22}, {0x1.a250d4cd03694p-22, -0x1.27ae82ffb9f57p-22}, {0x1.178f166d0307fp-22, -0x1.95f72207a6129p-23}, {0x1.71aa3652a3fc4p-23, -0x1.1369557d3cb34p-23}, {0x1.e3ab098a5d25ap-24, -0x1.7161d310bea09p-24}, {0x1.39211c963981dp-24, -0x1.e9d332e2d4b5bp-25}, {0x1.91494d8c2d8c8p-25, -0x1.412bf64121c3dp-25}, {0x1.fd0d35f68e564p-26, -0x1.a0966755e30cbp-26}, {0x1.3fa47558ae6b5p-26, -0x1.0b46e4403e2e2p-26}, {0x1.8d6f8287b1b53p-27, -0x1.535606383f7e1p-27}, {0x1.e94e37c537417p-28, -0x1.aa53c50c38231p-28}, {0x1.2a45b227b4655p-28, -0x1.090ca821d55b1p-28}, {0x1.68218991c99d4p-29, -0x1.4634f4f126c8cp-29}, {0x1.aea6e02b14709p-30, -0x1.8d6dc557e255cp-30}, {0x1.fe1561b8d4373p-31, -0x1.df5e6355dbfe4p-31}, {0x1.2b3ac24909bddp-31, -0x1.1e3e3c25774fep-31}, {0x1.5bc7590e067bfp-32, -0x1.527ef338c5387p-32}, {0x1.906f76a187184p-33, -0x1.8c659ac17f8a2p-33}, {0x1.c8ca563e47693p-34, -0x1.cbb9bbde5f30ap-34}, {0x1.0222e4bc4dc87p-34, -0x1.0808a638fdad1p-34}, {0x1.21132711bd421p-35, -0x1.2c66c12dcaae3p-35}, {0x1.40c48a0e4f461p-36, -0x1.528cded6a8233p-36}, {0x1.60b4080926d30p-37, -0x1.79f6700237b95p-37}, {0x1.80500ce6edb33p-38, -0x1.a206a46e7f8d4p-38}, {0x1.9efc797d4dcbbp-39, -0x1.ca0bc45bca122p-39}, {0x1.bc177898d9baap-40, -0x1.f143d8c00b46cp-40}, {0x1.d6fef2ff3bc09p-41, -0x1.0b713f39ab0e7p-40}, {0x1.ef166229d53a2p-42, -0x1.1d0bd535b0289p-41}, {0x1.01e65bc2d4784p-42, -0x1.2d0b88aac04fdp-42}, {0x1.0a51046396da1p-43, -0x1.3b0feaaf00632p-43}, {0x1.109658fd57d96p-44, -0x1.46c2099f68059p-44}, {0x1.148ed1d1b6cf7p-45, -0x1.4fd7f26eea8b5p-45}, {0x1.1621cf1917f24p-46, -0x1.5617ba2e15046p-46}, {0x1.154695d314aabp-47, -0x1.5959e33068b02p-47}},
};
__device__ __forceinline__ double half_erfc_tab(double a) {
  const double y = fma(a, 16.0, -0.5) + 0x1.8p52;   // 1.5*2^52 + rint(16a - 1/2): the interval
  const double jd = y - 0x1.8p52;
  const int j = min(max(__double2loint(y), 0), 99);  // out of range only where the select discards it
  const double2* t = reinterpret_cast<const double2*>(&kErfcTab[0][j][0]);
  const double2 t01 = __ldg(t), t23 = __ldg(t + 100), t45 = __ldg(t + 200), t67 = __ldg(t + 300),
                t89 = __ldg(t + 400);
  const double d = a - fma(jd, 0.0625, 0.03125);
  double p = fma(t89.y, d, t89.x);
  p = fma(p, d, t67.y);
  p = fma(p, d, t67.x);
  p = fma(p, d, t45.y);
  p = fma(p, d, t45.x);
  p = fma(p, d, t23.y);
  p = fma(p, d, t23.x);
  p = fma(p, d, t01.y);
  p = fma(p, d, t01.x);
  return a > 6.2 ? 0.0 : (a == 0.0 ? 0.5 : p);
}
__device__ __forceinline__ double half_erfc_fit(double a) {
  constexpr double K = 3.0;
  const double r = rcp_lcp(a + K);
  const double q = (a - K) * r;
  double p = kErfcLcpHalf[16];
#pragma unroll
  for (int k = 15; k >= 0; --k) p = fma(p, q, kErfcLcpHalf[k]);
  const double s = a * a;
  const double lo = fma(a, a, -s);
  double y = p * r * exp_neg_lcp(-s);
  y = fma(y, -lo, y);
  return a > 6.2 ? 0.0 : (a == 0.0 ? 0.5 : y);
}
__device__ __forceinline__ double half_erfc_lcp(double a) {
#if DIVUQ_LCP_ERFC_TAB
  return half_erfc_tab(a);
#else
  return half_erfc_fit(a);
#endif
}

// the tail argument (theta - mu) / sigma * sqrt(1/2) for the LCP kernels,
// rounded as before (lcp_div, then the multiply): the CLI's LCP CSV must stay
// within 1e-12 relative + 1e-15 absolute of the reference's (tests/test_cli.py),
// which a one-Newton quotient without the residual step (~2^-46) misses
__device__ __forceinline__ double lcp_arg(double n, double sigma) {
  return div_pos<1>(n, sigma) * 0.70710678118654752440;
}

// (theta - mu) / sigma: fp64 by reciprocal + one Newton step + one residual
// correction (~1 ulp; no IEEE-division slow path: sigma > 0 and finite
// here).  Two edges follow the reference's "overflow allowed" division
// (lcp.py:62-65) exactly: a tiny sigma (rcp.approx.ftz flushes subnormals and
// 1/sigma overflows below 2^-1022) takes the IEEE division, and a quotient
// that overflows stays +-inf (the residual step would turn inf into NaN).
// Both found by the reference's own test_lcp.py run through the drop-in hook
// (tests/test_reference_boundary.py).
__device__ __forceinline__ double lcp_div(double n, double d) { return div_pos<1>(n, d); }
__device__ __forceinline__ float lcp_div(float n, float d) { return __fdiv_rn(n, d); }

// tail pair of one vertex for the LCP kernels: _tail_probs semantics
// (lcp.py:48-68) with the branch-free erfc above (fp32: the shared fp32 erfc)
// fp64, branch-free: sigma = 0 (the reference's step function, lcp.py:58-61:
// below = mu <= theta) becomes x = +inf for theta - mu >= 0 and -inf below,
// which the erfc maps to exactly (1, 0) / (0, 1)
__device__ __forceinline__ void tail_pair_lcp(double mu, double sigma, double theta, double& below,
                                              double& above) {
  const double n = theta - mu;
  const double xs = lcp_arg(n, sigma);
  const double x = sigma == 0.0 ? (n >= 0.0 ? __longlong_as_double(0x7ff0000000000000ll)
                                            : __longlong_as_double(0xfff0000000000000ll))
                                : xs;
  const double y = half_erfc_lcp(fabs(x));
  const double c = 1.0 - y;
  below = x > 0.0 ? c : y;
  above = x > 0.0 ? y : c;
}

// the pair stored in place: the larger tail c goes to `below` when x > 0 and
// to `above` otherwise -- the store addresses are selected (2 integer selects)
// instead of the two fp64 values (4 FSEL)
__device__ __forceinline__ void tail_store_lcp(double mu, double sigma, double theta, double* below,
                                               double* above) {
  const double n = theta - mu;
  const double xs = lcp_arg(n, sigma);
  const double x = sigma == 0.0 ? (n >= 0.0 ? __longlong_as_double(0x7ff0000000000000ll)
                                            : __longlong_as_double(0xfff0000000000000ll))
                                : xs;
  const double y = half_erfc_lcp(fabs(x));
  const bool pos = x > 0.0;
  *(pos ? above : below) = y;
  *(pos ? below : above) = 1.0 - y;
}
__device__ __forceinline__ void tail_store_lcp(float mu, float sigma, float theta, float* below, float* above);

template <typename T>
__device__ __forceinline__ void tail_pair_lcp(T mu, T sigma, T theta, T& below, T& above) {
  using A = Arith<T>;
  if (sigma == T(0)) {
    below = mu <= theta ? T(1) : T(0);
    above = T(1) - below;
    return;
  }
  const T x = A::mul(lcp_div(A::sub(theta, mu), sigma), T(0.70710678118654752440));
  const T y = A::mul(T(0.5), erfc_abs_lcp(x));
  const T c = A::sub(T(1), y);
  below = x > T(0) ? c : y;
  above = x > T(0) ? y : c;
}

__device__ __forceinline__ void tail_store_lcp(float mu, float sigma, float theta, float* below, float* above) {
  float b, a;
  tail_pair_lcp(mu, sigma, theta, b, a);
  *below = b;
  *above = a;
}

#ifndef DIVUQ_LCP_UNROLL
#define DIVUQ_LCP_UNROLL 2   // with 6 CTAs/SM (40 regs): 123.3 -> 121.3 us; 5 + 4 CTAs: 179 us
#endif
constexpr int kLcpUnroll = DIVUQ_LCP_UNROLL;
#ifndef DIVUQ_LCP_MINB
#define DIVUQ_LCP_MINB 6
#endif
constexpr int kLcpTX = 64, kLcpTY = 16, kLcpBX = 32, kLcpBY = 8;
#ifndef DIVUQ_LCP_TMA_TY
#define DIVUQ_LCP_TMA_TY 32   // fit tails: 16: 121.5 us, 24: 114.8, 32: 113.7, 40: 112.6; table tails + row-run epilogue: 32: 100.5, 40: 101.0 (4096^2)
#endif
constexpr int kLcpTYT = DIVUQ_LCP_TMA_TY;   // cell rows per CTA of lcp2d_tma_kernel

// max(r, 0) keeping NaN: r = 1 - (pb + pa) is never -0, and the GPU's NaN
// is positive, so the sign bit alone says r < 0 (fp32: the plain compare)
__device__ __forceinline__ double lcp_clip0(double r) { return __double2hiint(r) < 0 ? 0.0 : r; }
__device__ __forceinline__ float lcp_clip0(float r) { return r < 0.0f ? 0.0f : r; }

// the tile's cells from its tail tables (row pitch W): lcp.py:88-100, corners
// v00, v00+1, v00+nx, v00+nx+1, np.prod's order.  clip(r, 0, 1): r <= 1 always
// (1 minus a sum of products of tails in [0, 1]; the erfc fit is relative, so
// no tail is ever below 0), so only the lower clip is evaluated; NaN passes
// through both ways like np.clip.  Bounds and addressing in 32-bit per tile.
template <typename T, int W, int TY = kLcpTY>
__device__ __forceinline__ void lcp_tile_cells(const T* below, const T* above, int64_t ci0, int64_t cj0,
                                               int64_t nx, int64_t ny, T* __restrict__ out) {
  // a thread walks RPT consecutive cell rows down one column pair: each corner
  // row is read once and serves the cells above and below it (6 + 2 (RPT - 1)
  // table reads per RPT cells instead of 8 per cell; lanes stay on consecutive
  // x, so the reads are conflict-free and the stores coalesced per row)
  static_assert(TY % kLcpBY == 0, "whole row runs per thread");
  constexpr int RPT = TY / kLcpBY;
  using A = Arith<T>;
  const int xl = int(min(nx - 1 - ci0, int64_t(kLcpTX))), yl = int(min(ny - 1 - cj0, int64_t(TY)));
  const int64_t ld = nx - 1;
  T* const o = out + cj0 * ld + ci0;
  const int y0 = threadIdx.y * RPT;
#pragma unroll
  for (int rx = 0; rx < kLcpTX; rx += kLcpBX) {
    const int x = threadIdx.x + rx;
    if (x >= xl) continue;
    const T* b = below + y0 * W + x;
    const T* a = above + y0 * W + x;
    T b0 = b[0], b1 = b[1], a0 = a[0], a1 = a[1];
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      if (y0 + r >= yl) break;
      const T c0 = b[(r + 1) * W], c1 = b[(r + 1) * W + 1];
      const T d0 = a[(r + 1) * W], d1 = a[(r + 1) * W + 1];
      const T pb = A::mul(A::mul(A::mul(b0, b1), c0), c1);
      const T pa = A::mul(A::mul(A::mul(a0, a1), d0), d1);
      o[int64_t(y0 + r) * ld + x] = lcp_clip0(A::sub(T(1), A::add(pb, pa)));
      b0 = c0; b1 = c1; a0 = d0; a1 = d1;
    }
  }
}
constexpr int kLcpV = (kLcpTX + 1) * (kLcpTY + 1);
constexpr int kLcpNQ = (kLcpV + kLcpBX * kLcpBY - 1) / (kLcpBX * kLcpBY);

template <typename T>
__global__ void __launch_bounds__(kLcpBX * kLcpBY, DIVUQ_LCP_MINB)
lcp2d_kernel(const T* __restrict__ mu, const T* __restrict__ sigma, int64_t nx, int64_t ny,
             T theta, T* __restrict__ out, int* err) {
  using A = Arith<T>;
  __shared__ T below[kLcpTY + 1][kLcpTX + 1];
  __shared__ T above[kLcpTY + 1][kLcpTX + 1];
  const int tid = threadIdx.y * kLcpBX + threadIdx.x;
  const int64_t ci0 = int64_t(blockIdx.x) * kLcpTX, cj0 = int64_t(blockIdx.y) * kLcpTY;
  int nonfinite = 0, negative = 0;   // validation flags (check_value / check_sigma)
  T* const bl = &below[0][0];
  T* const ab = &above[0][0];
  T mv[kLcpNQ], sv[kLcpNQ];
#pragma unroll
  for (int k = 0; k < kLcpNQ; ++k) {  // all loads first: kLcpNQ x 2 in flight per thread
    const int v = tid + k * kLcpBX * kLcpBY;
    const int vy = v / (kLcpTX + 1), vx = v % (kLcpTX + 1);
    const int64_t i = ci0 + vx, j = cj0 + vy;
    mv[k] = T(0);
    sv[k] = T(1);
    if (v < kLcpV && i < nx && j < ny) {
      mv[k] = mu[j * nx + i];
      sv[k] = sigma[j * nx + i];
    }
  }
  // park (mu, sigma) in the tile's own slots (flat slot v = vy*(TX+1) + vx), so
  // the tail pairs run as a rolled loop: the erfc / exp coefficients stay in
  // uniform registers across iterations instead of being reloaded per copy
#pragma unroll
  for (int k = 0; k < kLcpNQ; ++k) {
    const int v = tid + k * kLcpBX * kLcpBY;
    if (v < kLcpV) { bl[v] = mv[k]; ab[v] = sv[k]; }
  }
#pragma unroll 1
  for (int v = tid; v < kLcpV; v += kLcpBX * kLcpBY) {   // own slots only: no barrier needed
    const T m = bl[v], sg = ab[v];
    nonfinite |= int(!isfinite(m)) | int(!isfinite(sg));
    negative |= int(sg < T(0));
    tail_store_lcp(m, sg, theta, bl + v, ab + v);
  }
  const int errbits = (nonfinite ? kErrNonFinite : 0) | (negative ? kErrNegativeSigma : 0);
  __syncthreads();
  lcp_tile_cells<T, kLcpTX + 1>(&below[0][0], &above[0][0], ci0, cj0, nx, ny, out);
  flush_error(err, errbits);
}

// TMA variant (nx * sizeof(T) % 16 == 0): one thread stages the tile's
// (mu, sigma) boxes of 17 x (64 + 16 B) vertices straight into the two tables
// with cp.async.bulk.tensor (out-of-grid vertices arrive as 0, 0: a finite
// step-function tail pair in cells that are never written), so the per-vertex
// index arithmetic, bounds checks and parking of the register-loaded kernel
// disappear (~40 of its ~200 instructions per vertex); the tail-pair loop runs
// over every table slot without coordinates.  Same arithmetic as above.
template <typename T>
struct LcpTma {
  static constexpr int W = kLcpTX + 16 / int(sizeof(T));   // box width: 16-byte multiple
  static constexpr int H = kLcpTYT + 1;
};

template <typename T>
__global__ void __launch_bounds__(kLcpBX * kLcpBY, DIVUQ_LCP_MINB)
lcp2d_tma_kernel(const __grid_constant__ CUtensorMap map_mu, const __grid_constant__ CUtensorMap map_sg,
                 int64_t nx, int64_t ny, T theta, T* __restrict__ out, int* err) {
  using A = Arith<T>;
  using L = LcpTma<T>;
  __shared__ __align__(128) T below[L::H][L::W];
  __shared__ __align__(128) T above[L::H][L::W];
  __shared__ uint64_t bar;
  const int tid = threadIdx.y * kLcpBX + threadIdx.x;
  const int64_t ci0 = int64_t(blockIdx.x) * kLcpTX, cj0 = int64_t(blockIdx.y) * kLcpTYT;
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
    mbar_expect_tx(&bar, 2 * L::H * L::W * sizeof(T));
    tma_load_3d(&below[0][0], &map_mu, &bar, int(ci0), int(cj0), 0);
    tma_load_3d(&above[0][0], &map_sg, &bar, int(ci0), int(cj0), 0);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  int nonfinite = 0, negative = 0;   // validation flags (check_value / check_sigma)
  T* const bl = &below[0][0];
  T* const ab = &above[0][0];
#pragma unroll kLcpUnroll
  for (int v = tid; v < L::H * L::W; v += kLcpBX * kLcpBY) {   // own slots only: no barrier needed
    const T m = bl[v], sg = ab[v];
    nonfinite |= int(!isfinite(m)) | int(!isfinite(sg));
    negative |= int(sg < T(0));
    tail_store_lcp(m, sg, theta, bl + v, ab + v);
  }
  const int errbits = (nonfinite ? kErrNonFinite : 0) | (negative ? kErrNegativeSigma : 0);
  __syncthreads();
  lcp_tile_cells<T, L::W, kLcpTYT>(&below[0][0], &above[0][0], ci0, cj0, nx, ny, out);
  flush_error(err, errbits);
}

// Odd nx (fp64 rows not 16-byte aligned: no tiled tensor map): the same tile
// on 1D tensor maps over the flat arrays, one row box per vertex row.  A box
// must start on a 16-byte boundary, so row y's box starts one element early
// when its offset is odd and the row sits at shift sh(y) = ((cj0 + y) nx) & 1
// in its table row (cj0 + y parity for odd nx; ci0 is even).  Out-of-range
// parts arrive as 0; a row's last two table columns hold the next row's
// first values, read only by cells that are never written.
constexpr int kLcpFTY = 32;   // cell rows per CTA (2 x 33 x 640 B tables: static shared memory)
struct LcpFlat {
  static constexpr int W = kLcpTX + 2;    // vertices per row used (65) rounded to even
  static constexpr int BOX = W + 2;       // row box: + 1 element of start slack, even
  static constexpr int P = 80;            // table pitch (640 B: 128-byte aligned rows)
  static constexpr int H = kLcpFTY + 1;
};

__global__ void __launch_bounds__(kLcpBX * kLcpBY, DIVUQ_LCP_MINB)
lcp2d_flat_kernel(const __grid_constant__ CUtensorMap map_mu, const __grid_constant__ CUtensorMap map_sg,
                  int64_t nx, int64_t ny, double theta, double* __restrict__ out, int* err) {
  using A = Arith<double>;
  using L = LcpFlat;
  __shared__ __align__(128) double below[L::H][L::P];
  __shared__ __align__(128) double above[L::H][L::P];
  __shared__ uint64_t bar;
  const int tid = threadIdx.y * kLcpBX + threadIdx.x;
  const int64_t ci0 = int64_t(blockIdx.x) * kLcpTX, cj0 = int64_t(blockIdx.y) * kLcpFTY;
  const int odd = int(nx & 1);
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
    mbar_expect_tx(&bar, 2u * L::H * L::BOX * sizeof(double));
  }
  __syncthreads();
  if (tid == 0 || tid == 32) {   // two issuing threads: one 1D load every ~72 cycles each
    const CUtensorMap* map = tid == 0 ? &map_mu : &map_sg;
    double* tab = tid == 0 ? &below[0][0] : &above[0][0];
    for (int r = 0; r < L::H; ++r) {
      const int64_t off = (cj0 + r) * nx + ci0;
      tma_load_1d(tab + r * L::P, map, &bar, int(off & ~int64_t(1)));
    }
  }
  mbar_wait(&bar, 0);
  int nonfinite = 0, negative = 0;
  double* const bl = &below[0][0];
  double* const ab = &above[0][0];
#pragma unroll kLcpUnroll
  for (int v = tid; v < L::H * L::W; v += kLcpBX * kLcpBY) {
    const int y = v / L::W, x = v - y * L::W;
    const int idx = y * L::P + (odd & int(cj0 + y)) + x;
    const double m = bl[idx], sg = ab[idx];
    nonfinite |= int(!isfinite(m)) | int(!isfinite(sg));
    negative |= int(sg < 0.0);
    tail_store_lcp(m, sg, theta, bl + idx, ab + idx);
  }
  const int errbits = (nonfinite ? kErrNonFinite : 0) | (negative ? kErrNegativeSigma : 0);
  __syncthreads();
  const int xl = int(min(nx - 1 - ci0, int64_t(kLcpTX))), yl = int(min(ny - 1 - cj0, int64_t(kLcpFTY)));
  const int64_t ld = nx - 1;
  double* const o = out + cj0 * ld + ci0;
#pragma unroll
  for (int ry = 0; ry < kLcpFTY; ry += kLcpBY) {
#pragma unroll
    for (int rx = 0; rx < kLcpTX; rx += kLcpBX) {
      const int x = threadIdx.x + rx, y = threadIdx.y + ry;
      if (x < xl && y < yl) {
        const int r0 = y * L::P + (odd & int(cj0 + y)) + x;
        const int r1 = (y + 1) * L::P + (odd & int(cj0 + y + 1)) + x;
        // corners in lcp.py order: v00, v00+1, v00+nx, v00+nx+1
        const double pb = A::mul(A::mul(A::mul(bl[r0], bl[r0 + 1]), bl[r1]), bl[r1 + 1]);
        const double pa = A::mul(A::mul(A::mul(ab[r0], ab[r0 + 1]), ab[r1]), ab[r1 + 1]);
        o[int64_t(y) * ld + x] = lcp_clip0(A::sub(1.0, A::add(pb, pa)));
      }
    }
  }
  flush_error(err, errbits);
}

// stacked cells: mu4 / sigma4 are (n, 4) row-major, corners in order
template <typename T>
__global__ void cell_crossing_kernel(const T* __restrict__ mu4, const T* __restrict__ sigma4,
                                     int64_t n, T theta, T* __restrict__ out, int* err) {
  using A = Arith<T>;
  int errbits = 0;
  for (int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < n;
       c += int64_t(gridDim.x) * blockDim.x) {
    T pb = T(1), pa = T(1);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const T m = mu4[c * 4 + k], s = sigma4[c * 4 + k];
      errbits |= check_value(m) | check_sigma(s);
      T b, a;
      tail_pair_lcp(m, s, theta, b, a);
      pb = k == 0 ? b : A::mul(pb, b);
      pa = k == 0 ? a : A::mul(pa, a);
    }
    const T r = A::sub(T(1), A::add(pb, pa));
    out[c] = r < T(0) ? T(0) : (r > T(1) ? T(1) : r);
  }
  flush_error(err, errbits);
}

}  // namespace divuq

namespace divuq {

// ---------------------------------------------------------------------------
// propagate_divergence -> lcp fused ("fused into the K2
// epilogue"): the (u, v) moments of a tile's 65 x 17 vertices plus their
// stencil halo are TMA-staged, every vertex's divergence (mu, sigma) is
// evaluated with K2's arithmetic (StencilMath<double>: the reference order,
// stencils.py:64-84, IEEE sqrt -- bitwise equal to propagate_divergence),
// its tail pair with the LCP kernels' tail_pair_lcp, and the cells' crossing
// probability with lcp.py:71-100's corner order -- so the result is bitwise
// K2 followed by lcp2d_tma_kernel, without writing (mu, sigma) to HBM and
// reading them back unless the caller asks for them.
// Boxes (fp64, 16-byte aligned starts): u moments rows j0..j0+16, columns
// i0-2..i0+65 (68 wide); v moments rows j0-1..j0+17, columns i0..i0+65
// (66 wide).  Out-of-grid slots arrive as 0 and feed only vertices that are
// never written and cells that are never written.
// ---------------------------------------------------------------------------
// row-run epilogue (lcp_tile_cells): 16 rows 172.2 us, 24 rows aliased 167.7,
// 32 aliased 178.8 (4096^2; before it: 16 rows 180.4, 24 aliased 179.8)
#ifndef DIVUQ_LCPF_TY
#define DIVUQ_LCPF_TY 24
#endif
#ifndef DIVUQ_LCPF_ALIAS
#define DIVUQ_LCPF_ALIAS 1
#endif
constexpr int kLcpFY = DIVUQ_LCPF_TY;           // cell rows per CTA of the fused kernel
constexpr bool kLcpFAlias = DIVUQ_LCPF_ALIAS;   // tail tables over the u boxes (tails held in registers)
struct LcpFused {
  static constexpr int UW = kLcpTX + 4, UH = kLcpFY + 1;   // u box: x from i0 - 2
  static constexpr int VW = kLcpTX + 2, VH = kLcpFY + 3;   // v box: y from j0 - 1
  static constexpr int W = kLcpTX + 2, H = kLcpFY + 1;     // vertex / tail tables
  static constexpr int NV = (H * (kLcpTX + 1) + kLcpBX * kLcpBY - 1) / (kLcpBX * kLcpBY);
  static constexpr uint32_t kBytes = uint32_t(2 * UW * UH + 2 * VW * VH) * 8u;
  static_assert(H * W <= UH * UW, "a tail table fits in a u box");
};

struct LcpFusedSmem {
  alignas(128) double mu_u[LcpFused::UH][LcpFused::UW];
  alignas(128) double s_u[LcpFused::UH][LcpFused::UW];
  alignas(128) double mu_v[LcpFused::VH][LcpFused::VW];
  alignas(128) double s_v[LcpFused::VH][LcpFused::VW];
#if !DIVUQ_LCPF_ALIAS
  alignas(16) double below[LcpFused::H][LcpFused::W];
  alignas(16) double above[LcpFused::H][LcpFused::W];
#endif
  uint64_t bar;
};

struct LcpFusedParams {
  int64_t nx, ny;
  double cx_in, cx_bd, cy_in, cy_bd, theta;
  double *out_mu, *out_sigma, *out_lcp;
  int* err;
};

// vertices (x, y) of the tile, x in [0, 65), y in [0, 17): global (i0 + x,
// j0 + y) -> (mu, sigma) with K2's arithmetic -> tail pair into the tables
template <bool EDGE>
__device__ __forceinline__ int lcpf_vertices(LcpFusedSmem& s, const LcpFusedParams& p, int tid,
                                             int64_t i0, int64_t j0, double* tb, double* ta) {
  using A = Arith<double>;
  using F = LcpFused;
  using SM = StencilMath<double, false>;
  const int64_t nx = p.nx, ny = p.ny;
  int nonfinite = 0, negative = 0;
  double rb[kLcpFAlias ? F::NV : 1], ra[kLcpFAlias ? F::NV : 1];   // tails held until the boxes are free
#pragma unroll
  for (int k = 0; k < (kLcpFAlias ? F::NV : 1); ++k) { rb[k] = 0.0; ra[k] = 0.0; }
#pragma unroll (kLcpFAlias ? F::NV : 1)
  for (int k = 0; k < F::NV; ++k) {
    const int v = tid + k * kLcpBX * kLcpBY;
    if (v >= F::H * (kLcpTX + 1)) break;
    const int y = v / (kLcpTX + 1), x = v - y * (kLcpTX + 1);
    const int64_t i = i0 + x, j = j0 + y;
    if (EDGE && (i >= nx || j >= ny)) continue;
    // stencils.py:46-51: the point itself at the global faces, c = 1/h there
    const bool ilo = EDGE && i == 0, ihi = EDGE && i == nx - 1;
    const bool jlo = EDGE && j == 0, jhi = EDGE && j == ny - 1;
    const int ux = x + 2, vy = y + 1;            // this vertex in the u / v boxes
    const double cx = (ilo || ihi) ? p.cx_bd : p.cx_in;
    const double cy = (jlo || jhi) ? p.cy_bd : p.cy_in;
    const int xl = ilo ? ux : ux - 1, xh = ihi ? ux : ux + 1;
    const int yl = jlo ? vy : vy - 1, yh = jhi ? vy : vy + 1;
    const double m = SM::mean(s.mu_u[y][xh], s.mu_u[y][xl], s.mu_v[yh][x], s.mu_v[yl][x], 0.0, 0.0,
                              cx, cy, 0.0);
    const double var = SM::var(s.s_u[y][xh], s.s_u[y][xl], s.s_v[yh][x], s.s_v[yl][x], 0.0, 0.0,
                               cx, cy, 0.0);
    const double sg = A::sqrt_(var);
    // validation: every in-grid input point is some tile's vertex exactly once
    const bool owned = (x < kLcpTX || (EDGE && i == nx - 1)) && (y < kLcpFY || (EDGE && j == ny - 1));
    if (owned) {
      const double mu = s.mu_u[y][ux], mv = s.mu_v[vy][x], su = s.s_u[y][ux], sv = s.s_v[vy][x];
      nonfinite |= int(!isfinite(mu)) | int(!isfinite(mv)) | int(!isfinite(su)) | int(!isfinite(sv));
      negative |= int(su < 0.0) | int(sv < 0.0);
      if (p.out_mu || p.out_sigma) {
        const int64_t o = j * nx + i;
        if (p.out_mu) p.out_mu[o] = m;
        if (p.out_sigma) p.out_sigma[o] = sg;
      }
    }
    if constexpr (kLcpFAlias) {
      tail_pair_lcp(m, sg, p.theta, rb[k], ra[k]);
    } else {
      tail_store_lcp(m, sg, p.theta, tb + y * F::W + x, ta + y * F::W + x);
    }
  }
  if constexpr (kLcpFAlias) {
    __syncthreads();   // every box read is done: the tables take over the u boxes
#pragma unroll
    for (int k = 0; k < F::NV; ++k) {
      const int v = tid + k * kLcpBX * kLcpBY;
      if (v >= F::H * (kLcpTX + 1)) break;
      const int y = v / (kLcpTX + 1), x = v - y * (kLcpTX + 1);
      tb[y * F::W + x] = rb[k];
      ta[y * F::W + x] = ra[k];
    }
  }
  return (nonfinite ? kErrNonFinite : 0) | (negative ? kErrNegativeSigma : 0);
}

__global__ void __launch_bounds__(kLcpBX * kLcpBY)
lcp2d_fused_kernel(const __grid_constant__ CUtensorMap m_mu_u, const __grid_constant__ CUtensorMap m_s_u,
                   const __grid_constant__ CUtensorMap m_mu_v, const __grid_constant__ CUtensorMap m_s_v,
                   const LcpFusedParams p) {
  using A = Arith<double>;
  using F = LcpFused;
  using SM = StencilMath<double, false>;
  extern __shared__ __align__(128) unsigned char lf_smem[];
  LcpFusedSmem& s = *reinterpret_cast<LcpFusedSmem*>(lf_smem);
  const int tid = threadIdx.y * kLcpBX + threadIdx.x;
  const int64_t i0 = int64_t(blockIdx.x) * kLcpTX, j0 = int64_t(blockIdx.y) * kLcpFY;
  if (tid == 0) {
    mbar_init(&s.bar, 1);
    mbar_fence_init();
    mbar_expect_tx(&s.bar, F::kBytes);
    tma_load_3d(&s.mu_u[0][0], &m_mu_u, &s.bar, int(i0) - 2, int(j0), 0);
    tma_load_3d(&s.s_u[0][0], &m_s_u, &s.bar, int(i0) - 2, int(j0), 0);
    tma_load_3d(&s.mu_v[0][0], &m_mu_v, &s.bar, int(i0), int(j0) - 1, 0);
    tma_load_3d(&s.s_v[0][0], &m_s_v, &s.bar, int(i0), int(j0) - 1, 0);
  }
  __syncthreads();
  mbar_wait(&s.bar, 0);
  const int64_t nx = p.nx, ny = p.ny;
  // tiles clear of the global faces and of the grid's end take the path
  // without boundary logic (CTA-uniform branch; same arithmetic)
  const bool interior = i0 >= 1 && i0 + kLcpTX <= nx - 2 && j0 >= 1 && j0 + kLcpFY <= ny - 2;
#if DIVUQ_LCPF_ALIAS
  double* const tb = &s.mu_u[0][0];
  double* const ta = &s.s_u[0][0];
#else
  double* const tb = &s.below[0][0];
  double* const ta = &s.above[0][0];
#endif
  const int errbits = interior ? lcpf_vertices<false>(s, p, tid, i0, j0, tb, ta)
                               : lcpf_vertices<true>(s, p, tid, i0, j0, tb, ta);
  __syncthreads();
  lcp_tile_cells<double, F::W, kLcpFY>(tb, ta, i0, j0, nx, ny, p.out_lcp);
  flush_error(p.err, errbits);
}

}  // namespace divuq
