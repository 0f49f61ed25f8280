"""Philox4x32-10 + Box-Muller stream and the MC estimator -- TEST INFRASTRUCTURE ONLY.

The north star (BASELINE.json) mandates a counter-based Philox RNG with
Box-Muller sampling for the GPU Monte Carlo kernel, replacing the reference's
splitmix64 + AS241 stream (rng.py:23-92).  The *semantics* of the reference
stream are kept: every draw is a pure function of
(seed, sample, component, vertex), one shared field per sample (mc.py:80-91),
so any partitioning of the work gives identical draws.

Stream contract (mirrored by csrc/mc.cu):
    key     = (seed & 0xffffffff, seed >> 32)
    counter = (vertex & 0xffffffff, vertex >> 32, sample & 0xffffffff, sample >> 32)
    r0..r3  = Philox4x32-10(counter, key)           # Salmon et al., SC'11
    U1      = (r1 << 32 | r0) >> 12                  # top 52 bits
    u1      = 2 - (1 + U1 * 2^-52)                    # in (0, 1]   (exact)
    u2      = (1 + ((r3 << 32 | r2) >> 12) * 2^-52) - 1   # in [0, 1)   (exact)
    rad     = sqrt(-2 ln u1)
    z_u     = rad * cos(2 pi u2);  z_v = rad * sin(2 pi u2)

Estimator contract (mirrors the reference's Welford in strict sample order,
mc.py:106-117, but over fixed chunks of CHUNK samples so the GPU can spread the
sample axis over thread blocks):
    chunk r = samples [r*CHUNK, min(n, (r+1)*CHUNK)), Welford in sample order
    with mean += delta * (1/count);
    slot l (0..min(chunks, 32)-1) left-folds chunks l, l+32, ... with Chan's
    merge (with fewer than 32 chunks every slot holds one chunk), then a
    fixed shuffle tree (offsets 16, 8, 4, 2, 1) merges the 32 lanes;
    std = sqrt(M2 / (n - 1)).
The chunking depends on n only, so results are invariant to launch shape and
GPU count.  The GPU evaluates log (table + log1p series, <= 1.6 ulp), sqrt and
sin/cos(2 pi u) (quadrant reduction + Taylor, more accurate than numpy's
cos(2*pi*u)) with its own in-range routines and fuses the draw mu + sigma*z and
the Welford updates into fmas, so GPU-vs-oracle agreement is tolerance-based
(tests state it); the Philox words and the uniforms are bit-exact, and
sigma = 0 still reproduces the deterministic divergence exactly.
"""

from __future__ import annotations

import numpy as np

from .ref2d import divergence2d

M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
W0, W1 = np.uint32(0x9E3779B9), np.uint32(0xBB67AE85)
CHUNK = 128
_MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32 with 10 rounds; all inputs uint32 arrays/scalars."""
    c0, c1, c2, c3 = (np.asarray(c, dtype=np.uint32) for c in (c0, c1, c2, c3))
    k0 = np.asarray(k0, dtype=np.uint32)
    k1 = np.asarray(k1, dtype=np.uint32)
    for r in range(10):
        if r:
            k0 = ((k0.astype(np.uint64) + np.uint64(W0)) & _MASK32).astype(np.uint32)
            k1 = ((k1.astype(np.uint64) + np.uint64(W1)) & _MASK32).astype(np.uint32)
        p0 = M0 * c0.astype(np.uint64)
        p1 = M1 * c2.astype(np.uint64)
        hi0 = (p0 >> np.uint64(32)).astype(np.uint32)
        lo0 = (p0 & _MASK32).astype(np.uint32)
        hi1 = (p1 >> np.uint64(32)).astype(np.uint32)
        lo1 = (p1 & _MASK32).astype(np.uint32)
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return c0, c1, c2, c3


def _one_plus_u52(lo, hi):
    """1 + (top 52 bits of hi:lo) * 2^-52 in [1, 2): the GPU builds this double
    from the bits directly (csrc/mc.cuh one_plus_u52)."""
    x = (hi.astype(np.uint64) << np.uint64(32)) | lo.astype(np.uint64)
    return 1.0 + (x >> np.uint64(12)).astype(np.float64) * (2.0**-52)


def uniforms(seed: int, vertex, sample):
    """(u1, u2) for the given vertex/sample counters (broadcasting)."""
    vertex = np.asarray(vertex, dtype=np.uint64)
    sample = np.asarray(sample, dtype=np.uint64)
    vertex, sample = np.broadcast_arrays(vertex, sample)
    r0, r1, r2, r3 = philox4x32_10(
        (vertex & _MASK32).astype(np.uint32),
        (vertex >> np.uint64(32)).astype(np.uint32),
        (sample & _MASK32).astype(np.uint32),
        (sample >> np.uint64(32)).astype(np.uint32),
        np.uint32(seed & 0xFFFFFFFF),
        np.uint32((seed >> 32) & 0xFFFFFFFF),
    )
    return 2.0 - _one_plus_u52(r0, r1), _one_plus_u52(r2, r3) - 1.0


def normals(seed: int, vertex, sample):
    """(z_u, z_v) Box-Muller pair for the given vertex/sample counters."""
    u1, u2 = uniforms(seed, vertex, sample)
    rad = np.sqrt(-2.0 * np.log(u1))
    ang = 2.0 * np.pi * u2
    return rad * np.cos(ang), rad * np.sin(ang)


def _chan(a, b):
    na, ma, qa = a
    nb, mb, qb = b
    n = na + nb
    safe = np.where(n > 0, n, 1.0)
    d = mb - ma
    mean = ma + d * (nb / safe)
    q = qa + qb + d * d * (na * nb / safe)
    mean = np.where(nb == 0, ma, np.where(na == 0, mb, mean))
    q = np.where(nb == 0, qa, np.where(na == 0, qb, q))
    return n, mean, q


def mc_divergence(mu_u, mu_v, s_u, s_v, nx, ny, dx, dy, n_samples, seed, batch=64):
    """(mean, std) per vertex with the GPU's stream and merge order."""
    if n_samples < 2:
        raise ValueError("mc_divergence needs n_samples >= 2")
    n = nx * ny
    vertex = np.arange(n, dtype=np.uint64)
    n_chunks = -(-n_samples // CHUNK)
    parts = []
    for r in range(n_chunks):
        s0, s1 = r * CHUNK, min(n_samples, (r + 1) * CHUNK)
        cnt, mean, m2 = 0, np.zeros(n), np.zeros(n)
        for b0 in range(s0, s1, batch):
            b1 = min(s1, b0 + batch)
            smp = np.arange(b0, b1, dtype=np.uint64)[:, None]
            zu, zv = normals(seed, vertex[None, :], smp)
            u = mu_u + s_u * zu
            v = mu_v + s_v * zv
            div = divergence2d(u, v, nx, ny, dx, dy)
            for row in div:
                cnt += 1
                delta = row - mean
                mean = mean + delta * (1.0 / cnt)
                m2 = m2 + delta * (row - mean)
        parts.append((np.full(n, float(cnt)), mean, m2))
    lanes = []
    for lane in range(32):
        st = (np.zeros(n), np.zeros(n), np.zeros(n))
        for r in range(lane, n_chunks, 32):
            st = _chan(st, parts[r])
        lanes.append(st)
    off = 16
    while off:
        for lane in range(off):
            lanes[lane] = _chan(lanes[lane], lanes[lane + off])
        off //= 2
    cnt, mean, m2 = lanes[0]
    return mean, np.sqrt(m2 / (n_samples - 1))
