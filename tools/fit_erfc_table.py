"""Table-driven erfc(a)/2 for the LCP kernels (csrc/lcp.cuh, half_erfc_tab).

erfc(a)/2 on [0, 6.25) as 100 intervals of width 1/16, each a degree-9 Taylor
polynomial in d = a - c_j about its centre c_j = (j + 1/2)/16 (|d| <= 1/32):
t_0 = erfc(c)/2, t_k = f^(k)(c)/k! with f^(k)(a) = -(-1)^(k-1) H_(k-1)(a)
e^(-a^2) / sqrt(pi) (H = physicists' Hermite), computed in mpmath at 60
digits and rounded once to fp64.  The truncation bound (|d|^10/10! *
max|f^(10)|) is < 2e-18 absolute; the check below evaluates the fp64 Horner
form (numpy, the kernel's operation order) against mpmath on 200k points.

    python tools/fit_erfc_table.py            # prints the C table and the check
"""
import mpmath as mp
import numpy as np

mp.mp.dps = 60
NJ, DEG, STEP = 100, 9, mp.mpf(1) / 16


def coeffs(j):
    c = (j + mp.mpf(1) / 2) * STEP
    t = [mp.erfc(c) / 2]
    e = mp.e ** (-c * c) / mp.sqrt(mp.pi)
    for k in range(1, DEG + 1):
        t.append(-((-1) ** (k - 1)) * mp.hermite(k - 1, c) * e / mp.factorial(k))
    return [float(x) for x in t]


TAB = np.array([coeffs(j) for j in range(NJ)])


def half_erfc_tab(a):
    a = np.asarray(a, dtype=np.float64)
    j = np.clip(np.rint(a * 16.0 - 0.5), 0, NJ - 1).astype(np.int64)
    c = j * 0.0625 + 0.03125
    d = a - c
    t = TAB[j]
    p = t[:, DEG]
    for k in range(DEG - 1, -1, -1):
        p = p * d + t[:, k]      # the kernel fuses these (fma): at least as accurate
    return np.where(a > 6.2, 0.0, np.where(a == 0.0, 0.5, p))


if __name__ == "__main__":
    xs = np.concatenate([np.linspace(0, 6.2, 200001), np.random.default_rng(0).uniform(0, 6.2, 20000)])
    got = half_erfc_tab(xs)
    ref = np.array([float(mp.erfc(mp.mpf(x)) / 2) for x in xs[::10]])
    err = np.abs(got[::10] - ref)
    print(f"// max abs error {err.max():.3g}, max rel error {(err / ref).max():.3g} on [0, 6.2]")
    print(f"__constant__ double kErfcTab[{NJ}][{DEG + 1}] = {{")
    for j in range(NJ):
        print("    {" + ", ".join(float(v).hex() for v in TAB[j]) + "},")
    print("};")
