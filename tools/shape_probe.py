"""Time propagate3d / ensemble_divergence2d on shapes the TMA kernels do not
take (nx % 4 != 0) next to aligned ones: the fallback paths' HBM fraction."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2510_01190_b200 import device as dev  # noqa: E402

PEAK = json.load(open("MEASURED_PEAKS.json")).get("hbm_gbs", 6534.5) if os.path.exists("MEASURED_PEAKS.json") else 6534.5


ERR = None  # set below: a device validation word, as bench.py (no per-call read-back)


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


ERR = torch.zeros(1, dtype=torch.int32, device="cuda")
for nx in (512, 510, 511):
    ny, nz = 512, 512
    n = nx * ny * nz
    f = [torch.randn(n, device="cuda") for _ in range(3)] + [torch.rand(n, device="cuda") * 0.3 + 0.05 for _ in range(3)]
    out = {k: torch.empty(n, device="cuda") for k in dev.ALL_OUTPUTS}
    ms = timeit(lambda: dev.propagate3d(*f, nx, ny, nz, 1.0, 1.0, 1.0, 0.0, out=out, check=ERR))
    print(f"propagate3d fp32 {nx}x{ny}x{nz}: {ms:.3f} ms, {40 * n / ms / 1e6 / PEAK * 100:.1f} % HBM")
    del f, out
for nx in (1024, 1022, 1023):
    ny, m = 1024, 20
    mem = torch.randn(m, 2, nx * ny, device="cuda")
    ms = timeit(lambda: dev.ensemble_divergence2d(mem, nx, ny, 1.0, 1.0, 0.0, check=ERR))
    print(f"ensemble_divergence2d M=20 {nx}x{ny}: {ms * 1e3:.1f} us, {(160 + 16) * nx * ny / ms / 1e6 / PEAK * 100:.1f} % HBM")
for nx in (1024, 1023):
    ny, m = 1024, 20
    mem = torch.randn(m, 2, nx * ny, device="cuda")
    ms = timeit(lambda: dev.gradient_ensemble_divergence2d(mem, nx, ny, 1.0, 1.0, 0.0, check=ERR))
    print(f"gradient_ensemble_divergence2d (K6) M=20 {nx}x{ny}: {ms * 1e3:.1f} us, {(160 + 16) * nx * ny / ms / 1e6 / PEAK * 100:.1f} % HBM")
for nx in (4096, 4095):
    ny = 4096
    mu, sg = torch.randn(nx * ny, device="cuda", dtype=torch.float64), torch.rand(nx * ny, device="cuda", dtype=torch.float64)
    ms = timeit(lambda: dev.lcp2d(mu, sg, nx, ny, 0.0, check=ERR))
    print(f"lcp2d fp64 {nx}x{ny}: {ms * 1e3:.1f} us, {24 * (nx - 1) * (ny - 1) / ms / 1e6 / PEAK * 100:.1f} % HBM")
for nx in (512, 511):
    ny, nz, m = 128, 64, 16
    mem = torch.randn(m, 3, nx * ny * nz, device="cuda")
    ms = timeit(lambda: dev.ensemble_divergence3d(mem, nx, ny, nz, 1.0, 1.0, 1.0, 0.1, check=ERR))
    print(f"ensemble_divergence3d M=16 {nx}x{ny}x{nz}: {ms * 1e3:.1f} us, {(192 + 16) * nx * ny * nz / ms / 1e6 / PEAK * 100:.1f} % HBM")
for nx in (128, 127):
    ny, nz = 128, 1024
    n = nx * ny * nz
    f = [torch.randn(n, device="cuda") for _ in range(3)] + [torch.rand(n, device="cuda") * 0.3 + 0.05 for _ in range(3)]
    out = {k: torch.empty(n, device="cuda") for k in dev.ALL_OUTPUTS}
    ms = timeit(lambda: dev.propagate3d(*f, nx, ny, nz, 1.0, 1.0, 1.0, 0.0, out=out, check=ERR))
    print(f"propagate3d fp32 small planes {nx}x{ny}x{nz}: {ms * 1e3:.1f} us, {40 * n / ms / 1e6 / PEAK * 100:.1f} % HBM")
for nx, ny, nz in ((256, 256, 512), (256, 200, 300), (512, 512, 512)):
    n = nx * ny * nz
    f = [torch.randn(n, device="cuda") for _ in range(3)] + [torch.rand(n, device="cuda") * 0.3 + 0.05 for _ in range(3)]
    out = {k: torch.empty(n, device="cuda") for k in dev.ALL_OUTPUTS}
    ms = timeit(lambda: dev.propagate3d(*f, nx, ny, nz, 1.0, 1.0, 1.0, 0.0, out=out, check=ERR))
    print(f"propagate3d fp32 {nx}x{ny}x{nz}: {ms * 1e3:.1f} us, {40 * n / ms / 1e6 / PEAK * 100:.1f} % HBM")
