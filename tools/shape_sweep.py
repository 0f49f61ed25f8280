"""HBM fraction of the device entry points over a spread of shapes (not only
the BASELINE configs): finds shapes a kernel's work decomposition handles
badly.  python tools/shape_sweep.py"""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_01190_b200 import device as dev  # noqa: E402

PEAK = json.load(open("MEASURED_PEAKS.json")).get("hbm_gbs", 6534.5) if os.path.exists("MEASURED_PEAKS.json") else 6534.5
ERR = torch.zeros(1, dtype=torch.int32, device="cuda")


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


def line(name, ms, nbytes):
    print(f"{name:58s} {ms * 1e3:9.1f} us  {nbytes / ms / 1e6 / PEAK * 100:5.1f} % HBM")


def main():
    for nx, ny in ((512, 512), (1024, 1024), (2048, 2048), (4096, 1024), (1000, 700), (256, 4096)):
        m = 20
        mem = torch.randn(m, 2, nx * ny, device="cuda")
        line(f"ensemble_divergence2d M=20 {nx}x{ny}", timeit(lambda: dev.ensemble_divergence2d(mem, nx, ny, 1.0, 1.0, 0.0, check=ERR)), (160 + 16) * nx * ny)
        line(f"gradient_ensemble_divergence2d M=20 {nx}x{ny}", timeit(lambda: dev.gradient_ensemble_divergence2d(mem, nx, ny, 1.0, 1.0, 0.0, check=ERR)), (160 + 16) * nx * ny)
        memd = mem.double()
        out = torch.empty(2, 2, nx * ny, device="cuda", dtype=torch.float64)
        line(f"fit_moments fp64 M=20 {nx}x{ny}", timeit(lambda: dev.fit_moments(memd, check=ERR)), (320 + 32) * nx * ny)
        mu, sg = torch.randn(nx * ny, device="cuda", dtype=torch.float64), torch.rand(nx * ny, device="cuda", dtype=torch.float64)
        line(f"lcp2d fp64 {nx}x{ny}", timeit(lambda: dev.lcp2d(mu, sg, nx, ny, 0.0, check=ERR)), 24 * (nx - 1) * (ny - 1))
        g = [torch.randn(nx * ny, device="cuda", dtype=torch.float64) for _ in range(2)] + [torch.rand(nx * ny, device="cuda", dtype=torch.float64) for _ in range(2)]
        line(f"propagate2d fp64 {nx}x{ny}", timeit(lambda: dev.propagate2d(*g, nx, ny, 1.0, 1.0, 0.0, check=ERR)), 64 * nx * ny)
        del mem, memd, out
    for nx, ny, nz, m in ((1024, 1024, 64, 16), (512, 512, 128, 16), (256, 256, 256, 8), (1024, 256, 128, 16)):
        mem = torch.randn(m, 3, nx * ny * nz, device="cuda")
        line(f"ensemble_divergence3d M={m} {nx}x{ny}x{nz}", timeit(lambda: dev.ensemble_divergence3d(mem, nx, ny, nz, 1.0, 1.0, 1.0, 0.1, check=ERR)), (12 * m + 16) * nx * ny * nz)
        del mem


if __name__ == "__main__":
    main()
