"""Per-call host cost of the device API pieces at 128^2 (wall clock, 2000
calls each): torch stream query, argument checks, output allocation, the
ctypes call itself, and the whole dev.propagate2d."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2510_01190_b200 import device as dev  # noqa: E402
from paper_2510_01190_b200._lib import lib  # noqa: E402

nx = ny = 128
n = nx * ny
g = [torch.randn(n, device="cuda", dtype=torch.float64) for _ in range(2)] + \
    [torch.rand(n, device="cuda", dtype=torch.float64) for _ in range(2)]
err = torch.zeros(1, dtype=torch.int32, device="cuda")
outs = {k: torch.empty(n, device="cuda", dtype=torch.float64) for k in dev.ALL_OUTPUTS}
s = torch.cuda.current_stream().cuda_stream
ptrs = [t.data_ptr() for t in g] + [outs[k].data_ptr() for k in dev.ALL_OUTPUTS]


def t(label, fn, k=2000):
    for _ in range(100):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        fn()
    torch.cuda.synchronize()
    print(f"{label:48s} {(time.perf_counter() - t0) / k * 1e6:7.2f} us")


t("torch.cuda.current_stream().cuda_stream", lambda: torch.cuda.current_stream().cuda_stream)
t("dev._stream() (raw getter)", dev._stream)
t("_req x4", lambda: [dev._req(x, "x", torch.float64, n) for x in g])
t("_outs (given)", lambda: dev._outs(g[0], n, dev.ALL_OUTPUTS, outs))
t("_outs (fresh)", lambda: dev._outs(g[0], n, dev.ALL_OUTPUTS, None))
t("data_ptr x8", lambda: [x.data_ptr() for x in g + list(outs.values())])
t("ctypes launch only", lambda: lib.divuq_propagate2d_f64(*ptrs[:4], nx, ny, 1.0, 1.0, 0.0, *ptrs[4:],
                                                          err.data_ptr(), s))
t("dev.propagate2d out= check=word", lambda: dev.propagate2d(*g, nx, ny, 1.0, 1.0, 0.0, check=err, out=outs))
t("dev.propagate2d fresh check=word", lambda: dev.propagate2d(*g, nx, ny, 1.0, 1.0, 0.0, check=err))
t("dev.propagate2d fresh check=True", lambda: dev.propagate2d(*g, nx, ny, 1.0, 1.0, 0.0), k=500)
