import time, sys, torch
sys.path.insert(0, '.')
from paper_2510_01190_b200 import configs, _lib
lib = _lib.lib
n = 512
f = configs.config3_slab(0, n)
host_in = [x.cpu().pin_memory() for x in f]
host_out = [torch.empty(n ** 3, dtype=torch.float32).pin_memory() for _ in range(4)]
for chunk in (8, 16, 32, 64, 128):
    def call():
        st = lib.divuq_host_propagate3d_f32(*(t.data_ptr() for t in host_in), n, n, n, 1.0, 1.0, 1.0, 0.0,
                                            *(t.data_ptr() for t in host_out), chunk, 0)
        assert st == 0, st
    call()
    t0 = time.perf_counter()
    for _ in range(3):
        call()
    print(chunk, (time.perf_counter() - t0) / 3 * 1e3, "ms", flush=True)
