import numpy as np, time, threading, torch
n = 32 << 20  # 32 MB
src = np.ones(n // 8); 
pin = torch.empty(n // 8, dtype=torch.float64).pin_memory().numpy()
dst = np.ones(n // 8)
def run(nt, d):
    per = len(src) // nt
    def w(i): np.copyto(d[i*per:(i+1)*per], src[i*per:(i+1)*per])
    ts = [threading.Thread(target=w, args=(i,)) for i in range(nt)]
    t0 = time.perf_counter(); [t.start() for t in ts]; [t.join() for t in ts]
    return n / (time.perf_counter() - t0) / 1e9
for nt in (1, 2, 4, 8, 16):
    b1 = max(run(nt, pin) for _ in range(5)); b2 = max(run(nt, dst) for _ in range(5))
    print(f"{nt:2d} threads: -> pinned {b1:5.1f} GB/s, -> pageable {b2:5.1f} GB/s")
