"""H2D bandwidth probe: pinned vs pageable, whole vs chunked (e2e planning)."""
import time
import numpy as np
import torch

n = 10000
nbytes = n * n * 8
dev = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
pin = torch.empty(nbytes // 8, dtype=torch.float64).pin_memory()
pin.fill_(1.0)
pag = np.ones(nbytes // 8)
pag_t = torch.from_numpy(pag)
s = torch.cuda.Stream()


def t(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


r = {}
r["pinned_whole"] = t(lambda: dev.copy_(pin, non_blocking=True))
r["pageable_whole"] = t(lambda: dev.copy_(pag_t))
for ch in (8, 32, 128):
    sz = nbytes // 8 // ch
    def f():
        with torch.cuda.stream(s):
            for k in range(ch):
                dev[k * sz:(k + 1) * sz].copy_(pin[k * sz:(k + 1) * sz], non_blocking=True)
    r[f"pinned_chunks{ch}"] = t(f)
for k, v in r.items():
    print(f"{k:20s} {v*1e3:8.2f} ms  {nbytes / v / 1e9:7.1f} GB/s")
