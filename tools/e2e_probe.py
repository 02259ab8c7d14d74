"""PCIe probe for the e2e leg: pinned H2D of 1.61 GB, D2H of 1.07 GB, both concurrently, in 16 slabs."""
import time
import torch
n = 512 ** 3
f_h = torch.empty(n, dtype=torch.float32, pin_memory=True)
fh_h = torch.empty(n, dtype=torch.float64, pin_memory=True)
g_h = torch.empty(n, dtype=torch.float64, pin_memory=True)
f_d = torch.empty(n, dtype=torch.float32, device="cuda")
fh_d = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def h2d():
    with torch.cuda.stream(s1):
        for c in range(16):
            a, b = n * c // 16, n * (c + 1) // 16
            f_d[a:b].copy_(f_h[a:b], non_blocking=True)
            fh_d[a:b].copy_(fh_h[a:b], non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        for c in range(16):
            a, b = n * c // 16, n * (c + 1) // 16
            g_h[a:b].copy_(fh_d[a:b], non_blocking=True)


for label, fns in (("H2D 1.61 GB", [h2d]), ("D2H 1.07 GB", [d2h]), ("both concurrently", [h2d, d2h])):
    for _ in range(2):
        for fn in fns:
            fn()
        torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        for fn in fns:
            fn()
        torch.cuda.synchronize()
    print(f"{label:20s} {(time.perf_counter() - t0) / 5 * 1e3:7.2f} ms", flush=True)
