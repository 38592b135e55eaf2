"""Host<->device copy ceilings on this box (pinned memory, torch streams):
H2D alone, D2H alone, both directions concurrently, at the bench's per-step
byte counts. Debug aid for the e2e number."""
import time

import torch

H2D, D2H = 157286400, 314572800
dev = torch.device("cuda", 0)
hi = torch.empty(H2D, dtype=torch.uint8).pin_memory()
ho = torch.empty(D2H, dtype=torch.uint8).pin_memory()
di = torch.empty(H2D, dtype=torch.uint8, device=dev)
do = torch.empty(D2H, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


def h2d():
    with torch.cuda.stream(s1):
        di.copy_(hi, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        ho.copy_(do, non_blocking=True)


def both():
    h2d()
    d2h()


for name, fn, b in (("h2d", h2d, H2D), ("d2h", d2h, D2H), ("both", both, H2D + D2H)):
    t = timed(fn)
    print(f"{name}: {t * 1e3:.2f} ms  {b / t / 1e9:.1f} GB/s")
