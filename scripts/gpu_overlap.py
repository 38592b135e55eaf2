"""Does a pinned H2D / D2H copy overlap our device-resident call? Debug aid."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2205_03133_b200 as P  # noqa: E402

B, W, H = 256, 640, 480
left, right = P.synth_batch(0, B, seed0=0)
dl, dr = torch.from_numpy(left).cuda(), torch.from_numpy(right).cuda()
dd = torch.empty((B, H, W), dtype=torch.float32, device="cuda")
hi = torch.empty(157286400, dtype=torch.uint8).pin_memory()
di = torch.empty_like(hi, device="cuda")
ho = torch.empty(314572800, dtype=torch.uint8).pin_memory()
do = torch.empty_like(ho, device="cuda")
m = P.Matcher(P.PipelineConfig.baseline(0), W, H, B)
sc, sx = torch.cuda.Stream(), torch.cuda.Stream()


def compute():
    m.run_device_u8(B, W, H, 1, dl.data_ptr(), dr.data_ptr(), {"disparity": dd.data_ptr()},
                    stream=sc.cuda_stream, invalid_value=float("nan"))


def h2d():
    with torch.cuda.stream(sx):
        di.copy_(hi, non_blocking=True)


def d2h():
    with torch.cuda.stream(sx):
        ho.copy_(do, non_blocking=True)


def timed(fns, reps=5):
    for f in fns:
        f()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        for f in fns:
            f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3


print("compute      %.2f ms" % timed([compute]))
print("h2d          %.2f ms" % timed([h2d]))
print("d2h          %.2f ms" % timed([d2h]))
print("compute+h2d  %.2f ms" % timed([compute, h2d]))
print("h2d+compute  %.2f ms" % timed([h2d, compute]))
print("compute+d2h  %.2f ms" % timed([compute, d2h]))
