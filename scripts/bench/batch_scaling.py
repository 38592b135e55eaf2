"""Device-resident call time vs batch size (launch / tail overheads). Debug aid."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2205_03133_b200 as P  # noqa: E402

W, H = 640, 480
left, right = P.synth_batch(0, 256, seed0=0)
dl, dr = torch.from_numpy(left).cuda(), torch.from_numpy(right).cuda()
dd = torch.empty((256, H, W), dtype=torch.float32, device="cuda")
m = P.Matcher(P.PipelineConfig.baseline(0), W, H, 256)
s = torch.cuda.Stream()
for B in (1, 2, 4, 8, 16, 32, 64, 128, 256):
    def call():
        m.run_device_u8(B, W, H, 1, dl.data_ptr(), dr.data_ptr(), {"disparity": dd.data_ptr()},
                        stream=s.cuda_stream, invalid_value=float("nan"))
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    reps = max(3, 256 // B)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.perf_counter()
    e0.record(s)
    for _ in range(reps):
        call()
    e1.record(s)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t) / reps * 1e3
    gpu = e0.elapsed_time(e1) / reps
    print(f"B={B:4d}: gpu {gpu:.3f} ms/call ({B / gpu * 1e3:.0f} pairs/s), wall {wall:.3f} ms/call")
