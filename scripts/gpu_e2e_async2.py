"""bench-like sequence: device-path steps with profiling, then async e2e. Debug aid."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2205_03133_b200 as P  # noqa: E402

B, W, H = 256, 640, 480
left, right = P.synth_batch(0, B, seed0=0)
dl, dr = torch.from_numpy(left).cuda(), torch.from_numpy(right).cuda()
disp = torch.empty((B, H, W), dtype=torch.float32, device="cuda")
hl = torch.from_numpy(left).pin_memory()
hr = torch.from_numpy(right).pin_memory()
hd = torch.empty((B, H, W), dtype=torch.float32).pin_memory()
m = P.Matcher(P.PipelineConfig.baseline(0), W, H, B)
s = torch.cuda.Stream()
mode = sys.argv[1] if len(sys.argv) > 1 else "full"
if mode in ("full", "noprof"):
    for _ in range(3):
        m.run_device_u8(B, W, H, 1, dl.data_ptr(), dr.data_ptr(), {"disparity": disp.data_ptr()},
                        stream=s.cuda_stream, invalid_value=float("nan"))
    torch.cuda.synchronize()
    if mode == "full":
        m.set_profiling(True)
    for _ in range(10):
        m.run_device_u8(B, W, H, 1, dl.data_ptr(), dr.data_ptr(), {"disparity": disp.data_ptr()},
                        stream=s.cuda_stream, invalid_value=float("nan"))
    torch.cuda.synchronize()
    if mode == "full":
        m.stage_times()
        m.set_profiling(False)


def e2e():
    m.run_host_u8(B, W, H, 1, hl.data_ptr(), hr.data_ptr(), {"disparity": hd.data_ptr()},
                  stream=s.cuda_stream, invalid_value=float("nan"), async_host=True)


for _ in range(2):
    e2e()
m.wait(s.cuda_stream)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    e2e()
m.wait(s.cuda_stream)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"{mode}: {dt / 10 * 1e3:.2f} ms/call, {B * 10 / dt:.0f} pairs/s", flush=True)
