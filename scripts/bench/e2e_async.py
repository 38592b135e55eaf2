"""K back-to-back async e2e calls, wall time per call (bench-like). Debug aid."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2205_03133_b200 as P  # noqa: E402

B, W, H = 256, 640, 480
left, right = P.synth_batch(0, B, seed0=0)
hl = torch.from_numpy(left).pin_memory()
hr = torch.from_numpy(right).pin_memory()
hd = torch.empty((B, H, W), dtype=torch.float32).pin_memory()
m = P.Matcher(P.PipelineConfig.baseline(0), W, H, B)
s = torch.cuda.Stream()
print(f"host threads {P.lib().pstereo_gpu_host_threads()}", flush=True)
for K in ([int(v) for v in sys.argv[1].split(",")] if len(sys.argv) > 1 else (1, 2, 5, 10, 20)):
    for _ in range(2):
        m.run_host_u8(B, W, H, 1, hl.data_ptr(), hr.data_ptr(), {"disparity": hd.data_ptr()},
                      stream=s.cuda_stream, invalid_value=float("nan"), async_host=True)
    m.wait(s.cuda_stream)
    t0 = time.perf_counter()
    enq = []
    for _ in range(K):
        a = time.perf_counter()
        m.run_host_u8(B, W, H, 1, hl.data_ptr(), hr.data_ptr(), {"disparity": hd.data_ptr()},
                      stream=s.cuda_stream, invalid_value=float("nan"), async_host=True)
        enq.append(time.perf_counter() - a)
    m.wait(s.cuda_stream)
    dt = time.perf_counter() - t0
    busy, frames = P.host_expand_stats()
    print(f"K={K}: {dt / K * 1e3:.2f} ms/call, {B * K / dt:.0f} pairs/s, enqueue ms/call "
          f"{sum(enq) / K * 1e3:.2f} (max {max(enq) * 1e3:.2f}); replication total "
          f"{busy:.1f} worker-ms / {frames} frames", flush=True)
