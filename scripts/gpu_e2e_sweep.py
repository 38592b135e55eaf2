"""e2e (pinned host in/out) time per 256-pair call vs chunk size. Debug aid."""
import os
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
cfg = P.PipelineConfig.baseline(0)
for chunk in [int(c) for c in sys.argv[1:]] or [16, 32, 64]:
    os.environ["PSTEREO_CHUNK_PAIRS"] = str(chunk)
    m = P.Matcher(cfg, W, H, B)
    s = torch.cuda.Stream()
    for _ in range(2):
        m.run_host_u8(B, W, H, 1, hl.data_ptr(), hr.data_ptr(), {"disparity": hd.data_ptr()},
                      stream=s.cuda_stream, invalid_value=float("nan"))
    torch.cuda.synchronize()
    t = time.perf_counter()
    reps = 5
    for _ in range(reps):
        m.run_host_u8(B, W, H, 1, hl.data_ptr(), hr.data_ptr(), {"disparity": hd.data_ptr()},
                      stream=s.cuda_stream, invalid_value=float("nan"))
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / reps
    print(f"chunk {chunk}: {dt * 1e3:.2f} ms/call  {B / dt:.0f} pairs/s")
    m.close()
