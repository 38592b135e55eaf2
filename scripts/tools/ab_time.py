"""A/B timing of alternative builds of the product library (development tool).

  PSTEREO_GPU_LIB=/path/to/variant.so python scripts/dev/ab_time.py [workload]

Times the bench step (device-resident inputs, disparity-only output) and the
per-stage device times, and prints a digest of every output plane (F64) so
two variants can be checked for identical results.
"""
import hashlib
import json
import os
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2205_03133_b200 as P  # noqa: E402

wl = bench.workload(sys.argv[1] if len(sys.argv) > 1 else "c2")
W, H, CH, B = wl["W"], wl["H"], wl["C"], wl["batch"]
cfg = P.PipelineConfig(**wl["params"])
dl, dr = P.synth_batch_gpu(wl["gen"], B, seed0=0, **wl["over"])
disp = torch.empty((B, H, W), dtype=torch.float32, device="cuda")
m = P.Matcher(cfg, W, H, B, device=0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
sh = stream.cuda_stream


def step():
    m.run_device_u8(B, W, H, CH, dl.data_ptr(), dr.data_ptr(), {"disparity": disp.data_ptr()},
                    stream=sh, invalid_value=float("nan"))


for _ in range(3):
    step()
torch.cuda.synchronize()
steps = int(os.environ.get("AB_STEPS", "20"))
best = None
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    best = ms if best is None else min(best, ms)
m.set_device_chunks(1)
step()
torch.cuda.synchronize()
m.set_profiling(True)
for _ in range(5):
    step()
torch.cuda.synchronize()
stages, calls = m.stage_times()
m.set_profiling(False)
m.set_device_chunks(2)
full = {k: torch.empty((B, H, W), dtype=torch.float64 if k not in ("disparity_valid", "depth_valid")
                       else torch.uint8, device="cuda")
        for k in ("disparity", "disparity_valid", "probability", "depth", "depth_valid")}
m.run_device_u8(B, W, H, CH, dl.data_ptr(), dr.data_ptr(), {k: v.data_ptr() for k, v in full.items()},
                stream=sh, focal=500.0, baseline=5.0, dtype=P.F64)
torch.cuda.synchronize()
h = hashlib.sha256()
for k in sorted(full):
    h.update(full[k].cpu().numpy().tobytes())
print(json.dumps({"lib": os.environ.get("PSTEREO_GPU_LIB", "default"), "workload": wl["name"],
                  "ms_per_step": best, "pairs_s": B / best * 1e3,
                  "stage_ms": {k: v / calls for k, v in stages.items()},
                  "digest": h.hexdigest()[:16]}), flush=True)
