"""BASELINE.json config 4 sweep on one B200: RGB inputs from the device
generator; resolutions 320x240 .. 1920x1080 at s=8 stride 4, and every
(patch size, stride) in {8,12,16} x {2,4,6} at 640x480; batch 1 (latency,
ms per call) and batch 1024 (throughput, pairs/s), device-resident, CUDA events.
Reference: run_pipeline on one host core for one pair of each case.
Prints one JSON line per case."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2205_03133_b200 as P  # noqa: E402
from oracle import pyoracle  # noqa: E402

orc = pyoracle.load("reference" if pyoracle.available("reference") else "port")


def exps_for(w, h, s):
    # deepest pyramid the sizes allow, at most 4 levels below full resolution,
    # finest 2^1 (the BASELINE reading of "3-scale" / "4 scales")
    ce = 1
    while ce < 4 and min(w >> (ce + 1), h >> (ce + 1)) >= 2 * s:
        ce += 1
    return ce


def case(w, h, s, stride, ref_pairs=1):
    ce = exps_for(w, h, s)
    cfg = P.PipelineConfig(coarsest_exp=ce, finest_exp=1, patch_size=s, overlap=1 - stride / s)
    out = {"size": f"{w}x{h}", "channels": 3, "patch": s, "stride": stride,
           "exps": f"{ce}..1"}
    for B in (1, 1024):
        dl, dr = P.synth_batch_gpu(4, B, seed0=0, width=w, height=h, channels=3)
        disp = torch.empty((B, h, w), dtype=torch.float32, device="cuda")
        st = torch.cuda.Stream()
        with P.Matcher(cfg, w, h, B) as m:
            def step():
                m.run_device_u8(B, w, h, 3, dl.data_ptr(), dr.data_ptr(),
                                {"disparity": disp.data_ptr()}, stream=st.cuda_stream,
                                invalid_value=float("nan"))
            for _ in range(3):
                step()
            torch.cuda.synchronize()
            reps = 20 if B == 1 else 3
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(reps):
                step()
            e1.record(st)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
        if B == 1:
            out["latency_ms_b1"] = round(ms, 4)
            l, r = dl[0].cpu().numpy(), dr[0].cpu().numpy()
        else:
            out["pairs_s_b1024"] = round(B / (ms / 1e3), 1)
        del dl, dr, disp
        torch.cuda.empty_cache()
    ocfg = pyoracle.Config(coarsest_exp=ce, finest_exp=1, patch_size=s, overlap=1 - stride / s)
    lf, _ = orc.to_grayscale(l)
    rf, _ = orc.to_grayscale(r)
    out["ref_ms_1core"] = round(orc.run_pipeline(lf, rf, ocfg, 500.0, 5.0)["runtime_ms"], 2)
    print(json.dumps(out), flush=True)


for w, h in ((320, 240), (640, 480), (1280, 1024), (1920, 1080)):
    case(w, h, 8, 4)
for s in (8, 12, 16):
    for stride in (2, 4, 6):
        if (s, stride) != (8, 4):
            case(640, 480, s, stride)
