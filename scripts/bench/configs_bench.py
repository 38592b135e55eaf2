"""Device-resident throughput for the other BASELINE.json configurations
(one GPU), beside the reference on one host core for the same pairs.
Prints one JSON line per configuration."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2205_03133_b200 as P  # noqa: E402
from oracle import pyoracle  # noqa: E402

CASES = [
    # name, synth config, overrides, batch, PipelineConfig
    ("c1 640x480 variance+stress", 1, {}, 256, P.PipelineConfig.baseline(1)),
    ("c3 1280x1024 s12 4 levels variance", 3, {}, 32, P.PipelineConfig.baseline(3)),
    ("c4 320x240 RGB s8 stride 2", 4, dict(width=320, height=240, channels=3), 512,
     P.PipelineConfig(coarsest_exp=3, finest_exp=1, patch_size=8, overlap=1 - 2 / 8)),
    ("c4 1920x1080 RGB s16 stride 6", 4, dict(width=1920, height=1080, channels=3), 16,
     P.PipelineConfig(coarsest_exp=4, finest_exp=1, patch_size=16, overlap=1 - 6 / 16)),
]
orc = pyoracle.load("reference" if pyoracle.available("reference") else "port")
for name, conf, ov, B, cfg in CASES:
    left, right = P.synth_batch(conf, B, seed0=0, **ov)
    h, w = left.shape[1], left.shape[2]
    ch = 1 if left.ndim == 3 else left.shape[3]
    dl, dr = torch.from_numpy(left).cuda(), torch.from_numpy(right).cuda()
    disp = torch.empty((B, h, w), dtype=torch.float32, device="cuda")
    m = P.Matcher(cfg, w, h, B)
    s = torch.cuda.Stream()

    def step():
        m.run_device_u8(B, w, h, ch, dl.data_ptr(), dr.data_ptr(), {"disparity": disp.data_ptr()},
                        stream=s.cuda_stream, invalid_value=float("nan"))

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    reps = 5
    for _ in range(reps):
        step()
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    # reference on one core, 2 pairs
    ocfg = pyoracle.Config(coarsest_exp=cfg.coarsest_exp, finest_exp=cfg.finest_exp,
                           patch_size=cfg.patch_size, overlap=cfg.overlap,
                           estimate_variance=cfg.estimate_variance)
    t = []
    for k in range(2):
        lf, _ = orc.to_grayscale(left[k])
        rf, _ = orc.to_grayscale(right[k])
        t.append(orc.run_pipeline(lf, rf, ocfg, 500.0, 5.0)["runtime_ms"])
    print(json.dumps({"config": name, "batch": B, "gpu_pairs_s": B / (ms / 1e3),
                      "gpu_ms_per_batch": ms, "ref_ms_per_pair_1core": float(np.median(t)),
                      "ref_pairs_s_1core": 1e3 / float(np.median(t))}), flush=True)
    m.close()
