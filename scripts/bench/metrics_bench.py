"""Throughput of the GPU compute_metrics on 256 frames of
640x480 double fields (device-resident, one call), beside the reference's
compute_metrics (oracle/_ref) on one core. Prints one JSON line."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2205_03133_b200 as P  # noqa: E402
from oracle import pyoracle  # noqa: E402

n, h, w = 256, 480, 640
rng = np.random.default_rng(0)
est = rng.normal(20, 5, (n, h, w))
ref = est + rng.normal(0, 0.5, (n, h, w))
sig = np.abs(rng.normal(0.5, 0.2, (n, h, w)))
ev = (rng.random((n, h, w)) < 0.9).astype(np.uint8)
ones = np.ones((n, h, w), np.uint8)
dev = torch.device("cuda", 0)
t = {k: torch.from_numpy(v).to(dev) for k, v in
     dict(est=est, ev=ev, ref=ref, rv=ones, sig=sig, sv=ones).items()}
m = P.Matcher(P.PipelineConfig(coarsest_exp=0, finest_exp=0, patch_size=2), w, h, 1)
out = (P.FrameMetricsC * n)()
s = torch.cuda.Stream()


def call():
    rc = P.lib().pstereo_gpu_metrics(m._h, n, w, h, t["est"].data_ptr(), t["ev"].data_ptr(),
                                     t["ref"].data_ptr(), t["rv"].data_ptr(), t["sig"].data_ptr(),
                                     t["sv"].data_ptr(), 1, out, s.cuda_stream)
    assert rc == 0, m.last_error()


for _ in range(3):
    call()
torch.cuda.synchronize()
reps = 10
t0 = time.perf_counter()
for _ in range(reps):
    call()
torch.cuda.synchronize()
gpu_ms = (time.perf_counter() - t0) / reps * 1e3
orc = pyoracle.load("reference" if pyoracle.available("reference") else "port")
k = 8
t0 = time.perf_counter()
for i in range(k):
    orc.compute_metrics(est[i], ev[i], ref[i], ones[i], sig[i], ones[i])
cpu_ms = (time.perf_counter() - t0) / k * 1e3
print(json.dumps({"metric": "compute_metrics frames/s (640x480 f64, sigma on)",
                  "gpu_frames_s": n / (gpu_ms / 1e3), "gpu_ms_per_256": gpu_ms,
                  "cpu_frames_s_1core": 1e3 / cpu_ms, "cpu_ms_per_frame": cpu_ms,
                  "cpu_kind": "reference" if pyoracle.available("reference") else "port"}))
