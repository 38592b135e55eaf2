"""Throughput of the on-device generator (pstereo_gpu_synth) against the host
generator (pstereo_synth_batch, all host cores) on BASELINE configs 0, 1, 3."""
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2205_03133_b200 as P  # noqa: E402


def dev_rate(config, n, reps=5):
    P.synth_batch_gpu(config, n)  # warm-up (allocator, module load)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = []
    for _ in range(reps):
        s.record()
        P.synth_batch_gpu(config, n, seed0=1000)
        e.record()
        e.synchronize()
        ms.append(s.elapsed_time(e))
    ms.sort()
    return n / (ms[len(ms) // 2] / 1e3), ms[len(ms) // 2]


def host_rate(config, n, threads):
    t = time.perf_counter()
    P.synth_batch(config, n, seed0=1000, threads=threads)
    return n / (time.perf_counter() - t)


cores = len(os.sched_getaffinity(0))
out = {}
for config, n, nh in ((0, 256, 64), (1, 256, 64), (3, 32, 8)):
    g, ms = dev_rate(config, n)
    h = host_rate(config, nh, cores)
    out[f"c{config}"] = {"gpu_pairs_s": round(g, 1), "gpu_ms_per_batch": round(ms, 3),
                         "batch": n, "host_pairs_s": round(h, 1), "host_threads": cores,
                         "host_sample": nh}
print(json.dumps(out))
