"""Throughput of the device renderer (pstereo_gpu_render) on the shipped
scenes at 640x480 against the reference's render_scene (oracle/_ref) on the
host cores, plus run_benchmark_gpu (src/bench.cpp flow) on all seven."""
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2205_03133_b200 as P  # noqa: E402
from oracle import pyoracle  # noqa: E402

SCENES = json.loads((ROOT / "tests" / "golden" / "scenes.json").read_text())
names = sorted(SCENES)
reps = 16
specs = []
for r in range(reps):
    for n in names:
        d = dict(SCENES[n])
        d["seed"] = 1 + r
        specs.append(P.scene_spec(**d))
P.render_scenes_gpu(specs[:7])
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
times = []
for _ in range(5):
    s.record()
    P.render_scenes_gpu(specs)
    e.record()
    e.synchronize()
    times.append(s.elapsed_time(e))
times.sort()
gpu_ms = times[2]
per_kind = {}
for n in names:
    sp = [x for x in specs if x.name.decode() == n]
    P.render_scenes_gpu(sp)
    torch.cuda.synchronize()
    s.record()
    P.render_scenes_gpu(sp)
    e.record()
    e.synchronize()
    per_kind[n] = round(s.elapsed_time(e) / len(sp), 4)

ref = pyoracle.load("reference") if pyoracle.available("reference") else pyoracle.load("port")
cores = len(os.sched_getaffinity(0))
sample = [specs[i % len(specs)] for i in range(cores)]
t0 = time.perf_counter()
with ThreadPoolExecutor(cores) as ex:  # ctypes releases the GIL during the call
    list(ex.map(ref.render_scene, sample))
cpu_s = time.perf_counter() - t0

cfg = P.PipelineConfig(coarsest_exp=5, finest_exp=1)
shipped = [P.scene_spec(**SCENES[n]) for n in names]
t0 = time.perf_counter()
frames, agg = P.run_benchmark_gpu(shipped, cfg, repetitions=10)
flow_s = time.perf_counter() - t0
print(json.dumps({
    "render": {"scenes": len(specs), "size": "640x480", "gpu_ms": round(gpu_ms, 3),
               "gpu_scenes_s": round(len(specs) / (gpu_ms / 1e3), 1),
               "gpu_ms_per_scene_by_kind": per_kind,
               "cpu_scenes_s": round(len(sample) / cpu_s, 2), "cpu_threads": cores,
               "cpu_kind": ref.kind},
    "run_benchmark_gpu": {"scenes": len(shipped), "repetitions": 10,
                          "wall_s": round(flow_s, 2),
                          "rows": frames + [agg]}}, default=float))
