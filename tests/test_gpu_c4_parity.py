"""BASELINE config 4 (the sweep bench.py --sweep c4 times): every case at its
full size -- 320x240 .. 1920x1080 RGB at s=8 stride 4, and s in {8,12,16} x
stride in {2,4,6} at 640x480 -- two seeds each, through the device path with
the same level choice as the bench, bit for bit against the reference."""
import os
from concurrent.futures import ThreadPoolExecutor

import pytest

from tests.parity import compare_pair, run_gpu_batch, run_oracle

pytestmark = pytest.mark.gpu

CASES = [(w, h, 8, 4) for w, h in ((320, 240), (640, 480), (1280, 1024), (1920, 1080))]
CASES += [(640, 480, s, st) for s in (8, 12, 16) for st in (2, 4, 6) if (s, st) != (8, 4)]


@pytest.mark.parametrize("w,h,s,st", CASES)
def test_config4_case(gpu, checker, w, h, s, st):
    import bench

    P = gpu
    wl = bench.workload(f"c4:{w}x{h}:{s}:{st}:3:2")
    cfg = P.PipelineConfig(**wl["params"])
    left, right = P.synth_batch(4, 2, seed0=0, **wl["over"])
    gpu_out = run_gpu_batch(P, cfg, left, right, 500.0, 5.0)

    def ref_of(k):
        lf, lv = checker.to_grayscale(left[k])
        rf, rv = checker.to_grayscale(right[k])
        return run_oracle(checker, lf, rf, cfg, 500.0, 5.0, lv, rv)

    with ThreadPoolExecutor(min(2, os.cpu_count() or 1)) as ex:
        refs = list(ex.map(ref_of, range(2)))
    for k, (pipe, match) in enumerate(refs):
        compare_pair(gpu_out, k, pipe, match, cfg)
