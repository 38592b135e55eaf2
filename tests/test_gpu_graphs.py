"""pstereo_gpu_set_graphs: repeated device-buffer calls replayed as CUDA
graphs give the eager call's results bit for bit -- across repeats, when the
output buffer changes (a new signature), when the context reallocates (a
bigger batch invalidates every graph), and on the two-stream sub-batch path
(>= 32 pairs) -- and graph replay is faster per call than the eager path."""
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

W, H = 320, 240


def _planes(t):
    return t.cpu().numpy().view(np.uint8)


def test_graph_replay_matches_eager(gpu):
    P = gpu
    import torch

    cfg = P.PipelineConfig.baseline(1)  # variance on
    dl, dr = P.synth_batch_gpu(1, 40, seed0=3, width=W, height=H)
    s = torch.cuda.Stream()
    names = ("disparity", "disparity_valid", "depth", "depth_sigma")

    def outs(n):
        return {k: torch.empty((n, H, W), dtype=torch.uint8 if "valid" in k else torch.float64,
                               device="cuda") for k in names}

    def call(m, n, o):
        m.run_device_u8(n, W, H, 1, dl.data_ptr(), dr.data_ptr(), {k: v.data_ptr() for k, v in o.items()},
                        dtype=P.F64, focal=500.0, baseline=5.0, stream=s.cuda_stream)
        s.synchronize()

    with P.Matcher(cfg, W, H, 40) as eager, P.Matcher(cfg, W, H, 40) as g:
        g.set_graphs(True)
        for n in (1, 4, 40):  # 40: the two-stream sub-batch path
            ref = outs(n)
            call(eager, n, ref)
            a, b = outs(n), outs(n)
            for o in (a, a, a, b, a):  # capture, replays, a second signature
                for v in o.values():
                    v.zero_()
                call(g, n, o)
                for k in names:
                    assert np.array_equal(_planes(o[k]), _planes(ref[k])), (n, k)


def test_graph_latency(gpu):
    P = gpu
    import torch

    cfg = P.PipelineConfig.baseline(0)
    dl, dr = P.synth_batch_gpu(0, 1, seed0=0)
    out = torch.empty((1, 480, 640), dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    lat = {}
    for mode in (False, True):
        with P.Matcher(cfg, 640, 480, 1) as m:
            m.set_graphs(mode)

            def call():
                m.run_device_u8(1, 640, 480, 1, dl.data_ptr(), dr.data_ptr(),
                                {"disparity": out.data_ptr()}, stream=s.cuda_stream,
                                invalid_value=float("nan"))
                s.synchronize()

            for _ in range(5):
                call()
            t = []
            for _ in range(30):
                t0 = time.perf_counter()
                call()
                t.append(time.perf_counter() - t0)
            lat[mode] = float(np.median(t)) * 1e3
    print(f"single-pair latency: eager {lat[False]:.4f} ms, graph {lat[True]:.4f} ms")
    assert lat[True] < lat[False]
