"""Stage times for s x stride grids at 640x480 (debug aid for the planner)."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2205_03133_b200 as P  # noqa: E402

W, H, B = 640, 480, 256
dl, dr = P.synth_batch_gpu(0, B, seed0=0, width=W, height=H)
disp = torch.empty((B, H, W), dtype=torch.float32, device="cuda")
tunes = [{}, {"PSTEREO_TUNE_THREADS": "192"}, {"PSTEREO_TUNE_THREADS": "256"},
         {"PSTEREO_TUNE_THREADS": "128"}]
for s, stride in ((8, 4), (8, 6), (12, 4), (12, 6)):
    for t in tunes:
        for k in ("PSTEREO_TUNE_THREADS",):
            os.environ.pop(k, None)
        os.environ.update(t)
        cfg = P.PipelineConfig(coarsest_exp=4, finest_exp=1, patch_size=s, overlap=1 - stride / s)
        with P.Matcher(cfg, W, H, B) as m:
            m.set_device_chunks(1)
            st = torch.cuda.Stream()

            def step():
                m.run_device_u8(B, W, H, 1, dl.data_ptr(), dr.data_ptr(),
                                {"disparity": disp.data_ptr()}, stream=st.cuda_stream,
                                invalid_value=float("nan"))
            for _ in range(2):
                step()
            torch.cuda.synchronize()
            m.set_profiling(True)
            for _ in range(3):
                step()
            torch.cuda.synchronize()
            stages, calls = m.stage_times()
            m.set_profiling(False)
        print(json.dumps({"s": s, "stride": stride, "tune": t,
                          "ms": {k: round(v / calls, 3) for k, v in stages.items()
                                 if k not in ("h2d", "d2h")}}), flush=True)
