"""Stage times for a few BASELINE configurations (debug aid)."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2205_03133_b200 as P  # noqa: E402

CASES = [("c3 1280x1024 s12 var", 3, {}, 32, P.PipelineConfig.baseline(3)),
         ("c4 1920x1080 s8 st4 RGB", 4, dict(width=1920, height=1080, channels=3), 64,
          P.PipelineConfig(coarsest_exp=4, finest_exp=1, patch_size=8, overlap=0.5)),
         ("c1 640x480 var stress", 1, {}, 256, P.PipelineConfig.baseline(1))]
for name, conf, ov, B, cfg in CASES:
    dl, dr = P.synth_batch_gpu(conf, B, **ov)
    h, w = dl.shape[1], dl.shape[2]
    ch = 1 if dl.dim() == 3 else dl.shape[3]
    disp = torch.empty((B, h, w), dtype=torch.float32, device="cuda")
    with P.Matcher(cfg, w, h, B) as m:
        m.set_device_chunks(1)
        st = torch.cuda.Stream()

        def step():
            m.run_device_u8(B, w, h, ch, dl.data_ptr(), dr.data_ptr(),
                            {"disparity": disp.data_ptr()}, stream=st.cuda_stream,
                            invalid_value=float("nan"))
        for _ in range(2):
            step()
        torch.cuda.synchronize()
        m.set_profiling(True)
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        t, calls = m.stage_times()
        m.set_profiling(False)
    print(json.dumps({"case": name, "batch": B,
                      "ms": {k: round(v / calls, 3) for k, v in t.items()
                             if k not in ("h2d", "d2h")}}), flush=True)
