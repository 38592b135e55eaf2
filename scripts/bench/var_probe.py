"""Stage times: config-0 data with / without variance, config-1 data (debug aid)."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2205_03133_b200 as P  # noqa: E402

B, W, H = 256, 640, 480
for data_cfg, var in ((0, False), (0, True), (1, False), (1, True)):
    dl, dr = P.synth_batch_gpu(data_cfg, B, seed0=0)
    disp = torch.empty((B, H, W), dtype=torch.float32, device="cuda")
    cfg = P.PipelineConfig(coarsest_exp=3, finest_exp=1, patch_size=8, overlap=0.5,
                           estimate_variance=var)
    with P.Matcher(cfg, W, H, B) as m:
        m.set_device_chunks(1)

        def step():
            m.run_device_u8(B, W, H, 1, dl.data_ptr(), dr.data_ptr(),
                            {"disparity": disp.data_ptr()}, invalid_value=float("nan"))
        for _ in range(2):
            step()
        torch.cuda.synchronize()
        m.set_profiling(True)
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        t, calls = m.stage_times()
        m.set_profiling(False)
    print(json.dumps({"data": f"c{data_cfg}", "variance": var,
                      "ms": {k: round(v / calls, 3) for k, v in t.items() if k not in ("h2d", "d2h")}}))
