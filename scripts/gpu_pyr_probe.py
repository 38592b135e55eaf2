"""Pyramid stage for large RGB / gray inputs (debug aid)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2205_03133_b200 as P  # noqa: E402

for ch in (3, 1):
    dl, dr = P.synth_batch_gpu(4, 16, width=1920, height=1080, channels=ch)
    disp = torch.empty((16, 1080, 1920), dtype=torch.float32, device="cuda")
    cfg = P.PipelineConfig(coarsest_exp=4, finest_exp=1, patch_size=8, overlap=0.5)
    with P.Matcher(cfg, 1920, 1080, 16) as m:
        m.run_device_u8(16, 1920, 1080, ch, dl.data_ptr(), dr.data_ptr(),
                        {"disparity": disp.data_ptr()}, invalid_value=float("nan"))
        torch.cuda.synchronize()
