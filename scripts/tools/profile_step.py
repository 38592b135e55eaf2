"""One bench step for profilers: the config-2 batch (256 pairs) matched twice
with one launch per stage (device chunks = 1), so an ncu capture with
--launch-skip 8 --launch-count 8 on the k_* kernels sees exactly one step:
k_pyramid, k_patches x3, k_fuse_ccl_local, k_ccl_border, k_ccl_merge,
k_output_disp_x4."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import bench  # noqa: E402
import paper_2205_03133_b200 as P  # noqa: E402

wl = bench.workload(sys.argv[1] if len(sys.argv) > 1 else "c2")
W, H, CH, B = wl["W"], wl["H"], wl["C"], wl["batch"]
dl, dr = P.synth_batch_gpu(wl["gen"], B, seed0=0, **wl["over"])
disp = torch.empty((B, H, W), dtype=torch.float32, device="cuda")
with P.Matcher(P.PipelineConfig(**wl["params"]), W, H, B) as m:
    m.set_device_chunks(1)
    for _ in range(2):
        m.run_device_u8(B, W, H, CH, dl.data_ptr(), dr.data_ptr(), {"disparity": disp.data_ptr()},
                        invalid_value=float("nan"))
    torch.cuda.synchronize()
print("ok")
