"""Pipelined call time by which side is on the host. Debug aid."""
import os
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2205_03133_b200 as P  # noqa: E402

B, W, H = 256, 640, 480
left, right = P.synth_batch(0, B, seed0=0)
hl = torch.from_numpy(left).pin_memory()
hr = torch.from_numpy(right).pin_memory()
hd = torch.empty((B, H, W), dtype=torch.float32).pin_memory()
dl, dr = hl.cuda(), hr.cuda()
dd = torch.empty((B, H, W), dtype=torch.float32, device="cuda")
cfg = P.PipelineConfig.baseline(0)
os.environ["PSTEREO_CHUNK_PAIRS"] = sys.argv[1] if len(sys.argv) > 1 else "32"
m = P.Matcher(cfg, W, H, B)
s = torch.cuda.Stream()
lib = P.lib()
import ctypes as C  # noqa: E402


def call(inp_dev, out_dev):
    o = P._Outputs()
    o.dtype = P.F32
    o.on_device = int(out_dev)
    o.fill_invalid, o.invalid_value = 1, float("nan")
    o.disparity = (dd if out_dev else hd).data_ptr()
    L, R = (dl, dr) if inp_dev else (hl, hr)
    rc = lib.pstereo_gpu_match_u8(m._h, B, W, H, 1, L.data_ptr(), R.data_ptr(), int(inp_dev),
                                  1.0, 1.0, C.byref(o), s.cuda_stream)
    assert rc == 0, m.last_error()


for inp_dev, out_dev in ((0, 0), (0, 1), (1, 0), (1, 1)):
    for _ in range(2):
        call(inp_dev, out_dev)
    torch.cuda.synchronize()
    t = time.perf_counter()
    reps = 5
    for _ in range(reps):
        call(inp_dev, out_dev)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / reps
    t = time.perf_counter()
    call(inp_dev, out_dev)
    t_ret = time.perf_counter() - t
    torch.cuda.synchronize()
    print(f"in_dev={inp_dev} out_dev={out_dev}: {dt * 1e3:.2f} ms/call (single call returns after {t_ret * 1e3:.2f} ms)")
