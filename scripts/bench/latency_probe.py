"""Stage times of single-pair calls (config-4 latency row), debug aid."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2205_03133_b200 as P  # noqa: E402

for (w, h, ch) in ((640, 480, 1), (640, 480, 3), (1920, 1080, 3)):
    dl, dr = P.synth_batch_gpu(4 if ch == 3 else 0, 1, width=w, height=h, channels=ch)
    disp = torch.empty((1, h, w), dtype=torch.float32, device="cuda")
    cfg = P.PipelineConfig(coarsest_exp=4 if w > 640 or ch == 3 else 3, finest_exp=1,
                           patch_size=8, overlap=0.5)
    with P.Matcher(cfg, w, h, 1) as m:
        st = torch.cuda.Stream()

        def step():
            m.run_device_u8(1, w, h, ch, dl.data_ptr(), dr.data_ptr(),
                            {"disparity": disp.data_ptr()}, stream=st.cuda_stream,
                            invalid_value=float("nan"))
        for _ in range(5):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(50):
            step()
        e1.record(st)
        torch.cuda.synchronize()
        total = e0.elapsed_time(e1) / 50
        m.set_profiling(True)
        for _ in range(20):
            step()
        torch.cuda.synchronize()
        stages, calls = m.stage_times()
        m.set_profiling(False)
    print(json.dumps({"size": f"{w}x{h}x{ch}", "ms_per_call": round(total, 4),
                      "stages_ms": {k: round(v / calls, 4) for k, v in stages.items()}}))
