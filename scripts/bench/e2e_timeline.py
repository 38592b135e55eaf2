"""Chunk timeline of a few back-to-back async e2e calls (PSTEREO_DEBUG_TIMELINE=1). Debug aid."""
import os
import sys

os.environ["PSTEREO_DEBUG_TIMELINE"] = "1"
import torch  # noqa: E402

sys.path.insert(0, ".")
import paper_2205_03133_b200 as P  # noqa: E402

B, W, H = 256, 640, 480
calls = int(sys.argv[1]) if len(sys.argv) > 1 else 4
left, right = P.synth_batch(0, B, seed0=0)
hl = torch.from_numpy(left).pin_memory()
hr = torch.from_numpy(right).pin_memory()
hd = torch.empty((B, H, W), dtype=torch.float32).pin_memory()
m = P.Matcher(P.PipelineConfig.baseline(0), W, H, B)
s = torch.cuda.Stream()
for rep in range(2):
    for _ in range(calls):
        m.run_host_u8(B, W, H, 1, hl.data_ptr(), hr.data_ptr(), {"disparity": hd.data_ptr()},
                      stream=s.cuda_stream, invalid_value=float("nan"), async_host=True)
    print(f"--- pass {rep}", file=sys.stderr, flush=True)
    m.wait(s.cuda_stream)
