# async_host staging race probe: optional arg = alternative library path
import sys
from pathlib import Path
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2205_03133_b200 as P
if len(sys.argv) > 1:
    P.LIB_PATH = Path(sys.argv[1])
n, w, h, calls = 32, 640, 480, 8
cfg = P.PipelineConfig.baseline(0)
planes = ("disparity", "disparity_valid", "probability", "depth")
with P.Matcher(cfg, w, h, n) as m:
    batches = [P.synth_batch(0, n, seed0=1000 + k * n) for k in range(calls)]
    want = [m.run_batch(l, r, focal=500.0, baseline=5.0, dtype=P.F64, want=planes) for l, r in batches]
    pinned = [(torch.from_numpy(l).pin_memory(), torch.from_numpy(r).pin_memory()) for l, r in batches]
    outs = [{k: torch.full((n, h, w), 7, dtype=torch.uint8 if "valid" in k else torch.float64).pin_memory() for k in planes} for _ in range(calls)]
    for (hl, hr), o in zip(pinned, outs):
        m.run_host_u8(n, w, h, 1, hl.data_ptr(), hr.data_ptr(), {k: v.data_ptr() for k, v in o.items()}, dtype=P.F64, focal=500.0, baseline=5.0, async_host=True)
    m.wait()
for k in range(calls):
    print(k, [bool(np.array_equal(want[k][nm].view(np.uint8), outs[k][nm].numpy().view(np.uint8))) for nm in planes])
