"""Per-level CTA-shape sweep of k_patches (threads x CTAs per SM) for the
config-4 patch-size x stride grid at 640x480, 256 device-resident pairs:
prints the default stage times and, per level, the best shape found.
Tuning aid (PSTEREO_TUNE_SPEC)."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2205_03133_b200 as P  # noqa: E402

# usage: gpu_shape_sweep.py [W H B "s:stride,s:stride,..."]
W, H, B = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (640, 480, 256)
GRID = ([tuple(int(v) for v in c.split(":")) for c in sys.argv[4].split(",")]
        if len(sys.argv) > 4 else [(s, st) for s in (8, 12, 16) for st in (2, 4, 6)])
dl, dr = P.synth_batch_gpu(0, B, seed0=0, width=W, height=H)
disp = torch.empty((B, H, W), dtype=torch.float32, device="cuda")
SHAPES = ["96x4", "128x2", "128x3", "128x4", "192x1", "192x2", "256x1", "256x2"]


def stages(cfg, spec):
    if spec:
        os.environ["PSTEREO_TUNE_SPEC"] = spec
    else:
        os.environ.pop("PSTEREO_TUNE_SPEC", None)
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
        t, calls = m.stage_times()
        m.set_profiling(False)
    return {k: v / calls for k, v in t.items() if k.startswith("patches_")}


for s, stride in GRID:
    if True:
        ce = int(os.environ.get("SWEEP_CE", 4 if (s <= 12 or W > 640) else 3))
        cfg = P.PipelineConfig(coarsest_exp=ce, finest_exp=1, patch_size=s, overlap=1 - stride / s)
        base = stages(cfg, None)
        best = {}
        for lvl in base:
            e = lvl.split("_e")[1]
            cand = []
            for sh in SHAPES:
                try:
                    t = stages(cfg, f"e{e}={sh}")[lvl]
                except Exception as ex:  # noqa: BLE001
                    continue
                cand.append((t, sh))
            cand.sort()
            best[lvl] = {"default_ms": round(base[lvl], 4), "best": cand[0][1],
                         "best_ms": round(cand[0][0], 4),
                         "all": {sh: round(t, 4) for t, sh in sorted(cand, key=lambda x: x[1])}}
        print(json.dumps({"size": f"{W}x{H}", "s": s, "stride": stride, "levels": best}),
              flush=True)
