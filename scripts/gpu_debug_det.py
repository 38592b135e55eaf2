"""Determinism / chunking check at the bench workload: device-resident runs
against each other and against the chunked host path; differing pairs are
checked against the CPU oracle. Debug aid, run under gpurun."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2205_03133_b200 as P  # noqa: E402
from tests.parity import run_oracle  # noqa: E402
from oracle import pyoracle  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
W, H = 640, 480
cfg = P.PipelineConfig.baseline(0)
left, right = P.synth_batch(0, B, seed0=0)
dev = torch.device("cuda", 0)
dl, dr = torch.from_numpy(left).to(dev), torch.from_numpy(right).to(dev)
m = P.Matcher(cfg, W, H, B)
keys = ["disparity", "match_disparity", "match_valid"]


def dev_run():
    outs = {k: torch.empty((B, H, W), dtype=torch.float32 if "valid" not in k else torch.uint8,
                           device=dev) for k in keys}
    m.run_device_u8(B, W, H, 1, dl.data_ptr(), dr.data_ptr(), {k: v.data_ptr() for k, v in outs.items()},
                    invalid_value=float("nan"))
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in outs.items()}


def host_run():
    outs = {k: np.empty((B, H, W), dtype=np.float32 if "valid" not in k else np.uint8) for k in keys}
    m.run_host_u8(B, W, H, 1, left.ctypes.data, right.ctypes.data,
                  {k: v.ctypes.data for k, v in outs.items()}, invalid_value=float("nan"))
    torch.cuda.synchronize()
    return outs


def diff(a, b, tag):
    bad = set()
    for k in keys:
        x, y = a[k], b[k]
        eq = (x == y) | (np.isnan(x) & np.isnan(y)) if x.dtype == np.float32 else (x == y)
        pairs = np.nonzero(~eq.reshape(B, -1).all(1))[0]
        print(f"{tag} {k}: {int((~eq).sum())} px differ in pairs {pairs[:20].tolist()}")
        bad |= set(pairs.tolist())
    return sorted(bad)


runs = [dev_run() for _ in range(3)]
bad = set()
bad |= set(diff(runs[0], runs[1], "dev0-dev1"))
bad |= set(diff(runs[0], runs[2], "dev0-dev2"))
h0 = host_run()
bad |= set(diff(runs[0], h0, "dev0-host0"))
h1 = host_run()
bad |= set(diff(h0, h1, "host0-host1"))
port = pyoracle.load("port")
for k in sorted(bad)[:4]:
    lf, lv = port.to_grayscale(left[k])
    rf, rv = port.to_grayscale(right[k])
    pipe, match = run_oracle(port, lf, rf, cfg, 1.0, 1.0, lv, rv)
    ov = np.asarray(pipe["disparity_valid"]).astype(bool)
    for tag, r in (("dev0", runs[0]), ("dev1", runs[1]), ("dev2", runs[2]), ("host0", h0), ("host1", h1)):
        gv = ~np.isnan(r["disparity"][k])
        mv = r["match_valid"][k].astype(bool)
        print(f"pair {k} {tag}: valid vs oracle {int((gv != ov).sum())} px, "
              f"match_valid vs oracle {int((mv != np.asarray(match['disparity_valid']).astype(bool)).sum())} px, "
              f"match disp max diff {float(np.nanmax(np.abs(r['match_disparity'][k] - match['disparity']))):.3g}")
print("done")
