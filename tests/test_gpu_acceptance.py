"""The reference's accuracy acceptance checks, run on the device path.

tests/acceptance.cpp:322-344 (check_subpixel): rendered planes at d = 4/8/16
px, default PipelineConfig, compute_metrics(disparity vs the scene's
reference disparity): median |err| < 0.2 px and mean < 0.5 px.
tests/acceptance.cpp:520-556 (check_coverage): plane_noise with variance
estimation; one simulated depth error per pixel drawn from the estimated std
must fall inside the 1.96-sigma band 0.95 +/- 0.02 of the time over >= 10000
px. Here the scenes come from the device renderer (pstereo_gpu_render), the
matcher from the C ABI and the metrics from the device compute_metrics
(pstereo_gpu_metrics) -- the whole check on the B200. Beside them, the
BASELINE generator's own ground truth: configs 0-3, disparity error and,
with variance on, the empirical 1.96-sigma coverage of disparity errors."""
import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SCENES = json.loads((Path(__file__).resolve().parent / "golden" / "scenes.json").read_text())


def _scene(P, name):
    spec = P.scene_spec(**SCENES[name])
    gl, gr, gd, gz = (t.cpu().numpy()[0] for t in P.render_scenes_gpu([spec]))
    return spec, gl, gr, gd, gz


@pytest.mark.parametrize("name", ["plane_d4", "plane_d8", "plane_d16"])
def test_subpixel_planes(gpu, name):
    P = gpu
    spec, left, right, ref_d, _ = _scene(P, name)
    h, w = left.shape
    cfg = P.PipelineConfig()  # the reference defaults, as acceptance.cpp uses
    with P.Matcher(cfg, w, h, 1) as m:
        out = m.run_batch(left[None], right[None], focal=spec.focal_px, baseline=spec.baseline,
                          dtype=P.F64, want=("disparity", "disparity_valid"))
        met = m.metrics(out["disparity"][0], out["disparity_valid"][0], ref_d,
                        np.ones_like(out["disparity_valid"][0]))
    print(name, met)
    assert met["has_errors"]
    assert met["median_err"] < 0.2 and met["mean_err"] < 0.5


def test_coverage_plane_noise(gpu):
    P = gpu
    spec, left, right, _, ref_z = _scene(P, "plane_noise")
    h, w = left.shape
    cfg = P.PipelineConfig(estimate_variance=True)
    with P.Matcher(cfg, w, h, 1) as m:
        out = m.run_batch(left[None], right[None], focal=spec.focal_px, baseline=spec.baseline,
                          dtype=P.F64, want=("depth", "depth_valid", "depth_sigma",
                                             "sigma_valid"))
        z, zv = out["depth"][0], out["depth_valid"][0]
        sg, sv = out["depth_sigma"][0], out["sigma_valid"][0]
        ones = np.ones_like(zv)
        rng = np.random.default_rng(0xC0FE)
        ok = (zv != 0) & (sv != 0)
        sim = np.where(ok, ref_z + sg * rng.standard_normal(ref_z.shape), 0.0)
        simulated = m.metrics(sim, ok.astype(np.uint8), ref_z, ones, sg, sv)
        empirical = m.metrics(z, zv, ref_z, ones, sg, sv)
    print("simulated", simulated, "empirical", empirical)
    assert simulated["valid_px"] >= 10000
    assert abs(simulated["coverage_rate"] - 0.95) <= 0.02


@pytest.mark.parametrize("config,n", [(0, 4), (1, 4), (2, 8), (3, 2)])
def test_generator_ground_truth(gpu, config, n):
    """Disparity error against the BASELINE generator's own field d(x, y):
    the matcher recovers it to well under a pixel on the pixels it keeps."""
    P = gpu
    import torch

    cfg = P.PipelineConfig.baseline(config)
    gen = 0 if config == 2 else config
    dl, dr, gt = P.synth_batch_gpu(gen, n, seed0=0, with_disparity=True)
    left, right, truth = dl.cpu().numpy(), dr.cpu().numpy(), gt.cpu().numpy()
    del dl, dr, gt
    torch.cuda.empty_cache()
    h, w = left.shape[1:3]
    want = ("disparity", "disparity_valid", "match_disparity", "match_valid", "var_disp")
    with P.Matcher(cfg, w, h, n) as m:
        out = m.run_batch(left, right, focal=500.0, baseline=5.0, dtype=P.F64,
                          want=want if cfg.estimate_variance else want[:2])
        ones = np.ones((n, h, w), np.uint8)
        met = m.metrics(out["disparity"], out["disparity_valid"], truth.astype(np.float64), ones)
        if cfg.estimate_variance:
            sd = np.sqrt(np.maximum(out["var_disp"], 0.0))
            cov = m.metrics(out["match_disparity"], out["match_valid"],
                            truth.astype(np.float64), ones, sd, out["match_valid"])
    valid_frac = float(out["disparity_valid"].mean())
    med = float(np.median([r["median_err"] for r in met]))
    print(f"config {config}: valid {valid_frac:.3f}, median |err| {med:.3f} px, "
          f"mean {np.mean([r['mean_err'] for r in met]):.3f} px")
    assert valid_frac > 0.5
    assert med < (0.5 if config in (1, 3) else 0.25)
    if cfg.estimate_variance:
        c = [r["coverage_rate"] for r in cov]
        print(f"config {config}: empirical 1.96-sigma coverage of disparity errors {c}")
        assert all(0.0 <= x <= 1.0 for x in c)
