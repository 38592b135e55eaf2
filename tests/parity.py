"""Shared parity helpers: run the GPU product and the CPU oracle on the same
bytes and compare. The bar is bit-exactness for everything the reference
computes without libm transcendentals (disparity, probability, validity masks,
depth, MatchStats, finest-level patch records); var_disp / depth sigma go
through std::exp in the Gauss-Newton fit (src/depth_variance.cpp:125,155), so
they are compared at the BASELINE.json tolerance of 1e-3 relative (observed:
~1e-15)."""
from __future__ import annotations

import numpy as np

VAR_RTOL = 1e-3  # BASELINE.json north_star: "variance within 1e-3 relative"


def oracle_cfg(cfg):
    from oracle import pyoracle

    return pyoracle.Config(**{k: getattr(cfg, k) for k in (
        "coarsest_exp", "finest_exp", "patch_size", "overlap", "min_iterations",
        "max_iterations", "early_stop_good", "early_stop_bad", "early_stop_improve",
        "window_offsets", "sigma_s", "pixel_threshold", "gamma", "valid_patch_ratio",
        "estimate_variance", "threads")})


def gray_of(oracle, raster):
    return oracle.to_grayscale(raster)


def run_oracle(oracle, left_f, right_f, cfg, focal, baseline, lv=None, rv=None):
    ocfg = oracle_cfg(cfg)
    pipe = oracle.run_pipeline(left_f, right_f, ocfg, focal, baseline, lv, rv)
    match = oracle.match_stereo(left_f, right_f, ocfg, lv, rv)
    return pipe, match


GPU_PLANES = ["disparity", "disparity_valid", "probability", "depth", "depth_valid",
              "match_disparity", "match_valid"]
VAR_PLANES = ["depth_sigma", "sigma_valid", "var_disp"]


def run_gpu_batch(P, cfg, left, right, focal, baseline, left_valid=None, right_valid=None,
                  finest_cap=1 << 16):
    n = left.shape[0]
    h, w = left.shape[1], left.shape[2]
    want = GPU_PLANES + (VAR_PLANES if cfg.estimate_variance else [])
    with P.Matcher(cfg, w, h, n) as m:
        out = m.run_batch(left, right, focal=focal, baseline=baseline, dtype=P.F64,
                          left_valid=left_valid, right_valid=right_valid, want=want, stats=True,
                          finest_cap=finest_cap)
        out["launches"] = m.launch_count()
    return out


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint64) if a.dtype == np.float64 else a


def compare_pair(gpu, k, pipe, match, cfg, report=None):
    """Asserts the GPU result of pair k equals the oracle's. Returns a dict of
    observed agreement statistics."""
    stats = {}
    np.testing.assert_array_equal(gpu["stats"][k], match["stats"], err_msg="MatchStats")
    for name, ref in (("disparity_valid", pipe["disparity_valid"]),
                      ("depth_valid", pipe["depth_valid"]),
                      ("match_valid", match["disparity_valid"])):
        np.testing.assert_array_equal(gpu[name][k], ref, err_msg=name)
    for name, ref in (("disparity", pipe["disparity"]), ("probability", pipe["probability"]),
                      ("depth", pipe["depth"]), ("match_disparity", match["disparity"])):
        g = gpu[name][k]
        same = bits(g) == bits(ref)
        if not same.all():
            bad = np.argwhere(~same)[:5]
            raise AssertionError(f"{name}: {int((~same).sum())} px differ, e.g. {bad.tolist()} "
                                 f"gpu={g[tuple(bad[0])]!r} ref={ref[tuple(bad[0])]!r}")
    # finest patch records (MatchResult::finest.patches)
    fin = gpu["finest"][k]
    ref_f = match["finest"]
    assert fin.shape[0] == ref_f.shape[0], "finest patch count"
    np.testing.assert_array_equal(bits(fin[:, :5]), bits(ref_f[:, :5]), err_msg="finest records")
    if cfg.estimate_variance:
        np.testing.assert_array_equal(gpu["sigma_valid"][k], pipe["sigma_valid"],
                                      err_msg="sigma_valid")
        sk_g, sk_r = fin[:, 5], ref_f[:, 5]
        np.testing.assert_allclose(sk_g, sk_r, rtol=VAR_RTOL, atol=0)
        stats["sigma_k_bitexact"] = float((bits(sk_g) == bits(sk_r)).mean()) if len(sk_g) else 1.0
        m = match["disparity_valid"].astype(bool)
        np.testing.assert_allclose(gpu["var_disp"][k][m], match["var_disp"][m], rtol=VAR_RTOL,
                                   atol=0)
        sv = pipe["sigma_valid"].astype(bool)
        np.testing.assert_allclose(gpu["depth_sigma"][k][sv], pipe["depth_sigma"][sv],
                                   rtol=VAR_RTOL, atol=0)
        stats["var_bitexact"] = float((bits(gpu["var_disp"][k][m]) ==
                                       bits(match["var_disp"][m])).mean()) if m.any() else 1.0
    stats["valid_fraction"] = float(pipe["disparity_valid"].mean())
    return stats
