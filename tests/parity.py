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


def random_case(P, seed):
    """A random valid PipelineConfig and pair (tests/test_gpu_parity.py's
    randomized sweep; tests/test_port_vs_ref.py pins the port to the reference
    on the same cases). Returns (cfg, left, right) uint8 rasters."""
    rng = np.random.default_rng(1000 + seed)
    size = int(rng.integers(2, 21))
    stride = int(rng.integers(1, size + 1))
    fe = int(rng.integers(0, 2))
    ce = fe + int(rng.integers(0, 4))
    minw = size << ce
    w = int(rng.integers(minw, minw + 120))
    h = int(rng.integers(minw, minw + 90))
    offs = sorted(set(float(x) for x in rng.choice([0.25, 0.5, 0.75, 1.0, 1.5, 2.0],
                                                   size=int(rng.integers(1, 4)), replace=False)))
    cfg = P.PipelineConfig(coarsest_exp=ce, finest_exp=fe, patch_size=size,
                           overlap=1.0 - stride / size,
                           min_iterations=int(rng.integers(1, 6)), max_iterations=12,
                           window_offsets=offs,
                           pixel_threshold=float(rng.uniform(0.05, 0.4)),
                           gamma=float(rng.uniform(0.1, 1.0)),
                           valid_patch_ratio=float(rng.uniform(0.5, 1.0)),
                           estimate_variance=bool(rng.integers(0, 2)))
    ch = int(rng.choice([1, 3, 4]))
    l, r = P.synth_pair(0, seed=seed, width=w, height=h, channels=min(ch, 3),
                        d_range=float(rng.uniform(2, 12)), d_min=float(rng.uniform(0, 3)))
    if ch == 4:  # RGBA: alpha == 0 marks invalid pixels (src/image.cpp:32-34)
        alpha = [np.full((h, w, 1), 255, np.uint8) for _ in range(2)]
        for a in alpha:
            a[rng.random((h, w)) < rng.uniform(0, 0.05)] = 0
            y0, x0 = int(rng.integers(0, h)), int(rng.integers(0, w))
            a[y0:y0 + int(rng.integers(1, h // 2 + 2)), x0:x0 + int(rng.integers(1, w // 2 + 2))] = 0
        l, r = np.concatenate([l, alpha[0]], axis=2), np.concatenate([r, alpha[1]], axis=2)
    return cfg, l, r


def compare_oracles(a, b, cfg, left, right, focal=500.0, baseline=5.0):
    """Runs run_pipeline + match_stereo of two checker libraries on the same
    raster pair and asserts every output identical (f64 bits; MatchStats and
    the finest records included)."""
    la, lva = a.to_grayscale(left)
    ra, rva = a.to_grayscale(right)
    lb, lvb = b.to_grayscale(left)
    rb, rvb = b.to_grayscale(right)
    for x, y in ((la, lb), (lva, lvb), (ra, rb), (rva, rvb)):
        assert np.array_equal(bits(x) if x.dtype == np.float64 else x, y)
    pa, ma = run_oracle(a, la, ra, cfg, focal, baseline, lva, rva)
    pb, mb = run_oracle(b, lb, rb, cfg, focal, baseline, lvb, rvb)
    for res_a, res_b in ((pa, pb), (ma, mb)):
        for k in res_a:
            if k == "runtime_ms":
                continue
            va, vb = res_a[k], res_b[k]
            if isinstance(va, np.ndarray):
                assert np.array_equal(bits(va), bits(vb)), k
            else:
                assert va == vb, k
