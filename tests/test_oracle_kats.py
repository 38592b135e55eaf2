"""The reference's own known-answer tests (proj/tests/test_*.cpp), restated in
pytest and run against BOTH checkers: the plain-C restatement ("port") and the
reference sources compiled in-tree ("reference", skipped where
/root/reference is absent). This pins the oracle before it is trusted as the
GPU's checker. Each test cites the reference test it follows."""
import math

import numpy as np
import pytest

from oracle import pyoracle


@pytest.fixture(params=["port", "reference"])
def orc(request, built):
    if not pyoracle.available(request.param):
        pytest.skip(f"{request.param} oracle not built")
    return pyoracle.load(request.param)


# ---- tests/test_fast_exp.cpp
def test_fast_exp_at_zero(orc):
    assert orc.fast_exp(0.0) == 0.9710078239440918  # :15
    assert abs(orc.fast_exp(0.0) - 1.0) < 0.04


def test_fast_exp_error_band(orc):
    rng = np.random.default_rng(7)
    xs = rng.uniform(-30.0, 0.0, 20000)
    worst = max(abs(orc.fast_exp(x) - math.exp(x)) / math.exp(x) for x in xs)
    assert 0.03 < worst < 0.04  # :20-33


def test_fast_exp_cutoff_and_monotone(orc):
    assert orc.fast_exp(-30.000001) == 0.0  # :36-40
    assert orc.fast_exp(-1e9) == 0.0
    assert orc.fast_exp(-30.0) > 0.0
    prev = orc.fast_exp(-30.0)
    for x in np.arange(-29.75, 0.0001, 0.25):  # :42-47
        v = orc.fast_exp(float(x))
        assert v >= prev
        prev = v


# ---- tests/test_image.cpp
def test_luma_weights(orc):
    g, _ = orc.to_grayscale(np.array([[[255, 0, 0]]], np.uint8))
    assert g[0, 0] == pytest.approx(0.299, rel=1e-6)  # :20-31
    g, _ = orc.to_grayscale(np.array([[[0, 255, 0]]], np.uint8))
    assert g[0, 0] == pytest.approx(0.587, rel=1e-6)
    g, _ = orc.to_grayscale(np.array([[[0, 0, 255]]], np.uint8))
    assert g[0, 0] == pytest.approx(0.114, rel=1e-6)


def test_gray_range_and_alpha(orc):
    g, v = orc.to_grayscale(np.array([[255], [0]], np.uint8))
    assert g[0, 0] == pytest.approx(1.0) and g[1, 0] == 0.0 and v.all()  # :33-40
    g, v = orc.to_grayscale(np.array([[[100, 100, 100, 255], [100, 100, 100, 0]]], np.uint8))
    assert v.tolist() == [[1, 0]]  # :42-48
    assert g[0, 0] == pytest.approx(100.0 / 255.0, rel=1e-6)


def test_bilinear_validity(orc):
    img = np.array([[0, 1], [2, 3]], np.float32)
    v, ok = orc.sample_bilinear(img, None, 0.5, 0.5)
    assert ok and v == pytest.approx(1.5)  # :50-56
    v, _ = orc.sample_bilinear(img, None, 1.0, 0.0)
    assert v == pytest.approx(1.0)
    assert not orc.sample_bilinear(img, None, -0.51, 0.0)[1]
    assert not orc.sample_bilinear(img, None, 0.0, 1.51)[1]
    valid = np.array([[1, 1], [1, 0]], np.uint8)
    assert not orc.sample_bilinear(img, valid, 0.5, 0.5)[1]
    big = np.full((3, 3), 0.5, np.float32)
    bv = np.ones((3, 3), np.uint8)
    bv[2, 2] = 0  # :65-71, zero-weight taps still count
    assert orc.sample_bilinear(big, bv, 0.5, 0.5)[1]
    assert not orc.sample_bilinear(big, bv, 1.5, 1.5)[1]
    assert not orc.sample_bilinear(big, bv, 2.0, 2.0)[1]


# ---- tests/test_pyramid.cpp
def test_downsample_dims_values_edges(orc):
    d, _ = orc.downsample_half(np.ones((4, 5), np.float32))
    assert d.shape == (2, 3)  # :8-14
    d, _ = orc.downsample_half(np.array([[0, 1], [2, 3]], np.float32))
    assert d.shape == (1, 1) and d[0, 0] == pytest.approx(1.5)  # :16-22
    d, _ = orc.downsample_half(np.array([[0, 4, 8]], np.float32))
    assert d[0, 1] == pytest.approx(8.0) and d[0, 0] == pytest.approx(2.0)  # :24-30
    lvl = np.full((480, 640), 0.37, np.float32)
    for _ in range(5):  # :33-42
        lvl, _ = orc.downsample_half(lvl)
        np.testing.assert_allclose(lvl, 0.37, rtol=1e-6)
    assert lvl.shape == (15, 20)
    v = np.ones((2, 2), np.uint8)
    v[0, 1] = 0
    _, dv = orc.downsample_half(np.ones((2, 2), np.float32), v)
    assert dv[0, 0] == 0  # :44-49


def test_gradient_central_differences(orc):
    g = orc.gradient_x(np.array([[0, 2, 6, 12]], np.float32))
    np.testing.assert_allclose(g[0], [2, 3, 5, 6])  # :51-58


# ---- tests/test_patch.cpp
def test_patch_constant_and_ramp(orc):
    p = orc.extract_patch(np.full((32, 32), 0.6, np.float32), None, 15.5, 15.5, 10)
    vals, ok, info = p
    assert info.mean == pytest.approx(0.6, rel=1e-6) and info.valid_count == 100  # :28-36
    np.testing.assert_allclose(vals, 0.0, atol=1e-6)
    ramp = (np.arange(32, dtype=np.float32) * np.float32(0.01))[None, :].repeat(32, 0)
    vals, _, _ = orc.extract_patch(ramp, None, 15.5, 15.5, 10)
    assert abs(vals.sum()) < 1e-5  # :38-46
    assert vals[1] - vals[0] == pytest.approx(0.01, rel=1e-4)


def test_patch_validity_fraction(orc):
    img = np.full((32, 32), 0.5, np.float32)
    v = np.ones((32, 32), np.uint8)
    v[:, 16:] = 0
    vals, ok, info = orc.extract_patch(img, v, 15.5, 15.5, 10)  # :48-62
    assert 0.4 <= info.valid_fraction < 0.6
    assert info.valid_count == round(info.valid_fraction * 100)
    assert vals[9] == 0.0
    assert orc.extract_patch(img, np.zeros((32, 32), np.uint8), 3.5, 3.5, 4) is None  # :64-67
    _, _, info = orc.extract_patch(img, None, 0.5, 15.5, 10)
    assert info.valid_fraction == pytest.approx(0.6, rel=1e-6)  # :69-78


# ---- tests/test_lk_solver.cpp
def _tex(x, y):
    return (0.5 + 0.2 * np.sin(x * 0.37 + 0.8) + 0.15 * np.sin(y * 0.29)
            + 0.1 * np.sin((x + y) * 0.143) + 0.05 * np.sin(x * 0.071 * y * 0.013))


def _analytic(w, h, shift):
    y, x = np.mgrid[0:h, 0:w].astype(np.float64)
    return _tex(x + shift, y).astype(np.float32)


def test_hessian_matches_direct_evaluation(orc):
    left = _analytic(64, 48, 0.0)
    grad = orc.gradient_x(left)
    jac, info = orc.patch_system(left, grad, 31.5, 23.5, 10)  # :35-56
    expected = 0.0
    for j in range(10):
        for i in range(10):
            g = float(grad[int(23.5 - 4.5 + j), int(31.5 - 4.5 + i)])
            assert jac[j * 10 + i] == g
            expected += g * g
    assert info.hessian == expected and not info.degenerate


def test_lk_identity_and_shifts(orc):
    left = _analytic(64, 48, 0.0)
    grad = orc.gradient_x(left)
    r = orc.solve_patch(left, grad, left, 31.5, 23.5, 10, 0.0)  # :58-68
    assert r["converged"] and r["iterations"] == 1 and abs(r["u"]) < 1e-12
    right = _analytic(64, 48, 3.0)
    r = orc.solve_patch(left, grad, right, 31.5, 23.5, 10, 0.0, min_iterations=60,
                        max_iterations=60, update_epsilon=1e-6)  # :70-85
    assert r["converged"] and r["u"] == pytest.approx(3.0, rel=1e-3)
    left96 = _analytic(96, 48, 0.0)
    g96 = orc.gradient_x(left96)
    for d in np.arange(0.25, 3.76, 0.5):  # :87-100
        right = _analytic(96, 48, d)
        for cx in (23.5, 47.5, 71.5):
            r = orc.solve_patch(left96, g96, right, cx, 23.5, 10, 0.0)
            assert r["converged"] and abs(r["u"] - d) < 0.05
    right = _analytic(96, 48, 2.5)
    for u0 in (0.5, 4.5):  # :102-113
        r = orc.solve_patch(left96, g96, right, 47.5, 23.5, 10, u0)
        assert r["converged"] and abs(r["u"] - 2.5) < 0.05


def test_lk_degenerate_and_out_of_bounds(orc):
    flat = np.full((48, 64), 0.5, np.float32)
    gflat = orc.gradient_x(flat)
    _, info = orc.patch_system(flat, gflat, 31.5, 23.5, 10)
    assert info.degenerate  # :115-124
    r = orc.solve_patch(flat, gflat, flat, 31.5, 23.5, 10, 0.0)
    assert not r["converged"] and r["iterations"] == 0
    left = _analytic(64, 48, 0.0)
    grad = orc.gradient_x(left)
    r = orc.solve_patch(left, grad, left, 5.5, 23.5, 10, 20.0)  # :126-134
    assert not r["converged"] and r["iterations"] == 0 and r["u"] == 20.0


def test_lk_early_stops(orc):
    left = _analytic(64, 48, 0.0)
    right = _analytic(64, 48, 2.0)
    grad = orc.gradient_x(left)
    r = orc.solve_patch(left, grad, right, 31.5, 23.5, 10, 0.25, min_iterations=1,
                        stop_good=1e9)  # :142-149
    assert r["converged"] and r["iterations"] == 1 and r["u"] == 0.25
    r = orc.solve_patch(left, grad, right, 31.5, 23.5, 10, 0.0, min_iterations=1,
                        stop_good=0.0, stop_bad=1e-12)  # :151-158
    assert not r["converged"] and r["iterations"] == 1
    r = orc.solve_patch(left, grad, right, 31.5, 23.5, 10, 0.0, min_iterations=1,
                        stop_good=0.0, stop_improve=1e9)  # :160-168
    assert r["iterations"] == 2 and not r["converged"]
    r = orc.solve_patch(left, grad, right, 31.5, 23.5, 10, 0.0)  # :170-176
    assert r["converged"] and abs(r["u"] - 2.0) < 0.05


# ---- tests/test_window_posterior.cpp
def test_dynamic_sigma(orc):
    assert orc.dynamic_sigma([0, 1, 2, 3, 4]) == pytest.approx(math.sqrt(2.0), rel=1e-12)
    assert orc.dynamic_sigma([0, 0, 0, 0, 1]) == pytest.approx(0.4, rel=1e-12)
    assert orc.dynamic_sigma([0.3] * 5) == 1e-4  # :50-54
    assert orc.dynamic_sigma([0] * 5) == 1e-4
    assert orc.dynamic_sigma([0, 1, 2, 3, 1e9], [1, 1, 1, 1, 0]) == pytest.approx(
        math.sqrt(1.25), rel=1e-12)  # :56-61


def test_priors_and_posterior(orc):
    pr = orc.window_priors([2, 1, 0, 1, 2], 1.0, 1, use_fast_exp=False)  # :63-72
    assert pr[2] == pytest.approx(1.0) and pr[1] == pytest.approx(math.exp(-0.5))
    assert pr[0] == pytest.approx(math.exp(-1.0)) and pr[1] == pr[3] and pr[0] == pr[4]
    pr = orc.window_priors([2, 1, 0, 1, 2], 1.0, 1, False, valid=[0, 1, 1, 1, 1])
    assert pr[0] == 0.0 and pr[4] > 0.0  # :74-80
    p, m = orc.patch_posterior([2, 1, 0, 1, 2], 1.0, 1, use_fast_exp=False)
    assert p == pytest.approx(0.3391189, rel=1e-6) and m  # :82-91
    p, _ = orc.patch_posterior([2, 1, 0, 1, 2], 1.0, 1, use_fast_exp=True)
    assert p == pytest.approx(0.3391189, rel=0.085)  # :93-99
    p, m = orc.patch_posterior([0.5] * 5, 1.0, 1, use_fast_exp=False)
    assert p == pytest.approx(0.2, rel=1e-12) and not m  # :101-107
    pa, _ = orc.patch_posterior([2, 1, 0, 1, 2], 1.0, 1, False)
    pb, _ = orc.patch_posterior([8, 4, 0, 4, 8], 2.0, 1, False)
    assert pa == pytest.approx(pb, rel=1e-12)  # :109-117
    w = [0, 1, 2, 1, 2]
    _, m = orc.patch_posterior(w, orc.dynamic_sigma(w), 1, False)
    assert not m  # :133-138
    assert orc.patch_posterior([1e9, 1e9, 1e8, 1e9, 1e9], 1e-4, 1, True) is None
    assert orc.patch_posterior([1e9, 1e9, 1e8, 1e9, 1e9], 1e-4, 1, False) is None  # :140-144


def test_window_sampling(orc):
    y, x = np.mgrid[0:48, 0:64].astype(np.float64)
    img = (0.5 + 0.2 * np.sin(x * 0.37 + 0.8) + 0.15 * np.sin(y * 0.29)
           + 0.1 * np.sin((x + y) * 0.143)).astype(np.float32)
    g = orc.gradient_x(img)
    w = orc.sample_window(img, g, img, 31.5, 23.5, 10, 0.0, [1.0, 0.5])  # :146-166
    assert w is not None and w["offsets"].tolist() == [-1.0, -0.5, 0.0, 0.5, 1.0]
    assert w["center_index"] == 2 and w["valid"].sum() == 5
    r = w["residuals"]
    assert abs(r[2]) < 1e-12 and r[0] > r[1] and r[4] > r[3] and r[1] > 0
    w = orc.sample_window(img, g, img, 5.5, 23.5, 10, 0.4, [0.5, 1.0])  # :168-181
    assert w is not None and w["valid"].sum() == 4 and w["valid"][4] == 0
    assert orc.sample_window(img, g, img, 5.5, 23.5, 10, 1.4, [0.5, 1.0]) is None
    assert orc.sample_window(img, g, img, 5.5, 23.5, 10, 7.0, [0.5, 1.0]) is None


# ---- tests/test_spatial_mask.cpp
def test_spatial_mask(orc):
    m9 = orc.spatial_mask(9, 4.0)
    assert m9[4, 4] == orc.fast_exp(0.0) and (m9 <= m9[4, 4]).all()  # :10-17
    assert m9[0, 0] == pytest.approx(math.exp(-1.0), rel=0.04)  # :19-25
    assert m9[4, 0] == pytest.approx(math.exp(-0.5), rel=0.04)
    m10 = orc.spatial_mask(10, 4.0)
    pk = m10[4, 4]
    assert m10[4, 5] == pk and m10[5, 4] == pk and m10[5, 5] == pk  # :27-37
    assert pk == pytest.approx(math.exp(-0.5 / 32.0), rel=0.04)
    assert (m10 == m10[:, ::-1]).all() and (m10 == m10[::-1, :]).all() and (m10 == m10.T).all()
    for i in range(4, 8):  # :50-54
        assert m9[4, i + 1] <= m9[4, i]
    nar, wid = orc.spatial_mask(9, 2.0), orc.spatial_mask(9, 8.0)
    assert wid[0, 0] > nar[0, 0]  # :56-61


# ---- tests/test_coarse_to_fine.cpp
def test_patch_grids(orc):
    st, xs, ys = orc.make_patch_grid(20, 15, 10, 0.55)  # :45-66
    assert st == 4 and xs.tolist() == [4.5, 8.5, 12.5, 14.5] and ys.tolist() == [4.5, 8.5, 9.5]
    st, xs, _ = orc.make_patch_grid(64, 48, 10, 0.0)  # :68-75
    assert st == 10 and len(xs) == 7 and xs[5] == 54.5 and xs[6] == 58.5
    _, xs, ys = orc.make_patch_grid(10, 10, 10, 0.55)
    assert xs.tolist() == [4.5] and ys.tolist() == [4.5]  # :77-82
    with pytest.raises(pyoracle.OracleError):
        orc.make_patch_grid(9, 20, 10, 0.55)  # :84-86


def test_level_weights(orc):
    lv = [5, 4, 3, 2, 1]  # :103-121
    assert orc.level_weight(5, lv) == pytest.approx(32 / 62, rel=1e-12)
    assert orc.level_weight(1, lv) == pytest.approx(2 / 62, rel=1e-12)
    assert sum(orc.level_weight(n, lv) for n in lv) == pytest.approx(1.0, rel=1e-12)
    assert orc.level_weight(0, [2, 1, 0]) == pytest.approx(1 / 7, rel=1e-12)
    assert orc.propagate_probability(1.0, 0.4, 1, lv) == pytest.approx(0.4 + 2 / 62, rel=1e-12)
    assert orc.propagate_probability(1.0, 0.99, 5, lv) == 1.0  # :123-130
    assert orc.propagate_probability(0.0, 0.25, 3, lv) == 0.25


def test_fusion_cases(orc):
    out, ok = orc.fuse_level([(14.5, 9.5, 3.25, 0.8)], 10, 4.0, 32, 20)  # :132-152
    assert ok["disp"].sum() == 100
    ys, xs = np.nonzero(ok["disp"])
    assert xs.min() == 10 and xs.max() == 19 and ys.min() == 5 and ys.max() == 14
    np.testing.assert_allclose(out["disp"][ok["disp"] == 1], 3.25, rtol=1e-12)
    out, ok = orc.fuse_level([(14.5, 9.5, 2.0, 0.8), (14.5, 9.5, 3.0, 0.2)], 10, 4.0, 32, 20)
    assert out["disp"][9, 14] == pytest.approx(2.2, rel=1e-9)  # :154-168
    assert out["prob"][9, 14] == pytest.approx(0.68, rel=1e-9)
    out, ok = orc.fuse_level([(14.5, 9.5, 2.0, 0.5, 1.0), (14.5, 9.5, 2.0, 0.5, 2.0)], 10, 4.0,
                             32, 20, with_variance=True)
    assert out["var"][9, 14] == pytest.approx(1.25, rel=1e-9)  # :182-196
    _, ok = orc.fuse_level([(4.5, 4.5, 1.0, 0.5)], 10, 4.0, 64, 48)
    assert not ok["disp"][30, 30] and not ok["disp"][0, 10] and ok["disp"][0, 0]  # :198-205


def test_init_and_upsample(orc):
    fine = orc.init_next_level(np.full((3, 4), 3.0), np.ones((3, 4), np.uint8), 8, 6)
    assert (fine == 6.0).all()  # :207-222
    fine = orc.init_next_level(np.full((2, 2), 5.0), np.zeros((2, 2), np.uint8), 4, 4)
    assert (fine == 0.0).all()  # :224-229
    small = np.array([[1.0, 2.0], [3.0, 4.0]])
    full, ok = orc.upsample_to_full(small, np.ones((2, 2), np.uint8), 8, 8, 2, 2.0)
    assert full[0, 0] == 4.0 and full[3, 3] == 4.0 and full[0, 4] == 8.0  # :231-252
    assert full[4, 0] == 12.0 and full[7, 7] == 16.0 and ok.sum() == 64
    v = np.ones((2, 2), np.uint8)
    v[1, 1] = 0
    _, ok = orc.upsample_to_full(np.ones((2, 2)), v, 4, 4, 1, 2.0)
    assert ok[0, 0] and not ok[2, 2] and not ok[3, 3]  # :254-261


def test_validate_rejects(orc):
    assert orc.validate(pyoracle.Config())[0] == 0  # :302-339
    bad = [dict(patch_size=1), dict(overlap=1.0), dict(min_iterations=13), dict(finest_exp=6),
           dict(window_offsets=[0.5, 0.5]), dict(window_offsets=[-0.5, 1.0]),
           dict(window_offsets=[]), dict(pixel_threshold=1.5), dict(valid_patch_ratio=0.0),
           dict(threads=0), dict(gamma=-0.1)]
    for kw in bad:
        assert orc.validate(pyoracle.Config(**kw))[0] == 2, kw


# ---- tests/test_depth_variance.cpp
def test_depth_and_sigma(orc):
    d, dv, _, _ = orc.disparity_to_depth(np.full((1, 2), 10.0), np.ones((1, 2), np.uint8),
                                         500.0, 5.0)
    assert d[0, 0] == pytest.approx(250.0, rel=1e-12)  # :30-35
    disp = np.array([[10.0, 0.05, 10.0]])
    d, dv, _, _ = orc.disparity_to_depth(disp, np.array([[1, 1, 0]], np.uint8), 500.0, 5.0)
    assert dv.tolist() == [[1, 0, 0]]  # :37-45
    d, dv, s, sv = orc.disparity_to_depth(np.full((1, 2), 10.0), np.ones((1, 2), np.uint8),
                                          500.0, 5.0, var=np.ones((1, 2)),
                                          var_valid=np.array([[1, 0]], np.uint8))
    assert s[0, 0] == pytest.approx(25.0, rel=1e-12) and dv[0, 1] and not sv[0, 1]  # :47-58


def test_components_and_filter(orc):
    v = np.zeros((4, 8), np.uint8)  # :60-84
    for x, y in [(0, 0), (1, 0), (2, 0), (3, 1), (4, 1), (4, 2), (7, 3)]:
        v[y, x] = 1
    k = orc.remove_small_components(v, 3)
    assert k[0, 0] and k[0, 2] and k[1, 3] and k[2, 4] and not k[3, 7]
    k = orc.remove_small_components(v, 4)
    assert not k[0, 0] and not k[1, 3]
    prob = np.full((20, 40), 0.5)  # :86-108
    prob[:, 30:32] = 0.05
    prob[8:20, 32:40] = 0.05
    prob[0:8, 32:40] = 0.5
    prob[8:, 32:] = 0.05
    out = orc.filter_validity(np.ones((20, 40), np.uint8), prob, np.ones((20, 40), np.uint8),
                              0.75, 0.15, 10)
    assert out[0, 0] and not out[5, 31] and not out[2, 35]
    loose = orc.filter_validity(np.ones((20, 40), np.uint8), prob, np.ones((20, 40), np.uint8),
                                0.0, 0.15, 10)
    assert loose[2, 35]


def test_gauss_newton_fit(orc):
    offs = [-1.0, -0.5, 0.0, 0.5, 1.0]

    def pri(c, s):
        return [c * math.exp(-o * o / (2 * s * s)) for o in offs]

    f = orc.estimate_variance(offs, pri(0.8, 2.0))  # :119-128
    assert f["accepted"] and f["reason"] == "none"
    assert f["sigma_k"] == pytest.approx(2.0, rel=1e-6) and f["c_k"] == pytest.approx(0.8, rel=1e-6)
    assert f["fit_residual"] < 1e-8
    for s in (0.4, 0.7, 1.5, 3.0):  # :130-138
        f = orc.estimate_variance(offs, pri(0.6, s))
        assert f["accepted"] and f["sigma_k"] == pytest.approx(s, rel=1e-5)
    f = orc.estimate_variance(offs, [0.5] * 5)  # :140-146
    assert not f["accepted"] and f["reason"] == "not_gaussian" and f["sigma_k"] == 2.0
    f = orc.estimate_variance(offs, [0.9, 0.5, 0.8, 0.5, 0.3])
    assert f["reason"] == "not_gaussian"  # :148-153
    f = orc.estimate_variance(offs, [0.9, 0.2, 1.0, 0.2, 0.9])  # :155-162
    assert f["reason"] == "residual_too_large" and f["fit_residual"] > 0.1 and f["sigma_k"] == 2.0
    f = orc.estimate_variance(offs, pri(0.8, 1.0), valid=[0, 0, 1, 1, 0])
    assert not f["accepted"] and f["reason"] == "not_gaussian"  # :164-171
    assert orc.estimate_variance(offs, [0.5] * 5, fallback=3.5)["sigma_k"] == 3.5


def test_gn_recovery_rate(orc):
    """acceptance.cpp:470-518: >= 990/1000 planted Gaussians recovered."""
    rng = np.random.default_rng(1234)
    offs = [-1.0, -0.5, 0.0, 0.5, 1.0]
    ok = 0
    for _ in range(1000):
        c, s = rng.uniform(0.2, 1.0), rng.uniform(0.3, 3.0)
        f = orc.estimate_variance(offs, [c * math.exp(-o * o / (2 * s * s)) for o in offs])
        ok += f["accepted"] and abs(f["sigma_k"] - s) < 1e-4 * s
    assert ok >= 990


# ---- compute_metrics (tests/test_metrics.cpp:9-84) ----

def _fields(vals, valid=None):
    v = np.asarray(vals, np.float64)[None, :]
    ok = np.ones_like(v, np.uint8) if valid is None else np.asarray(valid, np.uint8)[None, :]
    return v, ok


def test_metrics_kats(orc):
    est, ok = _fields([1.0, 2.0, 9.0])
    z = np.zeros_like(est)
    m = orc.compute_metrics(est, ok, z, ok)  # :9-23
    assert m["has_errors"] and m["mean_err"] == 4.0 and m["median_err"] == 2.0
    assert m["valid_px"] == 3 and np.isnan(m["coverage_rate"])
    est, ok = _fields([1.0, 2.0, 4.0, 9.0])  # :25-34 even count
    assert orc.compute_metrics(est, ok, np.zeros_like(est), ok)["median_err"] == 3.0
    e = np.full((8, 8), 3.0)  # :36-43 exact
    ok8 = np.ones((8, 8), np.uint8)
    m = orc.compute_metrics(e, ok8, e, ok8)
    assert m["mean_err"] == 0.0 and m["median_err"] == 0.0 and m["valid_px"] == 64
    est, ev = _fields([100.0, 5.0, 5.0], [0, 1, 1])  # :45-55 masks
    ref, rv = _fields([5.0, 5.0, 5.0], [1, 0, 1])
    m = orc.compute_metrics(est, ev, ref, rv)
    assert m["mean_err"] == 0.0 and m["valid_px"] == 2
    est, ev = _fields([1.0, 1.0], [0, 0])  # :57-65 nothing comparable
    m = orc.compute_metrics(est, ev, est, np.ones_like(ev))
    assert not m["has_errors"] and np.isnan(m["mean_err"]) and np.isnan(m["median_err"])
    assert m["valid_px"] == 0
    est, ok = _fields([1.0, -1.5, 2.5, 1.96])  # :67-76 coverage, boundary inclusive
    m = orc.compute_metrics(est, ok, np.zeros_like(est), ok, np.ones_like(est), ok)
    assert m["coverage_rate"] == 0.75
    est, ok = _fields([0.5, 0.5])  # :78-84 missing sigma counts as a miss
    m = orc.compute_metrics(est, ok, np.zeros_like(est), ok, np.ones_like(est),
                            np.array([[1, 0]], np.uint8))
    assert m["coverage_rate"] == 0.5


def test_metrics_port_matches_reference():
    if not pyoracle.available("reference"):
        pytest.skip("oracle/_ref not built")
    port, ref = pyoracle.load("port"), pyoracle.load("reference")
    rng = np.random.default_rng(5)
    for h, w in ((1, 1), (7, 9), (64, 48), (240, 320)):
        for quant in (None, 0.25):
            est = rng.normal(0, 3, (h, w))
            gt = rng.normal(0, 3, (h, w))
            if quant:
                est, gt = np.round(est / quant) * quant, np.round(gt / quant) * quant  # ties
            sig = np.abs(rng.normal(1, 1, (h, w)))
            ev = (rng.random((h, w)) < 0.8).astype(np.uint8)
            rv = (rng.random((h, w)) < 0.9).astype(np.uint8)
            sv = (rng.random((h, w)) < 0.7).astype(np.uint8)
            a = port.compute_metrics(est, ev, gt, rv, sig, sv)
            b = ref.compute_metrics(est, ev, gt, rv, sig, sv)
            for k in a:
                assert (np.isnan(a[k]) and np.isnan(b[k])) or a[k] == b[k], (h, w, k)
