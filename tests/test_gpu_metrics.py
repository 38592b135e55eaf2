"""compute_metrics on the GPU (src/metrics.cpp:10-52)
against the CPU oracle: the reference's own cases (tests/test_metrics.cpp),
randomised fields with masks and ties, batches, and the pipeline's depth
against the generator's ground truth. Every field must be identical (the mean
is the reference's sequential sum, the median an exact order statistic)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _same(a, b):
    for k in ("valid_px", "compared", "mean_err", "median_err", "coverage_rate"):
        x, y = a[k], b[k]
        assert (np.isnan(x) and np.isnan(y)) or x == y, (k, x, y)
    assert bool(a["has_errors"]) == bool(b["has_errors"])


def test_reference_cases(gpu, port):
    P = gpu
    cases = [
        ([1.0, 2.0, 9.0], None, [0, 0, 0], None, None, None),
        ([1.0, 2.0, 4.0, 9.0], None, [0, 0, 0, 0], None, None, None),
        ([100.0, 5.0, 5.0], [0, 1, 1], [5.0, 5.0, 5.0], [1, 0, 1], None, None),
        ([1.0, 1.0], [0, 0], [1.0, 1.0], None, None, None),
        ([1.0, -1.5, 2.5, 1.96], None, [0, 0, 0, 0], None, [1, 1, 1, 1], None),
        ([0.5, 0.5], None, [0, 0], None, [1.0, 1.0], [1, 0]),
    ]
    for est, ev, ref, rv, sg, sv in cases:
        e = np.array([est], np.float64)
        ones = np.ones_like(e, np.uint8)
        ev_ = ones if ev is None else np.array([ev], np.uint8)
        r = np.array([ref], np.float64)
        rv_ = ones if rv is None else np.array([rv], np.uint8)
        s = None if sg is None else np.array([sg], np.float64)
        sv_ = None if sg is None else (ones if sv is None else np.array([sv], np.uint8))
        _same(P.compute_metrics(e, ev_, r, rv_, s, sv_), port.compute_metrics(e, ev_, r, rv_, s, sv_))


@pytest.mark.parametrize("h,w", [(1, 1), (3, 5), (61, 47), (480, 640), (1080, 1920)])
@pytest.mark.parametrize("quant", [None, 0.125])
def test_random_fields(gpu, port, h, w, quant):
    P = gpu
    rng = np.random.default_rng(h * 7 + w)
    est = rng.normal(0, 4, (h, w))
    ref = rng.normal(0, 4, (h, w))
    if quant:  # many equal errors: ties at the median
        est, ref = np.round(est / quant) * quant, np.round(ref / quant) * quant
    sig = np.abs(rng.normal(1, 2, (h, w)))
    ev = (rng.random((h, w)) < 0.85).astype(np.uint8)
    rv = (rng.random((h, w)) < 0.9).astype(np.uint8)
    sv = (rng.random((h, w)) < 0.6).astype(np.uint8)
    _same(P.compute_metrics(est, ev, ref, rv, sig, sv), port.compute_metrics(est, ev, ref, rv, sig, sv))
    _same(P.compute_metrics(est, ev, ref, rv), port.compute_metrics(est, ev, ref, rv))


def test_batch_of_frames(gpu, port):
    P = gpu
    rng = np.random.default_rng(3)
    n, h, w = 6, 120, 160
    est = rng.gamma(2.0, 1.0, (n, h, w))
    ref = rng.gamma(2.0, 1.0, (n, h, w))
    ev = (rng.random((n, h, w)) < 0.7).astype(np.uint8)
    rv = np.ones((n, h, w), np.uint8)
    ev[2] = 0  # a frame with nothing comparable
    ev[3] = 0
    ev[3, 5, 7] = 1  # exactly one comparable pixel
    got = P.compute_metrics(est, ev, ref, rv)
    for k in range(n):
        _same(got[k], port.compute_metrics(est[k], ev[k], ref[k], rv[k]))


def test_pipeline_depth_against_ground_truth(gpu, port):
    """The reference's benchmark use (src/bench.cpp:27-30): depth and its sigma
    from run_pipeline against a ground-truth depth field."""
    P = gpu
    l, r, disp = P.synth_pair(1, seed=3, width=320, height=240, with_disparity=True)
    cfg = P.PipelineConfig(coarsest_exp=3, finest_exp=1, patch_size=8, overlap=0.5,
                           estimate_variance=True)
    focal, base = 500.0, 5.0
    with P.Matcher(cfg, 320, 240, 1) as m:
        out = m.run_batch(l[None], r[None], focal=focal, baseline=base, dtype=P.F64,
                          want=["depth", "depth_valid", "depth_sigma", "sigma_valid"])
        gt = np.where(disp >= 0.1, focal * base / np.maximum(disp.astype(np.float64), 1e-9), 0.0)
        gv = (disp >= 0.1).astype(np.uint8)
        got = m.metrics(out["depth"][0], out["depth_valid"][0], gt, gv, out["depth_sigma"][0],
                        out["sigma_valid"][0])
    want = port.compute_metrics(out["depth"][0], out["depth_valid"][0], gt, gv,
                                out["depth_sigma"][0], out["sigma_valid"][0])
    _same(got, want)
    assert got["has_errors"] and got["compared"] > 1000
