"""pstereo_multi: pairs sharded over several device contexts.

The box has one GPU, so the shards are several contexts on device 0 (each
with its own host thread, streams and staging) -- the host-side splitting,
slicing of every output plane, stats and finest records, and the worker
threads are what is under test; results must equal one context matching the
whole batch, bit for bit."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

WANT = ("disparity", "disparity_valid", "probability", "depth", "depth_valid", "depth_sigma",
        "sigma_valid", "match_disparity", "match_valid", "var_disp")


@pytest.mark.parametrize("n_dev,n_pairs", [(2, 7), (3, 2), (4, 9)])
def test_multi_equals_single_context(gpu, n_dev, n_pairs):
    P = gpu
    cfg = P.PipelineConfig.baseline(1)  # variance on: every plane is produced
    left, right = P.synth_batch(1, n_pairs, seed0=11, width=320, height=240)
    kw = dict(focal=500.0, baseline=5.0, dtype=P.F64, want=WANT, stats=True, finest_cap=6000)
    with P.Matcher(cfg, 320, 240, n_pairs, device=0) as m:
        one = m.run_batch(left, right, **kw)
    with P.MultiMatcher(cfg, 320, 240, n_pairs, devices=[0] * n_dev) as mm:
        many = mm.run_batch(left, right, **kw)
        again = mm.run_batch(left[:1], right[:1], **kw)  # fewer pairs than devices
    assert len(many["ms_per_device"]) == n_dev
    for k in WANT:
        assert np.array_equal(one[k].view(np.uint8), many[k].view(np.uint8)), k
        assert np.array_equal(one[k][:1].view(np.uint8), again[k].view(np.uint8)), k
    assert np.array_equal(one["stats"], many["stats"])
    assert np.array_equal(one["finest_count"], many["finest_count"])
    for a, b in zip(one["finest"], many["finest"]):
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_multi_errors(gpu):
    P = gpu
    cfg = P.PipelineConfig.baseline(0)
    with P.MultiMatcher(cfg, 64, 48, 4, devices=[0, 0]) as mm:
        tiny = np.zeros((2, 20, 20), np.uint8)
        with pytest.raises(P.DegenerateInputError):
            mm.run_batch(tiny, tiny, stats=True)
    bad = P.PipelineConfig.baseline(0)
    bad.overlap = 1.5
    with pytest.raises(P.ConfigError):
        P.MultiMatcher(bad, 64, 48, 4, devices=[0])
