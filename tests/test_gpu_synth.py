"""On-device generator: pstereo_gpu_synth must write the
same bytes as the host generator pstereo_synth_pair for every BASELINE.json
configuration (both evaluate csrc/synth_core.h with IEEE-exact operations)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _host(P, config, n, seed0, **kw):
    outs = [P.synth_pair(config, seed=seed0 + k, with_disparity=True, **kw) for k in range(n)]
    return [np.stack([o[i] for o in outs]) for i in range(3)]


def _check(P, config, n, seed0, **kw):
    hl, hr, hd = _host(P, config, n, seed0, **kw)
    gl, gr, gd = P.synth_batch_gpu(config, n, seed0=seed0, with_disparity=True, **kw)
    gl, gr, gd = gl.cpu().numpy(), gr.cpu().numpy(), gd.cpu().numpy()
    assert gl.shape == hl.shape and gr.shape == hr.shape
    assert np.array_equal(gd.view(np.uint32), hd.view(np.uint32)), "disparity bits differ"
    assert np.array_equal(gl, hl), f"left differs at {np.argwhere(gl != hl)[:5]}"
    assert np.array_equal(gr, hr), f"right differs at {np.argwhere(gr != hr)[:5]}"


def test_config0_full_size(gpu):
    _check(gpu, 0, 2, 0)


def test_config1_stress_full_size(gpu):
    _check(gpu, 1, 2, 1)


def test_config3_full_size(gpu):
    _check(gpu, 3, 1, 0)


def test_rgb_and_odd_sizes(gpu):
    _check(gpu, 0, 2, 11, width=320, height=240, channels=3)
    _check(gpu, 1, 2, 7, width=97, height=61, channels=3, blur_sigma=5.0)
    _check(gpu, 0, 1, 3, width=1920, height=1080, channels=3)


def test_chunk_boundary_and_empty(gpu):
    # 70 pairs cross the 64-pair scratch chunk
    _check(gpu, 0, 70, 100, width=64, height=48, blur_sigma=4.0)
    l, r = gpu.synth_batch_gpu(0, 0)
    assert l.shape[0] == 0 and r.shape[0] == 0


def test_bad_spec_is_config_error(gpu):
    with pytest.raises(gpu.ConfigError):
        gpu.synth_batch_gpu(0, 1, channels=2)


@pytest.mark.parametrize("seed", range(4))
def test_randomized_specs(gpu, seed):
    """Random generator specs (sizes, channels, octaves, wavelengths, blur,
    disparity range, noise, stress): byte-identical to the host."""
    rng = np.random.default_rng(2000 + seed)
    for _ in range(3):
        kw = dict(width=int(rng.integers(8, 300)), height=int(rng.integers(8, 200)),
                  channels=int(rng.choice([1, 3])), octaves=int(rng.integers(1, 7)),
                  base_wavelength=float(rng.uniform(2, 80)),
                  d_min=float(rng.uniform(0, 10)), d_range=float(rng.uniform(0, 40)),
                  blur_sigma=float(rng.uniform(0.5, 30)), noise_sigma=float(rng.uniform(0, 5)),
                  stress=int(rng.integers(0, 2)))
        _check(gpu, 0, int(rng.integers(1, 4)), int(rng.integers(0, 2**40)), **kw)
