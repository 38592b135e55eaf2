"""GPU parity: the sm_100a path through the C ABI against the reference itself
(oracle/_ref, the unmodified reference sources; the plain-C restatement
oracle/bdis_oracle.c, pinned bit-exact to it, where _ref was not built) on the
same seeded inputs. Bit-exact except var_disp / depth sigma (1e-3 rel, see
tests/parity.py)."""
import os

import numpy as np
import pytest

from tests.parity import compare_pair, random_case, run_gpu_batch, run_oracle

pytestmark = pytest.mark.gpu

FOCAL, BASELINE = 500.0, 5.0


def _check(P, checker, cfg, left_u8, right_u8, lv=None, rv=None):
    """left_u8/right_u8: [n,h,w(,c)] uint8 rasters."""
    gpu = run_gpu_batch(P, cfg, left_u8, right_u8, FOCAL, BASELINE)
    out = []
    for k in range(left_u8.shape[0]):
        lf, lvk = checker.to_grayscale(left_u8[k])
        rf, rvk = checker.to_grayscale(right_u8[k])
        pipe, match = run_oracle(checker, lf, rf, cfg, FOCAL, BASELINE, lvk, rvk)
        out.append(compare_pair(gpu, k, pipe, match, cfg))
    return out


def test_config0_pair_bitexact(gpu, checker):
    P = gpu
    l, r = P.synth_pair(0)
    _check(P, checker, P.PipelineConfig.baseline(0), l[None], r[None])


def test_config1_stress_variance(gpu, checker):
    P = gpu
    l, r = P.synth_pair(1)
    st = _check(P, checker, P.PipelineConfig.baseline(1), l[None], r[None])
    print("config1 agreement", st)


def test_reference_defaults(gpu, checker):
    P = gpu
    l, r = P.synth_pair(0, seed=7)
    _check(P, checker, P.PipelineConfig(), l[None], r[None])


def test_batch_of_seeds(gpu, checker):
    P = gpu
    left, right = P.synth_batch(0, 4, seed0=10, width=320, height=240)
    _check(P, checker, P.PipelineConfig.baseline(0), left, right)


@pytest.mark.parametrize("size,stride", [(8, 2), (12, 4), (16, 6), (10, 5), (9, 3)])
def test_patch_size_stride_sweep(gpu, checker, size, stride):
    P = gpu
    l, r = P.synth_pair(0, seed=3, width=200, height=150)
    cfg = P.PipelineConfig(coarsest_exp=2, finest_exp=1, patch_size=size,
                           overlap=1.0 - stride / size, estimate_variance=True)
    _check(P, checker, cfg, l[None], r[None])


@pytest.mark.parametrize("w,h", [(97, 75), (64, 48), (33, 17)])
def test_odd_dimensions(gpu, checker, w, h):
    P = gpu
    l, r = P.synth_pair(0, seed=5, width=w, height=h, blur_sigma=8.0, d_range=6.0, d_min=1.0)
    cfg = P.PipelineConfig(coarsest_exp=1, finest_exp=0, patch_size=6, overlap=0.5,
                           estimate_variance=True)
    _check(P, checker, cfg, l[None], r[None])


@pytest.mark.parametrize("w,h", [(97, 75), (131, 67)])
def test_odd_dimensions_upsampled(gpu, checker, w, h):
    """Odd full-resolution sizes with finest_exp 1: the last finest column/row
    covers one full-resolution pixel, which the component areas must weigh."""
    P = gpu
    l, r = P.synth_pair(0, seed=6, width=w, height=h, blur_sigma=8.0, d_range=6.0, d_min=1.0)
    cfg = P.PipelineConfig(coarsest_exp=2, finest_exp=1, patch_size=6, overlap=0.5,
                           estimate_variance=True, gamma=0.05)
    _check(P, checker, cfg, l[None], r[None])


def test_rgb_and_rgba_validity(gpu, checker):
    P = gpu
    l, r = P.synth_pair(0, seed=11, width=160, height=120, channels=3)
    cfg = P.PipelineConfig(coarsest_exp=2, finest_exp=1, patch_size=8, overlap=0.5)
    _check(P, checker, cfg, l[None], r[None])
    # RGBA: alpha == 0 marks invalid pixels (src/image.cpp:32-34)
    rng = np.random.default_rng(0)
    la = np.concatenate([l, np.full(l.shape[:2] + (1,), 255, np.uint8)], axis=2)
    ra = np.concatenate([r, np.full(r.shape[:2] + (1,), 255, np.uint8)], axis=2)
    la[30:60, 40:80, 3] = 0
    ra[rng.random(ra.shape[:2]) < 0.01, 3] = 0
    _check(P, checker, cfg, la[None], ra[None])


def test_float_api_with_mask(gpu, checker):
    """GrayImage entry point with an explicit validity mask."""
    P = gpu
    l, r = P.synth_pair(0, seed=2, width=128, height=96)
    lf, _ = checker.to_grayscale(l)
    rf, _ = checker.to_grayscale(r)
    lv = np.ones_like(l, np.uint8)
    lv[:, 100:] = 0
    cfg = P.PipelineConfig(coarsest_exp=2, finest_exp=1, patch_size=8, overlap=0.5,
                           estimate_variance=True)
    gpu_out = run_gpu_batch(P, cfg, lf[None], rf[None], FOCAL, BASELINE, left_valid=lv[None])
    pipe, match = run_oracle(checker, lf, rf, cfg, FOCAL, BASELINE, lv, None)
    compare_pair(gpu_out, 0, pipe, match, cfg)


def test_shifted_analytic_pair(gpu, checker):
    """The reference's own end-to-end case (tests/test_coarse_to_fine.cpp:253-287):
    64x48 sinusoid pair shifted by 2 px, exps 2..1, recovered within 0.2 px."""
    P = gpu
    y, x = np.mgrid[0:48, 0:64].astype(np.float64)

    def tex(xx):
        return (0.5 + 0.2 * np.sin(xx * 0.37 + 0.8) + 0.15 * np.sin(y * 0.29)
                + 0.1 * np.sin((xx + y) * 0.143)).astype(np.float32)

    left, right = tex(x), tex(x + 2.0)
    cfg = P.PipelineConfig(coarsest_exp=2, finest_exp=1)
    res = P.match_stereo(left, right, cfg)
    st = res["stats"]
    assert st[0][0] == 2 and st[1][0] == 1
    assert all(s[4] > 0 for s in st)
    valid = res["disparity_valid"].astype(bool)
    assert valid.sum() > 64 * 48 / 2
    assert np.abs(res["disparity"][valid] - 2.0).max() < 0.2
    pipe, match = run_oracle(checker, left, right, cfg, 1.0, 1.0)
    np.testing.assert_array_equal(res["disparity"], match["disparity"])


def test_config3_full_size(gpu, checker):
    """BASELINE config 3: 1280x1024, exps 4..1, 12x12 patches stride 4,
    variance on -- the largest single-pair configuration."""
    P = gpu
    l, r = P.synth_pair(3)
    _check(P, checker, P.PipelineConfig.baseline(3), l[None], r[None])


@pytest.mark.parametrize("w,h,ch,size,stride", [
    (320, 240, 3, 8, 2), (320, 240, 3, 12, 6), (320, 240, 1, 16, 4), (640, 480, 3, 12, 2),
    pytest.param(1920, 1080, 3, 16, 6, marks=pytest.mark.slow),
])
def test_config4_sweep(gpu, checker, w, h, ch, size, stride):
    """BASELINE config 4: sizes x patch sizes x strides, RGB through the
    Rec.601 conversion (src/image.cpp:36)."""
    P = gpu
    l, r = P.synth_pair(4, seed=size * 10 + stride, width=w, height=h, channels=ch)
    cfg = P.PipelineConfig(coarsest_exp=3, finest_exp=1, patch_size=size,
                           overlap=1.0 - stride / size)
    _check(P, checker, cfg, l[None], r[None])


@pytest.mark.parametrize("w,h,ch,size,stride,n", [
    (640, 480, 1, 16, 4, 16),    # starving bands -> one 256-thread CTA per SM
    (640, 480, 3, 8, 2, 12),     # dense wide grid
    (1280, 1024, 3, 8, 4, 6),    # wide s=8 levels, vectorised RGB pyramid
])
def test_planner_shapes_batches(gpu, checker, w, h, ch, size, stride, n):
    """Batches large enough that the band planner keeps its tall-band shapes
    (s >= 12 starving bands, dense or wide grids) and the RGB pyramid path:
    every pair bit-identical to the oracle."""
    P = gpu
    left, right = P.synth_batch(4, n, seed0=50 + size, width=w, height=h, channels=ch)
    cfg = P.PipelineConfig(coarsest_exp=4, finest_exp=1, patch_size=size,
                           overlap=1.0 - stride / size)
    _check(P, checker, cfg, left, right)


def test_empty_batch_and_limits(gpu):
    """n = 0 is a no-op; frames larger than the context's maximum are refused."""
    P = gpu
    cfg = P.PipelineConfig.baseline(0)
    with P.Matcher(cfg, 160, 120, 2) as m:
        out = m.run_batch(np.zeros((0, 120, 160), np.uint8), np.zeros((0, 120, 160), np.uint8))
        assert out["disparity"].shape == (0, 120, 160)
        with pytest.raises(P.GpuError):
            m.run_batch(np.zeros((1, 240, 320), np.uint8), np.zeros((1, 240, 320), np.uint8))


def test_determinism(gpu):
    P = gpu
    left, right = P.synth_batch(0, 2, seed0=0, width=320, height=240)
    cfg = P.PipelineConfig.baseline(1)
    a = run_gpu_batch(P, cfg, left, right, FOCAL, BASELINE)
    b = run_gpu_batch(P, cfg, left, right, FOCAL, BASELINE)
    for k in ("disparity", "disparity_valid", "depth", "var_disp"):
        assert np.array_equal(a[k], b[k]), k


def test_large_batch_determinism(gpu, checker):
    """Many CTAs per SM over several waves (stale shared memory from earlier
    CTAs, every SM busy): device-resident runs repeat bit-for-bit, the chunked
    host path agrees with them, and sampled pairs match the oracle."""
    import torch

    P = gpu
    n, w, h = 96, 320, 240
    left, right = P.synth_batch(0, n, seed0=40, width=w, height=h)
    cfg = P.PipelineConfig.baseline(0)
    dev = torch.device("cuda", 0)
    dl, dr = torch.from_numpy(left).to(dev), torch.from_numpy(right).to(dev)
    with P.Matcher(cfg, w, h, n) as m:
        runs = []
        for _ in range(2):
            d = torch.empty((n, h, w), dtype=torch.float32, device=dev)
            m.run_device_u8(n, w, h, 1, dl.data_ptr(), dr.data_ptr(), {"disparity": d.data_ptr()},
                            invalid_value=float("nan"))
            torch.cuda.synchronize()
            runs.append(d.cpu().numpy())
        hd = np.empty((n, h, w), np.float32)
        m.run_host_u8(n, w, h, 1, left.ctypes.data, right.ctypes.data,
                      {"disparity": hd.ctypes.data}, invalid_value=float("nan"))
        torch.cuda.synchronize()
    for other in (runs[1], hd):
        assert np.array_equal(np.isnan(runs[0]), np.isnan(other))
        assert np.array_equal(np.nan_to_num(runs[0]), np.nan_to_num(other))
    for k in (0, n - 1):
        lf, lv = checker.to_grayscale(left[k])
        rf, rv = checker.to_grayscale(right[k])
        pipe, _ = run_oracle(checker, lf, rf, cfg, 1.0, 1.0, lv, rv)
        ov = np.asarray(pipe["disparity_valid"]).astype(bool)
        assert np.array_equal(~np.isnan(runs[0][k]), ov)
        od = np.asarray(pipe["disparity"]).astype(np.float32)
        assert np.array_equal(runs[0][k][ov], od[ov])


def test_errors(gpu):
    P = gpu
    with pytest.raises(P.ConfigError):
        P.Matcher(P.PipelineConfig(patch_size=1), 64, 48)
    m = P.Matcher(P.PipelineConfig(coarsest_exp=5, finest_exp=1, patch_size=10), 64, 48)
    l = np.zeros((1, 48, 64), np.uint8)
    with pytest.raises(P.DegenerateInputError):
        m.run_batch(l, l)  # 64x48 at 1/32 is 2x2 < 10 px (tests/test_pyramid.cpp:90-92)
    m.close()


def test_chunked_host_pipeline(gpu, monkeypatch):
    """Host buffers are pipelined in chunks over three streams; the result must
    not depend on the chunking."""
    P = gpu
    left, right = P.synth_batch(0, 7, seed0=20, width=160, height=120)
    cfg = P.PipelineConfig(coarsest_exp=2, finest_exp=1, patch_size=8, overlap=0.5,
                           estimate_variance=True)
    want = ["disparity", "disparity_valid", "depth", "depth_valid", "var_disp"]
    with P.Matcher(cfg, 160, 120, 7) as m:
        whole = m.run_batch(left, right, dtype=P.F64, want=want, stats=True)
    monkeypatch.setenv("PSTEREO_CHUNK_PAIRS", "3")
    with P.Matcher(cfg, 160, 120, 7) as m:
        parts = m.run_batch(left, right, dtype=P.F64, want=want, stats=True)
    for k in want + ["stats"]:
        assert np.array_equal(whole[k], parts[k]), k


def test_async_host_calls_overlap_safely(gpu):
    """async_host: back-to-back calls return once queued and overlap; after
    wait() every host plane equals the synchronous result."""
    import torch

    P = gpu
    n, w, h = 12, 160, 120
    cfg = P.PipelineConfig(coarsest_exp=2, finest_exp=1, patch_size=8, overlap=0.5)
    batches = [P.synth_batch(0, n, seed0=100 * k, width=w, height=h) for k in range(3)]
    with P.Matcher(cfg, w, h, n) as m:
        sync = []
        for left, right in batches:
            d = np.empty((n, h, w), np.float32)
            m.run_host_u8(n, w, h, 1, left.ctypes.data, right.ctypes.data,
                          {"disparity": d.ctypes.data}, invalid_value=float("nan"))
            sync.append(d)
        pinned = [(torch.from_numpy(l).pin_memory(), torch.from_numpy(r).pin_memory())
                  for l, r in batches]
        outs = [torch.empty((n, h, w), dtype=torch.float32).pin_memory() for _ in batches]
        for (hl, hr), d in zip(pinned, outs):
            m.run_host_u8(n, w, h, 1, hl.data_ptr(), hr.data_ptr(), {"disparity": d.data_ptr()},
                          invalid_value=float("nan"), async_host=True)
        m.wait()
    for a, b in zip(sync, outs):
        b = b.numpy()
        assert np.array_equal(np.isnan(a), np.isnan(b))
        assert np.array_equal(np.nan_to_num(a), np.nan_to_num(b))


def test_async_host_many_large_calls(gpu):
    """Eight back-to-back async_host calls on distinct 32-pair 640x480 batches,
    each with its own pinned outputs, one wait() at the end. The outputs are
    three f64 planes + a mask (26 B/px down against 2 B/px up), so each call's
    downloads take several times its uploads and kernels: call k+2 reuses the
    staging set call k is still downloading -- every host plane
    must still equal the synchronous result of its own batch."""
    import torch

    P = gpu
    n, w, h, calls = 32, 640, 480, 8
    cfg = P.PipelineConfig.baseline(0)
    planes = ("disparity", "disparity_valid", "probability", "depth")
    with P.Matcher(cfg, w, h, n) as m:
        batches = [P.synth_batch(0, n, seed0=1000 + k * n) for k in range(calls)]
        want = [m.run_batch(l, r, focal=500.0, baseline=5.0, dtype=P.F64, want=planes)
                for l, r in batches]
        pinned = [(torch.from_numpy(l).pin_memory(), torch.from_numpy(r).pin_memory())
                  for l, r in batches]
        outs = [{k: torch.full((n, h, w), 7, dtype=torch.uint8 if "valid" in k
                               else torch.float64).pin_memory() for k in planes}
                for _ in range(calls)]
        for (hl, hr), o in zip(pinned, outs):
            m.run_host_u8(n, w, h, 1, hl.data_ptr(), hr.data_ptr(),
                          {k: v.data_ptr() for k, v in o.items()}, dtype=P.F64, focal=500.0,
                          baseline=5.0, async_host=True)
        m.wait()
    for k in range(calls):
        for name in planes:
            a = want[k][name]
            b = outs[k][name].numpy()
            assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), (k, name)


def test_device_sub_batches_are_invisible(gpu):
    """A device call split into sub-batches over two compute streams
    (pstereo_gpu_set_device_chunks, default 2 for >= 32 pairs) writes exactly
    what one launch sequence writes, for any split."""
    import torch

    P = gpu
    n, w, h = 70, 160, 120
    cfg = P.PipelineConfig(coarsest_exp=3, finest_exp=1, patch_size=8, overlap=0.5,
                           estimate_variance=True)
    dl, dr = P.synth_batch_gpu(1, n, seed0=300, width=w, height=h)
    names = ("disparity", "disparity_valid", "depth", "depth_sigma", "var_disp")
    res = {}
    with P.Matcher(cfg, w, h, n) as m:
        for chunks in (1, 2, 3, 5):
            m.set_device_chunks(chunks)
            outs = {k: torch.full((n, h, w), 7, dtype=torch.uint8 if "valid" in k
                                  else torch.float64, device="cuda") for k in names}
            m.run_device_u8(n, w, h, 1, dl.data_ptr(), dr.data_ptr(),
                            {k: v.data_ptr() for k, v in outs.items()}, dtype=P.F64,
                            focal=500.0, baseline=5.0)
            torch.cuda.synchronize()
            res[chunks] = {k: v.cpu().numpy() for k, v in outs.items()}
    for chunks in (2, 3, 5):
        for k in names:
            a, b = res[1][k], res[chunks][k]
            assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), (chunks, k)


def test_disparity_only_output_path(gpu, checker):
    """Requests of the disparity plane alone (+ validity) take a dedicated
    output kernel: same values as the full-plane request and the oracle."""
    P = gpu
    left, right = P.synth_batch(0, 3, seed0=70, width=320, height=240)
    cfg = P.PipelineConfig(coarsest_exp=3, finest_exp=1, patch_size=8, overlap=0.5)
    full = ["disparity", "disparity_valid", "probability", "depth", "depth_valid"]
    with P.Matcher(cfg, 320, 240, 3) as m:
        for dt in (P.F32, P.F64):
            a = m.run_batch(left, right, 500.0, 5.0, dtype=dt, want=full)
            b = m.run_batch(left, right, 500.0, 5.0, dtype=dt, want=("disparity", "disparity_valid"))
            c = m.run_batch(left, right, 500.0, 5.0, dtype=dt, want=("disparity",),
                            invalid_value=-1.0, flip_rows=True)
            assert np.array_equal(a["disparity"], b["disparity"])
            assert np.array_equal(a["disparity_valid"], b["disparity_valid"])
            want_c = np.where(a["disparity_valid"] != 0, a["disparity"], -1.0)[:, ::-1]
            assert np.array_equal(c["disparity"], want_c.astype(c["disparity"].dtype))
    _check(P, checker, cfg, left, right)


def test_invalid_value_fill(gpu):
    """fill_invalid writes the PFM-style sentinel (src/io.cpp:297-310) into
    invalid disparity/depth pixels and leaves valid ones untouched."""
    P = gpu
    left, right = P.synth_batch(1, 2, seed0=1, width=160, height=120)
    cfg = P.PipelineConfig.baseline(1)
    want = ["disparity", "disparity_valid", "depth", "depth_valid", "depth_sigma",
            "sigma_valid", "match_disparity"]
    with P.Matcher(cfg, 160, 120, 2) as m:
        a = m.run_batch(left, right, focal=500.0, baseline=5.0, want=want)
        b = m.run_batch(left, right, focal=500.0, baseline=5.0, want=want, invalid_value=-1.0)
    for plane, ok in (("disparity", "disparity_valid"), ("depth", "depth_valid"),
                      ("depth_sigma", "sigma_valid")):
        v = a[ok].astype(bool)
        assert np.array_equal(b[plane][v], a[plane][v])
        assert (b[plane][~v] == -1.0).all()
    assert np.array_equal(a["match_disparity"], b["match_disparity"])
    assert (~a["disparity_valid"].astype(bool)).any()


@pytest.mark.parametrize("seed", range(int(os.environ.get("PSTEREO_RANDOM_CASES", "16"))))
def test_randomized_configs(gpu, checker, seed):
    """Random valid PipelineConfigs and frame sizes (patch sizes 2..20, any
    stride, 1..4 levels, window offsets, thresholds, variance on/off, gray,
    RGB or RGBA with holes): bit-exact against the reference every time."""
    P = gpu
    cfg, l, r = random_case(P, seed)
    _check(P, checker, cfg, l[None], r[None])


def test_ccl_sure_chains(gpu, checker):
    """Components that cross 32x64 finest tiles as sure / not-sure / sure
    pieces (k_ccl_border skips unions between two sure pieces): the
    inputs hold such chains (tests/test_ccl_chains.py pins that on CPU) and
    every output, the validity masks first, equals the reference's."""
    from oracle import pyoracle
    from tests.ccl_chains import CASES, chain_count

    chains = 0
    for thr, gamma, seed in CASES:
        cfg = gpu.PipelineConfig(coarsest_exp=3, finest_exp=1, patch_size=8, overlap=0.5,
                                 pixel_threshold=thr, gamma=gamma)
        left, right = pyoracle.synth_batch(1, 1, seed0=seed)
        out = run_gpu_batch(gpu, cfg, left, right, 500.0, 5.0)
        lf, lv = checker.to_grayscale(left[0])
        rf, rv = checker.to_grayscale(right[0])
        pipe, match = run_oracle(checker, lf, rf, cfg, 500.0, 5.0, lv, rv)
        compare_pair(out, 0, pipe, match, cfg)
        chains += chain_count(match["probability"], match["disparity_valid"], thr, gamma, 8)
    assert chains >= 4


@pytest.mark.parametrize("w,h,size,overlap,levels", [
    (2048, 256, 32, 0.75, 2),   # s = 32 (the cap): one patch row of the level needs 413 KB of
                                # shared memory -> the global-memory instantiation
    (1536, 192, 24, 0.5, 2),    # runtime size 24 (the 32-entry instantiation), global path
    (640, 480, 32, 0.75, 2),    # s = 32 at the bench size
])
def test_max_patch_and_global_memory_path(gpu, checker, w, h, size, overlap, levels):
    """Patch sizes at the cap (32) and runtime sizes whose level bands do not
    fit in shared memory: the k_patches global-memory instantiation, bit for
    bit against the reference (a gray pair and an RGBA pair with holes)."""
    P = gpu
    cfg = P.PipelineConfig(coarsest_exp=levels, finest_exp=1, patch_size=size, overlap=overlap)
    l, r = P.synth_batch(4, 1, seed0=5, width=w, height=h, channels=1)
    _check(P, checker, cfg, l, r)
    l3, r3 = P.synth_batch(4, 1, seed0=6, width=w, height=h, channels=3)
    alpha = np.full((1, h, w, 1), 255, np.uint8)
    l4, r4 = np.concatenate([l3, alpha], 3), np.concatenate([r3, alpha], 3)
    l4[0, h // 3:h // 2, w // 5:w // 4, 3] = 0  # an invalid block (alpha 0)
    _check(P, checker, cfg, l4, r4)
