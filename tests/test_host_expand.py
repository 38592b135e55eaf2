"""Host-side replication of upsample_to_full (src/coarse_to_fine.cpp:166-180):
host-output calls download finest-resolution planes and a host thread pool
writes the 2^e x 2^e blocks (csrc/host_expand.cpp). CPU tests pin the
replication against numpy; the GPU test requires identical bytes with the
device-side replication it replaces."""
import numpy as np
import pytest

import paper_2205_03133_b200 as P


def _numpy_expand(src, W, H, e, flip):
    n, fh, fw = src.shape
    ys = np.minimum(np.arange(H) >> e, fh - 1)
    xs = np.minimum(np.arange(W) >> e, fw - 1)
    out = src[:, ys][:, :, xs]
    return out[:, ::-1] if flip else out


def _half(v, e):
    for _ in range(e):
        v = (v + 1) // 2
    return v


@pytest.mark.parametrize("dtype", [np.uint8, np.float32, np.float64])
@pytest.mark.parametrize("W,H,e", [(640, 480, 1), (64, 48, 1), (66, 49, 1), (67, 50, 1), (61, 47, 2),
                                   (128, 96, 2), (33, 17, 3), (16, 16, 0), (2, 2, 1), (1, 1, 1)])
@pytest.mark.parametrize("flip", [False, True])
def test_host_expand_matches_numpy(dtype, W, H, e, flip):
    rng = np.random.default_rng(W * 1000 + H + e)
    fw, fh = _half(W, e), _half(H, e)
    n = 3
    if dtype == np.uint8:
        src = rng.integers(0, 256, (n, fh, fw), dtype=np.uint8)
    else:
        src = rng.standard_normal((n, fh, fw)).astype(dtype)
        src[rng.random((n, fh, fw)) < 0.2] = np.nan  # payload bits must survive
    got = P.host_expand(src, W, H, e, flip)
    want = _numpy_expand(src, W, H, e, flip)
    assert got.shape == (n, H, W)
    assert np.array_equal(got.view(np.uint8), np.ascontiguousarray(want).view(np.uint8))


def test_host_expand_unaligned_destination():
    """Rows that are not 32-byte aligned take the plain-store path."""
    import ctypes as C

    src = np.arange(5 * 12 * 20, dtype=np.float32).reshape(5, 12, 20)
    raw = np.zeros(5 * 24 * 40 * 4 + 64, np.uint8)
    off = (-raw.ctypes.data) % 32 + 4  # 4 bytes past a 32-byte boundary
    dst = raw[off:off + 5 * 24 * 40 * 4].view(np.float32).reshape(5, 24, 40)
    rc = P.lib().pstereo_host_expand(src.ctypes.data, dst.ctypes.data, 4, 20, 12, 40, 24, 1, 5, 0)
    assert rc == 0
    assert np.array_equal(dst, _numpy_expand(src, 40, 24, 1, False))
    assert C.sizeof(C.c_float) == 4


def test_host_expand_rejects_bad_geometry():
    src = np.zeros((1, 4, 4), np.float32)
    with pytest.raises(P.GpuError):
        P.host_expand(src, 9, 8, 1)  # 9 halves to 5, not 4
    assert P.lib().pstereo_gpu_host_threads() >= 1


@pytest.mark.gpu
@pytest.mark.parametrize("w,h,ce,fe,dtype", [(160, 120, 3, 1, "f32"), (160, 120, 3, 1, "f64"),
                                             (163, 121, 3, 1, "f64"), (200, 152, 3, 2, "f32"),
                                             (96, 72, 2, 0, "f64")])
def test_host_outputs_identical_with_and_without_host_expand(gpu, w, h, ce, fe, dtype):
    P = gpu
    n = 9
    left, right = P.synth_batch(1, n, seed0=40, width=w, height=h)
    cfg = P.PipelineConfig(coarsest_exp=ce, finest_exp=fe, patch_size=8, overlap=0.5,
                           estimate_variance=True)
    want = ["disparity", "disparity_valid", "probability", "depth", "depth_valid", "depth_sigma",
            "sigma_valid", "match_disparity", "match_valid", "var_disp"]
    dt = P.F64 if dtype == "f64" else P.F32
    res = {}
    with P.Matcher(cfg, w, h, n) as m:
        for on in (False, True):
            m.set_host_expand(on)
            for flip in (False, True):
                res[on, flip] = m.run_batch(left, right, focal=500.0, baseline=5.0, dtype=dt,
                                            want=want, flip_rows=flip, invalid_value=-1.0)
    for flip in (False, True):
        for k in want:
            a, b = res[False, flip][k], res[True, flip][k]
            assert a.shape == b.shape == (n, h, w)
            assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), (k, flip)
    # flipped rows are the unflipped planes bottom to top
    assert np.array_equal(res[True, True]["disparity"].view(np.uint8),
                          np.ascontiguousarray(res[True, False]["disparity"][:, ::-1]).view(np.uint8))


@pytest.mark.gpu
def test_async_calls_alternating_download_modes(gpu):
    """Back-to-back async_host calls that alternate between the
    finest-resolution download (+ host replication) and the full-resolution
    download share the context's staging sets; every call's planes must equal
    the synchronous result of its own batch."""
    import torch

    P = gpu
    n, w, h, calls = 24, 320, 240, 6
    cfg = P.PipelineConfig.baseline(0)
    planes = ("disparity", "disparity_valid", "probability")
    with P.Matcher(cfg, w, h, n) as m:
        batches = [P.synth_batch(0, n, seed0=500 + k * n, width=w, height=h) for k in range(calls)]
        want = [m.run_batch(l, r, dtype=P.F32, want=planes, invalid_value=-1.0) for l, r in batches]
        pinned = [(torch.from_numpy(l).pin_memory(), torch.from_numpy(r).pin_memory())
                  for l, r in batches]
        outs = [{k: torch.full((n, h, w), 7, dtype=torch.uint8 if "valid" in k
                               else torch.float32).pin_memory() for k in planes}
                for _ in range(calls)]
        for k, ((hl, hr), o) in enumerate(zip(pinned, outs)):
            m.set_host_expand(k % 2 == 0)
            m.run_host_u8(n, w, h, 1, hl.data_ptr(), hr.data_ptr(),
                          {q: v.data_ptr() for q, v in o.items()}, dtype=P.F32,
                          invalid_value=-1.0, async_host=True)
        m.wait()
    for k in range(calls):
        for name in planes:
            a, b = want[k][name], outs[k][name].numpy()
            assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), (k, name)
