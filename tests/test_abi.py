"""CPU-side checks of the drop-in boundary: the C-ABI library loads without a
GPU, exports every entry point include/pstereo_gpu.h declares, validates
configs exactly like the reference, and reports errors with the reference's
exit-code classes -- no compute calls here."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle import pyoracle

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "pstereo_gpu.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pstereo_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_core_entry_points():
    fns = declared_functions()
    for f in ("pstereo_gpu_create", "pstereo_gpu_match_u8", "pstereo_gpu_match_f32",
              "pstereo_gpu_destroy", "pstereo_gpu_last_error", "pstereo_validate"):
        assert f in fns


def test_library_exports_every_declared_symbol(built):
    import paper_2205_03133_b200 as P

    lib = P.lib()
    missing = [f for f in declared_functions() if not hasattr(lib, f)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", str(P.LIB_PATH)], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r"\bT (pstereo_\w+)", out))
    assert set(declared_functions()) <= exported
    assert set(P.ABI_SYMBOLS) <= exported


def test_library_is_sm100a_only(built):
    import paper_2205_03133_b200 as P

    out = subprocess.run(["cuobjdump", "--list-elf", str(P.LIB_PATH)], capture_output=True,
                         text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_cpp_shim_compiles_and_links(built, tmp_path):
    """include/pstereo_gpu.hpp (reference-type C++ API) builds against the C ABI."""
    src = tmp_path / "t.cpp"
    src.write_text('#include "pstereo_gpu.hpp"\n'
                   "int main() { pstereo::gpu::PipelineConfig c; pstereo::gpu::validate(c);\n"
                   "  return c.patch_size == 10 ? 0 : 1; }\n")
    exe = tmp_path / "t"
    r = subprocess.run(["g++", "-std=c++17", "-I", str(ROOT / "include"), str(src), "-o", str(exe),
                        "-L", str(ROOT / "paper_2205_03133_b200"), "-lpstereo_gpu",
                        f"-Wl,-rpath,{ROOT / 'paper_2205_03133_b200'}"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert subprocess.run([str(exe)]).returncode == 0


BAD_CONFIGS = [dict(patch_size=1), dict(overlap=1.0), dict(overlap=-0.1), dict(min_iterations=0),
               dict(min_iterations=13), dict(finest_exp=6), dict(finest_exp=-1),
               dict(coarsest_exp=17, finest_exp=1), dict(window_offsets=[0.5, 0.5]),
               dict(window_offsets=[-0.5, 1.0]), dict(window_offsets=[]),
               dict(pixel_threshold=1.5), dict(valid_patch_ratio=0.0), dict(threads=0),
               dict(gamma=-0.1), dict(sigma_s=0.0), dict(early_stop_good=0.0),
               dict(early_stop_bad=0.0), dict(early_stop_improve=-1.0)]


@pytest.mark.parametrize("kw", BAD_CONFIGS + [dict()])
def test_validate_matches_reference(built, kw):
    import paper_2205_03133_b200 as P

    kind = "reference" if pyoracle.available("reference") else "port"
    rc, msg = pyoracle.load(kind).validate(pyoracle.Config(**kw))
    if rc == 0:
        P.validate(P.PipelineConfig(**kw))
    else:
        with pytest.raises(P.ConfigError) as e:
            P.validate(P.PipelineConfig(**kw))
        assert str(e.value) == msg


def test_gpu_patch_size_cap(built):
    import paper_2205_03133_b200 as P

    with pytest.raises(P.ConfigError):
        P.validate(P.PipelineConfig(patch_size=33, coarsest_exp=1, finest_exp=0))


def test_level_dims_and_degenerate(built):
    import paper_2205_03133_b200 as P

    dims = P.level_dims(P.PipelineConfig(), 640, 480)  # tests/test_pyramid.cpp:60-76
    assert dims[0] == (5, 20, 15) and dims[-1] == (1, 320, 240) and len(dims) == 5
    cfg = P.PipelineConfig.baseline(3)
    assert P.level_dims(cfg, 1920, 1080)[0] == (4, 120, 68)  # ceil halving of 1080 -> 68
    with pytest.raises(P.DegenerateInputError):
        P.level_dims(P.PipelineConfig(), 64, 48)  # tests/test_pyramid.cpp:90-92
    with pytest.raises(P.DegenerateInputError):
        P.level_dims(P.PipelineConfig(), 0, 0)


def test_create_without_gpu_fails_loudly(built):
    import torch

    import paper_2205_03133_b200 as P

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(P.GpuError):
        P.Matcher(P.PipelineConfig(), 64, 48)


def test_generator_deterministic_and_shaped(built):
    import paper_2205_03133_b200 as P

    a = P.synth_pair(0, seed=3, width=96, height=64, with_disparity=True)
    b = P.synth_pair(0, seed=3, width=96, height=64, with_disparity=True)
    c = P.synth_pair(0, seed=4, width=96, height=64)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    assert not np.array_equal(a[0], c[0])
    d = a[2]
    assert d.min() == pytest.approx(5.0, abs=1e-4) and d.max() == pytest.approx(40.0, abs=1e-4)
    l3, _ = P.synth_pair(0, seed=3, width=32, height=16, channels=3)
    assert l3.shape == (16, 32, 3)
    L, R = P.synth_batch(0, 3, seed0=3, width=96, height=64, threads=2)
    assert np.array_equal(L[0], a[0]) and np.array_equal(R[0], a[1])


def test_generator_right_view_follows_disparity(built):
    """right(x) ~= left(x + d): the reference convention x_right = x_left - d."""
    import paper_2205_03133_b200 as P

    l, r, d = P.synth_pair(0, seed=0, width=200, height=40, noise_sigma=0.0,
                           with_disparity=True)
    y, x = 20, 60
    xs = x + d[y, x]
    x0 = int(xs)
    f = xs - x0
    expect = (1 - f) * float(l[y, x0]) + f * float(l[y, x0 + 1])
    assert abs(float(r[y, x]) - expect) <= 0.6


def test_generator_noise_and_stress_statistics(built):
    """The portable Box-Muller (synth_core.h: polynomial log/cos) yields N(0, sigma):
    right - warped left has the configured spread; config-1 stress discs cover ~30%."""
    import paper_2205_03133_b200 as P

    l, r, d = P.synth_pair(0, seed=5, width=320, height=240, with_disparity=True)
    lq, rq = P.synth_pair(0, seed=5, width=320, height=240, noise_sigma=0.0)
    assert np.array_equal(l, lq)
    diff = r.astype(np.float64) - rq.astype(np.float64)
    assert abs(diff.mean()) < 0.05 and 1.9 < diff.std() < 2.15
    l1, r1 = P.synth_pair(1, seed=1, width=320, height=240)
    assert not np.array_equal(l1, P.synth_pair(0, seed=1, width=320, height=240)[0])
    # textureless discs: many constant 3x3 neighbourhoods
    flat = (np.abs(np.diff(l1.astype(int), axis=1)) == 0).mean()
    assert flat > 0.2
