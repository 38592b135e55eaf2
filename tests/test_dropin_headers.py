"""The C++ drop-in headers (include/pstereo/*.hpp) on CPU: they compile on
their own (C++17 and the reference's C++20), the drop-in caller binary carries
none of the reference's matcher code, and the reference build of the caller
(test infrastructure) behaves as the GPU test expects. The GPU comparison
itself is tests/test_gpu_dropin.py."""
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADERS = ["config", "errors", "fields", "image", "coarse_to_fine", "depth_variance", "pipeline",
           "gpu_runtime"]


@pytest.mark.parametrize("std", ["c++17", "gnu++20"])
def test_dropin_headers_compile_standalone(tmp_path, std):
    src = tmp_path / "tu.cpp"
    src.write_text("".join(f'#include "pstereo/{h}.hpp"\n' for h in HEADERS) +
                   '#include "pstereo_gpu.hpp"\n'
                   "int main() { pstereo::PipelineConfig c; pstereo::validate(c);\n"
                   "  pstereo::ScalarField f = pstereo::ScalarField::sized(3, 2, 1.5, true);\n"
                   "  return int(f.valid_count()) - 6 + int(f.at(2, 1) != 1.5); }\n")
    r = subprocess.run(["g++", f"-std={std}", "-Wall", "-Wextra", "-Werror", "-fsyntax-only",
                        "-I", str(ROOT / "include"), str(src)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def _symbols(exe):
    r = subprocess.run(["nm", "-C", str(exe)], capture_output=True, text=True)
    return r.stdout


def test_dropin_caller_has_no_reference_matcher():
    exe = ROOT / "build" / "caller_gpu"
    if not exe.exists():
        pytest.skip("build/caller_gpu not built (needs /root/reference at build time)")
    syms = _symbols(exe)
    for fn in ("solve_patch_disparity", "eval_patch_residual", "build_pyramid", "fuse_level",
               "remove_small_components", "estimate_patch_variance"):
        assert fn not in syms, fn
    needed = subprocess.run(["readelf", "-d", str(exe)], capture_output=True, text=True).stdout
    assert "libpstereo_gpu.so" in needed
    ref = _symbols(ROOT / "build" / "caller_ref")
    assert "solve_patch_disparity" in ref  # the reference build really is the reference


def _dump(path):
    from tests.test_gpu_dropin import read_dump

    return read_dump(path)


def test_reference_caller_runs_on_cpu(tmp_path):
    exe = ROOT / "build" / "caller_ref"
    if not exe.exists():
        pytest.skip("build/caller_ref not built (needs /root/reference at build time)")
    from oracle import pyoracle

    left, right = pyoracle.synth_batch(0, 1, seed0=3, width=160, height=120)
    for name, img in (("l.pgm", left[0]), ("r.pgm", right[0])):
        (tmp_path / name).write_bytes(b"P5\n160 120\n255\n" + img.tobytes())
    (tmp_path / "c.txt").write_text("focal_px = 500\nbaseline_mm = 5\nwidth = 160\nheight = 120\n")
    r = subprocess.run([str(exe), str(tmp_path / "out"), str(tmp_path / "l.pgm"),
                        str(tmp_path / "r.pgm"), str(tmp_path / "c.txt"), "0"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    d = _dump(tmp_path / "out" / "dump.bin")

    def text(k):
        return d[k][0][1].decode()

    def i64(k):
        return int(np.frombuffer(d[k][0][1], np.int64)[0])

    assert i64("run_match.rc") == 0 and i64("run_bench.rc") == 0
    assert text("err.validate") == "ConfigError"
    assert text("err.run_pipeline_config") == "ConfigError"
    assert text("err.size_mismatch") == "DegenerateInputError"
    assert text("err.too_small") == "DegenerateInputError"
    assert text("err.channels") == "invalid_argument"
    assert i64("err.run_match_missing") == 3  # kExitIoError (inc/runner.hpp:18)
    assert i64("finest.level_exp") == 1 and i64("finest.width") == 80
    assert i64("finest.n_patches") > 0
    assert (tmp_path / "out" / "match" / "disparity.pfm").exists()
