"""SURVEY.md 8f row 3 on the B200: PFM-ordered outputs (flip_rows) and the
reference's command line (src/runner.cpp) as pstereo_gpu_cli -- match writes
disparity/depth(/sigma) PFMs byte-identical to the reference's write_pfm of
the reference's run_pipeline; bench reproduces run_benchmark's metrics."""
import csv
import io
import json
import math
import subprocess
import zlib
import struct
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
CLI = ROOT / "paper_2205_03133_b200" / "pstereo_gpu_cli"
SCENES = json.loads((ROOT / "tests" / "golden" / "scenes.json").read_text())


def test_flip_rows_is_the_pfm_row_order(gpu):
    P = gpu
    left, right = P.synth_batch(1, 2, seed0=3, width=160, height=120)
    cfg = P.PipelineConfig(coarsest_exp=3, finest_exp=1, patch_size=8, overlap=0.5,
                           estimate_variance=True)
    want = ["disparity", "disparity_valid", "probability", "depth", "depth_valid",
            "depth_sigma", "sigma_valid", "match_disparity", "match_valid", "var_disp"]
    with P.Matcher(cfg, 160, 120, 2) as m:
        a = m.run_batch(left, right, 500.0, 5.0, dtype=P.F32, want=want, invalid_value=-1.0)
        b = m.run_batch(left, right, 500.0, 5.0, dtype=P.F32, want=want, invalid_value=-1.0,
                        flip_rows=True)
        # odd finest size (scalar output kernel)
        l2, r2 = P.synth_batch(0, 1, seed0=5, width=150, height=110)
        c = m.run_batch(l2, r2, 500.0, 5.0, dtype=P.F64, want=want)
        d = m.run_batch(l2, r2, 500.0, 5.0, dtype=P.F64, want=want, flip_rows=True)
    for k in want:
        assert np.array_equal(a[k][:, ::-1], b[k]), k
        assert np.array_equal(c[k][:, ::-1], d[k]), k


def _pgm(path, img):
    h, w = img.shape
    path.write_bytes(f"P5\n{w} {h}\n255\n".encode() + img.tobytes())


def _png_rgb(path, img):
    h, w, _ = img.shape
    raw = b"".join(b"\0" + img[y].tobytes() for y in range(h))

    def chunk(t, d):
        return struct.pack(">I", len(d)) + t + d + struct.pack(">I", zlib.crc32(t + d))
    path.write_bytes(b"\x89PNG\r\n\x1a\n" + chunk(b"IHDR", struct.pack(">IIBBBBB", w, h, 8, 2,
                                                                       0, 0, 0))
                     + chunk(b"IDAT", zlib.compress(raw)) + chunk(b"IEND", b""))


def _cli(*args, cwd=None):
    return subprocess.run([str(CLI), *map(str, args)], capture_output=True, text=True, cwd=cwd)


@pytest.mark.parametrize("variance", [False, True])
def test_cli_match_pfms_match_reference(gpu, ref, tmp_path, variance):
    from oracle import pyoracle

    P = gpu
    l, r = P.synth_pair(1 if variance else 0, seed=4, width=320, height=240)
    _pgm(tmp_path / "left.pgm", l)
    _pgm(tmp_path / "right.pgm", r)
    (tmp_path / "calib.txt").write_text("focal_px = 480\nbaseline_mm = 5.5\nwidth = 320\n"
                                        "height = 240\n")
    flags = ["--coarsest-exp", "4", "--finest-exp", "1", "--patch-size", "8", "--overlap", "0.5"]
    if variance:
        flags.append("--estimate-variance")
    p = _cli("match", tmp_path / "left.pgm", tmp_path / "right.pgm", "--calib",
             tmp_path / "calib.txt", "--out-dir", tmp_path / "out", *flags)
    assert p.returncode == 0, p.stderr
    lines = p.stdout.strip().splitlines()
    assert lines[0] == P.metrics_csv_header() and lines[1].startswith("left,nan,nan,")
    ocfg = pyoracle.Config(coarsest_exp=4, finest_exp=1, patch_size=8, overlap=0.5,
                           estimate_variance=variance)
    lf, _ = ref.to_grayscale(l)
    rf, _ = ref.to_grayscale(r)
    o = ref.run_pipeline(lf, rf, ocfg, 480.0, 5.5)
    assert int(lines[1].split(",")[3]) == int(o["disparity_valid"].sum())
    maps = [("disparity.pfm", "disparity", "disparity_valid"),
            ("depth.pfm", "depth", "depth_valid")]
    if variance:
        maps.append(("sigma.pfm", "depth_sigma", "sigma_valid"))
    for fname, key, vkey in maps:
        P.write_pfm(tmp_path / ("want_" + fname), o[key].astype(np.float32), o[vkey])
        got = (tmp_path / "out" / fname).read_bytes()
        want = (tmp_path / ("want_" + fname)).read_bytes()
        if key == "depth_sigma":  # libm exp in the variance fit: 1e-3 relative
            g, w_ = P.read_pfm(tmp_path / "out" / fname), P.read_pfm(tmp_path / ("want_" + fname))
            assert np.array_equal(g == -1, w_ == -1)
            np.testing.assert_allclose(g, w_, rtol=1e-3)
        else:
            assert got == want, fname
    assert not (tmp_path / "out" / "sigma.pfm").exists() or variance


def test_cli_match_png_and_errors(gpu, tmp_path):
    P = gpu
    l, r = P.synth_pair(0, seed=6, width=160, height=120, channels=3)
    for name, img in (("l", l), ("r", r)):
        _png_rgb(tmp_path / f"{name}.png", img)
        h, w, _ = img.shape
        (tmp_path / f"{name}.ppm").write_bytes(f"P6\n{w} {h}\n255\n".encode() + img.tobytes())
    (tmp_path / "calib.txt").write_text("focal_px = 500\nbaseline_mm = 5\nwidth = 160\n"
                                        "height = 120\n")
    base = ["--calib", tmp_path / "calib.txt", "--coarsest-exp", "3", "--patch-size", "8"]
    a = _cli("match", tmp_path / "l.png", tmp_path / "r.png", "--out-dir", tmp_path / "a", *base)
    b = _cli("match", tmp_path / "l.ppm", tmp_path / "r.ppm", "--out-dir", tmp_path / "b", *base)
    assert a.returncode == 0 and b.returncode == 0, a.stderr + b.stderr
    for f in ("disparity.pfm", "depth.pfm"):
        assert (tmp_path / "a" / f).read_bytes() == (tmp_path / "b" / f).read_bytes()
    (tmp_path / "bad.txt").write_text("focal_px = 500\nbaseline_mm = 5\nwidth = 64\nheight = 120\n")
    p = _cli("match", tmp_path / "l.png", tmp_path / "r.png", "--calib", tmp_path / "bad.txt")
    assert p.returncode == 2 and "calibration is for" in p.stderr
    p = _cli("match", tmp_path / "l.png", tmp_path / "missing.png", *base)
    assert p.returncode == 3
    small = np.zeros((8, 8), np.uint8)
    _pgm(tmp_path / "s.pgm", small)
    (tmp_path / "c8.txt").write_text("focal_px = 500\nbaseline_mm = 5\nwidth = 8\nheight = 8\n")
    p = _cli("match", tmp_path / "s.pgm", tmp_path / "s.pgm", "--calib", tmp_path / "c8.txt")
    assert p.returncode == 4, p.stderr
    p = _cli("match", tmp_path / "l.png", tmp_path / "r.png", *base, "--patch-size", "1")
    assert p.returncode == 2


def test_cli_bench_matches_reference_flow(gpu, ref, tmp_path):
    from oracle import pyoracle

    P = gpu
    names = ["plane_d8", "slanted", "sphere_shiny"]
    paths = []
    for n in names:
        text = (f"name = {n}\n" + "\n".join(
            f"{k} = {v}" for k, v in (("surface", ["plane", "slanted_plane", "sphere"]
                                       [SCENES[n]["surface"]]),
                                      ("disparity", SCENES[n]["disparity"]),
                                      ("disparity0", SCENES[n]["disparity0"]),
                                      ("disparity_gradient", SCENES[n]["disparity_gradient"]),
                                      ("shading", ["diffuse", "nonlambertian"]
                                       [SCENES[n]["shading"]]),
                                      ("width", 320), ("height", 240))) + "\n")
        f = tmp_path / f"{n}.txt"
        f.write_text(text)
        paths.append(f)
    (tmp_path / "run.ini").write_text("[bench]\ncoarsest-exp = 4\npatch_size = 9\nreps = 2\n")
    p = _cli("--config", tmp_path / "run.ini", "bench", *paths, "--patch-size", "8",
             "--out", tmp_path / "m.csv", "--seed", "3")
    assert p.returncode == 0, p.stderr
    rows = list(csv.DictReader(io.StringIO((tmp_path / "m.csv").read_text())))
    assert [r["frame"] for r in rows] == names + ["average"]
    ocfg = pyoracle.Config(coarsest_exp=4, finest_exp=1, patch_size=8)
    for n, row in zip(names, rows):
        s = P.load_scene_spec(tmp_path / f"{n}.txt")
        s.seed = 3  # no seed key: the --seed flag applies (src/runner.cpp:166-168)
        l, r, d, z = ref.render_scene(s)
        o = ref.run_pipeline(l, r, ocfg, s.focal_px, s.baseline)
        m = ref.compute_metrics(o["depth"], o["depth_valid"], z, np.ones_like(l, np.uint8))
        assert int(row["valid_px"]) == m["valid_px"], n
        assert float(row["mean_err"]) == m["mean_err"], n
        assert float(row["median_err"]) == m["median_err"], n
        assert math.isnan(float(row["coverage_rate"]))
