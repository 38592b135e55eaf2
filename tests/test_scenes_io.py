"""SURVEY.md 8f rows 3-4 on the CPU: scene files and the analytic renderer's
oracle (restatement pinned to the reference's render_scene), and the
caller-side formats (kv / calibration, PGM/PPM/PNG, PFM, metrics CSV) against
the reference's own known answers (tests/test_synth.cpp, test_scene_files.cpp,
test_io.cpp)."""
import json
import math
import struct
import zlib
from pathlib import Path

import numpy as np
import pytest

GOLDEN = Path(__file__).resolve().parent / "golden"
SCENES = json.loads((GOLDEN / "scenes.json").read_text())


def _spec(P, **kw):
    return P.scene_spec(**kw)


def _shipped(P, name, **over):
    d = dict(SCENES[name])
    d.update(over)
    return P.scene_spec(**d)


# ---- scene files (test_synth.cpp:209-245, test_scene_files.cpp)

def test_scene_file_parses_every_field(built, tmp_path):
    import paper_2205_03133_b200 as P

    f = tmp_path / "scene.txt"
    f.write_text(
        "name = demo\nsurface = sphere\nsphere_depth = 55\nsphere_radius = 18\n"
        "background_depth = 100\ntexture = checker\ntexture_scale = 12\n"
        "texture_octaves = 3\nshading = nonlambertian\nambient = 0.4\n"
        "highlight_strength = 0.5\nhighlight_falloff = 4\nnoise_std = 0.01\n"
        "seed = 7\nfocal_px = 450\nbaseline = 4.5\nwidth = 320\nheight = 240\n")
    s = P.load_scene_spec(f).as_dict()
    assert s["name"] == "demo" and s["surface"] == 2 and s["texture"] == 1 and s["shading"] == 1
    assert (s["sphere_depth"], s["sphere_radius"], s["background_depth"]) == (55.0, 18.0, 100.0)
    assert (s["texture_scale"], s["texture_octaves"], s["ambient"]) == (12.0, 3, 0.4)
    assert (s["highlight_strength"], s["highlight_falloff"], s["noise_std"]) == (0.5, 4.0, 0.01)
    assert (s["seed"], s["seed_explicit"], s["focal_px"], s["baseline"]) == (7, 1, 450.0, 4.5)
    assert (s["width"], s["height"]) == (320, 240)
    for bad in ("surface = plane\ndisparity = 8\nwavelength = 3\n", "surface = cube\n",
                "surface = plane\ndisparity = -2\n",
                "surface = sphere\nsphere_depth = 95\nbackground_depth = 90\n",
                "surface = plane\ndisparity = 8\ndisparity = 9\n", "just words\n",
                "surface = plane\ndisparity = eight\n"):
        f.write_text(bad)
        with pytest.raises(P.ConfigError):
            P.load_scene_spec(f)
    with pytest.raises(P.IoError):
        P.load_scene_spec(tmp_path / "missing.txt")


def test_shipped_scenes_pin_their_geometry(port):
    import paper_2205_03133_b200 as P

    for name, d in (("plane_d4", 4.0), ("plane_d8", 8.0), ("plane_d16", 16.0)):
        s = _shipped(P, name)
        assert s.surface == 0 and s.disparity == d and s.noise_std == 0.0
        assert port.scene_disparity_at(s, 0.0, 0.0) == pytest.approx(d)
        assert port.scene_disparity_at(s, 639.0, 479.0) == pytest.approx(d)
    s = _shipped(P, "plane_noise")
    assert s.disparity == 8.0 and s.noise_std == pytest.approx(0.01)
    s = _shipped(P, "slanted")
    assert s.surface == 1 and port.scene_disparity_at(s, 0.0, 240.0) == pytest.approx(6.0)
    a, b = _shipped(P, "sphere_diffuse").as_dict(), _shipped(P, "sphere_shiny").as_dict()
    diff = {k for k in a if a[k] != b[k]}
    assert diff <= {"name", "shading", "highlight_strength", "highlight_falloff", "ambient"}


# ---- renderer oracle pinned to the reference (src/synth.cpp:209-284)

@pytest.mark.parametrize("name", sorted(SCENES))
def test_render_port_matches_reference(port, ref, name):
    import paper_2205_03133_b200 as P

    for over in ({}, {"width": 97, "height": 61, "seed": 5}):
        s = _shipped(P, name, **over)
        a, b = port.render_scene(s), ref.render_scene(s)
        for x, y in zip(a, b):
            assert np.array_equal(x.view(np.uint8), y.view(np.uint8))


def test_render_reference_kats(port):
    """test_synth.cpp:36-165, restated on the port."""
    import paper_2205_03133_b200 as P

    s = _spec(P, width=64, height=48, disparity=8.0)
    l, r, d, z = port.render_scene(s)
    assert np.allclose(d, 8.0) and np.allclose(z, 500.0 * 5.0 / 8.0)
    s = _spec(P, surface="slanted_plane", disparity0=4.0, disparity_gradient=0.02,
              width=120, height=20)
    assert port.scene_disparity_at(s, 0.0, 10.0) == pytest.approx(4.0)
    assert port.scene_disparity_at(s, 50.0, 10.0) == pytest.approx(5.0)
    assert port.render_scene(s)[2][5, 80] == pytest.approx(4.0 + 0.02 * 80)
    s = _spec(P, surface="sphere", sphere_depth=60.0, sphere_radius=5.0,
              background_depth=90.0, width=96, height=64)
    cx, cy = 0.5 * 95, 0.5 * 63
    fb = 500.0 * 5.0
    assert fb / port.scene_disparity_at(s, cx, cy) == pytest.approx(60.0, rel=1e-9)
    assert fb / port.scene_disparity_at(s, 0.0, 0.0) == pytest.approx(90.0)
    # right(x, y) == left-view intensity at x + d on a fronto-parallel plane
    s = _spec(P, width=80, height=10, disparity=5.0)
    l, r, _, _ = port.render_scene(s)
    for x in range(0, 70, 7):
        assert r[3, x] == pytest.approx(l[3, x + 5], abs=1e-6)
    s = _spec(P, texture="checker", width=64, height=48)
    l = port.render_scene(s)[0]
    assert np.all(np.isclose(l, 0.2, atol=1e-6) | np.isclose(l, 0.8, atol=1e-6))
    g = np.array([port.gaussian_noise(3, 0, i) for i in range(20000)])
    assert abs(g.mean()) < 0.02 and g.var() == pytest.approx(1.0, rel=0.03)
    v = [port.value_noise(0.37 * i, 1.3, 1, 4, 16.0) for i in range(400)]
    assert min(v) >= 0.0 and max(v) <= 1.0 and max(np.abs(np.diff(v))) < 0.08


# ---- caller-side formats (src/io.cpp; test_io.cpp)

def test_pnm_decode_and_errors(built, tmp_path):
    import paper_2205_03133_b200 as P

    f = tmp_path / "gray.pgm"
    f.write_bytes(b"P5\n# a comment\n2 1\n255\n" + bytes([0, 255]))
    img = P.load_image(f)
    assert img.shape == (1, 2, 1) and img.ravel().tolist() == [0, 255]
    f = tmp_path / "rgb.ppm"
    f.write_bytes(b"P6\n1 1\n255\n" + bytes([255, 0, 0]))
    assert P.load_image(f).shape == (1, 1, 3)
    for name, data in (("short.pgm", b"P5\n4 4\n255\nxy"),
                       ("deep.pgm", b"P5\n1 1\n65535\n\0\0"),
                       ("garbage.bin", b"not an image at all")):
        (tmp_path / name).write_bytes(data)
        with pytest.raises(P.IoError):
            P.load_image(tmp_path / name)
    with pytest.raises(P.IoError, match="cannot open"):
        P.load_image(tmp_path / "definitely_not_here.png")


def _png(w, h, ctype, depth, rows, plte=None, trns=None, interlace=False):
    """Minimal PNG encoder for the decoder tests (filter 0 rows; `rows` are
    the packed scanlines of each pass, already laid out by the caller)."""
    def chunk(t, d):
        return struct.pack(">I", len(d)) + t + d + struct.pack(">I", zlib.crc32(t + d))
    raw = b"".join(b"\0" + r for r in rows)
    out = b"\x89PNG\r\n\x1a\n" + chunk(b"IHDR", struct.pack(">IIBBBBB", w, h, depth, ctype,
                                                            0, 0, int(interlace)))
    if plte is not None:
        out += chunk(b"PLTE", plte)
    if trns is not None:
        out += chunk(b"tRNS", trns)
    return out + chunk(b"IDAT", zlib.compress(raw)) + chunk(b"IEND", b"")


def test_png_decode(built, tmp_path):
    import paper_2205_03133_b200 as P

    cases = {
        # test_io.cpp:107-114: gray 2x2 {0, 85, 170, 255}
        "gray.png": (_png(2, 2, 0, 8, [bytes([0, 85]), bytes([170, 255])]),
                     (2, 2, 1), [0, 85, 170, 255]),
        # 2-bit gray expands by x85
        "gray2.png": (_png(4, 1, 0, 2, [bytes([0b00011011])]), (1, 4, 1), [0, 85, 170, 255]),
        # test_io.cpp:117-126: RGBA keeps alpha as the mask
        "rgba.png": (_png(2, 1, 6, 8, [bytes([255, 0, 0, 255, 0, 255, 0, 0])]), (1, 2, 4),
                     [255, 0, 0, 255, 0, 255, 0, 0]),
        # test_io.cpp:128-134: palette expands to RGB
        "pal.png": (_png(2, 1, 3, 8, [bytes([0, 1])], plte=bytes([0, 0, 255, 255, 255, 255])),
                    (1, 2, 3), [0, 0, 255, 255, 255, 255]),
        # palette + tRNS -> RGBA
        "paltrns.png": (_png(2, 1, 3, 8, [bytes([0, 1])],
                             plte=bytes([0, 0, 255, 255, 255, 255]), trns=bytes([0])),
                        (1, 2, 4), [0, 0, 255, 0, 255, 255, 255, 255]),
        # 16-bit gray: high byte
        "gray16.png": (_png(2, 1, 0, 16, [bytes([0x12, 0x34, 0xAB, 0xCD])]), (1, 2, 1),
                       [0x12, 0xAB]),
        # gray + alpha -> RGBA
        "ga.png": (_png(1, 1, 4, 8, [bytes([77, 10])]), (1, 1, 4), [77, 77, 77, 10]),
        # gray + tRNS key -> RGBA with alpha 0 at the key
        "graykey.png": (_png(2, 1, 0, 8, [bytes([5, 6])], trns=bytes([0, 5])), (1, 2, 4),
                        [5, 5, 5, 0, 6, 6, 6, 255]),
    }
    for name, (data, shape, want) in cases.items():
        (tmp_path / name).write_bytes(data)
        img = P.load_image(tmp_path / name)
        assert img.shape == shape, name
        assert img.ravel().tolist() == want, name
    # Adam7: 3x3 gray, passes laid out per the PNG spec
    full = np.arange(9, dtype=np.uint8).reshape(3, 3) * 20
    passes = [(0, 0, 8, 8), (4, 0, 8, 8), (0, 4, 4, 8), (2, 0, 4, 4), (0, 2, 2, 4),
              (1, 0, 2, 2), (0, 1, 1, 2)]
    rows = []
    for x0, y0, dx, dy in passes:
        for y in range(y0, 3, dy):
            r = bytes(full[y, x0::dx].tolist())
            if r:
                rows.append(r)
    (tmp_path / "adam7.png").write_bytes(_png(3, 3, 0, 8, rows, interlace=True))
    assert np.array_equal(P.load_image(tmp_path / "adam7.png")[:, :, 0], full)
    bad = bytearray(cases["gray.png"][0])
    bad[40] ^= 0xFF
    (tmp_path / "crc.png").write_bytes(bytes(bad))
    with pytest.raises(P.IoError):
        P.load_image(tmp_path / "crc.png")


def test_pfm_layout_and_round_trip(built, tmp_path):
    import paper_2205_03133_b200 as P

    # test_io.cpp:170-188: header + payload bytes pinned (1.5 and -1 for invalid)
    f = tmp_path / "pin.pfm"
    P.write_pfm(f, np.array([[1.5, 7.0]], np.float32), valid=np.array([[1, 0]], np.uint8))
    b = f.read_bytes()
    assert b == b"Pf\n2 1\n-1.0\n" + bytes([0, 0, 0xC0, 0x3F, 0, 0, 0x80, 0xBF])
    # test_io.cpp:190-209: rows bottom to top, read back top to bottom
    P.write_pfm(f, np.array([[1, 2], [3, 4]], np.float32))
    first = struct.unpack("<f", f.read_bytes()[len(b"Pf\n2 2\n-1.0\n"):][:4])[0]
    assert first == 3.0
    assert P.read_pfm(f).ravel().tolist() == [1.0, 2.0, 3.0, 4.0]
    # already bottom-up planes (a flip_rows match output) are written verbatim
    P.write_pfm(f, np.array([[3, 4], [1, 2]], np.float32), rows_bottom_up=True)
    assert P.read_pfm(f).ravel().tolist() == [1.0, 2.0, 3.0, 4.0]
    rng = np.random.default_rng(0)
    bits = rng.integers(0, 2**32, size=(5, 7), dtype=np.uint64).astype(np.uint32)
    vals = bits.view(np.float32)
    P.write_pfm(f, vals)
    assert np.array_equal(P.read_pfm(f).view(np.uint32), bits)
    (tmp_path / "bad.pfm").write_bytes(b"PF\n1 1\n-1.0\n\0\0\0\0")
    with pytest.raises(P.IoError):
        P.read_pfm(tmp_path / "bad.pfm")
    (tmp_path / "be.pfm").write_bytes(b"Pf\n1 1\n1.0\n\0\0\0\0")
    with pytest.raises(P.IoError):
        P.read_pfm(tmp_path / "be.pfm")


def test_metrics_csv(built, tmp_path):
    import paper_2205_03133_b200 as P

    assert P.metrics_csv_header() == \
        "frame,mean_err,median_err,valid_px,runtime_ms,coverage_rate"
    r = P.metrics_row("plane_d8", 0.0001, 0.25, 1234, 51.5, float("nan"))
    # std::to_chars shortest form (1e-04 is shorter than 0.0001)
    assert P.format_metrics_row(r) == "plane_d8,1e-04,0.25,1234,51.5,nan"
    rows = [r, P.metrics_row("average", float("nan"), float("nan"), 7, 1.0 / 3.0, 0.95)]
    f = tmp_path / "m.csv"
    P.write_metrics_csv(f, rows)
    text = f.read_text().splitlines()
    assert text[0] == P.metrics_csv_header() and text[2].startswith("average,nan,nan,7,")
    back = P.read_metrics_csv(f)
    assert [x.frame for x in back] == [b"plane_d8", b"average"]
    assert back[0].mean_err == 0.0001 and back[1].runtime_ms == 1.0 / 3.0
    assert back[0].has_errors == 1 and back[1].has_errors == 0 and math.isnan(back[1].mean_err)
    f.write_text("frame,oops\n")
    with pytest.raises(P.IoError):
        P.read_metrics_csv(f)


def test_calibration(built, tmp_path):
    import paper_2205_03133_b200 as P

    f = tmp_path / "calib.txt"
    f.write_text("# rig\nfocal_px = 500\nbaseline_mm = 5.5\nwidth = 640\nheight = 480\n")
    assert P.load_calibration(f) == {"focal_px": 500.0, "baseline_mm": 5.5, "width": 640,
                                     "height": 480}
    f.write_text("focal_px = 500\nbaseline_mm = -1\nwidth = 640\nheight = 480\n")
    with pytest.raises(P.ConfigError):
        P.load_calibration(f)
    f.write_text("focal_px = 500\nwidth = 640\nheight = 480\n")
    with pytest.raises(P.ConfigError, match="missing key"):
        P.load_calibration(f)


def test_cli_usage_and_file_errors_without_gpu(built, tmp_path):
    """pstereo_gpu_cli exit codes (inc/pstereo/runner.hpp:16-19) for errors that
    happen before any device work: usage / config 2, unreadable files 3."""
    import subprocess

    import paper_2205_03133_b200 as P

    cli = str(Path(P.__file__).resolve().parent / "pstereo_gpu_cli")

    def run(*a):
        return subprocess.run([cli, *map(str, a)], capture_output=True, text=True).returncode

    assert run() == 2
    assert run("frobnicate") == 2
    assert run("match", "only_one.png") == 2
    assert run("match", "a.png", "b.png") == 2                      # --calib missing
    assert run("match", "a.png", "b.png", "--calib", "c.txt", "--patch-size", "x") == 2
    assert run("match", "a.png", "b.png", "--calib", "c.txt", "--bogus", "1") == 2
    assert run("match", "a.png", "b.png", "--calib", "c.txt", "--patch-size", "1") == 2
    assert run("match", tmp_path / "no.png", tmp_path / "no2.png", "--calib", "c.txt") == 3
    assert run("bench") == 2
    assert run("bench", tmp_path / "missing_scene.txt") == 3
    (tmp_path / "bad.txt").write_text("surface = cube\n")
    assert run("bench", tmp_path / "bad.txt") == 2
    (tmp_path / "cfg.ini").write_text("[bench]\nreps = zero\n")
    assert run("--config", tmp_path / "cfg.ini", "bench", tmp_path / "bad.txt") == 2
