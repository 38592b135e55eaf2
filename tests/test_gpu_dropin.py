"""The C++ drop-in, proven on the reference's own caller code.

tests/cpp/caller_main.cpp is written only against the reference's API. It
drives the reference's own callers -- run_match (src/runner.cpp:128-161),
run_bench (:164-183), run_benchmark (src/bench.cpp) -- plus run_pipeline,
match_stereo (MatchResult::finest included), to_grayscale and the error
paths. tests/cpp/build.sh builds it twice: `caller_ref` from the unmodified
reference sources, and `caller_gpu` from the reference's caller-side sources
(unchanged) compiled against this repo's include/pstereo/ headers and linked
to libpstereo_gpu.so. Both run here on the same PGM/PPM inputs; every dump
record, the PFM files run_match writes and the bench CSV must agree
(bit-exact; variance-derived values within 1e-3 relative, BASELINE.json).
The binaries are built where /root/reference exists and travel with the
snapshot; the inputs come from the test-side generator (oracle/)."""
import math
import struct
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
REF_EXE = ROOT / "build" / "caller_ref"
GPU_EXE = ROOT / "build" / "caller_gpu"


def read_dump(path):
    """name -> list of (kind, payload) in file order."""
    data = path.read_bytes()
    out = {}
    pos = 0
    while pos < len(data):
        name = data[pos:pos + 64].split(b"\0", 1)[0].decode()
        kind = data[pos + 64]
        (count,) = struct.unpack_from("<Q", data, pos + 65)
        pos += 73
        size = {0: 8, 1: 8, 2: 1, 3: 8, 4: 1}[kind]
        payload = data[pos:pos + count * size]
        pos += count * size
        out.setdefault(name, []).append((kind, payload))
    return out


def compare_dumps(a, b):
    problems = []
    assert a.keys() == b.keys(), sorted(set(a) ^ set(b))
    for name in a:
        assert len(a[name]) == len(b[name]), name
        for (ka, pa), (kb, pb) in zip(a[name], b[name]):
            assert ka == kb, name
            if ka == 1:
                x = np.frombuffer(pa, np.float64)
                y = np.frombuffer(pb, np.float64)
                same_nan = np.isnan(x) == np.isnan(y)
                close = np.isclose(x, y, rtol=1e-3, atol=0.0) | (np.isnan(x) & np.isnan(y))
                if x.shape != y.shape or not (same_nan.all() and close.all()):
                    problems.append(f"{name}: beyond 1e-3 relative")
            elif pa != pb:
                problems.append(f"{name}: differs")
    return problems


def _write_pnm(path, img):
    h, w = img.shape[:2]
    magic = b"P5" if img.ndim == 2 else b"P6"
    path.write_bytes(magic + f"\n{w} {h}\n255\n".encode() + np.ascontiguousarray(img).tobytes())


def _pfm(path):
    raw = path.read_bytes()
    head = raw.split(b"\n", 3)
    w, h = (int(v) for v in head[1].split())
    return np.frombuffer(head[3], "<f4").reshape(h, w)


CASES = [  # (config, seed, width, height, channels); config 5 = generator 0
    # with the reference's default PipelineConfig (5 levels, s = 10, overlap
    # 0.55 -> stride lrint(4.5) = 4)
    (0, 0, 640, 480, 1),
    (1, 1, 640, 480, 1),
    (3, 0, 640, 512, 1),
    (0, 7, 320, 240, 3),
    (5, 2, 640, 480, 1),
]


@pytest.mark.gpu
@pytest.mark.parametrize("config,seed,w,h,ch", CASES)
def test_reference_callers_against_dropin(gpu, tmp_path, config, seed, w, h, ch):
    if not (REF_EXE.exists() and GPU_EXE.exists()):
        pytest.skip("build/caller_{ref,gpu} not built (needs /root/reference at build time)")
    from oracle import pyoracle

    over = dict(width=w, height=h)
    if ch != 1:
        over["channels"] = ch
    gen = 4 if ch != 1 else (0 if config == 5 else config)
    left, right = pyoracle.synth_batch(gen, 1, seed0=seed, **over)
    lp, rp, cp = tmp_path / "l.pnm", tmp_path / "r.pnm", tmp_path / "calib.txt"
    _write_pnm(lp, left[0])
    _write_pnm(rp, right[0])
    cp.write_text(f"focal_px = 500\nbaseline_mm = 5\nwidth = {w}\nheight = {h}\n")
    runs = {}
    for tag, exe in (("ref", REF_EXE), ("gpu", GPU_EXE)):
        wd = tmp_path / tag
        r = subprocess.run([str(exe), str(wd), str(lp), str(rp), str(cp),
                            str(4 if config == 5 else min(config, 3))], capture_output=True,
                           text=True, timeout=900)
        assert r.returncode == 0, f"{tag}: {r.stdout}{r.stderr}"
        runs[tag] = wd
    a = read_dump(runs["ref"] / "dump.bin")
    b = read_dump(runs["gpu"] / "dump.bin")
    problems = compare_dumps(a, b)
    assert not problems, problems
    # run_match's files: disparity / depth PFMs byte-identical, sigma within 1e-3
    for f in ("disparity.pfm", "depth.pfm"):
        assert (runs["ref"] / "match" / f).read_bytes() == (runs["gpu"] / "match" / f).read_bytes(), f
    sig = runs["ref"] / "match" / "sigma.pfm"
    assert sig.exists() == (runs["gpu"] / "match" / "sigma.pfm").exists()
    if sig.exists():
        x, y = _pfm(sig), _pfm(runs["gpu"] / "match" / "sigma.pfm")
        np.testing.assert_allclose(y, x, rtol=1e-3)
    # run_bench's CSV: every column but runtime_ms
    ra = (runs["ref"] / "bench.csv").read_text().splitlines()
    rb = (runs["gpu"] / "bench.csv").read_text().splitlines()
    assert len(ra) == len(rb) == 4 and ra[0] == rb[0]
    for la, lb in zip(ra[1:], rb[1:]):
        ca, cb = la.split(","), lb.split(",")
        assert ca[:4] == cb[:4] or all(
            x == y or (x != "nan" and math.isclose(float(x), float(y), rel_tol=1e-3))
            for x, y in zip(ca[:4], cb[:4])), (la, lb)
        assert ca[5:] == cb[5:] or math.isclose(float(ca[5]), float(cb[5]), rel_tol=1e-3), (la, lb)
    # the boundary's error behaviour is the reference's
    for k in ("err.validate", "err.run_pipeline_config", "err.size_mismatch", "err.too_small",
              "err.channels", "err.run_match_missing"):
        assert a[k] == b[k], k
    assert a["finest.n_patches"][0][1] != struct.pack("<q", 0)
