"""Generates tests/golden/*.npz with the REFERENCE ITSELF (oracle/_ref, the
unmodified reference sources compiled in this container). Run here, where
/root/reference exists:

    python tests/golden/make_golden.py

Each fixture holds the uint8 (or float) inputs, the PipelineConfig, and the
reference's run_pipeline + match_stereo outputs: small cases as full arrays,
larger ones as SHA-256 digests of the exact output bytes (bit-exactness makes
the digest a complete check) plus MatchStats.
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))

import paper_2205_03133_b200 as P  # noqa: E402  (generator only)
from oracle import pyoracle  # noqa: E402

FOCAL, BASELINE = 500.0, 5.0
FULL_LIMIT = 96 * 72  # store full arrays up to this many pixels


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def analytic_pair(w, h, d):
    y, x = np.mgrid[0:h, 0:w].astype(np.float64)

    def tex(xx):
        return (0.5 + 0.2 * np.sin(xx * 0.37 + 0.8) + 0.15 * np.sin(y * 0.29)
                + 0.1 * np.sin((xx + y) * 0.143)).astype(np.float32)

    return tex(x), tex(x + d)


CASES = {
    "c0_160x120": dict(kind="synth", config=0, seed=0, w=160, h=120,
                       cfg=dict(coarsest_exp=2, finest_exp=1, patch_size=8, overlap=0.5)),
    "c1_160x120_var": dict(kind="synth", config=1, seed=1, w=160, h=120,
                           cfg=dict(coarsest_exp=2, finest_exp=1, patch_size=8, overlap=0.5,
                                    estimate_variance=True)),
    "c3like_192x160_s12": dict(kind="synth", config=3, seed=2, w=192, h=160,
                               cfg=dict(coarsest_exp=2, finest_exp=1, patch_size=12,
                                        overlap=1 - 4 / 12, estimate_variance=True)),
    "shift2_64x48": dict(kind="analytic", d=2.0, w=64, h=48,
                         cfg=dict(coarsest_exp=2, finest_exp=1)),
    "rgba_96x72_fe0": dict(kind="rgba", seed=4, w=96, h=72,
                           cfg=dict(coarsest_exp=1, finest_exp=0, patch_size=6, overlap=0.5,
                                    estimate_variance=True)),
    "defaults_384x320": dict(kind="synth", config=0, seed=9, w=384, h=320, cfg=dict()),
}


def make_inputs(spec):
    if spec["kind"] == "synth":
        extra = {}
        if spec["config"] == 3:
            extra = dict(d_range=24.0, blur_sigma=16.0)
        l, r = P.synth_pair(spec["config"], seed=spec["seed"], width=spec["w"], height=spec["h"],
                            **extra)
        return {"left_u8": l, "right_u8": r}
    if spec["kind"] == "rgba":
        l, r = P.synth_pair(0, seed=spec["seed"], width=spec["w"], height=spec["h"], channels=3,
                            blur_sigma=8.0, d_min=1.0, d_range=5.0)
        la = np.concatenate([l, np.full(l.shape[:2] + (1,), 255, np.uint8)], axis=2)
        ra = np.concatenate([r, np.full(r.shape[:2] + (1,), 255, np.uint8)], axis=2)
        la[20:30, 30:45, 3] = 0
        ra[5:9, 60:70, 3] = 0
        return {"left_u8": la, "right_u8": ra}
    lf, rf = analytic_pair(spec["w"], spec["h"], spec["d"])
    return {"left_f32": lf, "right_f32": rf}


def gray_inputs(orc, inputs):
    if "left_u8" in inputs:
        lf, lv = orc.to_grayscale(inputs["left_u8"])
        rf, rv = orc.to_grayscale(inputs["right_u8"])
        return lf, lv, rf, rv
    return inputs["left_f32"], None, inputs["right_f32"], None


def main():
    ref = pyoracle.load("reference")
    for name, spec in CASES.items():
        inputs = make_inputs(spec)
        lf, lv, rf, rv = gray_inputs(ref, inputs)
        cfg = pyoracle.Config(**spec["cfg"])
        pipe = ref.run_pipeline(lf, rf, cfg, FOCAL, BASELINE, lv, rv)
        match = ref.match_stereo(lf, rf, cfg, lv, rv)
        outs = {
            "disparity": pipe["disparity"], "disparity_valid": pipe["disparity_valid"],
            "probability": pipe["probability"], "depth": pipe["depth"],
            "depth_valid": pipe["depth_valid"], "match_disparity": match["disparity"],
            "match_valid": match["disparity_valid"], "finest": match["finest"],
        }
        if cfg.estimate_variance:
            outs.update(depth_sigma=pipe["depth_sigma"], sigma_valid=pipe["sigma_valid"],
                        var_disp=match["var_disp"])
        full = spec["w"] * spec["h"] <= FULL_LIMIT
        data = {k: v for k, v in inputs.items()}
        data["stats"] = match["stats"]
        meta = {"name": name, "cfg": spec["cfg"], "focal": FOCAL, "baseline": BASELINE,
                "full": full, "digests": {k: digest(v) for k, v in outs.items()},
                "generated_by": "oracle/_ref (reference sources), tests/golden/make_golden.py"}
        if full:
            for k, v in outs.items():
                data["out_" + k] = v
        else:
            # exact bytes for masks (compress well); digests for the rest
            for k in ("disparity_valid", "depth_valid", "match_valid"):
                data["out_" + k] = outs[k]
        data["meta"] = np.frombuffer(json.dumps(meta).encode(), np.uint8)
        np.savez_compressed(HERE / f"{name}.npz", **data)
        print(name, match["stats"].tolist(), "valid", float(pipe["disparity_valid"].mean()))


if __name__ == "__main__":
    main()
