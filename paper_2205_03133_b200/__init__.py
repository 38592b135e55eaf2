"""B200-native BDIS matching core -- Python host mirror of the reference API.

The product is libpstereo_gpu.so (hand-written sm_100a kernels behind the C ABI
in include/pstereo_gpu.h). This module binds that ABI with ctypes and mirrors
the reference's interface for the hot path (proj/include/pstereo/*.hpp):

  PipelineConfig             inc/config.hpp:12-33      -> PipelineConfig
  validate                   src/coarse_to_fine.cpp:18-49 -> validate
  ConfigError / DegenerateInputError  inc/errors.hpp:9-31
  CameraParams               inc/depth_variance.hpp:20-23
  match_stereo               inc/coarse_to_fine.hpp:102-103 -> match_stereo
  run_pipeline               inc/pipeline.hpp:20-22    -> run_pipeline
  (batched)                                            -> Matcher.run_batch

There is no CPU fallback: loading fails loudly when the library is missing,
and every compute call needs an sm_100 device.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

PKG = Path(__file__).resolve().parent
# PSTEREO_GPU_LIB: an alternative build of the same library (A/B timing runs)
LIB_PATH = Path(os.environ.get("PSTEREO_GPU_LIB", PKG / "libpstereo_gpu.so"))

PSTEREO_OK, PSTEREO_EINTERNAL, PSTEREO_ECONFIG, PSTEREO_EDEGENERATE = 0, 1, 2, 4
MAX_OFF = 16
F32, F64 = 0, 1

u8p = C.POINTER(C.c_uint8)
f32p = C.POINTER(C.c_float)
i32p = C.POINTER(C.c_int)


class ConfigError(ValueError):
    """Bad parameter values (inc/errors.hpp:9-11)."""


class DegenerateInputError(ValueError):
    """Structurally unusable input, e.g. smaller than a patch (inc/errors.hpp:28-30)."""


class GpuError(RuntimeError):
    """CUDA / internal failure (exit code 1 in src/runner.cpp:107-124)."""


class _Params(C.Structure):
    _fields_ = [
        ("coarsest_exp", C.c_int), ("finest_exp", C.c_int), ("patch_size", C.c_int),
        ("overlap", C.c_double), ("min_iterations", C.c_int), ("max_iterations", C.c_int),
        ("early_stop_good", C.c_double), ("early_stop_bad", C.c_double),
        ("early_stop_improve", C.c_double), ("n_window_offsets", C.c_int),
        ("window_offsets", C.c_double * MAX_OFF), ("sigma_s", C.c_double),
        ("pixel_threshold", C.c_double), ("gamma", C.c_double),
        ("valid_patch_ratio", C.c_double), ("estimate_variance", C.c_int), ("threads", C.c_int),
    ]


class LevelStats(C.Structure):
    """MatchStats::Level (inc/coarse_to_fine.hpp:80-89)."""
    _fields_ = [("exp", C.c_int), ("grid_patches", C.c_int), ("extracted", C.c_int),
                ("converged", C.c_int), ("accepted", C.c_int)]

    def as_tuple(self):
        return (self.exp, self.grid_patches, self.extracted, self.converged, self.accepted)


class PatchEstimate(C.Structure):
    _fields_ = [("cx", C.c_double), ("cy", C.c_double), ("u", C.c_double),
                ("prob", C.c_double), ("posterior", C.c_double), ("sigma_k", C.c_double)]


class FrameMetricsC(C.Structure):
    """pstereo_frame_metrics (FrameMetrics, inc/metrics.hpp:14-25)."""
    _fields_ = [("valid_px", C.c_longlong), ("compared", C.c_longlong), ("has_errors", C.c_int),
                ("mean_err", C.c_double), ("median_err", C.c_double),
                ("coverage_rate", C.c_double)]


class _Outputs(C.Structure):
    _fields_ = [
        ("dtype", C.c_int), ("on_device", C.c_int), ("disparity", C.c_void_p),
        ("disparity_valid", C.c_void_p), ("probability", C.c_void_p), ("depth", C.c_void_p),
        ("depth_valid", C.c_void_p), ("depth_sigma", C.c_void_p), ("sigma_valid", C.c_void_p),
        ("match_disparity", C.c_void_p), ("match_valid", C.c_void_p), ("var_disp", C.c_void_p),
        ("stats", C.POINTER(LevelStats)), ("finest", C.POINTER(PatchEstimate)),
        ("finest_count", i32p), ("finest_cap", C.c_int), ("fill_invalid", C.c_int),
        ("invalid_value", C.c_double), ("async_host", C.c_int), ("flip_rows", C.c_int),
    ]


class SynthSpec(C.Structure):
    _fields_ = [("width", C.c_int), ("height", C.c_int), ("channels", C.c_int),
                ("seed", C.c_uint64), ("octaves", C.c_int), ("base_wavelength", C.c_double),
                ("d_min", C.c_double), ("d_range", C.c_double), ("blur_sigma", C.c_double),
                ("noise_sigma", C.c_double), ("stress", C.c_int)]


class SceneSpec(C.Structure):
    """pstereo_scene_spec = SceneSpec (inc/pstereo/synth.hpp:20-50)."""
    _fields_ = [("name", C.c_char * 64), ("surface", C.c_int), ("disparity", C.c_double),
                ("disparity0", C.c_double), ("disparity_gradient", C.c_double),
                ("sphere_depth", C.c_double), ("sphere_radius", C.c_double),
                ("background_depth", C.c_double), ("texture", C.c_int),
                ("texture_scale", C.c_double), ("texture_octaves", C.c_int),
                ("shading", C.c_int), ("ambient", C.c_double),
                ("highlight_strength", C.c_double), ("highlight_falloff", C.c_double),
                ("noise_std", C.c_double), ("seed", C.c_uint64), ("seed_explicit", C.c_int),
                ("focal_px", C.c_double), ("baseline", C.c_double), ("width", C.c_int),
                ("height", C.c_int)]

    SURFACES = {"plane": 0, "slanted_plane": 1, "sphere": 2}
    TEXTURES = {"perlin": 0, "checker": 1, "constant": 2}
    SHADINGS = {"diffuse": 0, "nonlambertian": 1}

    def as_dict(self) -> dict:
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["name"] = self.name.decode()
        return d


class MetricsRow(C.Structure):
    """pstereo_metrics_row = FrameMetrics as the CSV stores it (inc/metrics.hpp)."""
    _fields_ = [("frame", C.c_char * 128), ("mean_err", C.c_double),
                ("median_err", C.c_double), ("valid_px", C.c_longlong),
                ("runtime_ms", C.c_double), ("coverage_rate", C.c_double),
                ("has_errors", C.c_int)]


_LIB = None


def lib() -> C.CDLL:
    """The product library. Raises if it was not built -- no fallback."""
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} missing: run python -m paper_2205_03133_b200.build")
        L = C.CDLL(str(LIB_PATH))
        L.pstereo_gpu_last_error.restype = C.c_char_p
        L.pstereo_gpu_last_error.argtypes = [C.c_void_p]
        L.pstereo_gpu_stage_name.restype = C.c_char_p
        L.pstereo_gpu_stage_name.argtypes = [C.c_void_p, C.c_int]
        L.pstereo_gpu_create.argtypes = [C.c_int, C.POINTER(_Params), C.c_int, C.c_int, C.c_int,
                                         C.POINTER(C.c_void_p)]
        L.pstereo_gpu_destroy.argtypes = [C.c_void_p]
        L.pstereo_gpu_set_fill_target.argtypes = [C.c_void_p, C.c_int]
        L.pstereo_gpu_set_graphs.argtypes = [C.c_void_p, C.c_int]
        L.pstereo_multi_create.argtypes = [C.POINTER(C.c_int), C.c_int, C.POINTER(_Params),
                                           C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        L.pstereo_multi_destroy.argtypes = [C.c_void_p]
        L.pstereo_multi_last_error.restype = C.c_char_p
        L.pstereo_multi_last_error.argtypes = [C.c_void_p]
        L.pstereo_multi_match_u8.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                             C.c_void_p, C.c_void_p, C.c_double, C.c_double,
                                             C.POINTER(_Outputs), C.c_void_p]
        L.pstereo_gpu_last_launch_count.argtypes = [C.c_void_p]
        L.pstereo_gpu_set_profiling.argtypes = [C.c_void_p, C.c_int]
        L.pstereo_gpu_set_device_chunks.argtypes = [C.c_void_p, C.c_int]
        L.pstereo_gpu_set_host_expand.argtypes = [C.c_void_p, C.c_int]
        L.pstereo_gpu_host_threads.argtypes = []
        L.pstereo_host_expand_stats.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_longlong)]
        L.pstereo_host_expand.argtypes = [C.c_void_p, C.c_void_p] + [C.c_int] * 8
        L.pstereo_gpu_stage_times.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_int, i32p]
        L.pstereo_gpu_match_u8.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                           C.c_void_p, C.c_void_p, C.c_int, C.c_double,
                                           C.c_double, C.POINTER(_Outputs), C.c_void_p]
        L.pstereo_gpu_match_f32.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                            C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                            C.c_double, C.c_double, C.POINTER(_Outputs),
                                            C.c_void_p]
        L.pstereo_gpu_metrics.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                          C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.c_int, C.POINTER(FrameMetricsC),
                                          C.c_void_p]
        L.pstereo_gpu_wait.argtypes = [C.c_void_p, C.c_void_p]
        L.pstereo_validate.argtypes = [C.POINTER(_Params), C.c_char_p, C.c_size_t]
        L.pstereo_level_dims.argtypes = [C.POINTER(_Params), C.c_int, C.c_int, i32p, i32p,
                                         i32p, i32p]
        L.pstereo_synth_default.argtypes = [C.POINTER(SynthSpec), C.c_int]
        L.pstereo_synth_pair.argtypes = [C.POINTER(SynthSpec), C.c_uint64, u8p, u8p, f32p]
        L.pstereo_synth_batch.argtypes = [C.POINTER(SynthSpec), C.c_int, C.c_uint64, u8p, u8p,
                                          C.c_int]
        L.pstereo_gpu_synth.argtypes = [C.c_int, C.POINTER(SynthSpec), C.c_int, C.c_uint64,
                                        C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.pstereo_synth_last_error.restype = C.c_char_p
        L.pstereo_render_last_error.restype = C.c_char_p
        L.pstereo_gpu_render.argtypes = [C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_void_p, C.c_void_p]
        L.pstereo_scene_default.argtypes = [C.POINTER(SceneSpec)]
        L.pstereo_scene_validate.argtypes = [C.POINTER(SceneSpec), C.c_char_p, C.c_size_t]
        L.pstereo_load_scene_spec.argtypes = [C.c_char_p, C.POINTER(SceneSpec), C.c_char_p,
                                              C.c_size_t]
        L.pstereo_load_calibration.argtypes = [C.c_char_p, C.POINTER(C.c_double),
                                               C.POINTER(C.c_double), i32p, i32p, C.c_char_p,
                                               C.c_size_t]
        L.pstereo_load_image.argtypes = [C.c_char_p, i32p, i32p, i32p, C.c_void_p, C.c_size_t,
                                         C.c_char_p, C.c_size_t]
        L.pstereo_write_pfm.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                        C.c_int, C.c_char_p, C.c_size_t]
        L.pstereo_read_pfm.argtypes = [C.c_char_p, i32p, i32p, C.c_void_p, C.c_size_t,
                                       C.c_char_p, C.c_size_t]
        L.pstereo_metrics_csv_header.restype = C.c_char_p
        L.pstereo_format_metrics_row.argtypes = [C.POINTER(MetricsRow), C.c_char_p, C.c_size_t]
        L.pstereo_write_metrics_csv.argtypes = [C.c_char_p, C.POINTER(MetricsRow), C.c_int,
                                                C.c_char_p, C.c_size_t]
        L.pstereo_read_metrics_csv.argtypes = [C.c_char_p, C.POINTER(MetricsRow), C.c_int,
                                               i32p, C.c_char_p, C.c_size_t]
        L.pstereo_debug_eval_residual.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p,
                                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                                  C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                                  C.c_void_p, C.c_void_p, C.c_void_p]
        _LIB = L
    return _LIB


def debug_eval_residual(left, right, size, x0, y0, u, left_valid=None, right_valid=None,
                        device=0):
    """Test hook: (msq, jr, n) arrays of eval_patch_residual on the GPU."""
    left = np.ascontiguousarray(left, np.float32)
    right = np.ascontiguousarray(right, np.float32)
    h, w = left.shape
    x0 = np.ascontiguousarray(x0, np.int32)
    y0 = np.ascontiguousarray(y0, np.int32)
    u = np.ascontiguousarray(u, np.float64)
    nq = len(u)
    msq = np.zeros(nq, np.float64)
    jr = np.zeros(nq, np.float64)
    n = np.zeros(nq, np.int32)
    lv = None if left_valid is None else np.ascontiguousarray(left_valid, np.uint8)
    rv = None if right_valid is None else np.ascontiguousarray(right_valid, np.uint8)
    rc = lib().pstereo_debug_eval_residual(
        device, w, h, left.ctypes.data, None if lv is None else lv.ctypes.data, right.ctypes.data,
        None if rv is None else rv.ctypes.data, size, nq, x0.ctypes.data, y0.ctypes.data,
        u.ctypes.data, msq.ctypes.data, jr.ctypes.data, n.ctypes.data)
    if rc:
        raise GpuError("pstereo_debug_eval_residual failed")
    return msq, jr, n


# Exported symbols of include/pstereo_gpu.h (checked by tests/test_abi.py).
ABI_SYMBOLS = [
    "pstereo_default_params", "pstereo_validate", "pstereo_level_dims", "pstereo_gpu_create",
    "pstereo_gpu_destroy", "pstereo_gpu_last_error", "pstereo_gpu_match_u8",
    "pstereo_gpu_match_f32", "pstereo_gpu_last_launch_count", "pstereo_gpu_set_profiling",
    "pstereo_gpu_stage_times", "pstereo_gpu_stage_name", "pstereo_synth_default",
    "pstereo_gpu_synth", "pstereo_synth_last_error", "pstereo_gpu_set_device_chunks", "pstereo_gpu_render",
    "pstereo_gpu_set_host_expand", "pstereo_gpu_host_threads", "pstereo_host_expand",
    "pstereo_host_expand_stats",
    "pstereo_render_last_error", "pstereo_scene_default", "pstereo_scene_validate",
    "pstereo_load_scene_spec", "pstereo_load_calibration", "pstereo_load_image",
    "pstereo_write_pfm", "pstereo_read_pfm", "pstereo_metrics_csv_header",
    "pstereo_format_metrics_row", "pstereo_write_metrics_csv", "pstereo_read_metrics_csv",
    "pstereo_synth_pair", "pstereo_synth_batch", "pstereo_debug_eval_residual",
    "pstereo_gpu_metrics", "pstereo_gpu_wait",
]


@dataclass
class PipelineConfig:
    """inc/config.hpp:12-33, published defaults."""
    coarsest_exp: int = 5
    finest_exp: int = 1
    patch_size: int = 10
    overlap: float = 0.55
    min_iterations: int = 12
    max_iterations: int = 12
    early_stop_good: float = 0.05
    early_stop_bad: float = 0.95
    early_stop_improve: float = 0.10
    window_offsets: list = field(default_factory=lambda: [0.5, 1.0])
    sigma_s: float = 4.0
    pixel_threshold: float = 0.15
    gamma: float = 0.75
    valid_patch_ratio: float = 0.75
    estimate_variance: bool = False
    threads: int = 1

    def to_c(self) -> _Params:
        p = _Params()
        for k in ("coarsest_exp", "finest_exp", "patch_size", "min_iterations",
                  "max_iterations", "threads"):
            setattr(p, k, int(getattr(self, k)))
        for k in ("overlap", "early_stop_good", "early_stop_bad", "early_stop_improve",
                  "sigma_s", "pixel_threshold", "gamma", "valid_patch_ratio"):
            setattr(p, k, float(getattr(self, k)))
        p.estimate_variance = int(bool(self.estimate_variance))
        p.n_window_offsets = len(self.window_offsets)
        for i, v in enumerate(list(self.window_offsets)[:MAX_OFF]):
            p.window_offsets[i] = float(v)
        if len(self.window_offsets) > MAX_OFF:
            p.n_window_offsets = MAX_OFF + 1  # rejected by validate
        return p

    @staticmethod
    def baseline(config: int) -> "PipelineConfig":
        """BASELINE.json configs -> PipelineConfig (SURVEY.md section 8a mapping)."""
        if config in (0, 2):
            return PipelineConfig(coarsest_exp=3, finest_exp=1, patch_size=8, overlap=0.5)
        if config == 1:
            return PipelineConfig(coarsest_exp=3, finest_exp=1, patch_size=8, overlap=0.5,
                                  estimate_variance=True)
        if config == 3:
            return PipelineConfig(coarsest_exp=4, finest_exp=1, patch_size=12,
                                  overlap=1.0 - 4.0 / 12.0, estimate_variance=True)
        raise ValueError(f"no fixed PipelineConfig for config {config}")


@dataclass
class CameraParams:
    """inc/depth_variance.hpp:20-23."""
    focal_px: float = 0.0
    baseline: float = 0.0


def _raise(code: int, msg: str):
    if code == PSTEREO_ECONFIG:
        raise ConfigError(msg)
    if code == PSTEREO_EDEGENERATE:
        raise DegenerateInputError(msg)
    raise GpuError(msg or f"pstereo error {code}")


def validate(cfg: PipelineConfig) -> None:
    """Raises ConfigError like validate() (src/coarse_to_fine.cpp:18-49)."""
    p = cfg.to_c()
    buf = C.create_string_buffer(256)
    rc = lib().pstereo_validate(C.byref(p), buf, 256)
    if rc:
        _raise(rc, buf.value.decode())


def level_dims(cfg: PipelineConfig, width: int, height: int):
    p = cfg.to_c()
    n = C.c_int()
    ws, hs, es = (np.zeros(32, np.int32) for _ in range(3))
    rc = lib().pstereo_level_dims(C.byref(p), width, height, C.byref(n),
                                  ws.ctypes.data_as(i32p), hs.ctypes.data_as(i32p),
                                  es.ctypes.data_as(i32p))
    if rc:
        _raise(rc, "level_dims")
    return [(int(es[i]), int(ws[i]), int(hs[i])) for i in range(n.value)]


def synth_spec(config: int = 0, **overrides) -> SynthSpec:
    s = SynthSpec()
    lib().pstereo_synth_default(C.byref(s), config)
    for k, v in overrides.items():
        setattr(s, k, v)
    return s


def synth_pair(config: int = 0, seed: int | None = None, with_disparity=False, **overrides):
    """One deterministic BASELINE.json pair: (left, right[, disparity])."""
    s = synth_spec(config, **overrides)
    shape = (s.height, s.width) if s.channels == 1 else (s.height, s.width, s.channels)
    left = np.zeros(shape, np.uint8)
    right = np.zeros(shape, np.uint8)
    disp = np.zeros((s.height, s.width), np.float32)
    seed = s.seed if seed is None else seed
    rc = lib().pstereo_synth_pair(C.byref(s), seed, left.ctypes.data_as(u8p),
                                  right.ctypes.data_as(u8p), disp.ctypes.data_as(f32p))
    if rc:
        _raise(rc, "synth_pair")
    return (left, right, disp) if with_disparity else (left, right)


def synth_batch(config: int, n: int, seed0: int = 0, threads: int = 8, **overrides):
    s = synth_spec(config, **overrides)
    shape = (n, s.height, s.width) if s.channels == 1 else (n, s.height, s.width, s.channels)
    left = np.zeros(shape, np.uint8)
    right = np.zeros(shape, np.uint8)
    rc = lib().pstereo_synth_batch(C.byref(s), n, seed0, left.ctypes.data_as(u8p),
                                   right.ctypes.data_as(u8p), threads)
    if rc:
        _raise(rc, "synth_batch")
    return left, right


def synth_batch_gpu(config: int, n: int, seed0: int = 0, device: int = 0, with_disparity=False,
                    stream=None, **overrides):
    """The generator on the device (pstereo_gpu_synth): the same bytes as
    synth_batch for the same (config, seeds, overrides), returned as CUDA uint8
    tensors [n, H, W(, C)] (and the float32 ground-truth disparity)."""
    import torch
    s = synth_spec(config, **overrides)
    shape = (n, s.height, s.width) if s.channels == 1 else (n, s.height, s.width, s.channels)
    dev = torch.device("cuda", device)
    left = torch.empty(shape, dtype=torch.uint8, device=dev)
    right = torch.empty(shape, dtype=torch.uint8, device=dev)
    disp = torch.empty((n, s.height, s.width), dtype=torch.float32, device=dev) \
        if with_disparity else None
    st = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
    rc = lib().pstereo_gpu_synth(device, C.byref(s), n, seed0, left.data_ptr() if n else None,
                                 right.data_ptr() if n else None,
                                 disp.data_ptr() if disp is not None and n else None, st)
    if rc:
        _raise(rc, lib().pstereo_synth_last_error().decode())
    return (left, right, disp) if with_disparity else (left, right)


# ---- analytic scenes and caller-side formats (row 3)

class IoError(OSError):
    """The reference's IoError (inc/pstereo/errors.hpp), exit code 3."""


def _check_io(rc: int, msg) -> None:
    if rc == 0:
        return
    text = msg.value.decode(errors="replace") if hasattr(msg, "value") else str(msg)
    if rc == 3:
        raise IoError(text)
    _raise(rc, text)


def scene_spec(**fields) -> SceneSpec:
    """SceneSpec defaults (inc/pstereo/synth.hpp:20-50) with overrides; surface /
    texture / shading may be given by name."""
    s = SceneSpec()
    lib().pstereo_scene_default(C.byref(s))
    for k, v in fields.items():
        if k == "name":
            v = v.encode()
        elif k == "surface" and isinstance(v, str):
            v = SceneSpec.SURFACES[v]
        elif k == "texture" and isinstance(v, str):
            v = SceneSpec.TEXTURES[v]
        elif k == "shading" and isinstance(v, str):
            v = SceneSpec.SHADINGS[v]
        setattr(s, k, v)
    msg = C.create_string_buffer(256)
    _check_io(lib().pstereo_scene_validate(C.byref(s), msg, 256), msg)
    return s


def load_scene_spec(path) -> SceneSpec:
    """load_scene_spec (src/synth.cpp:301-393)."""
    s = SceneSpec()
    msg = C.create_string_buffer(512)
    _check_io(lib().pstereo_load_scene_spec(str(path).encode(), C.byref(s), msg, 512), msg)
    return s


def render_scenes_gpu(specs, device: int = 0, stream=None, fields=True):
    """render_scene (src/synth.cpp:209-284) on the device for scenes of one
    size: CUDA tensors left/right float32 [n, h, w] and, with fields, the
    reference disparity / depth float64 [n, h, w]."""
    import torch
    specs = [specs] if isinstance(specs, SceneSpec) else list(specs)
    n = len(specs)
    arr = (SceneSpec * max(n, 1))(*specs)
    h, w = (specs[0].height, specs[0].width) if n else (0, 0)
    dev = torch.device("cuda", device)
    left = torch.empty((n, h, w), dtype=torch.float32, device=dev)
    right = torch.empty((n, h, w), dtype=torch.float32, device=dev)
    disp = torch.empty((n, h, w), dtype=torch.float64, device=dev) if fields else None
    depth = torch.empty((n, h, w), dtype=torch.float64, device=dev) if fields else None
    st = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
    ptr = (lambda t: t.data_ptr() if t is not None and n else None)
    rc = lib().pstereo_gpu_render(device, arr, n, ptr(left), ptr(right), ptr(disp), ptr(depth),
                                  st)
    if rc:
        _raise(rc, lib().pstereo_render_last_error().decode())
    return left, right, disp, depth


def load_calibration(path) -> dict:
    """load_calibration (src/io.cpp:266-281)."""
    f, b = C.c_double(), C.c_double()
    w, h = C.c_int(), C.c_int()
    msg = C.create_string_buffer(512)
    _check_io(lib().pstereo_load_calibration(str(path).encode(), C.byref(f), C.byref(b),
                                             C.byref(w), C.byref(h), msg, 512), msg)
    return {"focal_px": f.value, "baseline_mm": b.value, "width": w.value, "height": h.value}


def load_image(path) -> np.ndarray:
    """load_image (src/io.cpp:253-263): uint8 [h, w, channels] (PGM/PPM/PNG)."""
    w, h, c = C.c_int(), C.c_int(), C.c_int()
    msg = C.create_string_buffer(512)
    p = str(path).encode()
    _check_io(lib().pstereo_load_image(p, C.byref(w), C.byref(h), C.byref(c), None, 0, msg,
                                       512), msg)
    out = np.zeros((h.value, w.value, c.value), np.uint8)
    _check_io(lib().pstereo_load_image(p, C.byref(w), C.byref(h), C.byref(c),
                                       out.ctypes.data, out.nbytes, msg, 512), msg)
    return out


def write_pfm(path, values, valid=None, rows_bottom_up=False) -> None:
    """write_pfm (src/io.cpp:297-310): -1 at invalid pixels, rows bottom to top."""
    v = np.ascontiguousarray(values, np.float32)
    ok = None if valid is None else np.ascontiguousarray(valid, np.uint8)
    h, w = v.shape
    msg = C.create_string_buffer(512)
    _check_io(lib().pstereo_write_pfm(str(path).encode(), w, h, v.ctypes.data,
                                      None if ok is None else ok.ctypes.data,
                                      int(bool(rows_bottom_up)), msg, 512), msg)


def read_pfm(path) -> np.ndarray:
    """read_pfm (src/io.cpp:312-341): float32 [h, w], top row first."""
    w, h = C.c_int(), C.c_int()
    msg = C.create_string_buffer(512)
    p = str(path).encode()
    _check_io(lib().pstereo_read_pfm(p, C.byref(w), C.byref(h), None, 0, msg, 512), msg)
    out = np.zeros((h.value, w.value), np.float32)
    _check_io(lib().pstereo_read_pfm(p, C.byref(w), C.byref(h), out.ctypes.data, out.size,
                                     msg, 512), msg)
    return out


def metrics_row(frame="", mean_err=float("nan"), median_err=float("nan"), valid_px=0,
                runtime_ms=0.0, coverage_rate=float("nan")) -> MetricsRow:
    r = MetricsRow()
    r.frame = frame.encode()
    r.mean_err, r.median_err, r.valid_px = mean_err, median_err, valid_px
    r.runtime_ms, r.coverage_rate = runtime_ms, coverage_rate
    r.has_errors = int(mean_err == mean_err)
    return r


def metrics_csv_header() -> str:
    return lib().pstereo_metrics_csv_header().decode()


def format_metrics_row(row: MetricsRow) -> str:
    buf = C.create_string_buffer(1024)
    n = lib().pstereo_format_metrics_row(C.byref(row), buf, 1024)
    if n < 0:
        raise GpuError("metrics row too long")
    return buf.value.decode()


def write_metrics_csv(path, rows) -> None:
    arr = (MetricsRow * max(len(rows), 1))(*rows)
    msg = C.create_string_buffer(512)
    _check_io(lib().pstereo_write_metrics_csv(str(path).encode(), arr, len(rows), msg, 512), msg)


def read_metrics_csv(path) -> list:
    n = C.c_int()
    msg = C.create_string_buffer(512)
    p = str(path).encode()
    _check_io(lib().pstereo_read_metrics_csv(p, None, 0, C.byref(n), msg, 512), msg)
    arr = (MetricsRow * max(n.value, 1))()
    _check_io(lib().pstereo_read_metrics_csv(p, arr, n.value, C.byref(n), msg, 512), msg)
    return list(arr[: n.value])


class Matcher:
    """A device context (pstereo_gpu_create) for batches up to max_pairs of
    at most max_width x max_height."""

    def __init__(self, cfg: PipelineConfig, max_width: int, max_height: int, max_pairs: int = 1,
                 device: int = 0):
        self.cfg = cfg
        validate(cfg)
        self._p = cfg.to_c()
        h = C.c_void_p()
        rc = lib().pstereo_gpu_create(device, C.byref(self._p), max_width, max_height,
                                      max_pairs, C.byref(h))
        if rc:
            _raise(rc, f"pstereo_gpu_create failed (device {device}: needs an sm_100 GPU)")
        self._h = h
        self.n_levels = cfg.coarsest_exp - cfg.finest_exp + 1

    def close(self):
        if getattr(self, "_h", None):
            lib().pstereo_gpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def handle(self):
        return self._h

    def last_error(self) -> str:
        return lib().pstereo_gpu_last_error(self._h).decode()

    def launch_count(self) -> int:
        return lib().pstereo_gpu_last_launch_count(self._h)

    def set_graphs(self, on: bool):
        """pstereo_gpu_set_graphs: replay repeated device-buffer calls as CUDA graphs."""
        rc = lib().pstereo_gpu_set_graphs(self._h, int(bool(on)))
        if rc:
            _raise(rc, self.last_error())

    def set_fill_target(self, ctas: int):
        """pstereo_gpu_set_fill_target: spread small launches over >= ctas CTAs
        (148 = one per SM, best single-call latency; 0 = off, best with
        several calls in flight)."""
        rc = lib().pstereo_gpu_set_fill_target(self._h, int(ctas))
        if rc:
            _raise(rc, self.last_error())

    def set_device_chunks(self, chunks: int):
        """Sub-batches per device call (pstereo_gpu_set_device_chunks)."""
        lib().pstereo_gpu_set_device_chunks(self._h, int(chunks))

    def set_host_expand(self, on: bool):
        """Host-output calls download finest-resolution planes and replicate them
        on host threads (pstereo_gpu_set_host_expand; default on)."""
        lib().pstereo_gpu_set_host_expand(self._h, int(on))

    def set_profiling(self, on: bool):
        lib().pstereo_gpu_set_profiling(self._h, int(on))

    def stage_times(self):
        """(total device ms per stage since set_profiling(True), number of calls)."""
        ms = np.zeros(32, np.float64)
        calls = C.c_int()
        n = lib().pstereo_gpu_stage_times(self._h, ms.ctypes.data_as(C.POINTER(C.c_double)), 32,
                                          C.byref(calls))
        names = [lib().pstereo_gpu_stage_name(self._h, i).decode() for i in range(n)]
        return dict(zip(names, (float(v) for v in ms[:n]))), calls.value

    # ---- host-memory batched API (numpy in, numpy out)
    def run_batch(self, left, right, focal=1.0, baseline=1.0, dtype=F32, left_valid=None,
                  right_valid=None, want=("disparity", "disparity_valid"), stats=False,
                  finest_cap=0, invalid_value=None, flip_rows=False):
        """Batched run_pipeline. left/right: uint8 [n,h,w] / [n,h,w,c], or float32
        [n,h,w] GrayImage planes (+ optional u8 validity)."""
        left = np.ascontiguousarray(left)
        right = np.ascontiguousarray(right)
        is_u8 = left.dtype == np.uint8
        if is_u8:
            if left.ndim == 3:
                n, h, w = left.shape
                ch = 1
            else:
                n, h, w, ch = left.shape
        else:
            left = np.ascontiguousarray(left, np.float32)
            right = np.ascontiguousarray(right, np.float32)
            n, h, w = left.shape
        o, res, st, fin, cnt = _host_outputs(n, h, w, want, dtype, stats, self.n_levels,
                                             finest_cap, invalid_value, flip_rows)
        if is_u8:
            rc = lib().pstereo_gpu_match_u8(self._h, n, w, h, ch, left.ctypes.data,
                                            right.ctypes.data, 0, focal, baseline, C.byref(o),
                                            None)
        else:
            lv = None if left_valid is None else np.ascontiguousarray(left_valid, np.uint8)
            rv = None if right_valid is None else np.ascontiguousarray(right_valid, np.uint8)
            rc = lib().pstereo_gpu_match_f32(self._h, n, w, h, left.ctypes.data,
                                             None if lv is None else lv.ctypes.data,
                                             right.ctypes.data,
                                             None if rv is None else rv.ctypes.data, 0, focal,
                                             baseline, C.byref(o), None)
        if rc:
            _raise(rc, self.last_error())
        return _finish_outputs(res, n, self.n_levels, st, fin, cnt, finest_cap)

    # ---- device-pointer batched API (the zero-copy path used by bench.py)
    def wait(self, stream=None):
        """pstereo_gpu_wait: every stream of the context (and `stream`) done."""
        rc = lib().pstereo_gpu_wait(self._h, stream)
        if rc:
            _raise(rc, self.last_error())

    def metrics(self, estimate, estimate_valid, reference, reference_valid, sigma=None,
                sigma_valid=None):
        """compute_metrics (src/metrics.cpp:10-52) on the GPU for [n,h,w] (or [h,w])
        double fields + u8 validity; returns one dict per frame (FrameMetrics)."""
        est = np.ascontiguousarray(estimate, np.float64)
        single = est.ndim == 2
        if single:
            est = est[None]
        n, h, w = est.shape

        def prep(a, dt):
            a = np.ascontiguousarray(a, dt)
            return a[None] if a.ndim == 2 else a

        ev = prep(estimate_valid, np.uint8)
        ref = prep(reference, np.float64)
        rv = prep(reference_valid, np.uint8)
        sg = None if sigma is None else prep(sigma, np.float64)
        sv = None if sigma is None else prep(sigma_valid, np.uint8)
        for a in (ev, ref, rv) + ((sg, sv) if sg is not None else ()):
            if a.shape != (n, h, w):
                raise ValueError("metrics: field shapes differ")
        out = (FrameMetricsC * max(n, 1))()
        ptr = (lambda a: a.ctypes.data if a is not None else None)
        rc = lib().pstereo_gpu_metrics(self._h, n, w, h, ptr(est), ptr(ev), ptr(ref), ptr(rv),
                                       ptr(sg), ptr(sv), 0, out, None)
        if rc:
            _raise(rc, self.last_error())
        res = [{k: getattr(out[i], k) for k, _ in FrameMetricsC._fields_} for i in range(n)]
        for r in res:
            r["has_errors"] = bool(r["has_errors"])
        return res[0] if single else res

    def run_device_f32(self, n, width, height, left_ptr, right_ptr, outputs: dict, dtype=F32,
                       focal=1.0, baseline=1.0, stream=None, left_valid_ptr=None,
                       right_valid_ptr=None, invalid_value=None, flip_rows=False):
        """GrayImage planes (fp32 [n,h,w] + optional u8 validity) and outputs in
        device memory: only enqueues work on `stream`."""
        o = _Outputs()
        o.dtype = dtype
        o.on_device = 1
        o.flip_rows = int(bool(flip_rows))
        if invalid_value is not None:
            o.fill_invalid, o.invalid_value = 1, float(invalid_value)
        for k, ptr in outputs.items():
            setattr(o, k, ptr)
        rc = lib().pstereo_gpu_match_f32(self._h, n, width, height, left_ptr, left_valid_ptr,
                                         right_ptr, right_valid_ptr, 1, focal, baseline,
                                         C.byref(o), stream)
        if rc:
            _raise(rc, self.last_error())

    def metrics_device(self, n, width, height, est, est_valid, ref, ref_valid, sigma=None,
                       sigma_valid=None, stream=None):
        """compute_metrics on device-resident double fields (pointers)."""
        out = (FrameMetricsC * max(n, 1))()
        rc = lib().pstereo_gpu_metrics(self._h, n, width, height, est, est_valid, ref,
                                       ref_valid, sigma, sigma_valid, 1, out, stream)
        if rc:
            _raise(rc, self.last_error())
        res = [{k: getattr(out[i], k) for k, _ in FrameMetricsC._fields_} for i in range(n)]
        for r in res:
            r["has_errors"] = bool(r["has_errors"])
        return res

    def run_device_u8(self, n, width, height, channels, left_ptr, right_ptr, outputs: dict,
                      dtype=F32, focal=1.0, baseline=1.0, stream=None, invalid_value=None, flip_rows=False):
        o = _Outputs()
        o.dtype = dtype
        o.on_device = 1
        o.flip_rows = int(bool(flip_rows))
        if invalid_value is not None:
            o.fill_invalid, o.invalid_value = 1, float(invalid_value)
        for k, ptr in outputs.items():
            setattr(o, k, ptr)
        rc = lib().pstereo_gpu_match_u8(self._h, n, width, height, channels, left_ptr, right_ptr,
                                        1, focal, baseline, C.byref(o), stream)
        if rc:
            _raise(rc, self.last_error())

    def run_host_u8(self, n, width, height, channels, left_ptr, right_ptr, outputs: dict,
                    dtype=F32, focal=1.0, baseline=1.0, stream=None, invalid_value=None,
                    async_host=False):
        """Host (ideally pinned) buffers in and out; H2D/D2H inside the call.
        async_host: return once queued; outputs complete after wait()."""
        o = _Outputs()
        o.dtype = dtype
        o.on_device = 0
        o.async_host = int(bool(async_host))
        if invalid_value is not None:
            o.fill_invalid, o.invalid_value = 1, float(invalid_value)
        for k, ptr in outputs.items():
            setattr(o, k, ptr)
        rc = lib().pstereo_gpu_match_u8(self._h, n, width, height, channels, left_ptr, right_ptr,
                                        0, focal, baseline, C.byref(o), stream)
        if rc:
            _raise(rc, self.last_error())


_MATCHERS: dict = {}


def _matcher_for(cfg: PipelineConfig, w: int, h: int) -> Matcher:
    key = (repr(cfg), w, h)
    m = _MATCHERS.get(key)
    if m is None:
        m = _MATCHERS[key] = Matcher(cfg, w, h, 1)
    return m


def _as_gray(img):
    """GrayImage-like input: (data fp32 [h,w], valid u8 or None)."""
    if isinstance(img, tuple):
        return np.ascontiguousarray(img[0], np.float32), img[1]
    return np.ascontiguousarray(img, np.float32), None


def run_pipeline(left, right, cfg: PipelineConfig, cam: CameraParams, dtype=F64) -> dict:
    """run_pipeline (inc/pipeline.hpp:20-22) on one GrayImage pair: left/right are
    float32 [h,w] planes or (plane, valid) tuples. Returns the PipelineOutput
    fields as numpy arrays plus per-level MatchStats."""
    validate(cfg)
    (l, lv), (r, rv) = _as_gray(left), _as_gray(right)
    if l.shape != r.shape:
        raise DegenerateInputError(f"build_pipeline: left is {l.shape} but right is {r.shape}")
    h, w = l.shape
    m = _matcher_for(cfg, max(w, 1), max(h, 1))
    want = ["disparity", "disparity_valid", "probability", "depth", "depth_valid"]
    if cfg.estimate_variance:
        want += ["depth_sigma", "sigma_valid"]
    out = m.run_batch(l[None], r[None], focal=cam.focal_px, baseline=cam.baseline, dtype=dtype,
                      left_valid=None if lv is None else np.asarray(lv)[None],
                      right_valid=None if rv is None else np.asarray(rv)[None], want=want,
                      stats=True)
    res = {k: v[0] for k, v in out.items() if k != "stats"}
    res["probability_valid"] = res["disparity_valid"]
    res["stats"] = out["stats"][0]
    res["has_sigma"] = bool(cfg.estimate_variance)
    return res


def match_stereo(left, right, cfg: PipelineConfig, dtype=F64, finest_cap=1 << 16) -> dict:
    """match_stereo (inc/coarse_to_fine.hpp:102-103): pre-filter full-resolution
    disparity/probability(/var_disp), MatchStats and the finest-level patches."""
    validate(cfg)
    (l, lv), (r, rv) = _as_gray(left), _as_gray(right)
    if l.shape != r.shape:
        raise DegenerateInputError(f"match_stereo: left is {l.shape} but right is {r.shape}")
    h, w = l.shape
    m = _matcher_for(cfg, max(w, 1), max(h, 1))
    want = ["match_disparity", "match_valid"]
    if cfg.estimate_variance:
        want.append("var_disp")
    out = m.run_batch(l[None], r[None], dtype=dtype,
                      left_valid=None if lv is None else np.asarray(lv)[None],
                      right_valid=None if rv is None else np.asarray(rv)[None], want=want,
                      stats=True, finest_cap=finest_cap)
    res = {"disparity": out["match_disparity"][0], "disparity_valid": out["match_valid"][0],
           "stats": out["stats"][0], "finest": out["finest"][0],
           "has_variance": bool(cfg.estimate_variance)}
    if cfg.estimate_variance:
        res["var_disp"] = out["var_disp"][0]
    return res


def compute_metrics(estimate, estimate_valid, reference, reference_valid, sigma=None,
                    sigma_valid=None):
    """compute_metrics (src/metrics.cpp:10-52) on the GPU; see Matcher.metrics."""
    est = np.asarray(estimate)
    h, w = est.shape[-2], est.shape[-1]
    return _matcher_for(PipelineConfig(coarsest_exp=0, finest_exp=0, patch_size=2), w, h).metrics(
        estimate, estimate_valid, reference, reference_valid, sigma, sigma_valid)


def run_benchmark_gpu(scenes, cfg: "PipelineConfig", repetitions: int = 10, device: int = 0):
    """run_benchmark (src/bench.cpp:11-67) on the device: every scene rendered
    by pstereo_gpu_render, matched `repetitions` times (runtime_ms = mean CUDA
    event time of one run_pipeline call), depth errors against the scene's
    reference depth by pstereo_gpu_metrics; returns the per-scene FrameMetrics
    rows plus the aggregate row ("average", NaN-aware means)."""
    import math

    import torch
    if repetitions < 1:
        raise ConfigError("benchmark repetitions must be >= 1")
    scenes = list(scenes)
    if not scenes:
        raise ConfigError("benchmark needs at least one scene")
    validate(cfg)
    dev = torch.device("cuda", device)
    stream = torch.cuda.Stream(dev)
    sh = stream.cuda_stream
    frames = []
    with torch.cuda.stream(stream):
        for spec in scenes:
            w, h = spec.width, spec.height
            left, right, _, ref_depth = render_scenes_gpu([spec], device=device, stream=sh)
            ones = torch.ones((1, h, w), dtype=torch.uint8, device=dev)
            depth = torch.empty((1, h, w), dtype=torch.float64, device=dev)
            dvalid = torch.empty((1, h, w), dtype=torch.uint8, device=dev)
            var = bool(cfg.estimate_variance)
            sig = torch.empty_like(depth) if var else None
            svalid = torch.empty_like(dvalid) if var else None
            outs = {"depth": depth.data_ptr(), "depth_valid": dvalid.data_ptr()}
            if var:
                outs.update(depth_sigma=sig.data_ptr(), sigma_valid=svalid.data_ptr())
            with Matcher(cfg, w, h, 1, device=device) as m:
                total = 0.0
                for _ in range(repetitions):
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    m.run_device_f32(1, w, h, left.data_ptr(), right.data_ptr(), outs,
                                     dtype=F64, focal=spec.focal_px, baseline=spec.baseline,
                                     stream=sh)
                    e1.record(stream)
                    e1.synchronize()
                    total += e0.elapsed_time(e1)
                r = m.metrics_device(1, w, h, depth.data_ptr(), dvalid.data_ptr(),
                                     ref_depth.data_ptr(), ones.data_ptr(),
                                     sig.data_ptr() if var else None,
                                     svalid.data_ptr() if var else None, stream=sh)[0]
            frames.append({"frame": spec.name.decode(), "mean_err": r["mean_err"],
                           "median_err": r["median_err"], "valid_px": r["valid_px"],
                           "runtime_ms": total / repetitions,
                           "coverage_rate": r["coverage_rate"] if var else float("nan"),
                           "has_errors": r["has_errors"]})
    # aggregate row, src/bench.cpp:37-65
    err = [f for f in frames if f["has_errors"]]
    cov = [f["coverage_rate"] for f in frames if not math.isnan(f["coverage_rate"])]
    agg = {"frame": "average", "mean_err": float("nan"), "median_err": float("nan"),
           "has_errors": False, "coverage_rate": float("nan")}
    if err:
        ms = ds = 0.0
        for f in err:
            ms += f["mean_err"]
            ds += f["median_err"]
        agg.update(mean_err=ms / len(err), median_err=ds / len(err), has_errors=True)
    if cov:
        c = 0.0
        for v in cov:
            c += v
        agg["coverage_rate"] = c / len(cov)
    px = ms_ = 0.0
    for f in frames:
        px += float(f["valid_px"])
        ms_ += f["runtime_ms"]
    agg["valid_px"] = int(px / len(frames) + 0.5)
    agg["runtime_ms"] = ms_ / len(frames)
    return frames, agg


def _host_outputs(n, h, w, want, dtype, stats, n_levels, finest_cap, invalid_value, flip_rows):
    """pstereo_outputs over freshly allocated host planes (numpy)."""
    vt = np.float64 if dtype == F64 else np.float32
    res = {}
    o = _Outputs()
    o.dtype = dtype
    o.on_device = 0
    o.flip_rows = int(bool(flip_rows))
    if invalid_value is not None:
        o.fill_invalid, o.invalid_value = 1, float(invalid_value)
    planes = {"disparity": vt, "disparity_valid": np.uint8, "probability": vt, "depth": vt,
              "depth_valid": np.uint8, "depth_sigma": vt, "sigma_valid": np.uint8,
              "match_disparity": vt, "match_valid": np.uint8, "var_disp": vt}
    for k in want:
        a = np.zeros((n, h, w), planes[k])
        res[k] = a
        setattr(o, k, a.ctypes.data)
    st = None
    if stats:
        st = (LevelStats * max(n * n_levels, 1))()
        o.stats = st
    fin = cnt = None
    if finest_cap:
        fin = (PatchEstimate * max(n * finest_cap, 1))()
        cnt = np.zeros(max(n, 1), np.int32)
        o.finest = fin
        o.finest_count = cnt.ctypes.data_as(i32p)
        o.finest_cap = finest_cap
    return o, res, st, fin, cnt


def _finish_outputs(res, n, n_levels, st, fin, cnt, finest_cap):
    if st is not None:
        res["stats"] = np.array([st[i].as_tuple() for i in range(n * n_levels)],
                                np.int64).reshape(n, n_levels, 5)
    if finest_cap:
        res["finest"] = []
        for p in range(n):
            rows = [(fin[p * finest_cap + k].cx, fin[p * finest_cap + k].cy,
                     fin[p * finest_cap + k].u, fin[p * finest_cap + k].prob,
                     fin[p * finest_cap + k].posterior, fin[p * finest_cap + k].sigma_k)
                    for k in range(min(int(cnt[p]), finest_cap))]
            res["finest"].append(np.array(rows, np.float64).reshape(-1, 6))
        res["finest_count"] = cnt[:n]
    return res


class MultiMatcher:
    """pstereo_multi: one context and one host thread per entry of `devices`
    (entries may repeat); a batch is split into contiguous pair blocks, one
    per device, each matched from host memory with no exchange between
    devices."""

    def __init__(self, cfg: PipelineConfig, max_width: int, max_height: int, max_pairs: int,
                 devices=(0,)):
        validate(cfg)
        self.cfg = cfg
        self._p = cfg.to_c()
        devs = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        rc = lib().pstereo_multi_create(devs, len(devices), C.byref(self._p), max_width,
                                        max_height, max_pairs, C.byref(h))
        if rc:
            _raise(rc, f"pstereo_multi_create failed (devices {list(devices)})")
        self._h = h
        self.n_devices = len(devices)
        self.n_levels = cfg.coarsest_exp - cfg.finest_exp + 1

    def close(self):
        if getattr(self, "_h", None):
            lib().pstereo_multi_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def run_batch(self, left, right, focal=1.0, baseline=1.0, dtype=F32,
                  want=("disparity", "disparity_valid"), stats=False, finest_cap=0,
                  invalid_value=None, flip_rows=False):
        """uint8 pairs [n,h,w] / [n,h,w,c] from host memory; returns the same
        dict as Matcher.run_batch plus "ms_per_device"."""
        left = np.ascontiguousarray(left, np.uint8)
        right = np.ascontiguousarray(right, np.uint8)
        if left.ndim == 3:
            (n, h, w), ch = left.shape, 1
        else:
            n, h, w, ch = left.shape
        o, res, st, fin, cnt = _host_outputs(n, h, w, want, dtype, stats, self.n_levels,
                                             finest_cap, invalid_value, flip_rows)
        ms = (C.c_double * self.n_devices)()
        rc = lib().pstereo_multi_match_u8(self._h, n, w, h, ch, left.ctypes.data,
                                          right.ctypes.data, focal, baseline, C.byref(o),
                                          C.cast(ms, C.c_void_p))
        if rc:
            _raise(rc, lib().pstereo_multi_last_error(self._h).decode())
        res = _finish_outputs(res, n, self.n_levels, st, fin, cnt, finest_cap)
        res["ms_per_device"] = list(ms)
        return res


def host_expand(src: np.ndarray, W: int, H: int, e: int, flip_rows: bool = False) -> np.ndarray:
    """upsample_to_full's block replication on the host pool (pstereo_host_expand):
    src is [frames, fh, fw] of a 1-, 4- or 8-byte dtype."""
    src = np.ascontiguousarray(src)
    n, fh, fw = src.shape
    dst = np.empty((n, H, W), src.dtype)
    rc = lib().pstereo_host_expand(src.ctypes.data, dst.ctypes.data, src.dtype.itemsize, fw, fh,
                                   W, H, e, n, int(flip_rows))
    if rc:
        _raise(rc, "pstereo_host_expand: bad arguments")
    return dst


def host_expand_stats():
    """(worker ms spent replicating, frames finished) since the pool started."""
    ms, fr = C.c_double(), C.c_longlong()
    lib().pstereo_host_expand_stats(C.byref(ms), C.byref(fr))
    return ms.value, fr.value
