"""ctypes bindings of oracle/bdis_oracle.h -- TEST INFRASTRUCTURE ONLY.

Loads either the plain-C restatement (oracle/libbdis_oracle.so, kind="port")
or the reference itself (oracle/_ref/libbdis_ref.so, kind="reference"); both
export the same symbols. Only tests/, __graft_entry__.smoke() and bench.py's
CPU legs may import this module -- never the product path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIBS = {"port": HERE / "libbdis_oracle.so", "reference": HERE / "_ref" / "libbdis_ref.so"}
MAX_OFF = 16

u8p = C.POINTER(C.c_uint8)
f32p = C.POINTER(C.c_float)
f64p = C.POINTER(C.c_double)
i32p = C.POINTER(C.c_int)


class BoConfig(C.Structure):
    _fields_ = [
        ("coarsest_exp", C.c_int), ("finest_exp", C.c_int), ("patch_size", C.c_int),
        ("overlap", C.c_double), ("min_iterations", C.c_int), ("max_iterations", C.c_int),
        ("early_stop_good", C.c_double), ("early_stop_bad", C.c_double),
        ("early_stop_improve", C.c_double), ("n_window_offsets", C.c_int),
        ("window_offsets", C.c_double * MAX_OFF), ("sigma_s", C.c_double),
        ("pixel_threshold", C.c_double), ("gamma", C.c_double),
        ("valid_patch_ratio", C.c_double), ("estimate_variance", C.c_int), ("threads", C.c_int),
    ]


class BoImage(C.Structure):
    _fields_ = [("width", C.c_int), ("height", C.c_int), ("data", f32p), ("valid", u8p)]


class BoLkParams(C.Structure):
    _fields_ = [("min_iterations", C.c_int), ("max_iterations", C.c_int),
                ("update_epsilon", C.c_double), ("stop_good", C.c_double),
                ("stop_bad", C.c_double), ("stop_improve", C.c_double)]


class BoPatchInfo(C.Structure):
    _fields_ = [("mean", C.c_double), ("valid_fraction", C.c_double), ("valid_count", C.c_int),
                ("hessian", C.c_double), ("template_msq", C.c_double), ("degenerate", C.c_int)]


class BoOutputs(C.Structure):
    _fields_ = [("disparity", f64p), ("disparity_valid", u8p), ("probability", f64p),
                ("probability_valid", u8p), ("depth", f64p), ("depth_valid", u8p),
                ("depth_sigma", f64p), ("sigma_valid", u8p), ("has_sigma", C.c_int),
                ("stats", i32p), ("n_levels", C.c_int), ("runtime_ms", C.c_double)]


class BoFrameMetrics(C.Structure):
    _fields_ = [("valid_px", C.c_longlong), ("compared", C.c_longlong), ("has_errors", C.c_int),
                ("mean_err", C.c_double), ("median_err", C.c_double),
                ("coverage_rate", C.c_double)]


class BoMatchOutputs(C.Structure):
    _fields_ = [("disparity", f64p), ("disparity_valid", u8p), ("probability", f64p),
                ("probability_valid", u8p), ("var_disp", f64p), ("var_valid", u8p),
                ("has_variance", C.c_int), ("stats", i32p), ("n_levels", C.c_int),
                ("finest_cap", C.c_int), ("finest_count", C.c_int), ("finest", f64p)]


def _p(a, t):
    return a.ctypes.data_as(t) if a is not None else None


@dataclass
class Config:
    """PipelineConfig (inc/config.hpp:12-33) with the published defaults."""
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

    def to_c(self) -> BoConfig:
        c = BoConfig()
        for k in ("coarsest_exp", "finest_exp", "patch_size", "min_iterations",
                  "max_iterations", "threads"):
            setattr(c, k, int(getattr(self, k)))
        for k in ("overlap", "early_stop_good", "early_stop_bad", "early_stop_improve",
                  "sigma_s", "pixel_threshold", "gamma", "valid_patch_ratio"):
            setattr(c, k, float(getattr(self, k)))
        c.estimate_variance = int(bool(self.estimate_variance))
        c.n_window_offsets = len(self.window_offsets)
        for i, v in enumerate(self.window_offsets[:MAX_OFF]):
            c.window_offsets[i] = float(v)
        return c


class BoScene(C.Structure):
    """bo_scene = SceneSpec (inc/pstereo/synth.hpp:20-50), same layout as the
    product's pstereo_scene_spec."""
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


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class Oracle:
    """One loaded checker library (kind = "port" or "reference")."""

    def __init__(self, kind: str = "port"):
        path = LIBS[kind]
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (python -m paper_2205_03133_b200.build)")
        self.kind = kind
        self.lib = L = C.CDLL(str(path))
        L.bo_fast_exp.restype = C.c_double
        L.bo_fast_exp.argtypes = [C.c_double]
        L.bo_dynamic_sigma.restype = C.c_double
        L.bo_level_weight.restype = C.c_double
        L.bo_propagate_probability.restype = C.c_double
        L.bo_propagate_probability.argtypes = [C.c_double, C.c_double, C.c_int, C.c_int, i32p]
        L.bo_level_weight.argtypes = [C.c_int, C.c_int, i32p]
        L.bo_dynamic_sigma.argtypes = [C.c_int, f64p, u8p, C.c_double]
        for fn in ("bo_scene_disparity_at", "bo_scene_intensity_at"):
            getattr(L, fn).restype = C.c_double
            getattr(L, fn).argtypes = [C.POINTER(BoScene), C.c_double, C.c_double]
        L.bo_value_noise.restype = C.c_double
        L.bo_value_noise.argtypes = [C.c_double, C.c_double, C.c_uint64, C.c_int, C.c_double]
        L.bo_gaussian_noise.restype = C.c_double
        L.bo_gaussian_noise.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.bo_render_scene.argtypes = [C.POINTER(BoScene), f32p, f32p, f64p, f64p]

    # ---- helpers
    @staticmethod
    def image(data: np.ndarray, valid: np.ndarray | None = None):
        data = np.ascontiguousarray(data, dtype=np.float32)
        h, w = data.shape
        if valid is not None:
            valid = np.ascontiguousarray(valid, dtype=np.uint8)
        img = BoImage(w, h, _p(data, f32p), _p(valid, u8p))
        img._keep = (data, valid)
        return img

    # ---- analytic scenes (src/synth.cpp)
    @staticmethod
    def scene(spec) -> "BoScene":
        """A bo_scene from a layout-identical ctypes struct (the product's
        SceneSpec) or a dict of fields."""
        if isinstance(spec, dict):
            b = BoScene()
            for k, v in spec.items():
                setattr(b, k, v.encode() if k == "name" else v)
            return b
        return BoScene.from_buffer_copy(bytes(spec))

    def render_scene(self, spec):
        b = self.scene(spec)
        n = b.width * b.height
        left = np.zeros((b.height, b.width), np.float32)
        right = np.zeros_like(left)
        disp = np.zeros((b.height, b.width), np.float64)
        depth = np.zeros_like(disp)
        self.lib.bo_render_scene(C.byref(b), _p(left, f32p), _p(right, f32p), _p(disp, f64p),
                                 _p(depth, f64p))
        assert n == left.size
        return left, right, disp, depth

    def scene_disparity_at(self, spec, x, y) -> float:
        return self.lib.bo_scene_disparity_at(C.byref(self.scene(spec)), x, y)

    def scene_intensity_at(self, spec, x, y) -> float:
        return self.lib.bo_scene_intensity_at(C.byref(self.scene(spec)), x, y)

    def value_noise(self, x, y, seed, octaves, base) -> float:
        return self.lib.bo_value_noise(x, y, seed, octaves, base)

    def gaussian_noise(self, seed, stream, index) -> float:
        return self.lib.bo_gaussian_noise(seed, stream, index)

    # ---- numerics
    def fast_exp(self, x: float) -> float:
        return self.lib.bo_fast_exp(float(x))

    def spatial_mask(self, size: int, sigma_s: float) -> np.ndarray:
        out = np.zeros(size * size, np.float64)
        self.lib.bo_spatial_mask(C.c_int(size), C.c_double(sigma_s), _p(out, f64p))
        return out.reshape(size, size)

    def to_grayscale(self, raster: np.ndarray):
        raster = np.ascontiguousarray(raster, np.uint8)
        if raster.ndim == 2:
            raster = raster[:, :, None]
        h, w, c = raster.shape
        out = np.zeros((h, w), np.float32)
        valid = np.zeros((h, w), np.uint8)
        self.lib.bo_to_grayscale(C.c_int(w), C.c_int(h), C.c_int(c), _p(raster, u8p),
                                 _p(out, f32p), _p(valid, u8p))
        return out, valid

    def sample_bilinear(self, data, valid, x, y):
        img = self.image(data, valid)
        v = C.c_double()
        ok = self.lib.bo_sample_bilinear(C.byref(img), C.c_double(x), C.c_double(y), C.byref(v))
        return v.value, bool(ok)

    def downsample_half(self, data, valid=None):
        data = np.ascontiguousarray(data, np.float32)
        h, w = data.shape
        if valid is None:
            valid = np.ones_like(data, np.uint8)
        valid = np.ascontiguousarray(valid, np.uint8)
        ow, oh = (w + 1) // 2, (h + 1) // 2
        out = np.zeros((oh, ow), np.float32)
        ov = np.zeros((oh, ow), np.uint8)
        self.lib.bo_downsample_half(C.c_int(w), C.c_int(h), _p(data, f32p), _p(valid, u8p),
                                    _p(out, f32p), _p(ov, u8p))
        return out, ov

    def gradient_x(self, data):
        data = np.ascontiguousarray(data, np.float32)
        h, w = data.shape
        out = np.zeros_like(data)
        self.lib.bo_gradient_x(C.c_int(w), C.c_int(h), _p(data, f32p), _p(out, f32p))
        return out

    # ---- patch level
    def extract_patch(self, data, valid, cx, cy, size):
        img = self.image(data, valid)
        vals = np.zeros(size * size, np.float64)
        ok = np.zeros(size * size, np.uint8)
        info = BoPatchInfo()
        r = self.lib.bo_extract_patch(C.byref(img), C.c_double(cx), C.c_double(cy),
                                      C.c_int(size), _p(vals, f64p), _p(ok, u8p), C.byref(info))
        if not r:
            return None
        return vals, ok, info

    def patch_system(self, left, grad, cx, cy, size, valid=None):
        img = self.image(left, valid)
        grad = np.ascontiguousarray(grad, np.float32)
        jac = np.zeros(size * size, np.float64)
        info = BoPatchInfo()
        r = self.lib.bo_patch_system(C.byref(img), _p(grad, f32p), C.c_double(cx),
                                     C.c_double(cy), C.c_int(size), _p(jac, f64p), C.byref(info))
        return (jac, info) if r else None

    def eval_residual(self, left, grad, right, cx, cy, size, u):
        li, ri = self.image(left), self.image(right)
        grad = np.ascontiguousarray(grad, np.float32)
        msq, jr, n = C.c_double(), C.c_double(), C.c_int()
        r = self.lib.bo_eval_residual(C.byref(li), _p(grad, f32p), C.byref(ri), C.c_double(cx),
                                      C.c_double(cy), C.c_int(size), C.c_double(u),
                                      C.byref(msq), C.byref(jr), C.byref(n))
        return (msq.value, jr.value, n.value) if r else None

    def solve_patch(self, left, grad, right, cx, cy, size, u_init, *, min_iterations=12,
                    max_iterations=12, update_epsilon=1e-2, stop_good=0.05, stop_bad=0.95,
                    stop_improve=0.10):
        li, ri = self.image(left), self.image(right)
        grad = np.ascontiguousarray(grad, np.float32)
        p = BoLkParams(min_iterations, max_iterations, update_epsilon, stop_good, stop_bad,
                       stop_improve)
        u, conv, it, fr = C.c_double(), C.c_int(), C.c_int(), C.c_double()
        r = self.lib.bo_solve_patch(C.byref(li), _p(grad, f32p), C.byref(ri), C.c_double(cx),
                                    C.c_double(cy), C.c_int(size), C.c_double(u_init), C.byref(p),
                                    C.byref(u), C.byref(conv), C.byref(it), C.byref(fr))
        if not r:
            return None
        return {"u": u.value, "converged": bool(conv.value), "iterations": it.value,
                "final_residual": fr.value}

    def sample_window(self, left, grad, right, cx, cy, size, u_k, mags):
        li, ri = self.image(left), self.image(right)
        grad = np.ascontiguousarray(grad, np.float32)
        mags = np.ascontiguousarray(mags, np.float64)
        n = 2 * len(mags) + 1
        offs = np.zeros(n, np.float64)
        res = np.zeros(n, np.float64)
        ok = np.zeros(n, np.uint8)
        c = C.c_int()
        r = self.lib.bo_sample_window(C.byref(li), _p(grad, f32p), C.byref(ri), C.c_double(cx),
                                      C.c_double(cy), C.c_int(size), C.c_double(u_k),
                                      C.c_int(len(mags)), _p(mags, f64p), _p(offs, f64p),
                                      _p(res, f64p), _p(ok, u8p), C.byref(c))
        if r <= 0:
            return None
        return {"offsets": offs, "residuals": res, "valid": ok, "center_index": c.value}

    def dynamic_sigma(self, residuals, valid=None, floor=1e-4):
        r = np.ascontiguousarray(residuals, np.float64)
        v = np.ones(len(r), np.uint8) if valid is None else np.ascontiguousarray(valid, np.uint8)
        return self.lib.bo_dynamic_sigma(len(r), _p(r, f64p), _p(v, u8p), floor)

    def window_priors(self, residuals, sigma_r, patch_size, use_fast_exp=True, valid=None):
        r = np.ascontiguousarray(residuals, np.float64)
        v = np.ones(len(r), np.uint8) if valid is None else np.ascontiguousarray(valid, np.uint8)
        out = np.zeros(len(r), np.float64)
        self.lib.bo_window_priors(C.c_int(len(r)), _p(r, f64p), _p(v, u8p), C.c_double(sigma_r),
                                  C.c_int(patch_size), C.c_int(int(use_fast_exp)), _p(out, f64p))
        return out

    def patch_posterior(self, residuals, sigma_r, patch_size, use_fast_exp=True, valid=None,
                        center=None):
        r = np.ascontiguousarray(residuals, np.float64)
        v = np.ones(len(r), np.uint8) if valid is None else np.ascontiguousarray(valid, np.uint8)
        c = len(r) // 2 if center is None else center
        prob, is_min = C.c_double(), C.c_int()
        ok = self.lib.bo_patch_posterior(C.c_int(len(r)), _p(r, f64p), _p(v, u8p), C.c_int(c),
                                         C.c_double(sigma_r), C.c_int(patch_size),
                                         C.c_int(int(use_fast_exp)), C.byref(prob), C.byref(is_min))
        if not ok:
            return None
        return prob.value, bool(is_min.value)

    def estimate_variance(self, offsets, priors, valid=None, center=None, fallback=2.0):
        o = np.ascontiguousarray(offsets, np.float64)
        p = np.ascontiguousarray(priors, np.float64)
        v = np.ones(len(o), np.uint8) if valid is None else np.ascontiguousarray(valid, np.uint8)
        c = len(o) // 2 if center is None else center
        sk, ck, fr = C.c_double(), C.c_double(), C.c_double()
        acc, reason = C.c_int(), C.c_int()
        self.lib.bo_estimate_variance(C.c_int(len(o)), _p(o, f64p), _p(v, u8p), C.c_int(c),
                                      _p(p, f64p), C.c_double(fallback), C.byref(sk), C.byref(ck),
                                      C.byref(acc), C.byref(reason), C.byref(fr))
        return {"sigma_k": sk.value, "c_k": ck.value, "accepted": bool(acc.value),
                "reason": ("none", "residual_too_large", "not_gaussian")[reason.value],
                "fit_residual": fr.value}

    # ---- level / grid
    def make_patch_grid(self, w, h, size, overlap):
        cap = 4096
        xs = np.zeros(cap, np.float64)
        ys = np.zeros(cap, np.float64)
        st, nx, ny = C.c_int(), C.c_int(), C.c_int()
        rc = self.lib.bo_make_patch_grid(C.c_int(w), C.c_int(h), C.c_int(size),
                                         C.c_double(overlap), C.byref(st), C.byref(nx),
                                         C.byref(ny), _p(xs, f64p), _p(ys, f64p), C.c_int(cap))
        if rc:
            raise OracleError(rc, "make_patch_grid: level smaller than one patch")
        return st.value, xs[: nx.value].copy(), ys[: ny.value].copy()

    def level_weight(self, n, levels):
        lv = np.ascontiguousarray(levels, np.int32)
        return self.lib.bo_level_weight(n, len(lv), _p(lv, i32p))

    def propagate_probability(self, posterior, inherited, n, levels):
        lv = np.ascontiguousarray(levels, np.int32)
        return self.lib.bo_propagate_probability(posterior, inherited, n, len(lv), _p(lv, i32p))

    def fuse_level(self, patches, size, sigma_s, w, h, with_variance=False):
        """patches: list of (cx, cy, u, prob[, sigma_k])."""
        arr = np.zeros((max(len(patches), 1), 5), np.float64)
        for i, p in enumerate(patches):
            arr[i, : len(p)] = p
        cols = [np.ascontiguousarray(arr[:, k]) for k in range(5)]
        out = {k: np.zeros(h * w, np.float64) for k in ("disp", "prob", "var")}
        ok = {k: np.zeros(h * w, np.uint8) for k in ("disp", "prob", "var")}
        self.lib.bo_fuse_level(C.c_int(len(patches)), *(_p(c, f64p) for c in cols[:4]),
                               _p(cols[4], f64p) if with_variance else None, C.c_int(size),
                               C.c_double(sigma_s), C.c_int(w), C.c_int(h),
                               C.c_int(int(with_variance)), _p(out["disp"], f64p),
                               _p(ok["disp"], u8p), _p(out["prob"], f64p), _p(ok["prob"], u8p),
                               _p(out["var"], f64p), _p(ok["var"], u8p))
        return ({k: v.reshape(h, w) for k, v in out.items()},
                {k: v.reshape(h, w) for k, v in ok.items()})

    def init_next_level(self, values, valid, fw, fh):
        v = np.ascontiguousarray(values, np.float64)
        ok = np.ascontiguousarray(valid, np.uint8)
        ch, cw = v.shape
        out = np.zeros((fh, fw), np.float64)
        self.lib.bo_init_next_level(C.c_int(cw), C.c_int(ch), _p(v, f64p), _p(ok, u8p),
                                    C.c_int(fw), C.c_int(fh), _p(out, f64p))
        return out

    def upsample_to_full(self, values, valid, fw, fh, e, scale):
        v = np.ascontiguousarray(values, np.float64)
        ok = np.ascontiguousarray(valid, np.uint8)
        h, w = v.shape
        out = np.zeros((fh, fw), np.float64)
        ov = np.zeros((fh, fw), np.uint8)
        self.lib.bo_upsample_to_full(C.c_int(w), C.c_int(h), _p(v, f64p), _p(ok, u8p),
                                     C.c_int(fw), C.c_int(fh), C.c_int(e), C.c_double(scale),
                                     _p(out, f64p), _p(ov, u8p))
        return out, ov

    # ---- filter / depth
    def compute_metrics(self, est, est_valid, ref, ref_valid, sigma=None, sigma_valid=None):
        """src/metrics.cpp:10-52 -> dict(valid_px, compared, has_errors, mean_err,
        median_err, coverage_rate)."""
        e = np.ascontiguousarray(est, np.float64)
        ev = np.ascontiguousarray(est_valid, np.uint8)
        r = np.ascontiguousarray(ref, np.float64)
        rv = np.ascontiguousarray(ref_valid, np.uint8)
        sg = None if sigma is None else np.ascontiguousarray(sigma, np.float64)
        sv = None if sigma is None else np.ascontiguousarray(sigma_valid, np.uint8)
        h, w = e.shape
        m = BoFrameMetrics()
        self.lib.bo_compute_metrics(C.c_int(w), C.c_int(h), _p(e, f64p), _p(ev, u8p), _p(r, f64p),
                                    _p(rv, u8p), _p(sg, f64p), _p(sv, u8p), C.byref(m))
        return {k: getattr(m, k) for k, _ in BoFrameMetrics._fields_}

    def remove_small_components(self, valid, min_px):
        v = np.ascontiguousarray(valid, np.uint8)
        h, w = v.shape
        out = np.zeros_like(v)
        self.lib.bo_remove_small_components(_p(v, u8p), C.c_int(w), C.c_int(h),
                                            C.c_longlong(min_px), _p(out, u8p))
        return out

    def filter_validity(self, disp_valid, prob, prob_valid, gamma, threshold, patch_size):
        dv = np.ascontiguousarray(disp_valid, np.uint8)
        p = np.ascontiguousarray(prob, np.float64)
        pv = np.ascontiguousarray(prob_valid, np.uint8)
        h, w = dv.shape
        out = np.zeros_like(dv)
        self.lib.bo_filter_validity(C.c_int(w), C.c_int(h), _p(dv, u8p), _p(p, f64p),
                                    _p(pv, u8p), C.c_double(gamma), C.c_double(threshold),
                                    C.c_int(patch_size), _p(out, u8p))
        return out

    def disparity_to_depth(self, disp, disp_valid, focal, baseline, var=None, var_valid=None,
                           min_disparity=0.1):
        d = np.ascontiguousarray(disp, np.float64)
        dv = np.ascontiguousarray(disp_valid, np.uint8)
        h, w = d.shape
        depth = np.zeros_like(d)
        depth_ok = np.zeros_like(dv)
        sig = np.zeros_like(d)
        sig_ok = np.zeros_like(dv)
        vv = None if var is None else np.ascontiguousarray(var, np.float64)
        vok = None if var_valid is None else np.ascontiguousarray(var_valid, np.uint8)
        self.lib.bo_disparity_to_depth(C.c_int(w), C.c_int(h), _p(d, f64p), _p(dv, u8p),
                                       _p(vv, f64p), _p(vok, u8p), C.c_double(focal),
                                       C.c_double(baseline), C.c_double(min_disparity),
                                       _p(depth, f64p), _p(depth_ok, u8p), _p(sig, f64p),
                                       _p(sig_ok, u8p))
        return depth, depth_ok, sig, sig_ok

    # ---- whole path
    def validate(self, cfg: Config):
        c = cfg.to_c()
        msg = C.create_string_buffer(256)
        rc = self.lib.bo_validate(C.byref(c), msg, C.c_int(256))
        return rc, msg.value.decode()

    def match_stereo(self, left, right, cfg: Config, left_valid=None, right_valid=None,
                     finest_cap=1 << 20):
        left = np.ascontiguousarray(left, np.float32)
        h, w = left.shape
        li, ri = self.image(left, left_valid), self.image(right, right_valid)
        c = cfg.to_c()
        o = BoMatchOutputs()
        bufs = {k: np.zeros(h * w, np.float64) for k in ("disparity", "probability", "var_disp")}
        oks = {k: np.zeros(h * w, np.uint8) for k in ("disparity_valid", "probability_valid",
                                                      "var_valid")}
        stats = np.zeros(5 * 32, np.int32)
        finest = np.zeros(7 * finest_cap, np.float64)
        for k, v in bufs.items():
            setattr(o, k, _p(v, f64p))
        for k, v in oks.items():
            setattr(o, k, _p(v, u8p))
        o.stats = _p(stats, i32p)
        o.finest_cap = finest_cap
        o.finest = _p(finest, f64p)
        msg = C.create_string_buffer(256)
        rc = self.lib.bo_match_stereo(C.byref(li), C.byref(ri), C.byref(c), C.byref(o), msg,
                                      C.c_int(256))
        if rc:
            raise OracleError(rc, msg.value.decode())
        nl, nf = o.n_levels, o.finest_count
        res = {k: v.reshape(h, w) for k, v in bufs.items()}
        res.update({k: v.reshape(h, w) for k, v in oks.items()})
        res["has_variance"] = bool(o.has_variance)
        res["stats"] = stats[: 5 * nl].reshape(nl, 5).copy()
        res["finest"] = finest[: 7 * min(nf, finest_cap)].reshape(-1, 7).copy()
        return res

    def run_pipeline(self, left, right, cfg: Config, focal=1.0, baseline=1.0,
                     left_valid=None, right_valid=None):
        left = np.ascontiguousarray(left, np.float32)
        h, w = left.shape
        li, ri = self.image(left, left_valid), self.image(right, right_valid)
        c = cfg.to_c()
        o = BoOutputs()
        bufs = {k: np.zeros(h * w, np.float64) for k in ("disparity", "probability", "depth",
                                                         "depth_sigma")}
        oks = {k: np.zeros(h * w, np.uint8) for k in ("disparity_valid", "probability_valid",
                                                      "depth_valid", "sigma_valid")}
        stats = np.zeros(5 * 32, np.int32)
        for k, v in bufs.items():
            setattr(o, k, _p(v, f64p))
        for k, v in oks.items():
            setattr(o, k, _p(v, u8p))
        o.stats = _p(stats, i32p)
        msg = C.create_string_buffer(256)
        rc = self.lib.bo_run_pipeline(C.byref(li), C.byref(ri), C.byref(c), C.c_double(focal),
                                      C.c_double(baseline), C.byref(o), msg, C.c_int(256))
        if rc:
            raise OracleError(rc, msg.value.decode())
        res = {k: v.reshape(h, w) for k, v in bufs.items()}
        res.update({k: v.reshape(h, w) for k, v in oks.items()})
        res["has_sigma"] = bool(o.has_sigma)
        res["stats"] = stats[: 5 * o.n_levels].reshape(o.n_levels, 5).copy()
        res["runtime_ms"] = o.runtime_ms
        return res


_CACHE: dict[str, Oracle] = {}


def load(kind: str = "port") -> Oracle:
    if kind not in _CACHE:
        _CACHE[kind] = Oracle(kind)
    return _CACHE[kind]


def available(kind: str) -> bool:
    return LIBS[kind].exists()


# ---- BASELINE.json input generator, test side (oracle/libbdis_synth.so) ----
# The same plain-C generator the product ships (csrc/synth.c), compiled into a
# separate library so the reference arm of bench.py never loads the product.

class SynthSpec(C.Structure):
    _fields_ = [("width", C.c_int), ("height", C.c_int), ("channels", C.c_int),
                ("seed", C.c_uint64), ("octaves", C.c_int), ("base_wavelength", C.c_double),
                ("d_min", C.c_double), ("d_range", C.c_double), ("blur_sigma", C.c_double),
                ("noise_sigma", C.c_double), ("stress", C.c_int)]


_SYNTH = None


def _synth_lib():
    global _SYNTH
    if _SYNTH is None:
        path = HERE / "libbdis_synth.so"
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (make -C oracle)")
        L = C.CDLL(str(path))
        L.pstereo_synth_default.argtypes = [C.POINTER(SynthSpec), C.c_int]
        L.pstereo_synth_batch.argtypes = [C.POINTER(SynthSpec), C.c_int, C.c_uint64, u8p, u8p,
                                          C.c_int]
        _SYNTH = L
    return _SYNTH


def synth_batch(config: int, n: int, seed0: int = 0, threads: int = 8, **overrides):
    """Pairs seed0..seed0+n-1 of BASELINE.json configs[config]: (left, right)
    uint8 arrays [n, H, W(, C)], byte-identical to the product's generator."""
    L = _synth_lib()
    s = SynthSpec()
    L.pstereo_synth_default(C.byref(s), config)
    for k, v in overrides.items():
        setattr(s, k, v)
    shape = (n, s.height, s.width) if s.channels == 1 else (n, s.height, s.width, s.channels)
    left = np.zeros(shape, np.uint8)
    right = np.zeros(shape, np.uint8)
    rc = L.pstereo_synth_batch(C.byref(s), n, seed0, left.ctypes.data_as(u8p),
                               right.ctypes.data_as(u8p), threads)
    if rc:
        raise OracleError(rc, "synth_batch")
    return left, right
