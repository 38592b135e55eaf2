"""Adversarial parity of the residual evaluation (src/lk_solver.cpp:38-81):
the GPU evaluates x_i = (x0 + i) - u with a per-binade constant-fraction fast
path (see bdis_patches.cu). These queries put disparities exactly on and
around binade boundaries, image borders and integer positions, where that
argument is most delicate, and require bit-identical (msq, jr, n) against the
CPU oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _queries(w, h, s, rng):
    xs0 = sorted({0, 1, 2, 3, 5, 7, 13, 15, 16, 17, 24, 31, 32, 33, 57, 63, 64, 65, w - s - 1,
                  w - s})
    xs0 = [x for x in xs0 if 0 <= x <= w - s]
    qx, qy, qu = [], [], []
    tiny = [0.0, 1e-300, 5e-324, 1e-16, -1e-16, 2.0 ** -40, -(2.0 ** -40), 2.0 ** -52,
            -(2.0 ** -52), 0.25, -0.25, 0.5, -0.5, 1e-9, -1e-9]
    for x0 in xs0:
        y0 = int(rng.integers(0, h - s + 1))
        for i in range(s):
            for B in [2.0 ** k for k in range(-2, 8)]:
                for d in tiny:
                    u = (x0 + i) - B + d
                    qx.append(x0)
                    qy.append(y0)
                    qu.append(u)
                    # the neighbouring representable values of u
                    for nu in (np.nextafter(u, np.inf), np.nextafter(u, -np.inf)):
                        qx.append(x0)
                        qy.append(y0)
                        qu.append(float(nu))
        # borders: first / last sample exactly at 0 and w-1, and just beyond
        for base in (float(x0), float(x0 + s - 1) - (w - 1)):
            for d in tiny + [1.0, -1.0, 3.5, -3.5]:
                qx.append(x0)
                qy.append(y0)
                qu.append(base + d)
        for u in rng.uniform(-w, w, 40).tolist() + [1e12, -1e12, 2.0 ** 40 + 0.5]:
            qx.append(x0)
            qy.append(y0)
            qu.append(u)
    return np.array(qx), np.array(qy), np.array(qu)


@pytest.mark.parametrize("s", [2, 5, 8, 12, 16, 32])
@pytest.mark.parametrize("masked", [False, True])
def test_eval_residual_adversarial(gpu, port, s, masked):
    P = gpu
    rng = np.random.default_rng(s + 100 * masked)
    w, h = 100, s + 3
    left = rng.random((h, w)).astype(np.float32)
    right = rng.random((h, w)).astype(np.float32)
    lv = rv = None
    if masked:
        lv = (rng.random((h, w)) > 0.05).astype(np.uint8)
        rv = (rng.random((h, w)) > 0.05).astype(np.uint8)
    qx, qy, qu = _queries(w, h, s, rng)
    msq, jr, n = P.debug_eval_residual(left, right, s, qx, qy, qu, lv, rv)
    grad = port.gradient_x(left)
    half = (s - 1) * 0.5
    bad = []
    li = port.image(left, lv)
    ri = port.image(right, rv)
    import ctypes as C

    from oracle.pyoracle import _p, f32p

    m_, j_, n_ = C.c_double(), C.c_double(), C.c_int()
    for q in range(len(qu)):
        ok = port.lib.bo_eval_residual(C.byref(li), _p(grad, f32p), C.byref(ri),
                                       C.c_double(qx[q] + half), C.c_double(qy[q] + half),
                                       C.c_int(s), C.c_double(qu[q]), C.byref(m_), C.byref(j_),
                                       C.byref(n_))
        if not ok:
            continue  # template without valid pixels: never evaluated on the path
        same = (n_.value == n[q] and
                np.float64(m_.value).view(np.uint64) == np.float64(msq[q]).view(np.uint64) and
                np.float64(j_.value).view(np.uint64) == np.float64(jr[q]).view(np.uint64))
        if not same:
            bad.append((int(qx[q]), float(qu[q]), n_.value, int(n[q]), m_.value, msq[q]))
    assert not bad, f"{len(bad)}/{len(qu)} queries differ, e.g. {bad[:3]}"
