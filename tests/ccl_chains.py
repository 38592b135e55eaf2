"""Test helper: the tile structure of the finest-level keep mask that the
GPU's component labelling sees (csrc/bdis_kernels.cu: 32x64 finest tiles,
k_fuse_ccl_local / k_ccl_border / k_ccl_merge). A tile-local component is
"sure" when its own area (full-resolution pixels, 4 per finest pixel at even
sizes) already meets the area rule of remove_small_components
(src/depth_variance.cpp:87-90); k_ccl_border skips unions between two sure
pieces. A "chain" is a global component holding at least two sure pieces and
at least one piece that is not sure -- the case where that shortcut must not
change which pixels survive."""
import math

import numpy as np

TILE_W, TILE_H = 32, 64


def min_area(gamma, size):
    return max(int(math.floor(math.ceil(gamma * size * size - 1e-9) + 0.5)), 1)


def chain_count(probability, valid, threshold, gamma, size):
    from scipy import ndimage

    keep = (valid != 0) & ~(probability < threshold)
    k = keep[::2, ::2]
    h, w = k.shape
    need = min_area(gamma, size)
    loc = np.zeros(k.shape, np.int64)
    sure = {}
    nid = 0
    for ty in range(0, h, TILE_H):
        for tx in range(0, w, TILE_W):
            lab, n = ndimage.label(k[ty:ty + TILE_H, tx:tx + TILE_W])
            for c in range(1, n + 1):
                m = lab == c
                nid += 1
                loc[ty:ty + TILE_H, tx:tx + TILE_W][m] = nid
                sure[nid] = 4 * int(m.sum()) >= need
    glab, gn = ndimage.label(k)
    chains = 0
    for g in range(1, gn + 1):
        ids = np.unique(loc[glab == g])
        n_sure = sum(sure[i] for i in ids)
        if n_sure >= 2 and len(ids) - n_sure >= 1:
            chains += 1
    return chains


# stress-generator pairs at 640x480 with a high threshold and a large area
# rule: the kept mask breaks into pieces that cross tile borders
CASES = [(0.7, 3.0, 0), (0.7, 3.0, 2), (0.6, 2.0, 0), (0.4, 4.0, 0)]
