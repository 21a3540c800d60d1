"""Seeded test inputs, in the spirit of the reference's testutil:: helpers
(proj/tests/helpers.hpp:82-130) and pipeline_test's smooth image (:16-25)."""
import numpy as np

SUPPORT, MISSING, OUTSIDE = 0, 1, 2


def random_grid(rng, h, w, lo=-1.0, hi=1.0):
    return rng.uniform(lo, hi, (h, w))


def random_mask(rng, h, w, missing_prob=0.4, min_support=0.25):
    while True:
        m = np.where(rng.uniform(0, 1, (h, w)) < missing_prob, MISSING, SUPPORT).astype(np.uint8)
        s = int((m == SUPPORT).sum())
        if s > 0 and s >= min_support * h * w:
            return m


def smooth_test_image(rng, size):
    r = np.arange(size)[:, None]
    c = np.arange(size)[None, :]
    v = 128.0 + 90.0 * np.sin(0.09 * r) * np.cos(0.07 * c) + rng.uniform(-6, 6, (size, size))
    return np.clip(np.round(v), 0, 255)


def block_mask(h, w, missing=(), outside=()):
    m = np.zeros((h, w), np.uint8)
    for (r, c, hh, ww) in missing:
        m[r:r + hh, c:c + ww] = MISSING
    for (r, c, hh, ww) in outside:
        m[r:r + hh, c:c + ww] = OUTSIDE
    return m


def rects(pattern_blocks):
    return [tuple(int(x) for x in b) for b in pattern_blocks]
