"""Per-selection latency of the fp64 / fp32 iteration kernels for a single lost
block (one CTA): the time difference between two iteration counts."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2207_01205_b200 as P  # noqa: E402
from helpers import smooth_test_image  # noqa: E402


def run(prec, iters, t=64, reps=20):
    img = smooth_test_image(np.random.default_rng(5), 96)
    pat = P.LossPattern(96, 96, 16, 16, [P.Rect(40, 40, 16, 16)])
    cfg = P.ConcealConfig(gamma=0.5, iterations=iters, precision=prec, transform_size=t)
    P.conceal(img, pat, cfg)
    best = 1e9
    for _ in range(reps):
        out = P.conceal(img, pat, cfg)
        best = min(best, out.report.device["total_ms"])
    return best


if __name__ == "__main__":
    for prec in ("fp64", "fp32"):
        a, b = run(prec, 100), run(prec, 1100)
        print(f"{prec}: {1e3 * (b - a) / 1000:.2f} us per selection (I=100: {a:.3f} ms, I=1100: {b:.3f} ms)")
