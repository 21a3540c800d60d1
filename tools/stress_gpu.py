"""Randomised GPU stress of the public conceal path (not a unit test; a sweep
run on the B200 box): random transform sizes, block / support sizes, iteration
counts, gamma / rho, loss densities with neighbouring and border blocks.
Checks per case: GPU fp64 vs the C oracle (same selections -> pixels within
1e-9), GPU fp32 vs GPU fp64 (within 0.5 px), the frames batch path (f64
frames) vs the image path in fp32 (within fp32 noise).

usage: python tools/stress_gpu.py [cases] [seed]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle  # test infrastructure (the checker)
import paper_2207_01205_b200 as P

GEOMS = [(8, 4, 2), (16, 8, 4), (32, 8, 8), (32, 16, 8), (64, 16, 16), (64, 32, 16), (64, 8, 8), (128, 32, 16),
         (128, 64, 32), (48, 16, 16)]


def image(rng, h, w):
    y, x = np.mgrid[0:h, 0:w]
    f = 120 + 40 * np.cos(2 * np.pi * x / rng.uniform(20, 90) + rng.uniform(0, 6)) * np.cos(
        2 * np.pi * y / rng.uniform(20, 90)) + 20 * (x > rng.integers(0, w)) + rng.normal(0, 3, (h, w))
    return np.clip(np.round(f), 0, 255)


def main(cases=60, seed=1):
    rng = np.random.default_rng(seed)
    orc = oracle.Oracle()
    worst64 = worst32 = worstb = 0.0
    fails = []
    for c in range(cases):
        t, b, s = GEOMS[rng.integers(len(GEOMS))]
        size = int(rng.choice([t * 2, t * 3, 160, 256])) // b * b
        size = max(size, 2 * b)
        img = image(rng, size, size)
        cells = [(r, cc) for r in range(0, size, b) for cc in range(0, size, b)]
        frac = rng.uniform(0.03, 0.3)
        pick = [cells[i] for i in rng.choice(len(cells), max(1, int(frac * len(cells))), replace=False)]
        rects = [(r, cc, b, b) for r, cc in pick]
        # a window must keep some support: drop blocks whose whole window is lost
        pat = P.LossPattern(size, size, b, b, [P.Rect(*x) for x in rects])
        its = int(rng.choice([1, 7, 50, 150]))
        gamma = float(rng.choice([0.2, 0.5, 1.0]))
        rho = float(rng.choice([0.7, 0.8, 0.9]))
        algo = "ofse" if rng.random() < 0.2 else "fofse"
        kw = dict(algorithm=algo, gamma=gamma, iterations=its, transform_size=t, rho_hat=rho, support_width=s)
        try:
            o64 = P.conceal(img, pat, P.ConcealConfig(**kw))
            ref = orc.conceal(img, rects, b, b, algorithm=oracle.ALGO_OFSE if algo == "ofse" else oracle.ALGO_FOFSE,
                              gamma=gamma, iterations=its, t=t, rho_hat=rho, support=s)
            d64 = float(np.abs(o64.restored - ref["restored"]).max())
            o32 = P.conceal(img, pat, P.ConcealConfig(precision="fp32", **kw))
            d32 = float(np.abs(o32.restored - o64.restored).max())
            fr, _, _ = P.conceal_frames(img[None].astype(np.float64), [pat], P.ConcealConfig(precision="fp32", **kw))
            db = float(np.abs(fr[0] - o32.restored).max())
        except Exception as e:  # report, go on
            fails.append((c, t, b, s, size, its, repr(e)[:120]))
            continue
        worst64, worst32, worstb = max(worst64, d64), max(worst32, d32), max(worstb, db)
        bad = d64 > 1e-9 or d32 > 0.5 or db > 0.05
        print(f"case {c:3d} {algo:5s} T={t:3d} b={b:2d} S={s:2d} {size}x{size} blocks={len(rects):4d} I={its:3d} "
              f"g={gamma} rho={rho}: fp64-oracle {d64:.2e} fp32-fp64 {d32:.3f} batch-image {db:.2e}"
              f"{'  <-- FAIL' if bad else ''}", flush=True)
        if bad:
            fails.append((c, t, b, s, size, its, f"d64={d64} d32={d32} db={db}"))
    print(f"worst fp64-oracle {worst64:.2e}, fp32-fp64 {worst32:.3f}, batch-image {worstb:.2e}; failures: {len(fails)}")
    for f in fails:
        print("FAIL", f)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 60, int(sys.argv[2]) if len(sys.argv) > 2 else 1)
