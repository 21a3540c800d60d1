"""Small concealment cases for compute-sanitizer (racecheck / synccheck /
memcheck): every production kernel family on a C2 slice — K1f + K2d head +
K2v2r or K2v2h (FOFSE_V2_REAL_GW) + K2v2c borders + guard re-runs (fp32), K2d
/ K2dc with the near-tie guard (fp64), K1x + strict kernel (exact path), and
T = 128 (K1w, K2v2h<128>, K2d<128>)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2207_01205_b200 as P  # noqa: E402
from paper_2207_01205_b200 import workloads as WL  # noqa: E402


def main():
    img, pat = WL.C2.frame(seed=5)
    sub = P.LossPattern(pat.image_width, pat.image_height, 16, 16, pat.blocks[::24])  # ~85 blocks, borders too
    img = img.astype(np.float64)
    for prec in ("fp32", "fp64"):
        cfg = WL.C2.config(prec)
        cfg.iterations = 40
        out = P.conceal(img, sub, cfg)
        print(prec, len(sub.blocks), out.report.psnr_db, out.report.device["guard_reruns"], flush=True)
    cfg = WL.C2.config("fp64", guard_tau=1.0)  # every block on the exact path
    cfg.iterations = 20
    out = P.conceal(img, P.LossPattern(sub.image_width, sub.image_height, 16, 16, sub.blocks[:6]), cfg)
    print("exact", out.report.device["guard_reruns"], flush=True)
    img5, pat5 = WL.C5.frame(seed=9)
    sub5 = P.LossPattern(pat5.image_width, pat5.image_height, 32, 32, pat5.blocks[::200])
    for prec in ("fp32", "fp64"):
        cfg = WL.C5.config(prec)
        cfg.iterations = 30
        out = P.conceal(img5.astype(np.float64), sub5, cfg)
        print("C5", prec, len(sub5.blocks), out.report.psnr_db, flush=True)


if __name__ == "__main__":
    main()
