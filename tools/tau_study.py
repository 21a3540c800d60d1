"""Guard threshold study (GPU box): fp32 fast mode with near-tie guard tau vs
the fp64 path on whole C4 frames. Reports, per tau, the re-run fraction, the
max |pixel error| over all lost pixels, the number of blocks above 0.5 and the
worst per-frame PSNR difference (the fp32 bar: <= 0.5 px, <= 0.05 dB)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2207_01205_b200 as P  # noqa: E402
from paper_2207_01205_b200 import workloads as WL  # noqa: E402


def main(frames=64, seed=9100, taus=(1e-5, 5e-6, 3e-6, 2e-6), head=-1):
    wl = WL.C4
    stats = {t: dict(reruns=0, maxerr=0.0, bad=0, dpsnr=0.0) for t in taus}
    nblocks = 0
    t0 = time.time()
    for f in range(frames):
        img, pat = wl.frame(seed, f)
        img = img.astype(np.float64)
        o64 = P.conceal(img, pat, wl.config("fp64"))
        lost = np.zeros(img.shape, bool)
        for b in pat.blocks:
            lost[b.row:b.row + 16, b.col:b.col + 16] = True
        nblocks += len(pat.blocks)
        for t in taus:
            cfg = wl.config("fp32")
            cfg.guard_tau = t
            cfg.fp64_head = head
            o32 = P.conceal(img, pat, cfg)
            d = np.abs(o32.restored - o64.restored)
            s = stats[t]
            s["reruns"] += int(o32.report.device["guard_reruns"])
            s["maxerr"] = max(s["maxerr"], float(d[lost].max()))
            for b in pat.blocks:
                if d[b.row:b.row + 16, b.col:b.col + 16].max() > 0.5:
                    s["bad"] += 1
            s["dpsnr"] = max(s["dpsnr"], abs(o32.report.psnr_db - o64.report.psnr_db))
    for t in taus:
        s = stats[t]
        print(f"head={head} tau={t:g}: blocks={nblocks} reruns={s['reruns']} ({100 * s['reruns'] / nblocks:.2f}%) "
              f"maxerr={s['maxerr']:.4f} blocks>0.5px={s['bad']} max|dPSNR|={s['dpsnr']:.5f} dB", flush=True)
    print(f"done {time.time() - t0:.1f}s")


if __name__ == "__main__":
    frames = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    head = int(sys.argv[2]) if len(sys.argv) > 2 else -1
    taus = tuple(float(x) for x in sys.argv[3].split(",")) if len(sys.argv) > 3 else (1e-5, 5e-6, 3e-6, 2e-6)
    main(frames, head=head, taus=taus)
