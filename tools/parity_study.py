"""fp32 guard study (GPU box): for each (head, tau) the fp32 fast mode vs
the fp64 path over whole frames of a workload. Prints, per setting, the re-run
fraction, max |pixel error|, blocks above 0.5 px and |dPSNR| over all frames.

usage: python tools/parity_study.py WORKLOAD FRAMES SEED head:tau [...]  (head/tau -1 = default)
"""
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2207_01205_b200 as P  # noqa: E402
from paper_2207_01205_b200 import workloads as WL  # noqa: E402
from paper_2207_01205_b200.parity import _block_max  # noqa: E402


def main(wname, frames, seed, settings):
    wl = WL.ALL[wname]
    combos = []
    for s in settings:
        h, t = s.split(":")
        combos.append((int(h), float(t)))
    st = {c: dict(reruns=0, maxpx=0.0, bad=0, sq=0.0, worst=None) for c in combos}
    sq64 = 0.0
    npx = nblocks = 0
    t0 = time.time()
    for f in range(frames):
        img, pat = wl.frame(seed, f)
        img = img.astype(np.float64)
        o64 = P.conceal(img, pat, wl.config("fp64"))
        e = o64.restored - img
        sq64 += float((e * e).sum())
        npx += len(pat.blocks) * wl.block * wl.block
        nblocks += len(pat.blocks)
        for c in combos:
            cfg = wl.config("fp32")
            cfg.fp64_head, cfg.guard_tau = c
            o32 = P.conceal(img, pat, cfg)
            bm = _block_max(np.abs(o32.restored - o64.restored), pat.blocks, wl.block, wl.block)
            s = st[c]
            s["reruns"] += int(o32.report.device["guard_reruns"])
            s["bad"] += int((bm > 0.5).sum())
            if bm.size and bm.max() > s["maxpx"]:
                s["maxpx"] = float(bm.max())
                s["worst"] = (f, int(bm.argmax()))
            e = o32.restored - img
            s["sq"] += float((e * e).sum())

    def db(sq):
        return 10 * math.log10(255.0 ** 2 / (sq / npx)) if sq > 0 else math.inf

    for c in combos:
        s = st[c]
        print(f"{wname} seed={seed} frames={frames} head={c[0]} tau={c[1]:g}: blocks={nblocks} "
              f"reruns={s['reruns']} ({100 * s['reruns'] / nblocks:.2f}%) max_px={s['maxpx']:.4f} "
              f"blocks>0.5px={s['bad']} |dPSNR|={abs(db(s['sq']) - db(sq64)):.2e} dB worst={s['worst']}",
              flush=True)
    print(f"done {time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4:])
