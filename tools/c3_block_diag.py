"""Diagnose one block's fp32-vs-fp64 difference in a workload frame: traces of both
precisions through the image path, first divergent selection, top-2 gap there.

usage: python tools/c3_block_diag.py WORKLOAD SEED FRAME BLOCK
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2207_01205_b200 as P  # noqa: E402
from paper_2207_01205_b200 import workloads as WL  # noqa: E402


def main(wname, seed, frame, blk):
    wl = WL.ALL[wname]
    imgs, rects, offs = wl.batch(seed, frames=1, first=frame)
    rr = rects[offs[0]:offs[1]]
    pat = P.LossPattern(wl.width, wl.height, wl.block, wl.block,
                        [P.Rect(int(r["row"]), int(r["col"]), wl.block, wl.block) for r in rr])
    img = imgs[0].astype(np.float64)
    out = {}
    for prec in ("fp64", "fp32"):
        cfg = wl.config(prec)
        cfg.record_traces = True
        o = P.conceal(img, pat, cfg)
        out[prec] = o
    b = pat.blocks[blk]
    r0, c0 = b.row, b.col
    d = np.abs(out["fp32"].restored[r0:r0 + wl.block, c0:c0 + wl.block] -
               out["fp64"].restored[r0:r0 + wl.block, c0:c0 + wl.block])
    print(f"block {blk} at ({r0},{c0}): max |dpx| {d.max():.4f}; fp32 reruns {out['fp32'].report.device.get('guard_reruns')}")
    t64, t32 = out["fp64"].report.traces[blk], out["fp32"].report.traces[blk]
    u64 = list(zip(t64["u1"], t64["u2"]))
    u32 = list(zip(t32["u1"], t32["u2"]))
    print("selections", len(u64), len(u32))
    first = next((i for i, (a, c) in enumerate(zip(u64, u32)) if a != c), None)
    print("first divergence", first)
    if first is not None:
        for i in range(max(0, first - 2), min(len(u64), first + 3)):
            print(i, "fp64", u64[i], "fp32", u32[i] if i < len(u32) else None)
    print("fp64 reruns (exact)", out["fp64"].report.device.get("guard_reruns"))
    print("fp64 trace keys", list(t64.keys()))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]))
