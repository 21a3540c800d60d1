"""Same-box output comparison of two library builds (FOFSE_LIB_PATH): conceal a
workload batch in fp32 with each and compare restored frames / block errors.

usage: python tools/lib_ab_outputs.py WORKLOAD FRAMES LIB_A LIB_B
"""
import os
import subprocess
import sys

import numpy as np

CHILD = r'''
import sys, numpy as np
sys.path.insert(0, ".")
import paper_2207_01205_b200 as P
from paper_2207_01205_b200 import workloads as WL
wl = WL.ALL[sys.argv[1]]
frames, rects, offs = wl.batch(seed=2207, frames=int(sys.argv[2]))
pats = []
for f in range(len(frames)):
    rr = rects[offs[f]:offs[f + 1]]
    pats.append(P.LossPattern(wl.width, wl.height, wl.block, wl.block,
                              [P.Rect(*map(int, (r["row"], r["col"], wl.block, wl.block))) for r in rr]))
out, sq, rep = P.conceal_frames(frames, pats, wl.config("fp32"))
np.savez(sys.argv[3], out=out, sq=sq, reruns=rep.device["guard_reruns"])
'''


def main(w, n, la, lb):
    res = []
    for i, lib in enumerate((la, lb)):
        path = f"gpurun_out/lib_ab_{i}.npz"
        subprocess.run([sys.executable, "-c", CHILD, w, n, path], check=True,
                       env={**os.environ, "FOFSE_LIB_PATH": lib})
        res.append(np.load(path))
    a, b = res
    d = np.abs(a["out"].astype(int) - b["out"].astype(int))
    print(f"{w} frames={n}: restored bytes differing {int((d > 0).sum())} (max {int(d.max())}); "
          f"block sq max rel diff {float(np.max(np.abs(a['sq'] - b['sq']) / np.maximum(np.abs(a['sq']), 1e-300))):.3g}; "
          f"reruns {int(a['reruns'])} vs {int(b['reruns'])}")


if __name__ == "__main__":
    main(*sys.argv[1:5])
