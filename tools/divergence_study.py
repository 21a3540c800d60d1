"""Where does the fp32 fast mode leave the fp64 selection sequence? (GPU box)

For whole frames of a workload: GPU fp64 (the oracle-pinned path) vs GPU fp32
with the near-tie guard OFF and an fp64 head of H selections. Per block it
records the first divergent selection n_d and, for candidate guard rules, the
smallest normalised top-2 gap over the whole run and over n <= n_d:

  g_n  = (|R1|^2 - |R2|^2) / |R1|^2            relative gap (guard_tau's rule)
  D_n  = g_n |R1| / M0,  M0 = |R1| at n = H    gap in |R| units of M0 (x2)
  D_n / f(n) for f = sqrt(n-H+1), n-H+1, A_n = 1 + gamma sum_{H<=i<n} |R1_i| / M0

A rule "flag when x_n < thr" catches a divergent block iff min_{n<=n_d} x_n < thr
and re-runs a block iff min_n x_n < thr; the per-block minima are all an
offline threshold sweep needs (tools/divergence_analyse.py).

usage: python tools/divergence_study.py WORKLOAD FRAMES SEED HEAD OUT.npz
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from guard_study import diag  # noqa: E402
from paper_2207_01205_b200 import workloads as WL  # noqa: E402
from paper_2207_01205_b200.parity import _block_max  # noqa: E402

RULES = ["g", "D", "D/sqrt", "D/lin", "D/A"]


def main(wname, frames, seed, head, out):
    wl = WL.ALL[wname]
    t0 = time.time()
    rows = []
    for f in range(frames):
        img, pat = wl.frame(seed, f)
        img = img.astype(np.float64)
        r64, t64, c64, _ = diag(img, pat, wl.config("fp64"))
        r32, t32, c32, g32 = diag(img, pat, wl.config("fp32", guard_tau=0.0, fp64_head=head))
        n, it = t64.shape
        px = _block_max(np.abs(r32 - r64), pat.blocks, wl.block, wl.block)
        u64 = t64["u1"].astype(np.int64) * 4096 + t64["u2"]
        u32 = t32["u1"].astype(np.int64) * 4096 + t32["u2"]
        mag = np.hypot(t32["p_re"], t32["p_im"])  # |R1_n| / w0
        for i in range(n):
            m = min(c64[i], c32[i])
            d = np.nonzero(u64[i, :m] != u32[i, :m])[0]
            nd = int(d[0]) if d.size else -1
            e = int(c32[i])
            if e <= head:
                rows.append([f, i, nd, px[i], e] + [np.inf] * (2 * len(RULES)))
                continue
            k = np.arange(head, e)
            g = g32[i, head:e].astype(np.float64)
            r1 = mag[i, head:e]
            m0 = r1[0] if r1[0] > 0 else 1.0
            D = g * r1 / m0
            j = (k - head + 1).astype(np.float64)
            A = 1.0 + wl.gamma * np.concatenate([[0.0], np.cumsum(r1[:-1])]) / m0
            xs = [g, D, D / np.sqrt(j), D / j, D / A]
            mins = [float(x.min()) for x in xs]
            if nd >= head:
                lim = nd - head + 1
                mins_d = [float(x[:lim].min()) for x in xs]
            else:
                mins_d = [np.inf] * len(xs)
            rows.append([f, i, nd, px[i], e] + mins + mins_d)
        print(f"frame {f}: {n} blocks, divergent {(np.array([r[2] for r in rows[-n:]]) >= 0).sum()}, "
              f"{time.time() - t0:.1f}s", flush=True)
    a = np.array(rows, np.float64)
    np.savez_compressed(out, data=a, rules=np.array(RULES), head=head, workload=wname, seed=seed,
                        iterations=wl.iterations)
    print(f"saved {out}: {a.shape}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5])
