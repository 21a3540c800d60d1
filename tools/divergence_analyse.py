"""Offline threshold sweep over tools/divergence_study.py outputs.

For each rule and threshold: the fraction of blocks re-run, the divergent blocks
the rule misses (no flag at or before the first divergence) and how many of the
missed ones end above 0.5 px.

usage: python tools/divergence_analyse.py a.npz [b.npz ...]
"""
import sys

import numpy as np


def analyse(path, extra_tau=1e-5):
    z = np.load(path)
    a = z["data"]
    rules = list(z["rules"])
    nr = len(rules)
    n = len(a)
    nd = a[:, 2]
    px = a[:, 3]
    mins = a[:, 5:5 + nr]
    mins_d = a[:, 5 + nr:5 + 2 * nr]
    div = nd >= 0
    print(f"== {path}: {z['workload']} head={int(z['head'])} blocks={n} divergent={int(div.sum())} "
          f"(in head: {int((div & np.isinf(mins_d[:, 0])).sum())}) over0.5={int((px > 0.5).sum())} max_px={px.max():.3f}")
    gi = rules.index("g")
    base_flag = mins[:, gi] < extra_tau
    base_safe = mins_d[:, gi] < extra_tau
    print(f"   tau={extra_tau:g} alone: rerun {base_flag.mean() * 100:.2f}%  missed {int((div & ~base_safe).sum())} "
          f"(>0.5px {int((div & ~base_safe & (px > 0.5)).sum())})")
    for k, r in enumerate(rules):
        if r == "g":
            continue
        finite = mins[:, k][np.isfinite(mins[:, k])]
        for q in (1e-7, 3e-7, 1e-6, 3e-6, 1e-5, 3e-5, 1e-4):
            thr = q
            flag = base_flag | (mins[:, k] < thr)
            safe = base_safe | (mins_d[:, k] < thr)
            miss = div & ~safe
            print(f"   tau + {r:7s} < {thr:7.1e}: rerun {flag.mean() * 100:6.2f}%  missed {int(miss.sum()):5d} "
                  f"(>0.5px {int((miss & (px > 0.5)).sum())}, max px of missed {px[miss].max() if miss.any() else 0:.3f})")
        del finite


if __name__ == "__main__":
    for p in sys.argv[1:]:
        analyse(p)
