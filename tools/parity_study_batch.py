"""fp32 guard study through the batch path (what bench.py times and its parity
block checks): for each head:tau, fp32 vs fp64 over a workload's frames.

usage: python tools/parity_study_batch.py WORKLOAD FRAMES SEED head:tau [...]
"""
import dataclasses
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2207_01205_b200 import parity as PAR  # noqa: E402
from paper_2207_01205_b200 import workloads as WL  # noqa: E402


def main(wname, frames, seed, settings):
    wl = dataclasses.replace(WL.ALL[wname], frames=frames)
    for st in settings:
        h, t = st.split(":")
        cfg = wl.config("fp32")
        cfg.fp64_head, cfg.guard_tau = int(h), float(t)
        r = PAR.fp32_vs_fp64(wl, seed, cfg32=cfg, per_call=64)
        print(f"{wname} seed={seed} frames={frames} head={h} tau={t}: blocks={r['blocks']} reruns={r['guard_reruns']} "
              f"({100 * r['rerun_frac']:.2f}%) max_px={r['max_px']:.4f} blocks>0.5px={r['blocks_over_0.5']} "
              f"|dPSNR|={r['dpsnr_db']:.2e} dB worst={r['worst']}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4:])
