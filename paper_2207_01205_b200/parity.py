"""fp32 fast mode vs the fp64 path on whole workloads (north_star fp32 bar:
max |pixel error| <= 0.5 and PSNR of the concealed blocks within 0.05 dB).

Both arms run on the GPU through the batch path the bench times
(``fse.conceal_frames`` on fp64 frames = fofse_conceal_frames_f64: the same
plan, chunk pipeline, kernels — K2v2r / K2v2h / K2v2t, guard, exact near-tie
resolution — and parameters as the u8 frames API, with the unrounded pixels
out), ``per_call`` frames at a time. The fp64 arm is the path pinned to the
oracle by the GPU parity tests, so a block within 0.5 px of it is within
0.5 px of the reference up to the fp64 path's own 1e-9.
"""
from __future__ import annotations

import math

import numpy as np

from . import fse


def _block_max(d: np.ndarray, rects, bh: int, bw: int) -> np.ndarray:
    h, w = d.shape
    if h % bh == 0 and w % bw == 0 and all(r.row % bh == 0 and r.col % bw == 0 for r in rects):
        g = d.reshape(h // bh, bh, w // bw, bw).max(axis=(1, 3))
        return np.array([g[r.row // bh, r.col // bw] for r in rects], np.float64)
    return np.array([d[r.row:r.row + bh, r.col:r.col + bw].max() for r in rects], np.float64)


def fp32_vs_fp64(wl, seed: int, frames: int | None = None, cfg32=None, device: int = 0,
                 per_call: int = 32) -> dict:
    """Run every frame of workload `wl` (frame f from seed + f) in fp32 (``cfg32``,
    default: the workload's fp32 config with the library's default head / guard)
    and in fp64, ``per_call`` frames per batch call; compare pixel by pixel over
    all lost blocks."""
    nf = wl.frames if frames is None else frames
    cfg64 = wl.config("fp64")
    cfg32 = cfg32 or wl.config("fp32")
    bh = bw = wl.block
    blocks = over = reruns = 0
    max_px = 0.0
    sq32 = sq64 = 0.0
    npx = 0
    dpsnr_frame = 0.0
    worst = None

    def db(sq, n):
        return math.inf if sq == 0.0 else 10.0 * math.log10(255.0 * 255.0 / (sq / max(n, 1)))

    for f0 in range(0, nf, max(1, per_call)):
        nb = min(nf - f0, max(1, per_call))
        imgs, rects, offs = wl.batch(seed, frames=nb, first=f0)
        imgs = imgs.astype(np.float64)
        pats = []
        for f in range(nb):
            rr = rects[offs[f]:offs[f + 1]]
            pats.append(fse.LossPattern(wl.width, wl.height, bh, bw,
                                        [fse.Rect(int(r["row"]), int(r["col"]), bh, bw) for r in rr]))
        o64, s64, _ = fse.conceal_frames(imgs, pats, cfg64, device)
        o32, s32, rep32 = fse.conceal_frames(imgs, pats, cfg32, device)
        reruns += int(rep32.device["guard_reruns"])
        for f in range(nb):
            pat = pats[f]
            d = np.abs(o32[f] - o64[f])
            bm = _block_max(d, pat.blocks, bh, bw)
            blocks += len(bm)
            over += int((bm > 0.5).sum())
            if len(bm) and bm.max() > max_px:
                max_px = float(bm.max())
                worst = {"frame": f0 + f, "block": int(bm.argmax())}
            e32 = float(s32[offs[f]:offs[f + 1]].sum())  # per-block squared errors vs the input
            e64 = float(s64[offs[f]:offs[f + 1]].sum())
            sq32 += e32
            sq64 += e64
            n = len(pat.blocks) * bh * bw
            npx += n
            if e32 > 0.0 and e64 > 0.0:
                dpsnr_frame = max(dpsnr_frame, abs(db(e32, n) - db(e64, n)))

    return {"frames": nf, "blocks": blocks, "max_px": max_px, "blocks_over_0.5": over,
            "dpsnr_db": abs(db(sq32, npx) - db(sq64, npx)), "max_frame_dpsnr_db": dpsnr_frame,
            "guard_reruns": reruns, "rerun_frac": reruns / max(blocks, 1), "worst": worst,
            "psnr_fp32_db": db(sq32, npx), "psnr_fp64_db": db(sq64, npx), "per_call": per_call}
