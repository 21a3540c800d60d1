"""fp32 fast mode vs the fp64 path on whole workloads (north_star fp32 bar:
max |pixel error| <= 0.5 and PSNR of the concealed blocks within 0.05 dB).

Both arms run on the GPU through ``fse.conceal`` (fofse_conceal_f64: the same
kernels and parameters as the frames API, with unrounded f64 pixels out).
The fp64 arm is the path pinned to the oracle by the GPU parity tests, so a
block within 0.5 px of it is within 0.5 px of the reference up to the fp64
path's own 1e-9.
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


def fp32_vs_fp64(wl, seed: int, frames: int | None = None, cfg32=None, device: int = 0) -> dict:
    """Run every frame of workload `wl` (frame f from seed + f) in fp32 (``cfg32``,
    default: the workload's fp32 config with the library's default head / guard)
    and in fp64; compare pixel by pixel over all lost blocks."""
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
    for f in range(nf):
        img, pat = wl.frame(seed, f)
        img = img.astype(np.float64)
        o64 = fse.conceal(img, pat, cfg64, device)
        o32 = fse.conceal(img, pat, cfg32, device)
        d = np.abs(o32.restored - o64.restored)
        bm = _block_max(d, pat.blocks, bh, bw)
        blocks += len(bm)
        over += int((bm > 0.5).sum())
        if len(bm) and bm.max() > max_px:
            max_px = float(bm.max())
            worst = {"frame": f, "block": int(bm.argmax())}
        reruns += int(o32.report.device["guard_reruns"])
        e32 = o32.restored - img
        e64 = o64.restored - img
        sq32 += float((e32 * e32).sum())  # restored == image outside the lost blocks
        sq64 += float((e64 * e64).sum())
        npx += len(pat.blocks) * bh * bw
        if not (o32.report.psnr_identical or o64.report.psnr_identical):
            dpsnr_frame = max(dpsnr_frame, abs(o32.report.psnr_db - o64.report.psnr_db))

    def db(sq):
        return math.inf if sq == 0.0 else 10.0 * math.log10(255.0 * 255.0 / (sq / max(npx, 1)))

    return {"frames": nf, "blocks": blocks, "max_px": max_px, "blocks_over_0.5": over,
            "dpsnr_db": abs(db(sq32) - db(sq64)), "max_frame_dpsnr_db": dpsnr_frame,
            "guard_reruns": reruns, "rerun_frac": reruns / max(blocks, 1), "worst": worst,
            "psnr_fp32_db": db(sq32), "psnr_fp64_db": db(sq64)}
