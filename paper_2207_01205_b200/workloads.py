"""BASELINE.json configs C1-C5 as concrete seeded inputs.

Seeded synthetic images stand in for the reference's (absent) image fixtures;
losses are isolated blocks on a random parity sublattice.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _capi as capi
from .fse import ConcealConfig, LossPattern, Rect


@dataclass(frozen=True)
class Workload:
    name: str
    width: int
    height: int
    frames: int
    block: int
    support: int
    transform_size: int
    rho_hat: float
    gamma: float
    iterations: int
    loss_frac: float
    precision: str

    @property
    def window(self) -> int:
        return self.block + 2 * self.support

    def config(self, precision: str | None = None, **kw) -> ConcealConfig:
        return ConcealConfig(algorithm="fofse", gamma=self.gamma, iterations=self.iterations,
                             transform_size=self.transform_size, rho_hat=self.rho_hat,
                             support_width=self.support, precision=precision or self.precision,
                             **kw)

    def frame(self, seed: int, f: int = 0):
        """(image u8 (H, W), LossPattern) of frame f; frame f uses seed + f."""
        img = capi.gen_image_u8(seed + f, self.width, self.height)
        rects = capi.gen_losses(seed + f, self.width // self.block, self.height // self.block,
                                self.loss_frac, self.block, self.block)
        pat = LossPattern(self.width, self.height, self.block, self.block,
                          [Rect(int(r["row"]), int(r["col"]), int(r["height"]), int(r["width"]))
                           for r in rects])
        return img, pat

    def batch(self, seed: int, frames: int | None = None, first: int = 0, out: np.ndarray | None = None):
        """Frames first .. first+F-1 of the batch: (F, H, W) u8 (written into `out`
        when given), rects (structured), frame offsets (F+1,)."""
        nf = self.frames if frames is None else frames
        imgs = np.empty((nf, self.height, self.width), np.uint8) if out is None else out
        rects, offs = [], [0]
        for f in range(nf):
            imgs[f] = capi.gen_image_u8(seed + first + f, self.width, self.height)
            r = capi.gen_losses(seed + first + f, self.width // self.block, self.height // self.block,
                                self.loss_frac, self.block, self.block)
            rects.append(r)
            offs.append(offs[-1] + len(r))
        return imgs, np.concatenate(rects) if rects else np.zeros(0, capi.RECT_DTYPE), \
            np.asarray(offs, np.int64)


C1 = Workload("C1", 512, 512, 1, 16, 16, 64, 0.8, 0.5, 100, 0.10, "fp64")
C2 = Workload("C2", 1920, 1088, 1, 16, 16, 64, 0.8, 0.5, 200, 0.25, "fp32")
C3 = Workload("C3", 4096, 4096, 1, 8, 8, 32, 0.7, 0.5, 50, 0.20, "fp32")
C4 = Workload("C4", 1920, 1088, 256, 16, 16, 64, 0.8, 0.5, 200, 0.10, "fp32")
C5 = Workload("C5", 8192, 8192, 1, 32, 16, 128, 0.85, 0.5, 300, 0.05, "fp32")
ALL = {w.name: w for w in (C1, C2, C3, C4, C5)}
