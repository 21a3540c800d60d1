"""B200-native FOFSE block concealment (arXiv 2207.01205), drop-in for the
reference `fse` library's concealment hot path.

Product = paper_2207_01205_b200/_lib/libfofse.so (sm_100a CUDA kernels behind
the C ABI in include/fofse.h); this package is a thin reference-shaped
Python mirror over it (see fse.py).
"""
from . import _capi
from ._capi import (FofseCudaError, FofseError, Context, context, gen_image_u8, gen_losses,
                    LIB_PATH)
from .fse import (ConcealConfig, ConcealmentReport, ConcealOutput, CurveSeries, LossPattern, Rect, Region,
                  WindowRun, build_isotropic_weight, conceal, conceal_frames, conceal_shard, extrapolate_window,
                  extrapolate_windows, parse_algorithm, psnr, psnr_vs_iterations, series_label, spectral)

__all__ = [
    "ConcealConfig", "ConcealmentReport", "ConcealOutput", "CurveSeries", "LossPattern", "Rect", "Region",
    "WindowRun", "build_isotropic_weight", "conceal", "conceal_frames", "conceal_shard", "extrapolate_window",
    "extrapolate_windows", "parse_algorithm", "psnr", "psnr_vs_iterations", "series_label", "spectral",
    "FofseCudaError", "FofseError", "Context", "context", "gen_image_u8", "gen_losses", "LIB_PATH",
]
