"""Reference-shaped Python API over the B200 library (drop-in for the hot path).

Mirrors the reference C++ interface of /root/reference/proj:
  * ``conceal(image, pattern, config)``          <- fse::conceal (pipeline.hpp:83-84)
  * ``extrapolate_window(window, mask, config)`` <- fse::extrapolate_window (pipeline.hpp:74-77)
  * ``spectral.init_spectra / fast_iterate / synthesize_model``
                                                <- engine_spectral.hpp:38-51
  * ``ConcealConfig``, ``LossPattern``, ``Rect``, ``Region`` <- pipeline.hpp:19-33,
    pattern.hpp:11-17, grid.hpp:26-38
Exceptions follow the reference: ValueError for std::invalid_argument,
RuntimeError for std::runtime_error. Everything computes on the GPU through
the C ABI; nothing here falls back to the CPU.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from enum import IntEnum

import numpy as np

from . import _capi as capi


class Region(IntEnum):
    support = 0
    missing = 1
    outside = 2


@dataclass(frozen=True)
class Rect:
    row: int
    col: int
    height: int
    width: int

    def __iter__(self):
        return iter((self.row, self.col, self.height, self.width))


@dataclass
class LossPattern:
    image_width: int = 0
    image_height: int = 0
    block_height: int = 0
    block_width: int = 0
    blocks: list = field(default_factory=list)


_ALGOS = {"fse": capi.ALGO_FSE, "ofse": capi.ALGO_OFSE, "fofse": capi.ALGO_FOFSE}
_PRECS = {"fp64": capi.PREC_FP64, "fp32": capi.PREC_FP32}


def parse_algorithm(name: str) -> str:
    """pipeline.cpp:27-32."""
    if name not in _ALGOS:
        raise ValueError(f"unknown algorithm '{name}' (expected fse, ofse or fofse)")
    return name


@dataclass
class ConcealConfig:
    """fse::ConcealConfig (pipeline.hpp:19-33) + precision / guard knobs."""
    algorithm: str = "fofse"
    gamma: float = 0.2
    iterations: int = 200
    transform_size: int = 64
    rho_hat: float = 0.8
    support_width: int = 16
    threads: int = 1
    record_traces: bool = False
    precision: str = "fp64"
    guard_tau: float = -1.0
    fp64_head: int = -1
    basis: str = "dft2d"  # fse::BasisKind (basis.hpp:17): dft2d or dct2d

    def validate(self):
        """pipeline.cpp:34-38 + engine_spatial.cpp:8-15 (same messages)."""
        parse_algorithm(self.algorithm)
        if self.iterations < 0:
            raise ValueError("config: iterations must be >= 0")
        if self.transform_size < 1:
            raise ValueError("config: transform size must be >= 1")
        if not (self.rho_hat > 0.0) or not (self.rho_hat < 1.0):
            raise ValueError("config: rho_hat must lie in (0, 1)")
        if self.algorithm == "fofse" and (not (self.gamma > 0.0) or self.gamma > 1.0):
            raise ValueError("config: gamma must lie in (0, 1]")
        if self.support_width < 1:
            raise ValueError("config: support width must be >= 1")
        if self.threads < 1:
            raise ValueError("config: thread count must be >= 1")

    def params(self) -> capi.Params:
        p = capi.default_params()
        p.algorithm = _ALGOS[parse_algorithm(self.algorithm)]
        p.gamma = self.gamma
        p.iterations = self.iterations
        p.transform_size = self.transform_size
        p.rho_hat = self.rho_hat
        p.support_width = self.support_width
        p.threads = self.threads
        p.record_traces = int(bool(self.record_traces))
        if self.precision not in _PRECS:
            raise ValueError("config: precision must be 'fp64' or 'fp32'")
        p.precision = _PRECS[self.precision]
        p.guard_tau = self.guard_tau
        p.fp64_head = self.fp64_head
        if self.basis not in ("dft2d", "dct2d"):
            raise ValueError("config: basis must be 'dft2d' or 'dct2d'")
        p.basis = capi.BASIS_DCT if self.basis == "dct2d" else capi.BASIS_DFT
        return p


def series_label(config: ConcealConfig) -> str:
    """pipeline.cpp:63-68."""
    if config.algorithm != "fofse":
        return config.algorithm
    return "fofse_g%g" % config.gamma


@dataclass
class ConcealmentReport:
    algorithm: str
    gamma: float
    iterations: int
    psnr_db: float
    psnr_identical: bool
    mean_seconds_per_block: float
    traces: list | None = None
    device: dict | None = None


@dataclass
class ConcealOutput:
    restored: np.ndarray
    report: ConcealmentReport


def _report(config, rep: capi.Report, traces=None) -> ConcealmentReport:
    return ConcealmentReport(
        algorithm=config.algorithm,
        gamma=config.gamma if config.algorithm == "fofse" else 1.0,
        iterations=config.iterations, psnr_db=rep.psnr_db,
        psnr_identical=bool(rep.psnr_identical),
        mean_seconds_per_block=rep.mean_seconds_per_block, traces=traces, device=rep.as_dict())


@dataclass
class CurveSeries:
    """fse::CurveSeries (pipeline.hpp:86-96): label + (iterations, psnr_db) points."""
    label: str
    points: list


def psnr_vs_iterations(image: np.ndarray, pattern: LossPattern, algorithms, max_iterations: int,
                       stride: int, device: int = 0) -> list:
    """fse::psnr_vs_iterations (pipeline.cpp:264-369): the PSNR over all MISSING
    samples after stride, 2 stride, ... <= max_iterations selections, per config
    (the paper's Fig. 4/5 gamma sweep). Resumable fp64 phases on the GPU."""
    if stride < 1:
        raise ValueError("psnr_vs_iterations: stride must be >= 1")
    if max_iterations < 0:
        raise ValueError("psnr_vs_iterations: iterations must be >= 0")
    algorithms = list(algorithms)
    image = np.ascontiguousarray(image, np.float64)
    h, w = image.shape
    nck = max_iterations // stride
    if nck == 0:
        return [CurveSeries(series_label(c), []) for c in algorithms]
    rects = capi.rects_array(pattern.blocks)
    params = (capi.Params * max(len(algorithms), 1))(*[c.params() for c in algorithms])
    cks = np.zeros(nck, np.int32)
    db = np.zeros((len(algorithms), nck), np.float64)
    ctx = capi.context(device)
    capi.check(capi.lib().fofse_psnr_curves(
        ctx.handle, capi.ptr(image), w, h, rects.ctypes.data_as(C.POINTER(capi.Rect_)), C.c_int64(len(rects)),
        pattern.block_height, pattern.block_width, params, len(algorithms), int(max_iterations), int(stride),
        capi.ptr(cks, C.c_int32), capi.ptr(db)))
    return [CurveSeries(series_label(c), [(int(cks[k]), float(db[i, k])) for k in range(nck)])
            for i, c in enumerate(algorithms)]


def conceal(image: np.ndarray, pattern: LossPattern, config: ConcealConfig | None = None,
            device: int = 0) -> ConcealOutput:
    """fse::conceal: restored image (MISSING samples replaced, clamped, unrounded) + report."""
    config = config or ConcealConfig()
    image = np.ascontiguousarray(image, np.float64)
    if image.ndim != 2:
        raise ValueError("image must be 2-D")
    h, w = image.shape
    if pattern.image_width != w or pattern.image_height != h:
        # pipeline.cpp:126-127 (checked after validate + validate_pattern)
        config.validate()
        raise ValueError("conceal: pattern dimensions do not match the image")
    rects = capi.rects_array(pattern.blocks)
    n = len(rects)
    restored = np.empty_like(image)
    traces = counts = None
    if config.record_traces and config.iterations > 0:
        traces = np.zeros(n * config.iterations, capi.RECORD_DTYPE)
        counts = np.zeros(n, np.int32)
    rep = capi.Report()
    ctx = capi.context(device)
    capi.check(capi.lib().fofse_conceal_f64(
        ctx.handle, capi.ptr(image), w, h, rects.ctypes.data_as(C.POINTER(capi.Rect_)), C.c_int64(n),
        pattern.block_height, pattern.block_width, C.byref(config.params()), capi.ptr(restored),
        capi.vptr(traces), capi.ptr(counts, C.c_int32), C.byref(rep)))
    tr = None
    if traces is not None:
        it = config.iterations
        tr = [traces[i * it: i * it + counts[i]] for i in range(n)]
    elif config.record_traces:
        tr = [np.zeros(0, capi.RECORD_DTYPE) for _ in range(n)]
    return ConcealOutput(restored, _report(config, rep, tr))


def conceal_shard(image: np.ndarray, pattern: LossPattern, first: int, count: int,
                  config: ConcealConfig | None = None, device: int = 0):
    """Conceal blocks[first:first+count] only; every block of the pattern stays
    lost (OUTSIDE in the others' windows). Returns (restored, report)."""
    config = config or ConcealConfig()
    image = np.ascontiguousarray(image, np.float64)
    h, w = image.shape
    rects = capi.rects_array(pattern.blocks)
    restored = np.empty_like(image)
    rep = capi.Report()
    ctx = capi.context(device)
    capi.check(capi.lib().fofse_conceal_shard_f64(
        ctx.handle, capi.ptr(image), w, h, rects.ctypes.data_as(C.POINTER(capi.Rect_)),
        C.c_int64(len(rects)), C.c_int64(int(first)), C.c_int64(int(count)), pattern.block_height, pattern.block_width, C.byref(config.params()),
        capi.ptr(restored), C.byref(rep)))
    return restored, _report(config, rep)


def conceal_frames(frames: np.ndarray, patterns: list, config: ConcealConfig | None = None,
                   device: int = 0, inplace: bool = False):
    """Batched frames (video). uint8 frames: restored uint8 (rounded like write_pgm);
    float64 frames: the same pipeline with the unrounded concealed pixels.
    Returns (restored frames, per-block sq errors, report)."""
    config = config or ConcealConfig()
    f64 = np.asarray(frames).dtype == np.float64
    frames = np.ascontiguousarray(frames, np.float64 if f64 else np.uint8)
    f, h, w = frames.shape
    if len(patterns) != f:
        raise ValueError("one LossPattern per frame is required")
    bh = patterns[0].block_height if patterns else 0
    bw = patterns[0].block_width if patterns else 0
    offs = np.zeros(f + 1, np.int64)
    allb = []
    for i, p in enumerate(patterns):
        if (p.block_height, p.block_width) != (bh, bw):
            raise ValueError("pattern: blocks must share one size")
        allb.extend(p.blocks)
        offs[i + 1] = len(allb)
    rects = capi.rects_array(allb)
    out = frames if inplace else np.empty_like(frames)
    sq = np.zeros(len(rects), np.float64)
    rep = capi.Report()
    ctx = capi.context(device)
    if f64:
        capi.check(capi.lib().fofse_conceal_frames_f64(
            ctx.handle, capi.ptr(frames), f, w, h,
            rects.ctypes.data_as(C.POINTER(capi.Rect_)), capi.ptr(offs, C.c_int64), bh, bw,
            C.byref(config.params()), capi.ptr(out), capi.ptr(sq), C.byref(rep)))
    else:
        capi.check(capi.lib().fofse_conceal_frames_u8(
            ctx.handle, capi.ptr(frames, C.c_uint8), f, w, h,
            rects.ctypes.data_as(C.POINTER(capi.Rect_)), capi.ptr(offs, C.c_int64), bh, bw,
            C.byref(config.params()), capi.ptr(out, C.c_uint8), capi.ptr(sq), C.byref(rep)))
    return out, sq, _report(config, rep)


@dataclass
class WindowRun:
    model: np.ndarray
    trace: np.ndarray


def extrapolate_windows(windows: np.ndarray, masks: np.ndarray, config: ConcealConfig | None = None,
                        device: int = 0):
    """Batched fse::extrapolate_window: (n, h, w) windows + Region labels -> models, traces."""
    config = config or ConcealConfig()
    windows = np.ascontiguousarray(windows, np.float64)
    masks = np.ascontiguousarray(masks, np.uint8)
    n, wh, ww = windows.shape
    models = np.zeros_like(windows)
    traces = counts = None
    if config.iterations > 0:
        traces = np.zeros(n * config.iterations, capi.RECORD_DTYPE)
        counts = np.zeros(n, np.int32)
    ctx = capi.context(device)
    capi.check(capi.lib().fofse_extrapolate_windows(
        ctx.handle, capi.ptr(windows), capi.ptr(masks, C.c_uint8), C.c_int64(n), wh, ww,
        C.byref(config.params()), capi.ptr(models), capi.vptr(traces), capi.ptr(counts, C.c_int32)))
    it = config.iterations
    runs = []
    for i in range(n):
        tr = traces[i * it: i * it + counts[i]] if traces is not None else np.zeros(0, capi.RECORD_DTYPE)
        runs.append(WindowRun(models[i], tr))
    return runs


def extrapolate_window(window: np.ndarray, mask: np.ndarray, config: ConcealConfig | None = None,
                       device: int = 0) -> WindowRun:
    return extrapolate_windows(window[None], mask[None], config, device)[0]


def build_isotropic_weight(mask: np.ndarray, rho_hat: float) -> np.ndarray:
    """grid.cpp:75-92 (host helper; libm pow/hypot like the reference)."""
    if not (rho_hat > 0.0 and rho_hat < 1.0):
        raise ValueError("rho_hat must lie in (0,1)")
    h, w = mask.shape
    cr, cc = (h - 1) / 2.0, (w - 1) / 2.0
    out = np.zeros((h, w), np.float64)
    for r in range(h):
        for c in range(w):
            if mask[r, c] == Region.support:
                out[r, c] = math.pow(rho_hat, math.hypot(r - cr, c - cc))
    return out


def psnr(original: np.ndarray, reconstructed: np.ndarray, mask: np.ndarray, evaluate_on: int,
         peak: float = 255.0):
    """grid.cpp:103-121 -> (db, identical)."""
    sel = mask == evaluate_on
    if not sel.any():
        raise ValueError("psnr: no samples carry the evaluated label")
    e = original[sel] - reconstructed[sel]
    sq = float(np.sum(e * e))
    if sq == 0.0:
        return 0.0, True
    return 10.0 * math.log10(peak * peak / (sq / int(sel.sum()))), False


class spectral:
    """Engine level (engine_spectral.hpp:16-51) on the GPU, batched."""

    @dataclass
    class Spectrum:
        t: int
        window_width: int
        window_height: int
        rw: np.ndarray
        w: np.ndarray
        g: np.ndarray
        w0: float = 0.0
        weighted_energy: float = 0.0
        initial_energy: float = 0.0
        initial_max: float = 0.0
        nu: int = 0
        converged: bool = False
        trace: list = field(default_factory=list)

    @staticmethod
    def init_spectra(f: np.ndarray, mask: np.ndarray, weight: np.ndarray, t: int, device: int = 0):
        f = np.ascontiguousarray(f, np.float64)
        mask = np.ascontiguousarray(mask, np.uint8)
        weight = np.ascontiguousarray(weight, np.float64)
        if f.shape != mask.shape or f.shape != weight.shape:
            raise ValueError("init_spectra: signal, mask and weight shapes differ")
        h, w = f.shape
        rw = np.zeros((t, t), np.complex128)
        ws = np.zeros((t, t), np.complex128)
        w0 = np.zeros(1)
        e = np.zeros(1)
        m = np.zeros(1)
        ctx = capi.context(device)
        capi.check(capi.lib().fofse_spectral_init(
            ctx.handle, capi.ptr(f), capi.ptr(mask, C.c_uint8), capi.ptr(weight), C.c_int64(1), h, w, t,
            capi.ptr(rw.view(np.float64)), capi.ptr(ws.view(np.float64)), capi.ptr(w0), capi.ptr(e),
            capi.ptr(m)))
        return spectral.Spectrum(t, w, h, rw, ws, np.zeros((t, t), np.complex128), float(w0[0]),
                                 float(e[0]), float(e[0]), float(m[0]))

    @staticmethod
    def fast_iterate_full_od(spec, iterations: int, device: int = 0):
        """OFSE (engine_spectral.cpp:191-193): full orthogonality-deficiency
        compensation, gamma_eff = min(|p w0^2 / d|, 1); fp64. Resumable."""
        return spectral._iterate(spec, 1.0, iterations, "fp64", device, full_od=True)

    @staticmethod
    def fast_iterate(spec, gamma: float, iterations: int, precision: str = "fp64", device: int = 0):
        """Resumable like the reference: runs at most `iterations` more selections."""
        return spectral._iterate(spec, gamma, iterations, precision, device)

    @staticmethod
    def _iterate(spec, gamma, iterations, precision, device, full_od=False):
        t = spec.t
        rw = np.ascontiguousarray(spec.rw, np.complex128)
        g = np.ascontiguousarray(spec.g, np.complex128)
        ws = np.ascontiguousarray(spec.w, np.complex128)
        w0 = np.array([spec.w0])
        e = np.array([spec.weighted_energy])
        ei = np.array([spec.initial_energy])
        im = np.array([spec.initial_max])
        nu = np.array([spec.nu], np.int32)
        cv = np.array([int(spec.converged)], np.int32)
        its = max(int(iterations), 0)
        tr = np.zeros(max(its, 1), capi.RECORD_DTYPE)
        tc = np.zeros(1, np.int32)
        ctx = capi.context(device)
        if full_od:
            capi.check(capi.lib().fofse_spectral_iterate_full_od(
                ctx.handle, t, C.c_int64(1), spec.window_height, spec.window_width,
                capi.ptr(rw.view(np.float64)), capi.ptr(ws.view(np.float64)), capi.ptr(g.view(np.float64)),
                capi.ptr(w0), capi.ptr(e), capi.ptr(ei), capi.ptr(im), capi.ptr(nu, C.c_int32),
                capi.ptr(cv, C.c_int32), int(iterations), capi.vptr(tr), capi.ptr(tc, C.c_int32)))
        else:
            capi.check(capi.lib().fofse_spectral_iterate(
                ctx.handle, t, C.c_int64(1), spec.window_height, spec.window_width, capi.ptr(rw.view(np.float64)),
                capi.ptr(ws.view(np.float64)), capi.ptr(g.view(np.float64)), capi.ptr(w0), capi.ptr(e),
                capi.ptr(ei), capi.ptr(im), capi.ptr(nu, C.c_int32), capi.ptr(cv, C.c_int32),
                C.c_double(gamma), int(iterations), _PRECS[precision], capi.vptr(tr),
                capi.ptr(tc, C.c_int32)))
        spec.rw, spec.g = rw, g
        spec.weighted_energy = float(e[0])
        spec.nu = int(nu[0])
        spec.converged = bool(cv[0])
        spec.trace.extend(tr[: tc[0]].tolist())
        return tr[: tc[0]]

    @staticmethod
    def synthesize_model(spec, device: int = 0) -> np.ndarray:
        t = spec.t
        g = np.ascontiguousarray(spec.g, np.complex128)
        out = np.zeros((spec.window_height, spec.window_width), np.float64)
        mi = np.zeros(1)
        ctx = capi.context(device)
        capi.check(capi.lib().fofse_spectral_synthesize(
            ctx.handle, t, C.c_int64(1), capi.ptr(g.view(np.float64)), spec.window_height, spec.window_width,
            capi.ptr(out), capi.ptr(mi)))
        return out
