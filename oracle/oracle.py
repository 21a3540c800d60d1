"""ORACLE / TEST INFRASTRUCTURE ONLY.

ctypes bindings for
  * ``_build/libfofse_oracle.so`` — the plain-C restatement of the reference
    FOFSE path (fofse_oracle.c), and
  * ``_ref/libfse_ref.so`` — the UNMODIFIED reference sources compiled from
    /root/reference/proj/src with our FFT stand-in + extern "C" shim.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline
leg and ``--impl reference``) may import this module, and only as the checker
or the CPU baseline. The product path (paper_2207_01205_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libfofse_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfse_ref.so")
REF_SRC = "/root/reference/proj"

SUPPORT, MISSING, OUTSIDE = 0, 1, 2
ALGO_FSE, ALGO_OFSE, ALGO_FOFSE = 0, 1, 2


class OrRect(C.Structure):
    _fields_ = [("row", C.c_int), ("col", C.c_int), ("height", C.c_int), ("width", C.c_int)]


class OrSpectrum(C.Structure):
    _fields_ = [
        ("t", C.c_int), ("window_width", C.c_int), ("window_height", C.c_int),
        ("rw", C.POINTER(C.c_double)), ("w", C.POINTER(C.c_double)), ("g", C.POINTER(C.c_double)),
        ("w0", C.c_double), ("weighted_energy", C.c_double), ("initial_energy", C.c_double),
        ("initial_max", C.c_double), ("nu", C.c_int), ("converged", C.c_int),
    ]


class OrRecord(C.Structure):
    _fields_ = [
        ("nu", C.c_int), ("u1", C.c_int), ("u2", C.c_int),
        ("p_re", C.c_double), ("p_im", C.c_double), ("c_re", C.c_double), ("c_im", C.c_double),
        ("gamma_effective", C.c_double), ("weighted_energy", C.c_double), ("degenerate", C.c_int),
    ]


RECORD_DTYPE = np.dtype([
    ("nu", np.int32), ("u1", np.int32), ("u2", np.int32), ("_pad", np.int32),
    ("p_re", np.float64), ("p_im", np.float64), ("c_re", np.float64), ("c_im", np.float64),
    ("gamma_effective", np.float64), ("weighted_energy", np.float64),
    ("degenerate", np.int32), ("_pad2", np.int32),
])
assert RECORD_DTYPE.itemsize == C.sizeof(OrRecord)


class OracleError(Exception):
    pass


class OracleInvalidArgument(OracleError, ValueError):
    pass


def build(ref: bool | None = None) -> None:
    """Compile the C restatement (always) and the reference (when its sources exist)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if ref is None:
        ref = os.path.isdir(os.path.join(REF_SRC, "src"))
    if ref:
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _u8p(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_ubyte))


@dataclass
class Spectrum:
    """Mirror of fse::spectral::Spectrum (engine_spectral.hpp:16-35)."""
    t: int
    window_width: int
    window_height: int
    rw: np.ndarray  # complex128 (t, t)
    w: np.ndarray
    g: np.ndarray
    w0: float = 0.0
    weighted_energy: float = 0.0
    initial_energy: float = 0.0
    initial_max: float = 0.0
    nu: int = 0
    converged: bool = False

    @classmethod
    def empty(cls, t):
        z = lambda: np.zeros((t, t), np.complex128)
        return cls(t, 0, 0, z(), z(), z())

    def copy(self):
        return Spectrum(self.t, self.window_width, self.window_height, self.rw.copy(),
                        self.w.copy(), self.g.copy(), self.w0, self.weighted_energy,
                        self.initial_energy, self.initial_max, self.nu, self.converged)

    def _to_c(self) -> OrSpectrum:
        for a in (self.rw, self.w, self.g):
            assert a.dtype == np.complex128 and a.flags.c_contiguous
        return OrSpectrum(self.t, self.window_width, self.window_height,
                          self.rw.ctypes.data_as(C.POINTER(C.c_double)),
                          self.w.ctypes.data_as(C.POINTER(C.c_double)),
                          self.g.ctypes.data_as(C.POINTER(C.c_double)),
                          self.w0, self.weighted_energy, self.initial_energy, self.initial_max,
                          self.nu, int(self.converged))

    def _from_c(self, s: OrSpectrum):
        self.t, self.window_width, self.window_height = s.t, s.window_width, s.window_height
        self.w0, self.weighted_energy = s.w0, s.weighted_energy
        self.initial_energy, self.initial_max = s.initial_energy, s.initial_max
        self.nu, self.converged = s.nu, bool(s.converged)


class _Lib:
    prefix = ""
    path = ""

    def __init__(self):
        if not os.path.exists(self.path):
            raise OracleError(f"{self.path} not built (run oracle.build())")
        self.lib = C.CDLL(self.path)
        getattr(self.lib, self.prefix + "last_error").restype = C.c_char_p

    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)  # cached attribute keeps restype

    def _check(self, rc):
        if rc == 0:
            return
        msg = self._fn("last_error")().decode()
        raise (OracleInvalidArgument if rc == 1 else OracleError)(msg)

    # --- shared API -------------------------------------------------------
    def build_isotropic_weight(self, labels: np.ndarray, rho_hat: float) -> np.ndarray:
        labels = np.ascontiguousarray(labels, np.uint8)
        h, w = labels.shape
        out = np.zeros((h, w), np.float64)
        self._check(self._fn("build_isotropic_weight")(_u8p(labels), h, w, C.c_double(rho_hat),
                                                       _dp(out)))
        return out

    def init_spectra(self, f, labels, weight, t) -> Spectrum:
        f = np.ascontiguousarray(f, np.float64)
        labels = np.ascontiguousarray(labels, np.uint8)
        weight = np.ascontiguousarray(weight, np.float64)
        h, w = f.shape
        s = Spectrum.empty(t)
        cs = s._to_c()
        self._check(self._fn("init_spectra")(_dp(f), _u8p(labels), _dp(weight), h, w, t,
                                             C.byref(cs)))
        s._from_c(cs)
        return s

    def _iterate(self, name, s: Spectrum, *args):
        iters = args[-1]
        recs = np.zeros(max(iters, 0), RECORD_DTYPE)
        cnt = C.c_int(0)
        cs = s._to_c()
        self._check(self._fn(name)(C.byref(cs), *args,
                                   recs.ctypes.data_as(C.POINTER(OrRecord)), max(iters, 0),
                                   C.byref(cnt)))
        s._from_c(cs)
        return recs[: cnt.value]

    def fast_iterate(self, s: Spectrum, gamma: float, iterations: int):
        return self._iterate("fast_iterate", s, C.c_double(gamma), iterations)

    def fast_iterate_full_od(self, s: Spectrum, iterations: int):
        return self._iterate("fast_iterate_full_od", s, iterations)

    def conceal(self, image, blocks, block_h, block_w, *, algorithm=ALGO_FOFSE, gamma=0.2,
                iterations=200, t=64, rho_hat=0.8, support=16, threads=1, traces=False, basis=0):
        image = np.ascontiguousarray(image, np.float64)
        h, w = image.shape
        rects = (OrRect * max(len(blocks), 1))(*[OrRect(*map(int, b)) for b in blocks])
        n = len(blocks)
        restored = np.zeros_like(image)
        recs = np.zeros(n * max(iterations, 0), RECORD_DTYPE) if traces else None
        counts = np.zeros(n, np.int32)
        db, ident = C.c_double(0), C.c_int(0)
        extra = self._conceal_extra()
        fn = "conceal"
        if basis:  # DCT (spatial engine): the compiled reference only
            if not isinstance(self, Reference):
                raise OracleError("the DCT basis is pinned on the compiled reference (oracle/_ref) only")
            fn, extra = "conceal_basis", extra + (int(basis),)
        rc = self._fn(fn)(
            _dp(image), w, h, rects, n, block_h, block_w, algorithm, C.c_double(gamma),
            iterations, t, C.c_double(rho_hat), support, threads, _dp(restored),
            recs.ctypes.data_as(C.POINTER(OrRecord)) if traces else None,
            counts.ctypes.data_as(C.POINTER(C.c_int)), C.byref(db), C.byref(ident), *extra)
        self._check(rc)
        out = {"restored": restored, "psnr_db": db.value, "psnr_identical": bool(ident.value)}
        if traces:
            its = max(iterations, 0)
            out["traces"] = [recs[i * its: i * its + counts[i]] for i in range(n)]
        return out


class Oracle(_Lib):
    """The plain-C restatement (fofse_oracle.c)."""
    prefix = "or_"
    path = ORACLE_SO

    def _conceal_extra(self):
        return (None,)  # block_sq

    def dft2d(self, x: np.ndarray, inverse=False) -> np.ndarray:
        x = np.ascontiguousarray(x, np.complex128)
        out = np.zeros_like(x)
        fn = self._fn("dft2d_inverse" if inverse else "dft2d_forward")
        self._check(fn(x.shape[0], x.ctypes.data_as(C.POINTER(C.c_double)),
                       out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def synthesize_model(self, s: Spectrum):
        out = np.zeros((s.window_height, s.window_width), np.float64)
        mi = C.c_double(0)
        cs = s._to_c()
        self._check(self._fn("synthesize_model")(C.byref(cs), _dp(out), C.byref(mi)))
        return out

    def build_window(self, image, lost, block, support):
        image = np.ascontiguousarray(image, np.float64)
        lost = np.ascontiguousarray(lost, np.uint8)
        h, w = image.shape
        r = OrRect(*map(int, block))
        wh, ww = r.height + 2 * support, r.width + 2 * support
        win = np.zeros((wh, ww), np.float64)
        lab = np.zeros((wh, ww), np.uint8)
        self._check(self._fn("build_window")(_dp(image), w, h, _u8p(lost), r, support, _dp(win),
                                             _u8p(lab)))
        return win, lab


class Reference(_Lib):
    """The unmodified reference library (oracle/_ref/libfse_ref.so)."""
    prefix = "ref_"
    path = REF_SO

    def _conceal_extra(self):
        return (None,)  # mean_seconds_per_block

    def dft2d(self, x: np.ndarray, inverse=False) -> np.ndarray:
        x = np.ascontiguousarray(x, np.complex128)
        out = np.zeros_like(x)
        self._check(self._fn("dft2d")(x.shape[0], int(inverse),
                                      x.ctypes.data_as(C.POINTER(C.c_double)),
                                      out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def transform_counts(self):
        f, i = C.c_longlong(0), C.c_longlong(0)
        self._fn("transform_counts")(C.byref(f), C.byref(i))
        return f.value, i.value

    def synthesize_model(self, s: Spectrum):
        out = np.zeros((s.window_height, s.window_width), np.float64)
        cs = s._to_c()
        self._check(self._fn("synthesize_model")(C.byref(cs), _dp(out)))
        return out

    def spatial_run(self, f, labels, t, rho_hat, iterations, selection, compensation, gamma):
        f = np.ascontiguousarray(f, np.float64)
        labels = np.ascontiguousarray(labels, np.uint8)
        h, w = f.shape
        model = np.zeros((h, w), np.float64)
        recs = np.zeros(max(iterations, 0), RECORD_DTYPE)
        cnt = C.c_int(0)
        self._check(self._fn("spatial_run")(_dp(f), _u8p(labels), h, w, t, C.c_double(rho_hat),
                                            iterations, selection, compensation,
                                            C.c_double(gamma), _dp(model),
                                            recs.ctypes.data_as(C.POINTER(OrRecord)),
                                            max(iterations, 0), C.byref(cnt)))
        return model, recs[: cnt.value]

    def psnr(self, original, reconstructed, labels, evaluate_on, peak=255.0):
        o = np.ascontiguousarray(original, np.float64)
        r = np.ascontiguousarray(reconstructed, np.float64)
        lab = np.ascontiguousarray(labels, np.uint8)
        db, ident = C.c_double(0), C.c_int(0)
        self._check(self._fn("psnr")(_dp(o), _dp(r), _u8p(lab), o.shape[0], o.shape[1],
                                     evaluate_on, C.c_double(peak), C.byref(db), C.byref(ident)))
        return db.value, bool(ident.value)

    def generate_grid_pattern(self, img_w, img_h, block, spacing, limit=81):
        cap = 1 << 16
        out = (OrRect * cap)()
        n = C.c_int(0)
        self._check(self._fn("generate_grid_pattern")(img_w, img_h, block, spacing, limit, out,
                                                      cap, C.byref(n)))
        return [(out[i].row, out[i].col, out[i].height, out[i].width) for i in range(n.value)]

    def extract_windows(self, image, blocks, block_h, block_w, support):
        image = np.ascontiguousarray(image, np.float64)
        h, w = image.shape
        n = len(blocks)
        wh, ww = block_h + 2 * support, block_w + 2 * support
        wins = np.zeros((n, wh, ww), np.float64)
        labs = np.zeros((n, wh, ww), np.uint8)
        rects = (OrRect * max(n, 1))(*[OrRect(*map(int, b)) for b in blocks])
        self._check(self._fn("extract_windows")(_dp(image), w, h, rects, n, block_h, block_w,
                                                support, _dp(wins), _u8p(labs)))
        return wins, labs


def have_reference() -> bool:
    return os.path.exists(REF_SO)
