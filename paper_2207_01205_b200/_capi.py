"""ctypes binding of the C ABI (include/fofse.h) of _lib/libfofse.so.

The library is the product: CUDA kernels for sm_100a behind a plain C ABI.
There is no CPU fallback — if the library or a CUDA device is missing, calls
raise FofseCudaError.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

# FOFSE_LIB_PATH: another build of the library (same-box A/B of kernel variants)
LIB_PATH = os.environ.get("FOFSE_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib",
                                                            "libfofse.so")
# synthetic-input generator (include/fofse_gen.h): its own host-only library, so
# generating a workload never maps the product library
GEN_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libfofse_gen.so")
GEN_EXPORTS = ["fofse_gen_image_u8", "fofse_gen_losses"]

OK, EINVAL, ERUNTIME, ECUDA, EUNSUPPORTED = 0, 1, 2, 3, 4
ALGO_FSE, ALGO_OFSE, ALGO_FOFSE = 0, 1, 2
PREC_FP64, PREC_FP32 = 0, 1
BASIS_DFT, BASIS_DCT = 0, 1
SUPPORT, MISSING, OUTSIDE = 0, 1, 2

# Every symbol include/fofse.h declares (checked by tests/test_capi.py).
EXPORTS = [
    "fofse_abi_version", "fofse_last_error", "fofse_params_default", "fofse_create",
    "fofse_destroy", "fofse_set_stream", "fofse_conceal_f64", "fofse_conceal_frames_u8", "fofse_conceal_frames_f64",
    "fofse_plan_frames_u8", "fofse_plan_execute_device", "fofse_plan_destroy",
    "fofse_extrapolate_windows", "fofse_spectral_init", "fofse_spectral_iterate",
    "fofse_spectral_synthesize",
    "fofse_validate_conceal", "fofse_plan_info", "fofse_plan_block_labels", "fofse_microbench",
    "fofse_diag_conceal_f64", "fofse_diag_spectral_iterate",
    "fofse_conceal_shard_f64", "fofse_conceal_shard_tiles_f64", "fofse_host_register", "fofse_host_unregister", "fofse_spectral_iterate_full_od", "fofse_psnr_curves",
]


class FofseError(RuntimeError):
    pass


class FofseCudaError(FofseError):
    pass


class Rect_(C.Structure):
    _fields_ = [("row", C.c_int32), ("col", C.c_int32), ("height", C.c_int32), ("width", C.c_int32)]


class Params(C.Structure):
    _fields_ = [
        ("algorithm", C.c_int32), ("gamma", C.c_double), ("iterations", C.c_int32),
        ("transform_size", C.c_int32), ("rho_hat", C.c_double), ("support_width", C.c_int32),
        ("threads", C.c_int32), ("record_traces", C.c_int32), ("precision", C.c_int32),
        ("guard_tau", C.c_double), ("fp64_head", C.c_int32), ("basis", C.c_int32),
    ]


class Report(C.Structure):
    _fields_ = [
        ("psnr_db", C.c_double), ("psnr_identical", C.c_int32), ("pad0", C.c_int32),
        ("mean_seconds_per_block", C.c_double), ("blocks", C.c_int64), ("classes", C.c_int64),
        ("guard_reruns", C.c_int64), ("converged_blocks", C.c_int64), ("init_ms", C.c_double),
        ("iterate_ms", C.c_double), ("total_ms", C.c_double), ("kernel_launches", C.c_int64),
        ("rerun_ms", C.c_double), ("fp64_head", C.c_int64), ("real_blocks", C.c_int64),
        ("real_iterate_ms", C.c_double), ("k1_ms", C.c_double),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if not k.startswith("pad")}


RECORD_DTYPE = np.dtype([
    ("nu", np.int32), ("u1", np.int32), ("u2", np.int32), ("_pad", np.int32),
    ("p_re", np.float64), ("p_im", np.float64), ("c_re", np.float64), ("c_im", np.float64),
    ("gamma_effective", np.float64), ("weighted_energy", np.float64),
    ("degenerate", np.int32), ("_pad2", np.int32),
])
RECT_DTYPE = np.dtype([("row", np.int32), ("col", np.int32), ("height", np.int32), ("width", np.int32)])

_lib = None


def lib():
    """Load libfofse.so (raises FofseCudaError if it is not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FofseCudaError(f"{LIB_PATH} is not built; run paper_2207_01205_b200.build.build()")
        L = C.CDLL(LIB_PATH)
        L.fofse_last_error.restype = C.c_char_p
        L.fofse_plan_destroy.restype = None
        L.fofse_destroy.restype = None
        L.fofse_params_default.restype = None
        _lib = L
    return _lib


_gen = None


def gen_lib():
    """Load libfofse_gen.so (host-only synthetic inputs)."""
    global _gen
    if _gen is None:
        if not os.path.exists(GEN_LIB_PATH):
            raise FofseError(f"{GEN_LIB_PATH} is not built; run paper_2207_01205_b200.build.build()")
        G = C.CDLL(GEN_LIB_PATH)
        G.fofse_gen_losses.restype = C.c_int64
        _gen = G
    return _gen


def check(rc: int):
    if rc == OK:
        return
    msg = lib().fofse_last_error().decode()
    if rc == EINVAL:
        raise ValueError(msg)
    if rc == EUNSUPPORTED:
        raise NotImplementedError(msg)
    if rc == ECUDA:
        raise FofseCudaError(msg)
    raise RuntimeError(msg)


def ptr(a: np.ndarray | None, ctype=C.c_double):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ctype))


def vptr(a: np.ndarray | None):
    return None if a is None else C.c_void_p(a.ctypes.data)


def default_params() -> Params:
    p = Params()
    lib().fofse_params_default(C.byref(p))
    return p


class Context:
    """One device + one stream + cached device workspaces (fofse_ctx)."""

    def __init__(self, device: int = 0):
        self.device = device
        self._h = C.c_void_p()
        check(lib().fofse_create(device, C.byref(self._h)))

    @property
    def handle(self):
        if not self._h:
            raise FofseError("context destroyed")
        return self._h

    def set_stream(self, cuda_stream_ptr: int | None):
        check(lib().fofse_set_stream(self.handle, C.c_void_p(cuda_stream_ptr or 0)))

    def close(self):
        if self._h:
            lib().fofse_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_contexts: dict[int, Context] = {}


def context(device: int = 0) -> Context:
    ctx = _contexts.get(device)
    if ctx is None:
        ctx = _contexts[device] = Context(device)
    return ctx


def rects_array(blocks) -> np.ndarray:
    arr = np.zeros(len(blocks), RECT_DTYPE)
    for i, b in enumerate(blocks):
        r, c, h, w = b  # Rect, tuple or structured row
        arr[i] = (int(r), int(c), int(h), int(w))
    return arr


def gen_image_u8(seed: int, width: int, height: int) -> np.ndarray:
    out = np.empty((height, width), np.uint8)
    if gen_lib().fofse_gen_image_u8(C.c_uint64(seed), width, height, ptr(out, C.c_uint8)) != OK:
        raise ValueError("gen_image_u8: bad arguments")
    return out


def gen_losses(seed: int, grid_w: int, grid_h: int, frac: float, block_h: int, block_w: int):
    n = gen_lib().fofse_gen_losses(C.c_uint64(seed), grid_w, grid_h, C.c_double(frac), block_h, block_w,
                               None, 0)
    if n < 0:
        raise ValueError("gen_losses: bad arguments")
    out = np.zeros(n, RECT_DTYPE)
    gen_lib().fofse_gen_losses(C.c_uint64(seed), grid_w, grid_h, C.c_double(frac), block_h, block_w,
                           out.ctypes.data_as(C.POINTER(Rect_)), n)
    return out


def ptr_dev(t, ctype=C.c_double):
    """Device pointer of a torch tensor as a typed ctypes pointer (plumbing only)."""
    return C.cast(C.c_void_p(t.data_ptr()), C.POINTER(ctype))


def microbench(device: int, kind: int) -> float:
    v = C.c_double(0)
    check(lib().fofse_microbench(device, kind, C.byref(v)))
    return v.value
