"""fp32 near-tie guard study (runs on the GPU box).

For seeded C2/C3/C4/C5 inputs: GPU fp64 (reference-parity path) vs GPU fp32
with the guard OFF, recording per block the selected-basis sequences, the fp32
top-2 relative gaps at every selection and the pixel errors. The guard rule
and its tau are chosen offline from this data ("fp32 guard").
"""
import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2207_01205_b200 as P  # noqa: E402
from paper_2207_01205_b200 import _capi as capi  # noqa: E402
from paper_2207_01205_b200 import workloads as WL  # noqa: E402


def diag(img, pat, cfg):
    n = len(pat.blocks)
    it = cfg.iterations
    rects = capi.rects_array(pat.blocks)
    restored = np.empty_like(img)
    tr = np.zeros(n * it, capi.RECORD_DTYPE)
    tc = np.zeros(n, np.int32)
    gap = np.zeros(n * it, np.float32)
    capi.check(capi.lib().fofse_diag_conceal_f64(
        capi.context(0).handle, capi.ptr(img), img.shape[1], img.shape[0],
        rects.ctypes.data_as(C.POINTER(capi.Rect_)), C.c_int64(n), pat.block_height, pat.block_width,
        C.byref(cfg.params()), capi.ptr(restored), capi.vptr(tr), capi.ptr(tc, C.c_int32),
        capi.ptr(gap, C.c_float)))
    return restored, tr.reshape(n, it), tc, gap.reshape(n, it)


def study(name, img, pat, out):
    wl = WL.ALL[name]
    img = img.astype(np.float64)
    r64, t64, c64, _ = diag(img, pat, wl.config("fp64"))
    r32, t32, c32, g32 = diag(img, pat, wl.config("fp32", guard_tau=0.0))
    n, it = t64.shape
    b = wl.block
    maxerr = np.zeros(n)
    sq64 = np.zeros(n)
    sq32 = np.zeros(n)
    for i, blk in enumerate(pat.blocks):
        a = r64[blk.row:blk.row + b, blk.col:blk.col + b]
        z = r32[blk.row:blk.row + b, blk.col:blk.col + b]
        o = img[blk.row:blk.row + b, blk.col:blk.col + b]
        maxerr[i] = np.abs(a - z).max()
        sq64[i] = ((a - o) ** 2).sum()
        sq32[i] = ((z - o) ** 2).sum()
    u64 = t64["u1"].astype(np.int32) * 1024 + t64["u2"]
    u32 = t32["u1"].astype(np.int32) * 1024 + t32["u2"]
    first_div = np.full(n, -1, np.int32)
    for i in range(n):
        m = min(c64[i], c32[i])
        d = np.nonzero(u64[i, :m] != u32[i, :m])[0]
        if len(d):
            first_div[i] = d[0]
        elif c64[i] != c32[i]:
            first_div[i] = m
    out[name] = dict(maxerr=maxerr, first_div=first_div, gap=g32, count64=c64, count32=c32,
                     e64=t64["weighted_energy"], sq64=sq64, sq32=sq32)
    print(f"{name}: {n} blocks, diverged {np.mean(first_div >= 0):.3%}, max px err {maxerr.max():.3f}, "
          f">0.5: {(maxerr > 0.5).sum()}", flush=True)


def main():
    out = {}
    t0 = time.time()
    img, pat = WL.C2.frame(seed=101)
    study("C2", img, pat, out)
    for f in range(6):  # C4 frames
        img, pat = WL.C4.frame(seed=303, f=f)
        study("C4", img, pat, tmp := {})
        for k, v in tmp["C4"].items():
            out.setdefault("C4", {}).setdefault(k, []).append(v)
    out["C4"] = {k: np.concatenate(v) for k, v in out["C4"].items()}
    img, pat = WL.C3.frame(seed=505)
    pat.blocks = pat.blocks[:8000]
    study("C3", img, pat, out)
    img, pat = WL.C5.frame(seed=707)
    pat.blocks = pat.blocks[:1200]
    study("C5", img, pat, out)
    flat = {f"{k}_{kk}": vv for k, v in out.items() for kk, vv in v.items()}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    np.savez_compressed(os.path.join(ROOT, "gpurun_out", "guard_study.npz"), **flat)
    print(f"done in {time.time() - t0:.1f} s")


if __name__ == "__main__":
    main()
