"""Precision study (GPU box): fp64 'head' of N selections, then fp32, vs pure fp64.

Uses the engine-level C ABI (spectral init / iterate / synthesize), batched.
Reports per N: divergence rate vs fp64, pixel errors, and the fp32-phase gap
statistics that a near-tie guard would threshold."""
import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle  # noqa: E402  (window extraction for the study only)
from paper_2207_01205_b200 import _capi as capi  # noqa: E402
from paper_2207_01205_b200 import workloads as WL  # noqa: E402

L = capi.lib()
ctx = capi.context(0)


def windows(wl, img, pat):
    orc = oracle.Oracle()
    lost = np.zeros(img.shape, np.uint8)
    for b in pat.blocks:
        lost[b.row:b.row + b.height, b.col:b.col + b.width] = 1
    ws, ls = [], []
    for b in pat.blocks:
        w, l = orc.build_window(img.astype(np.float64), lost, tuple(b), wl.support)
        ws.append(w)
        ls.append(l)
    ws, ls = np.stack(ws), np.stack(ls)
    Lh = ws.shape[1]
    r = np.arange(Lh)[:, None] - (Lh - 1) / 2
    c = np.arange(Lh)[None, :] - (Lh - 1) / 2
    wf = wl.rho_hat ** np.hypot(r, c)
    wt = np.where(ls == 0, wf[None], 0.0)
    return ws, ls, wt


def init(t, ws, ls, wt):
    n, h, w = ws.shape
    rw = np.zeros((n, t, t), np.complex128)
    W = np.zeros((n, t, t), np.complex128)
    w0, e, m = np.zeros(n), np.zeros(n), np.zeros(n)
    capi.check(L.fofse_spectral_init(ctx.handle, capi.ptr(ws), capi.ptr(ls, C.c_uint8), capi.ptr(wt), C.c_int64(n), h, w, t,
                                     capi.ptr(rw.view(np.float64)), capi.ptr(W.view(np.float64)), capi.ptr(w0),
                                     capi.ptr(e), capi.ptr(m)))
    return dict(rw=rw, W=W, w0=w0, e=e, e0=e.copy(), m=m, g=np.zeros_like(rw), nu=np.zeros(n, np.int32),
                cv=np.zeros(n, np.int32))


def iterate(st, t, h, w, gamma, its, prec):
    n = st["rw"].shape[0]
    tr = np.zeros(n * max(its, 1), capi.RECORD_DTYPE)
    tc = np.zeros(n, np.int32)
    gap = np.zeros(n * max(its, 1), np.float32)
    capi.check(L.fofse_diag_spectral_iterate(
        ctx.handle, t, C.c_int64(n), h, w, capi.ptr(st["rw"].view(np.float64)), capi.ptr(st["W"].view(np.float64)),
        capi.ptr(st["g"].view(np.float64)), capi.ptr(st["w0"]), capi.ptr(st["e"]), capi.ptr(st["e0"]),
        capi.ptr(st["m"]), capi.ptr(st["nu"], C.c_int32), capi.ptr(st["cv"], C.c_int32), C.c_double(gamma), its,
        prec, capi.vptr(tr), capi.ptr(tc, C.c_int32), capi.ptr(gap, C.c_float)))
    return tr.reshape(n, max(its, 1)), tc, gap.reshape(n, max(its, 1))


def synth(st, t, h, w):
    n = st["g"].shape[0]
    out = np.zeros((n, h, w))
    mi = np.zeros(n)
    capi.check(L.fofse_spectral_synthesize(ctx.handle, t, C.c_int64(n), capi.ptr(st["g"].view(np.float64)), h, w,
                                           capi.ptr(out), capi.ptr(mi)))
    return out


def copy(st):
    return {k: v.copy() for k, v in st.items()}


def study(wl, img, pat, heads, res):
    ws, ls, wt = windows(wl, img, pat)
    n, h, w = ws.shape
    t, I = wl.transform_size, wl.iterations
    base = init(t, ws, ls, wt)
    ref = copy(base)
    tr_ref, tc_ref, _ = iterate(ref, t, h, w, wl.gamma, I, 0)
    model_ref = np.clip(synth(ref, t, h, w), 0, 255)
    hole = (ls == 1)
    u_ref = tr_ref["u1"].astype(np.int64) * 4096 + tr_ref["u2"]
    for N in heads:
        st = copy(base)
        if N:
            tr_h, tc_h, _ = iterate(st, t, h, w, wl.gamma, N, 0)
        tr_t, tc_t, gap = iterate(st, t, h, w, wl.gamma, I - N, 1)
        model = np.clip(synth(st, t, h, w), 0, 255)
        err = np.where(hole, np.abs(model - model_ref), 0).reshape(n, -1).max(1)
        u = tr_t["u1"].astype(np.int64) * 4096 + tr_t["u2"]
        div = np.full(n, -1)
        for i in range(n):
            m = max(0, min(tc_ref[i] - N, tc_t[i]))
            d = np.nonzero(u[i, :m] != u_ref[i, N:N + m])[0]
            div[i] = d[0] if len(d) else (-1 if tc_ref[i] - N == tc_t[i] else m)
        gmask = np.arange(I - N)[None, :] < tc_t[:, None]
        gmin = np.where(gmask, gap, 1.0).min(1)
        gdiv = np.array([gap[i, div[i]] if 0 <= div[i] < I - N else np.nan for i in range(n)])
        key = f"{wl.name}_N{N}"
        res.setdefault(key, {"err": [], "div": [], "gmin": [], "gdiv": []})
        for k, v in (("err", err), ("div", div), ("gmin", gmin), ("gdiv", gdiv)):
            res[key][k].append(v)


def main():
    heads = [0, 10, 25, 50, 100]
    res = {}
    t0 = time.time()
    img, pat = WL.C2.frame(seed=101)
    study(WL.C2, img, pat, heads, res)
    for f in range(4):
        img, pat = WL.C4.frame(seed=909, f=f)
        study(WL.C4, img, pat, heads, res)
    img, pat = WL.C5.frame(seed=707)
    pat.blocks = pat.blocks[:800]
    study(WL.C5, img, pat, [0, 25, 50, 100, 150], res)
    img, pat = WL.C3.frame(seed=505)
    pat.blocks = pat.blocks[:6000]
    study(WL.C3, img, pat, [0, 5, 10, 20], res)
    flat = {}
    for key, d in res.items():
        for k, v in d.items():
            flat[f"{key}_{k}"] = np.concatenate(v)
        err = flat[f"{key}_err"]
        div = flat[f"{key}_div"]
        print(f"{key}: n={len(err)} div={np.mean(div >= 0):.3%} >0.5px={np.sum(err > 0.5)} maxerr={err.max():.3f}", flush=True)
    np.savez_compressed(os.path.join(ROOT, "gpurun_out", "head_study.npz"), **flat)
    for k in range(4):
        print("microbench", k, capi.microbench(0, k))
    print(f"done {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
