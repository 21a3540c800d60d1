"""Race / synchronisation evidence without compute-sanitizer (closed on the GPU
pool): every kernel family runs the same inputs repeatedly — with the fp32
real path forced onto each of its two forms — and must reproduce its outputs
bit for bit. The kernels synchronise through named barriers, parity
double-buffered slots, mbarrier-completed bulk copies and warp shuffles; a
missing barrier or a slot reuse race shows up as run-to-run differences in
the selections or pixels (each case runs ~10^4-10^6 barrier phases)."""
import os

import numpy as np
import pytest

import paper_2207_01205_b200 as P
from paper_2207_01205_b200 import workloads as WL

pytestmark = pytest.mark.gpu


def _runs(img, pat, cfg, n=4):
    outs = [P.conceal(img, pat, cfg) for _ in range(n)]
    for o in outs[1:]:
        assert np.array_equal(o.restored, outs[0].restored)
        assert o.report.psnr_db == outs[0].report.psnr_db
        if cfg.record_traces:
            for a, b in zip(o.report.traces, outs[0].report.traces):
                assert np.array_equal(a, b)
    return outs[0]


@pytest.mark.parametrize("gw", ["1", "2"])
@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_c2_slice_is_deterministic(gpu, prec, gw, monkeypatch):
    monkeypatch.setenv("FOFSE_V2_REAL_GW", gw)  # K2v2r (one warp / block) or K2v2h (two)
    img, pat = WL.C2.frame(seed=5)
    sub = P.LossPattern(pat.image_width, pat.image_height, 16, 16, pat.blocks[::3])  # ~680, borders too
    _runs(img.astype(np.float64), sub, WL.C2.config(prec, record_traces=True))


def test_exact_path_is_deterministic(gpu):
    img, pat = WL.C2.frame(seed=6)
    sub = P.LossPattern(pat.image_width, pat.image_height, 16, 16, pat.blocks[:40])
    cfg = WL.C2.config("fp64", guard_tau=1.0, record_traces=True)
    cfg.iterations = 60
    o = _runs(img.astype(np.float64), sub, cfg, n=3)
    assert o.report.device["guard_reruns"] == 40


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_t128_is_deterministic(gpu, prec):
    img, pat = WL.C5.frame(seed=9)
    sub = P.LossPattern(pat.image_width, pat.image_height, 32, 32, pat.blocks[::12])  # ~270, borders too
    cfg = WL.C5.config(prec)
    cfg.iterations = 120
    _runs(img.astype(np.float64), sub, cfg, n=3)


def test_frames_api_is_deterministic(gpu):
    imgs, rects, offs = WL.C4.batch(31, frames=6)
    pats = [P.LossPattern(1920, 1088, 16, 16, [P.Rect(int(r["row"]), int(r["col"]), 16, 16)
                                                for r in rects[offs[f]:offs[f + 1]]]) for f in range(6)]
    cfg = WL.C4.config("fp32")
    ref = None
    for _ in range(3):
        out, sq, rep = P.conceal_frames(imgs, pats, cfg)
        if ref is None:
            ref = (out.copy(), sq.copy())
        assert np.array_equal(out, ref[0]) and np.array_equal(sq, ref[1])
