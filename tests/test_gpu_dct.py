"""The DCT basis family on the GPU: ConcealConfig.basis =
dct2d runs the spatial engine (engine_spatial.cpp:254-381) in the reference's
operation order (csrc/kernels_dct.cu). Checked against the compiled reference:
every trace field bit for bit and the restored pixels, for the three
algorithms (max portion + gamma, min distance, min distance + full OD),
interior and border blocks, several transform sizes (any T, not only powers
of two)."""
import numpy as np
import pytest

import paper_2207_01205_b200 as P
from helpers import random_grid

pytestmark = pytest.mark.gpu

ALGO = {"fse": 0, "ofse": 1, "fofse": 2}


@pytest.mark.parametrize("algo,t,blk,sup,its", [("fofse", 32, 8, 8, 25), ("fse", 32, 8, 8, 20), ("ofse", 16, 4, 4, 15),
                                               ("fofse", 24, 8, 8, 20), ("fofse", 64, 16, 16, 6)])
def test_conceal_dct_bit_exact_vs_reference(gpu, ref, algo, t, blk, sup, its):
    rng = np.random.default_rng(t * 3 + its)
    h, w = 6 * blk + 2 * sup, 7 * blk + 2 * sup
    img = np.clip(np.round(110 + 70 * random_grid(rng, h, w)), 0, 255)
    blocks = [(0, 0, blk, blk), (sup + blk, sup + 2 * blk, blk, blk), (h - blk, w - blk, blk, blk)]
    pat = P.LossPattern(w, h, blk, blk, [P.Rect(*b) for b in blocks])
    cfg = P.ConcealConfig(algorithm=algo, gamma=0.5, iterations=its, transform_size=t, rho_hat=0.75,
                          support_width=sup, record_traces=True, basis="dct2d")
    out = P.conceal(img, pat, cfg)
    r = ref.conceal(img, blocks, blk, blk, algorithm=ALGO[algo], gamma=0.5, iterations=its, t=t, rho_hat=0.75,
                    support=sup, traces=True, basis=1)
    for a, b in zip(out.report.traces, r["traces"]):
        assert len(a) == len(b)
        for k in ("u1", "u2", "p_re", "p_im", "c_re", "c_im", "gamma_effective", "weighted_energy", "degenerate"):
            np.testing.assert_array_equal(a[k], b[k], err_msg=k)
    np.testing.assert_array_equal(out.restored, r["restored"])
    assert out.report.psnr_db == pytest.approx(r["psnr_db"], rel=1e-13)  # summation order of the MSE


def test_dct_window_level_and_frames(gpu, ref):
    """extrapolate_window with the DCT basis returns the window model; the u8
    frames API routes the DCT config through the same engine."""
    rng = np.random.default_rng(5)
    img = np.clip(np.round(100 + 60 * random_grid(rng, 40, 48)), 0, 255)
    blocks = [(16, 16, 8, 8)]
    pat = P.LossPattern(48, 40, 8, 8, [P.Rect(*b) for b in blocks])
    cfg = P.ConcealConfig(gamma=0.5, iterations=12, transform_size=32, rho_hat=0.8, support_width=8, basis="dct2d")
    r = ref.conceal(img, blocks, 8, 8, gamma=0.5, iterations=12, t=32, rho_hat=0.8, support=8, basis=1)
    win = img[8:32, 8:32].copy()
    mask = np.zeros((24, 24), np.uint8)
    mask[8:16, 8:16] = P.Region.missing
    run = P.extrapolate_window(win, mask, cfg)
    got = np.clip(run.model[8:16, 8:16], 0, 255)
    np.testing.assert_array_equal(got, r["restored"][16:24, 16:24])
    out, sq, rep = P.conceal_frames(img.astype(np.uint8)[None], [pat], cfg)
    # write_pgm rounding: std::round (half away from zero) of the clamped value
    np.testing.assert_array_equal(out[0], np.floor(np.clip(r["restored"], 0, 255) + 0.5).astype(np.uint8))
