"""Any transform size (the reference accepts every T >= the window,
pipeline.cpp:128-131): T outside {8, 16, 32, 64, 128} runs the generic path
(csrc/kernels_generic.cu) in the reference's arithmetic — the FFT stand-in's
direct DFT for non-powers of two, radix-2 for 256 — and must select exactly
the compiled reference's basis sequence with bit-identical records."""
import numpy as np
import pytest

import paper_2207_01205_b200 as P
from helpers import random_grid

pytestmark = pytest.mark.gpu

ALGO = {"fse": 0, "ofse": 1, "fofse": 2}


@pytest.mark.parametrize("algo,t,blk,sup,its", [("fofse", 48, 16, 16, 40), ("fse", 40, 8, 12, 30),
                                               ("fofse", 96, 16, 16, 25), ("fofse", 256, 32, 16, 12),
                                               ("ofse", 36, 8, 8, 20)])
def test_generic_t_matches_reference(gpu, ref, algo, t, blk, sup, its):
    rng = np.random.default_rng(t + its)
    h, w = 4 * blk + 2 * sup + 16, 5 * blk + 2 * sup
    img = np.clip(np.round(120 + 70 * random_grid(rng, h, w)), 0, 255)
    blocks = [(0, 0, blk, blk), (sup + blk, sup + blk, blk, blk), (h - blk, w - blk, blk, blk)]
    pat = P.LossPattern(w, h, blk, blk, [P.Rect(*b) for b in blocks])
    cfg = P.ConcealConfig(algorithm=algo, gamma=0.5, iterations=its, transform_size=t, rho_hat=0.8,
                          support_width=sup, record_traces=True)
    out = P.conceal(img, pat, cfg)
    r = ref.conceal(img, blocks, blk, blk, algorithm=ALGO[algo], gamma=0.5, iterations=its, t=t, rho_hat=0.8,
                    support=sup, traces=True)
    fields = ("u1", "u2", "p_re", "p_im", "weighted_energy") if algo == "ofse" else \
        ("u1", "u2", "p_re", "p_im", "c_re", "c_im", "weighted_energy")
    for a, b in zip(out.report.traces, r["traces"]):
        assert len(a) == len(b)
        for k in fields if algo != "ofse" else ("u1", "u2"):
            np.testing.assert_array_equal(a[k], b[k], err_msg=k)
    assert np.abs(out.restored - r["restored"]).max() <= 1e-9
