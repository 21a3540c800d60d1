"""K1p (persistent K1 with cp.async-staged windows, the u8 frames path at T = 64)
against K1f, the kernel it replaces: the spectra are bit-identical, so the
frames API's outputs (every restored byte, every block error) are too — in
fp64 and fp32, interior and border windows, misaligned rows (odd widths).

The parity evidence gathered through the f64 frames path (K1f<double>, e.g.
bench.py's `parity` block) therefore carries over to the u8 path the bench
times. FOFSE_K1P is read once per process, so each arm runs in a subprocess.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_2207_01205_b200 as P
from paper_2207_01205_b200 import workloads as WL
import dataclasses
wl = dataclasses.replace(WL.C4, width={w}, height={h}, loss_frac={lf})
frames, rects, offs = wl.batch(seed={seed}, frames={nf})
pats = []
for f in range({nf}):
    rr = rects[offs[f]:offs[f + 1]]
    pats.append(P.LossPattern(wl.width, wl.height, 16, 16, [P.Rect(int(r["row"]), int(r["col"]), 16, 16) for r in rr]))
out, sq, rep = P.conceal_frames(frames, pats, wl.config({prec!r}))
np.savez({path!r}, out=out, sq=sq)
"""


def _run(tmp_path, k1p, prec, w, h, seed, nf, lf=0.1):
    path = str(tmp_path / f"k1p{k1p}_{prec}_{w}.npz")
    code = _SCRIPT.format(root=ROOT, w=w, h=h, seed=seed, nf=nf, prec=prec, path=path, lf=lf)
    env = dict(os.environ, FOFSE_K1P=str(k1p))
    subprocess.run([sys.executable, "-c", code], env=env, check=True, timeout=600)
    d = np.load(path)
    return d["out"], d["sq"]


@pytest.mark.parametrize("prec,w,h,nf", [("fp64", 1920, 1088, 4), ("fp32", 1920, 1088, 4), ("fp64", 643, 389, 6),
                                         ("fp32", 1001, 517, 6)])
def test_k1p_matches_k1f_bitwise(tmp_path, prec, w, h, nf):
    a_out, a_sq = _run(tmp_path, 0, prec, w, h, 77, nf)
    b_out, b_sq = _run(tmp_path, 1, prec, w, h, 77, nf)
    np.testing.assert_array_equal(a_out, b_out)
    np.testing.assert_array_equal(a_sq, b_sq)


def test_k1p_small_frames_match_k1f(tmp_path):
    """Frames smaller than the window (57 x 45: every window clipped on two or more
    sides, misaligned rows), half the cells lost."""
    a_out, a_sq = _run(tmp_path, 0, "fp64", 57, 45, 5, 8, lf=0.5)
    b_out, b_sq = _run(tmp_path, 1, "fp64", 57, 45, 5, 8, lf=0.5)
    assert a_sq.size > 0
    np.testing.assert_array_equal(a_out, b_out)
    np.testing.assert_array_equal(a_sq, b_sq)
