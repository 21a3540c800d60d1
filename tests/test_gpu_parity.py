"""GPU parity tests: the CUDA path (through the C ABI) vs the oracle.

Bars (BASELINE.json north_star):
  * fp64: identical selected-basis sequence, pixels within 1e-9 absolute;
    the iteration kernel fed the oracle's own spectra is bit-exact.
  * fp32 fast mode: max |pixel error| <= 0.5, PSNR within 0.05 dB.
"""
import numpy as np
import pytest

import paper_2207_01205_b200 as P
from paper_2207_01205_b200 import workloads as WL
from helpers import MISSING, OUTSIDE, SUPPORT, block_mask, random_grid, random_mask, smooth_test_image

pytestmark = pytest.mark.gpu

FP64_PX_TOL = 1e-9
FP32_PX_TOL = 0.5
FP32_PSNR_TOL = 0.05


def _oracle_spectrum(orc, rng, t, h, w, masked=True):
    f = random_grid(rng, h, w) * 100.0
    m = random_mask(rng, h, w) if masked else np.zeros((h, w), np.uint8)
    wt = orc.build_isotropic_weight(m, 0.8)
    return orc.init_spectra(f, m, wt, t), f, m, wt


def _gpu_iterate(spec, gamma, iters, precision="fp64"):
    s = P.spectral.Spectrum(spec.t, spec.window_width, spec.window_height, spec.rw.copy(),
                            spec.w.copy(), spec.g.copy(), spec.w0, spec.weighted_energy,
                            spec.initial_energy, spec.initial_max, spec.nu, spec.converged)
    tr = P.spectral.fast_iterate(s, gamma, iters, precision)
    return s, tr


def _canonical(t):
    k1, k2 = np.meshgrid(np.arange(t), np.arange(t), indexing="ij")
    return (k1 * t + k2) <= (((t - k1) % t) * t + (t - k2) % t)


@pytest.mark.parametrize("t,h,w,gamma,iters", [
    (8, 6, 7, 0.2, 20), (16, 14, 13, 0.5, 40), (32, 24, 24, 0.5, 50),
    (64, 48, 48, 0.5, 200), (64, 40, 47, 0.2, 120), (128, 64, 64, 0.5, 60),
])
def test_iterate_bit_exact_vs_oracle(gpu, orc, t, h, w, gamma, iters):
    """K2 strict fp64 fed the oracle's init_spectra reproduces fast_iterate bit for bit
    (engine_spectral.cpp:51-144): u, p, c, energies, G and the canonical R_w."""
    rng = np.random.default_rng(1000 + t + h)
    spec, *_ = _oracle_spectrum(orc, rng, t, h, w)
    ref = spec.copy()
    rec_ref = orc.fast_iterate(ref, gamma, iters)
    got, rec = _gpu_iterate(spec, gamma, iters)
    assert len(rec) == len(rec_ref) > 0
    for k in ("u1", "u2", "p_re", "p_im", "c_re", "c_im", "weighted_energy"):
        np.testing.assert_array_equal(rec[k], rec_ref[k], err_msg=k)
    assert got.nu == ref.nu and got.converged == ref.converged
    assert got.weighted_energy == ref.weighted_energy
    np.testing.assert_array_equal(got.g, ref.g)
    can = _canonical(t)
    np.testing.assert_array_equal(got.rw[can], ref.rw[can])


@pytest.mark.parametrize("t,h,w,iters", [(8, 6, 7, 20), (32, 24, 24, 50), (64, 48, 48, 120), (64, 40, 47, 80),
                                          (128, 64, 64, 40)])
def test_iterate_full_od_vs_oracle(gpu, orc, t, h, w, iters):
    """OFSE (fast_iterate_full_od, engine_spectral.cpp:79-97): the strict kernel with
    the block-wide d = sum_l R_w[l] W[u-l] reduction gives the oracle's selections;
    gamma_eff / p / c / energies agree to rounding (the reduction order differs)."""
    rng = np.random.default_rng(2000 + t + h)
    spec, *_ = _oracle_spectrum(orc, rng, t, h, w)
    ref = spec.copy()
    rec_ref = orc.fast_iterate_full_od(ref, iters)
    got = P.spectral.Spectrum(spec.t, spec.window_width, spec.window_height, spec.rw.copy(), spec.w.copy(),
                              spec.g.copy(), spec.w0, spec.weighted_energy, spec.initial_energy,
                              spec.initial_max, spec.nu, spec.converged)
    rec = P.spectral.fast_iterate_full_od(got, iters)
    assert len(rec) == len(rec_ref) > 0
    for k in ("u1", "u2", "degenerate"):
        np.testing.assert_array_equal(rec[k], rec_ref[k], err_msg=k)
    for k in ("p_re", "p_im", "c_re", "c_im", "gamma_effective"):
        np.testing.assert_allclose(rec[k], rec_ref[k], rtol=1e-9, atol=1e-12 * np.abs(rec_ref["p_re"]).max(),
                                   err_msg=k)
    assert (rec["gamma_effective"] < 1.0).any()  # the compensation is active
    np.testing.assert_allclose(rec["weighted_energy"], rec_ref["weighted_energy"], rtol=1e-9,
                               atol=1e-9 * spec.initial_energy)
    assert np.abs(got.g - ref.g).max() <= 1e-9 * np.abs(ref.g).max()


def test_iterate_resumes_like_reference(gpu, orc):
    """fast_iterate runs at most `iterations` more selections (engine_spectral.hpp:41-43)."""
    rng = np.random.default_rng(7)
    spec, *_ = _oracle_spectrum(orc, rng, 64, 48, 48)
    ref = spec.copy()
    orc.fast_iterate(ref, 0.5, 90)
    s = P.spectral.Spectrum(64, spec.window_width, spec.window_height, spec.rw.copy(), spec.w.copy(),
                            spec.g.copy(), spec.w0, spec.weighted_energy, spec.initial_energy,
                            spec.initial_max)
    P.spectral.fast_iterate(s, 0.5, 40)
    P.spectral.fast_iterate(s, 0.5, 50)
    assert s.nu == 90
    np.testing.assert_array_equal(s.g, ref.g)
    assert s.weighted_energy == ref.weighted_energy


def test_zero_signal_converges_immediately(gpu, orc):
    """engine_spectral_test.cpp:298-308."""
    m = np.zeros((8, 8), np.uint8)
    wt = orc.build_isotropic_weight(m, 0.8)
    spec = orc.init_spectra(np.zeros((8, 8)), m, wt, 8)
    s, tr = _gpu_iterate(spec, 0.5, 10)
    assert s.converged and len(tr) == 0 and s.nu == 0


def test_constant_window_collapses_to_dc(gpu, orc):
    """engine_spectral_test.cpp:98-115: u=(0,0), p=c, model == c."""
    c = 4.0
    m = block_mask(6, 6, missing=[(2, 2, 2, 2)])
    wt = orc.build_isotropic_weight(m, 0.8)
    spec = orc.init_spectra(np.full((6, 6), c), m, wt, 8)
    s, tr = _gpu_iterate(spec, 1.0, 1)
    assert len(tr) == 1 and tr[0]["u1"] == 0 and tr[0]["u2"] == 0
    assert abs(complex(tr[0]["p_re"], tr[0]["p_im"]) - c) < 1e-9
    assert np.abs(s.rw).max() < 1e-9 * spec.initial_max
    model = P.spectral.synthesize_model(s)
    np.testing.assert_allclose(model, c, rtol=1e-9)


@pytest.mark.parametrize("t,h,w", [(8, 6, 7), (16, 16, 16), (64, 48, 48), (128, 64, 64), (32, 24, 17)])
def test_init_spectra_vs_oracle(gpu, orc, t, h, w):
    """K1 (batched real-input 2-D FFT, fp64) vs init_spectra (engine_spectral.cpp:148-183)."""
    rng = np.random.default_rng(t * 31 + w)
    f = random_grid(rng, h, w) * 50.0
    m = random_mask(rng, h, w)
    wt = orc.build_isotropic_weight(m, 0.8)
    ref = orc.init_spectra(f, m, wt, t)
    got = P.spectral.init_spectra(f, m, wt, t)
    scale = np.abs(ref.rw).max()
    assert np.abs(got.rw - ref.rw).max() <= 1e-13 * scale
    assert np.abs(got.w - ref.w).max() <= 1e-13 * np.abs(ref.w).max()
    assert got.w0 == pytest.approx(ref.w0, rel=1e-14)
    assert got.weighted_energy == pytest.approx(ref.weighted_energy, rel=1e-13)
    assert got.initial_max == pytest.approx(ref.initial_max, rel=1e-13)


def test_synthesize_vs_oracle(gpu, orc):
    rng = np.random.default_rng(5)
    spec, *_ = _oracle_spectrum(orc, rng, 64, 48, 48)
    orc.fast_iterate(spec, 0.5, 150)
    ref = orc.synthesize_model(spec)
    got = P.spectral.synthesize_model(P.spectral.Spectrum(64, 48, 48, spec.rw, spec.w, spec.g))
    assert np.abs(got - ref).max() <= 1e-10


def _oracle_conceal(orc, img, pat, cfg, traces=True):
    return orc.conceal(img.astype(np.float64), [tuple(b) for b in pat.blocks], pat.block_height,
                       pat.block_width, algorithm={"fse": 0, "ofse": 1, "fofse": 2}[cfg.algorithm],
                       gamma=cfg.gamma, iterations=cfg.iterations, t=cfg.transform_size,
                       rho_hat=cfg.rho_hat, support=cfg.support_width, traces=traces)


def _assert_same_selections(got_traces, ref_traces):
    assert len(got_traces) == len(ref_traces)
    for i, (a, b) in enumerate(zip(got_traces, ref_traces)):
        assert len(a) == len(b), f"block {i}: {len(a)} vs {len(b)} records"
        np.testing.assert_array_equal(a["u1"], b["u1"], err_msg=f"block {i}")
        np.testing.assert_array_equal(a["u2"], b["u2"], err_msg=f"block {i}")


def test_conceal_fp64_C1(gpu, orc):
    """BASELINE C1 (512x512, 10% isolated 16x16 losses, T=64, 100 it, fp64): same
    selected-basis sequence for every block and pixels within 1e-9."""
    img, pat = WL.C1.frame(seed=11)
    cfg = WL.C1.config(record_traces=True)
    out = P.conceal(img.astype(np.float64), pat, cfg)
    ref = _oracle_conceal(orc, img, pat, cfg)
    _assert_same_selections(out.report.traces, ref["traces"])
    assert np.abs(out.restored - ref["restored"]).max() <= FP64_PX_TOL
    assert out.report.psnr_db == pytest.approx(ref["psnr_db"], rel=1e-12)


def test_conceal_fp64_borders_and_neighbours(gpu, orc):
    """Border windows + lost neighbours inside windows (OUTSIDE labels,
    pipeline.cpp:95-110), rectangular blocks, the reference's grid pattern."""
    rng = np.random.default_rng(409)
    img = smooth_test_image(rng, 160)
    blocks = [(0, 0, 12, 16), (0, 24, 12, 16), (20, 10, 12, 16), (148, 144, 12, 16),
              (70, 70, 12, 16), (82, 90, 12, 16), (40, 140, 12, 16)]
    pat = P.LossPattern(160, 160, 12, 16, [P.Rect(*b) for b in blocks])
    cfg = P.ConcealConfig(gamma=0.3, iterations=80, transform_size=64, support_width=14,
                          record_traces=True)
    out = P.conceal(img, pat, cfg)
    ref = _oracle_conceal(orc, img, pat, cfg)
    _assert_same_selections(out.report.traces, ref["traces"])
    assert np.abs(out.restored - ref["restored"]).max() <= FP64_PX_TOL


def test_conceal_fp64_k2d_vs_oracle_C2_slice(gpu, orc):
    """K2d (fp64 rotated frame, symmetric masks) on 400 C2 blocks at 200
    iterations: the oracle's selected-basis sequence for every block, pixels
    within 1e-9."""
    img, pat = WL.C2.frame(seed=23)
    sub = P.LossPattern(pat.image_width, pat.image_height, 16, 16, pat.blocks[::5])
    cfg = WL.C2.config("fp64", record_traces=True)
    out = P.conceal(img.astype(np.float64), sub, cfg)
    ref = _oracle_conceal(orc, img, sub, cfg)
    _assert_same_selections(out.report.traces, ref["traces"])
    assert np.abs(out.restored - ref["restored"]).max() <= FP64_PX_TOL


def test_conceal_fp64_k2d_matches_strict_full_C2(gpu, monkeypatch):
    """All 2040 C2 blocks: K2d vs the strict (reference operation order) kernel —
    identical selections, pixels within 1e-9."""
    img, pat = WL.C2.frame(seed=24)
    cfg = WL.C2.config("fp64", record_traces=True)
    fast = P.conceal(img.astype(np.float64), pat, cfg)
    monkeypatch.setenv("FOFSE_F64_KERNEL", "strict")
    strict = P.conceal(img.astype(np.float64), pat, cfg)
    _assert_same_selections(fast.report.traces, strict.report.traces)
    assert np.abs(fast.restored - strict.restored).max() <= FP64_PX_TOL


def _c5_crop(seed, size, nblocks, border=True):
    wl = WL.C5
    img = P.gen_image_u8(seed, size, size)
    rects = P.gen_losses(seed, size // wl.block, size // wl.block, wl.loss_frac, wl.block, wl.block)
    blocks = [tuple(map(int, (r["row"], r["col"], r["height"], r["width"]))) for r in rects][:nblocks]
    if border:  # windows clipped by the image edge (asymmetric masks: the strict kernel at T = 128)
        extra = [(0, 0, 32, 32), (size - 32, 96, 32, 32)]
        near = lambda b, e: abs(b[0] - e[0]) < 64 and abs(b[1] - e[1]) < 64  # noqa: E731
        blocks = [b for b in blocks if not any(near(b, e) for e in extra)] + extra
    return img, P.LossPattern(size, size, wl.block, wl.block, [P.Rect(*b) for b in blocks])


def test_conceal_fp64_T128_vs_oracle(gpu, orc):
    """C5 blocks (32x32, T = 128, 300 iterations) in fp64: K2d at T = 128 (one
    fp64 V copy, 16 warps per block, 14-bit key index) for interior windows and
    the strict kernel for border windows give the oracle's selected-basis
    sequence for every block, pixels within 1e-9."""
    img, pat = _c5_crop(57, 768, 14)
    cfg = WL.C5.config("fp64", record_traces=True)
    out = P.conceal(img.astype(np.float64), pat, cfg)
    ref = _oracle_conceal(orc, img, pat, cfg)
    _assert_same_selections(out.report.traces, ref["traces"])
    assert np.abs(out.restored - ref["restored"]).max() <= FP64_PX_TOL


def test_conceal_fp64_T128_k2d_matches_strict(gpu, monkeypatch):
    """160 C5 blocks: K2d (T = 128) vs the strict kernel — identical selections,
    pixels within 1e-9."""
    img, pat = _c5_crop(58, 2048, 160, border=False)
    cfg = WL.C5.config("fp64", record_traces=True)
    fast = P.conceal(img.astype(np.float64), pat, cfg)
    monkeypatch.setenv("FOFSE_F64_KERNEL", "strict")
    strict = P.conceal(img.astype(np.float64), pat, cfg)
    _assert_same_selections(fast.report.traces, strict.report.traces)
    assert np.abs(fast.restored - strict.restored).max() <= FP64_PX_TOL


def _c5_border_crop(seed, size=1024):
    """32 x 32 blocks on all four image edges (asymmetric windows, 300 iterations)."""
    img = P.gen_image_u8(seed, size, size)
    blocks = set()
    for x in range(0, size - 31, 96):
        blocks |= {(0, x), (size - 32, x), (x, 0), (x, size - 32)}
    pat = P.LossPattern(size, size, 32, 32, [P.Rect(r, c, 32, 32) for r, c in sorted(blocks)])
    return img, pat


def test_conceal_fp64_T128_border_cluster_matches_strict(gpu, monkeypatch):
    """T = 128 asymmetric (border) windows run K2dcx — the 2-CTA cluster kernel with
    the W image split across the pair's shared memory (DSMEM gathers): identical
    selections to the strict kernel (reference op order), pixels within 1e-9."""
    img, pat = _c5_border_crop(61)
    cfg = WL.C5.config("fp64", record_traces=True)
    fast = P.conceal(img.astype(np.float64), pat, cfg)
    monkeypatch.setenv("FOFSE_F64_KERNEL", "strict")
    strict = P.conceal(img.astype(np.float64), pat, cfg)
    _assert_same_selections(fast.report.traces, strict.report.traces)
    assert np.abs(fast.restored - strict.restored).max() <= FP64_PX_TOL


def test_conceal_T128_border_cluster_vs_oracle_both_precisions(gpu, orc):
    """Border windows at T = 128 against the oracle: fp64 selections + 1e-9 px; the
    fp32 mode (borders run fp64 outright on K2dcx, interior fp32) within 0.5 px."""
    img, pat = _c5_border_crop(62, 512)
    pat = P.LossPattern(pat.image_width, pat.image_height, 32, 32, pat.blocks[:8])
    cfg = WL.C5.config("fp64", record_traces=True)
    cfg.iterations = 150
    out = P.conceal(img.astype(np.float64), pat, cfg)
    ref = _oracle_conceal(orc, img, pat, cfg)
    _assert_same_selections(out.report.traces, ref["traces"])
    assert np.abs(out.restored - ref["restored"]).max() <= FP64_PX_TOL
    cfg32 = WL.C5.config("fp32")
    cfg32.iterations = 150
    o32 = P.conceal(img.astype(np.float64), pat, cfg32)
    lost = np.zeros(img.shape, bool)
    for b in pat.blocks:
        lost[b.row:b.row + 32, b.col:b.col + 32] = True
    assert _fp32_vs_ref(o32.restored, ref["restored"], lost) <= FP32_PX_TOL


@pytest.mark.parametrize("name", ["C2", "C3", "C5"])
def test_k1_register_fft_matches_radix2(gpu, monkeypatch, name):
    """The register K1 (T = 64: radix-8x8; T = 32: radix-8 then two radix-4 per
    lane; T = 128: 16 lanes x 8, output-parity split second stage, canonical
    half written from the registers) vs the shared-memory radix-2 K1 (both
    fp64): identical selections on C2 / C3 / C5 blocks (borders included),
    pixels within 1e-9."""
    wl = WL.ALL[name]
    if name == "C5":
        img, pat = _c5_crop(61, 1024, 24)
    else:
        img, pat = wl.frame(seed=25)
    step = {"C2": 3, "C3": 40, "C5": 1}[name]
    sub = P.LossPattern(pat.image_width, pat.image_height, wl.block, wl.block, pat.blocks[::step])
    cfg = wl.config("fp64", record_traces=True)
    fast = P.conceal(img.astype(np.float64), sub, cfg)
    monkeypatch.setenv("FOFSE_K1", "slow")
    slow = P.conceal(img.astype(np.float64), sub, cfg)
    _assert_same_selections(fast.report.traces, slow.report.traces)
    assert np.abs(fast.restored - slow.restored).max() <= FP64_PX_TOL


@pytest.mark.parametrize("t,b,sw", [(8, 4, 2), (16, 8, 4), (32, 8, 8), (32, 16, 8)])
def test_conceal_fp64_small_transforms(gpu, orc, t, b, sw):
    """K2d at T = 8/16/32 (one warp per block, idle lanes for T < 32) vs the oracle."""
    rng = np.random.default_rng(449 + t + b)
    img = smooth_test_image(rng, 96)
    cells = [(r, c) for r in range(b, 96 - 2 * b, 3 * b) for c in range(b, 96 - 2 * b, 3 * b)]
    pat = P.LossPattern(96, 96, b, b, [P.Rect(r, c, b, b) for r, c in cells])
    cfg = P.ConcealConfig(gamma=0.5, iterations=40, transform_size=t, support_width=sw, record_traces=True)
    out = P.conceal(img, pat, cfg)
    ref = _oracle_conceal(orc, img, pat, cfg)
    _assert_same_selections(out.report.traces, ref["traces"])
    assert np.abs(out.restored - ref["restored"]).max() <= FP64_PX_TOL


@pytest.mark.parametrize("t,b,sw", [(8, 4, 2), (16, 8, 4), (32, 16, 8)])
def test_conceal_fp32_small_transforms(gpu, orc, t, b, sw):
    """fp32 fast mode at T = 8/16/32 (K2v2r with idle lanes for T < 32, the
    fp64 head, the guard) vs the fp64 oracle: <= 0.5 px, <= 0.05 dB."""
    rng = np.random.default_rng(503 + t + b)
    img = smooth_test_image(rng, 128)
    cells = [(r, c) for r in range(0, 128 - b + 1, 3 * b) for c in range(0, 128 - b + 1, 3 * b)]
    pat = P.LossPattern(128, 128, b, b, [P.Rect(r, c, b, b) for r, c in cells])
    cfg = P.ConcealConfig(gamma=0.5, iterations=60, transform_size=t, support_width=sw, precision="fp32")
    out = P.conceal(img, pat, cfg)
    ref = _oracle_conceal(orc, img, pat, P.ConcealConfig(gamma=0.5, iterations=60, transform_size=t,
                                                         support_width=sw), traces=False)
    lost = np.zeros(img.shape, bool)
    for r, c in cells:
        lost[r:r + b, c:c + b] = True
    assert _fp32_vs_ref(out.restored, ref["restored"], lost) <= FP32_PX_TOL
    assert abs(out.report.psnr_db - ref["psnr_db"]) <= FP32_PSNR_TOL


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("case", ["zero_iterations", "constant", "black", "white", "corners"])
def test_conceal_edge_cases_vs_oracle(gpu, orc, precision, case):
    """Edge inputs through the whole path in both precisions, against the oracle:
    I = 0 (empty model: the hole is 0 after the clamp), constant / black /
    saturated images (black: zero energy converges at once; constant: the
    selections approach the DC value), and lost blocks in all four corners
    (every border class)."""
    rng = np.random.default_rng(509)
    img = smooth_test_image(rng, 96)
    iters = 0 if case == "zero_iterations" else 40
    if case == "constant":
        img = np.full((96, 96), 137.0)
    elif case == "black":
        img = np.zeros((96, 96))
    elif case == "white":
        img = np.full((96, 96), 255.0)
    blocks = [(0, 0), (0, 80), (80, 0), (80, 80), (40, 40)] if case == "corners" else [(16, 16), (48, 64)]
    pat = P.LossPattern(96, 96, 16, 16, [P.Rect(r, c, 16, 16) for r, c in blocks])
    cfg = P.ConcealConfig(gamma=0.5, iterations=iters, precision=precision)
    out = P.conceal(img, pat, cfg)
    ref = _oracle_conceal(orc, img, pat, P.ConcealConfig(gamma=0.5, iterations=iters), traces=False)
    lost = np.zeros(img.shape, bool)
    for r, c in blocks:
        lost[r:r + 16, c:c + 16] = True
    tol = FP64_PX_TOL if precision == "fp64" else FP32_PX_TOL
    assert np.abs(out.restored - ref["restored"]).max() <= tol
    np.testing.assert_array_equal(out.restored[~lost], img[~lost])
    if case == "black":  # zero residual energy: converged before the first selection
        assert not out.restored[lost].any()
    elif case in ("constant", "white"):  # the DC-led selections approach the constant
        np.testing.assert_allclose(out.restored[lost], img[lost], atol=1e-3)


def test_conceal_ofse_vs_oracle(gpu, orc):
    """pipeline ofse (fast_iterate_full_od per window, pipeline.cpp:194-196): K2d with
    the rotated-frame d reduction (interior masks) and the strict kernel (border and
    neighbour masks) give the oracle's selections; pixels within 1e-9."""
    rng = np.random.default_rng(457)
    img = smooth_test_image(rng, 160)
    blocks = [(0, 0, 16, 16), (0, 48, 16, 16), (48, 48, 16, 16), (48, 80, 16, 16), (96, 16, 16, 16),
              (112, 128, 16, 16), (144, 144, 16, 16)]
    pat = P.LossPattern(160, 160, 16, 16, [P.Rect(*b) for b in blocks])
    cfg = P.ConcealConfig(algorithm="ofse", iterations=60, transform_size=64, support_width=16,
                          record_traces=True)
    out = P.conceal(img, pat, cfg)
    ref = _oracle_conceal(orc, img, pat, cfg)
    _assert_same_selections(out.report.traces, ref["traces"])
    assert np.abs(out.restored - ref["restored"]).max() <= FP64_PX_TOL
    # an fp32 request runs the same fp64 OFSE kernels
    out32 = P.conceal(img, pat, P.ConcealConfig(algorithm="ofse", iterations=60, transform_size=64,
                                                support_width=16, precision="fp32"))
    np.testing.assert_array_equal(out32.restored, out.restored)


def test_conceal_ofse_C1(gpu, orc):
    """BASELINE C1 frame with algorithm = ofse (100 iterations): oracle selections, pixels <= 1e-9."""
    img, pat = WL.C1.frame(seed=12)
    cfg = WL.C1.config(record_traces=True)
    cfg.algorithm = "ofse"
    out = P.conceal(img.astype(np.float64), pat, cfg)
    ref = _oracle_conceal(orc, img, pat, cfg)
    _assert_same_selections(out.report.traces, ref["traces"])
    assert np.abs(out.restored - ref["restored"]).max() <= FP64_PX_TOL


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_conceal_ofse_T128_borders_vs_oracle(gpu, orc, precision):
    """OFSE at T = 128 with border (asymmetric) windows: the strict kernel serves
    them (the cluster kernel has no full-OD reduction) — oracle selections,
    pixels <= 1e-9; an fp32 request runs the same fp64 OFSE kernels."""
    rng = np.random.default_rng(557)
    img = smooth_test_image(rng, 256)
    blocks = [(0, 0, 32, 32), (96, 64, 32, 32), (224, 128, 32, 32), (128, 224, 32, 32)]
    pat = P.LossPattern(256, 256, 32, 32, [P.Rect(*b) for b in blocks])
    cfg = P.ConcealConfig(algorithm="ofse", gamma=0.5, iterations=40, transform_size=128, rho_hat=0.85,
                          support_width=16, record_traces=True, precision=precision)
    out = P.conceal(img, pat, cfg)
    ref = _oracle_conceal(orc, img, pat, cfg)
    _assert_same_selections(out.report.traces, ref["traces"])
    assert np.abs(out.restored - ref["restored"]).max() <= FP64_PX_TOL


def test_psnr_curves_vs_oracle(gpu, orc):
    """psnr_vs_iterations (pipeline.cpp:264-369): checkpointed PSNR after every
    `stride` selections for a gamma sweep + fse + ofse equals, point by point, the
    PSNR of a plain conceal run with that many iterations (oracle)."""
    rng = np.random.default_rng(461)
    img = smooth_test_image(rng, 128)
    blocks = [(16, 16, 16, 16), (16, 80, 16, 16), (64, 48, 16, 16), (96, 96, 16, 16), (0, 112, 16, 16)]
    pat = P.LossPattern(128, 128, 16, 16, [P.Rect(*b) for b in blocks])
    algos = [P.ConcealConfig(gamma=g) for g in (0.2, 0.5, 1.0)] + [P.ConcealConfig(algorithm="fse"),
                                                                   P.ConcealConfig(algorithm="ofse")]
    curves = P.psnr_vs_iterations(img, pat, algos, max_iterations=45, stride=15)
    assert [c.label for c in curves] == ["fofse_g0.2", "fofse_g0.5", "fofse_g1", "fse", "ofse"]
    for cfg, cur in zip(algos, curves):
        assert [it for it, _ in cur.points] == [15, 30, 45]
        for it, db in cur.points:
            c2 = P.ConcealConfig(algorithm=cfg.algorithm, gamma=cfg.gamma, iterations=it)
            ref = _oracle_conceal(orc, img, pat, c2, traces=False)
            assert db == pytest.approx(ref["psnr_db"], rel=1e-9), (cur.label, it)
    assert P.psnr_vs_iterations(img, pat, algos[:1], max_iterations=5, stride=10)[0].points == []


def test_conceal_empty_pattern_is_identity(gpu):
    """pipeline_test.cpp:171-183."""
    img = smooth_test_image(np.random.default_rng(421), 64)
    out = P.conceal(img, P.LossPattern(64, 64, 16, 16, []), P.ConcealConfig(algorithm="fse"))
    np.testing.assert_array_equal(out.restored, img)
    assert out.report.psnr_identical


def test_conceal_rewrites_only_missing_samples(gpu):
    """pipeline_test.cpp:140-169."""
    img = smooth_test_image(np.random.default_rng(419), 96)
    pat = P.LossPattern(96, 96, 16, 16, [P.Rect(16, 16, 16, 16), P.Rect(16, 64, 16, 16),
                                         P.Rect(64, 16, 16, 16), P.Rect(64, 64, 16, 16)])
    out = P.conceal(img, pat, P.ConcealConfig(iterations=5))
    lost = np.zeros_like(img, bool)
    for b in pat.blocks:
        lost[b.row:b.row + 16, b.col:b.col + 16] = True
    np.testing.assert_array_equal(out.restored[~lost], img[~lost])
    assert (out.restored[lost] >= 0).all() and (out.restored[lost] <= 255).all()
    assert (out.restored[lost] != img[lost]).any()


@pytest.mark.parametrize("algo,gamma", [("fse", 0.0), ("fofse", 1.0), ("fofse", 0.2)])
def test_conceal_fp64_algorithms(gpu, orc, algo, gamma):
    rng = np.random.default_rng(433)
    img = smooth_test_image(rng, 96)
    pat = P.LossPattern(96, 96, 16, 16, [P.Rect(16, 16, 16, 16), P.Rect(64, 64, 16, 16)])
    cfg = P.ConcealConfig(algorithm=algo, gamma=gamma, iterations=30, record_traces=True)
    out = P.conceal(img, pat, cfg)
    ref = _oracle_conceal(orc, img, pat, cfg)
    _assert_same_selections(out.report.traces, ref["traces"])
    assert np.abs(out.restored - ref["restored"]).max() <= FP64_PX_TOL


def _fp32_vs_ref(got_img, ref_img, lost):
    err = np.abs(got_img[lost].astype(np.float64) - ref_img[lost])
    return err.max()


def test_conceal_fp32_C2_vs_oracle(gpu, orc):
    """BASELINE C2 fp32 fast mode vs the fp64 oracle on a 400-block slice:
    max pixel error <= 0.5, PSNR within 0.05 dB."""
    img, pat = WL.C2.frame(seed=21)
    sub = P.LossPattern(pat.image_width, pat.image_height, 16, 16, pat.blocks[::5])
    cfg32 = WL.C2.config("fp32")
    out = P.conceal(img.astype(np.float64), sub, cfg32)
    ref = _oracle_conceal(orc, img, sub, WL.C2.config("fp64"), traces=False)
    lost = np.zeros(img.shape, bool)
    for b in sub.blocks:
        lost[b.row:b.row + 16, b.col:b.col + 16] = True
    assert _fp32_vs_ref(out.restored, ref["restored"], lost) <= FP32_PX_TOL
    assert abs(out.report.psnr_db - ref["psnr_db"]) <= FP32_PSNR_TOL


def test_conceal_fp32_vs_fp64_full_C2(gpu):
    """All 2040 blocks of C2: GPU fp32 vs GPU fp64 (the fp64 path is pinned to the
    oracle above)."""
    img, pat = WL.C2.frame(seed=22)
    o64 = P.conceal(img.astype(np.float64), pat, WL.C2.config("fp64"))
    o32 = P.conceal(img.astype(np.float64), pat, WL.C2.config("fp32"))
    lost = np.zeros(img.shape, bool)
    for b in pat.blocks:
        lost[b.row:b.row + 16, b.col:b.col + 16] = True
    assert np.abs(o32.restored[lost] - o64.restored[lost]).max() <= FP32_PX_TOL
    assert abs(o32.report.psnr_db - o64.report.psnr_db) <= FP32_PSNR_TOL


def test_fp32_default_on_c4_frames_vs_fp64(gpu):
    """The shipped fp32 default (fp64 head, guard tau) on 48 whole C4 frames
    (39,168 blocks) against the fp64 path: no block above 0.5 px, |dPSNR| of the
    concealed blocks <= 0.05 dB (north_star fp32 bar; bench.py reports the same
    check over all 256 frames of the timed batch)."""
    import dataclasses

    from paper_2207_01205_b200 import parity
    r = parity.fp32_vs_fp64(dataclasses.replace(WL.C4, frames=48), seed=4242)
    assert r["blocks"] == 48 * 816
    assert r["blocks_over_0.5"] == 0 and r["max_px"] <= FP32_PX_TOL, r
    assert r["dpsnr_db"] <= FP32_PSNR_TOL and r["max_frame_dpsnr_db"] <= FP32_PSNR_TOL, r


def test_fp32_head_exact_ties_follow_the_reference(gpu):
    """C3 seed 300 (T = 32, 52,429 blocks of one 4096^2 image) holds exact
    argmax ties inside the fp64 head (windows over saturated content): the
    head's near-tie guard sends those blocks to the exact path, as the fp64
    mode does, so no block ends far from the fp64 path (without it: block 212
    of frame 0 at 0.63 px)."""
    import dataclasses

    from paper_2207_01205_b200 import parity
    r = parity.fp32_vs_fp64(dataclasses.replace(WL.C3, frames=1), seed=300, per_call=1)
    assert r["blocks"] == 52429
    assert r["blocks_over_0.5"] == 0 and r["max_px"] <= 0.01, r
    assert r["dpsnr_db"] <= FP32_PSNR_TOL, r


def test_fp32_default_on_c5_vs_fp64(gpu):
    """T = 128 (C5, 3,277 blocks of one 8192^2 image, 300 iterations) at the shipped
    fp32 default against the fp64 path."""
    import dataclasses

    from paper_2207_01205_b200 import parity
    r = parity.fp32_vs_fp64(dataclasses.replace(WL.C5, frames=2), seed=777)
    assert r["blocks_over_0.5"] == 0 and r["max_px"] <= FP32_PX_TOL, r
    assert r["dpsnr_db"] <= FP32_PSNR_TOL, r


def test_extrapolate_windows_vs_oracle(gpu, orc):
    """Window level (pipeline.cpp:181-203) with arbitrary per-window masks."""
    rng = np.random.default_rng(99)
    n, h, w = 6, 40, 44
    wins = np.stack([random_grid(rng, h, w) * 80 + 100 for _ in range(n)])
    masks = np.stack([random_mask(rng, h, w, 0.3) for _ in range(n)])
    cfg = P.ConcealConfig(gamma=0.4, iterations=60, transform_size=64, rho_hat=0.75)
    runs = P.extrapolate_windows(wins, masks, cfg)
    for i in range(n):
        wt = orc.build_isotropic_weight(masks[i], cfg.rho_hat)
        s = orc.init_spectra(wins[i], masks[i], wt, 64)
        rec = orc.fast_iterate(s, cfg.gamma, cfg.iterations)
        model = orc.synthesize_model(s)
        np.testing.assert_array_equal(runs[i].trace["u1"], rec["u1"])
        np.testing.assert_array_equal(runs[i].trace["u2"], rec["u2"])
        assert np.abs(runs[i].model - model).max() <= 1e-9


@pytest.mark.parametrize("name", ["C3", "C5"])
def test_small_and_large_blocks_fp32(gpu, orc, name):
    """C3 (8x8, T=32, 50 it) and C5 (32x32, T=128, 300 it) on a cropped image."""
    wl = WL.ALL[name]
    size = 512 if name == "C3" else 1024
    img = P.gen_image_u8(31, size, size)
    rects = P.gen_losses(31, size // wl.block, size // wl.block, wl.loss_frac, wl.block, wl.block)
    rects = rects[: 120 if name == "C3" else 40]
    pat = P.LossPattern(size, size, wl.block, wl.block,
                        [P.Rect(*map(int, (r["row"], r["col"], r["height"], r["width"]))) for r in rects])
    out = P.conceal(img.astype(np.float64), pat, wl.config("fp32"))
    ref = _oracle_conceal(orc, img, pat, wl.config("fp64"), traces=False)
    lost = np.zeros(img.shape, bool)
    for b in pat.blocks:
        lost[b.row:b.row + wl.block, b.col:b.col + wl.block] = True
    assert _fp32_vs_ref(out.restored, ref["restored"], lost) <= FP32_PX_TOL
    assert abs(out.report.psnr_db - ref["psnr_db"]) <= FP32_PSNR_TOL
    o64 = P.conceal(img.astype(np.float64), pat, wl.config("fp64"))
    assert np.abs(o64.restored - ref["restored"]).max() <= FP64_PX_TOL


@pytest.mark.parametrize("name", ["C2", "C5"])
def test_guard_resume_matches_rerun_from_scratch(gpu, monkeypatch, name):
    """fp32 mode: near-tie blocks resumed at the flagged selection (k2d_replay
    rebuilds the fp64 state from the K1 spectrum and the recorded selections,
    K2d continues) give the pixels of re-running them from scratch in fp64 —
    the selections made before the near-tie are the fp64 path's own — within
    fp64 rounding, and within the fp32 bar of the fp64 path."""
    wl = WL.ALL[name]
    if name == "C2":
        img, pat = wl.frame(seed=27)
    else:
        size = 1024
        img = P.gen_image_u8(33, size, size)
        rects = P.gen_losses(33, size // wl.block, size // wl.block, wl.loss_frac, wl.block, wl.block)
        pat = P.LossPattern(size, size, wl.block, wl.block,
                            [P.Rect(*map(int, (r["row"], r["col"], r["height"], r["width"]))) for r in rects])
    cfg = wl.config("fp32")
    default = P.conceal(img.astype(np.float64), pat, cfg)  # K2v2r chunks: exact tie resolution (K2v2x)
    assert default.report.device["guard_reruns"] > 0
    monkeypatch.setenv("FOFSE_ETR", "0")
    resumed = P.conceal(img.astype(np.float64), pat, cfg)
    monkeypatch.setenv("FOFSE_RESUME", "0")
    scratch = P.conceal(img.astype(np.float64), pat, cfg)
    assert resumed.report.device["guard_reruns"] == scratch.report.device["guard_reruns"] == \
        default.report.device["guard_reruns"]
    assert np.abs(resumed.restored - scratch.restored).max() <= 1e-6
    # the exact resolution goes on in fp32 after each tie: within fp32 noise of the
    # fp64 re-run, not bit-identical
    assert np.abs(default.restored - scratch.restored).max() <= 0.02
    o64 = P.conceal(img.astype(np.float64), pat, wl.config("fp64"))
    lost = np.zeros(img.shape, bool)
    for b in pat.blocks:
        lost[b.row:b.row + wl.block, b.col:b.col + wl.block] = True
    for out in (default, resumed):
        assert _fp32_vs_ref(out.restored, o64.restored, lost) <= FP32_PX_TOL
        assert abs(out.report.psnr_db - o64.report.psnr_db) <= FP32_PSNR_TOL


def test_fp32_traces_are_complete_with_guard_reruns(gpu):
    """fp32 mode with record_traces: near-tie blocks re-run on a path that records
    every selection (the exact-resolution continuation records none, so traces
    route those blocks to the fp64 re-run): each block's trace is 1..nu without
    gaps, selections on the canonical half."""
    img, pat = WL.C2.frame(seed=29)
    cfg = WL.C2.config("fp32", record_traces=True)
    out = P.conceal(img.astype(np.float64), pat, cfg)
    assert out.report.device["guard_reruns"] > 0
    for tr in out.report.traces:
        assert len(tr) >= 1
        np.testing.assert_array_equal(tr["nu"], np.arange(1, len(tr) + 1))
        assert (tr["u1"] >= 0).all() and (tr["u1"] <= 32).all() and (tr["u2"] >= 0).all() and (tr["u2"] < 64).all()


@pytest.mark.parametrize("iters", [24, 400])
def test_fp32_batch_parity_short_and_long_runs(gpu, iters):
    """The batch path (K2v2r, head, guard, exact near-tie resolution) at a short
    run (the head is a third of it) and a long one (records / exact coefficients
    sized by the iteration count): within the fp32 bar of the fp64 path."""
    from paper_2207_01205_b200 import parity as PAR
    import dataclasses
    wl = dataclasses.replace(WL.C4, frames=24, iterations=iters)
    r = PAR.fp32_vs_fp64(wl, 933, per_call=24)
    assert r["blocks_over_0.5"] == 0 and r["dpsnr_db"] <= FP32_PSNR_TOL


def test_device_planned_guard_matches_host_planned(gpu, monkeypatch):
    """C2 (one chunk): the re-runs planned on the device (guard plan kernel,
    device-sized launches) equal the host-planned ones bit for bit."""
    img, pat = WL.C2.frame(seed=31)
    cfg = WL.C2.config("fp32")
    dev = P.conceal(img.astype(np.float64), pat, cfg)
    monkeypatch.setenv("FOFSE_DEVICE_GUARD", "0")
    host = P.conceal(img.astype(np.float64), pat, cfg)
    assert dev.report.device["guard_reruns"] == host.report.device["guard_reruns"] > 0
    np.testing.assert_array_equal(dev.restored, host.restored)


def test_frames_u8_matches_f64_and_is_deterministic(gpu):
    """Video entry point: u8 frames give write_pgm-rounded results of the f64 path;
    repeated runs and frame-order changes are bitwise identical."""
    wl = WL.C4
    frames, rects, offs = wl.batch(seed=40, frames=3)
    pats = []
    for f in range(3):
        rr = rects[offs[f]:offs[f + 1]]
        pats.append(P.LossPattern(wl.width, wl.height, 16, 16,
                                  [P.Rect(*map(int, (r["row"], r["col"], 16, 16))) for r in rr]))
    cfg = wl.config("fp32")
    a, sq_a, rep = P.conceal_frames(frames, pats, cfg)
    b, sq_b, _ = P.conceal_frames(frames, pats, cfg)
    np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(sq_a, sq_b)
    # reversed frame order -> same per-frame results
    c, _, _ = P.conceal_frames(frames[::-1].copy(), pats[::-1], cfg)
    np.testing.assert_array_equal(c[::-1], a)
    # f64 path on frame 1, rounded like write_pgm
    o = P.conceal(frames[1].astype(np.float64), pats[1], cfg)
    np.testing.assert_array_equal(np.clip(np.floor(o.restored + 0.5), 0, 255).astype(np.uint8), a[1])
    assert rep.device["blocks"] == offs[-1]


@pytest.mark.parametrize("nframes", [40, 130])
def test_frame_groups_match_single_frames(gpu, nframes):
    """The pipelined frames API with frame groups (40 frames: 2 groups; 130: 4
    groups, first/last a quarter of the others; lazily queued uploads, per-group
    downloads, two-copy border kernel) gives, frame by frame, the bytes (and the
    block errors to rounding) of concealing each frame on its own."""
    rng = np.random.default_rng(487)
    H = W = 160
    frames = np.stack([np.clip(smooth_test_image(rng, H) + 0.0, 0, 255).astype(np.uint8) for _ in range(nframes)])
    pats = []
    for f in range(nframes):
        rr = P.gen_losses(500 + f, W // 16, H // 16, 0.12, 16, 16)
        pats.append(P.LossPattern(W, H, 16, 16, [P.Rect(*map(int, (r["row"], r["col"], 16, 16))) for r in rr]))
    cfg = WL.C4.config("fp32")
    out, sq, rep = P.conceal_frames(frames, pats, cfg)
    k = 0
    for f in range(0, nframes, 7):
        one, sq1, _ = P.conceal_frames(frames[f:f + 1], pats[f:f + 1], cfg)
        np.testing.assert_array_equal(one[0], out[f])
        n0 = sum(len(p.blocks) for p in pats[:f])
        # per-block squared errors: fp64 sums whose reduction order follows the
        # kernel form chosen for the job (e.g. the tail's WIDE re-runs)
        np.testing.assert_allclose(sq1, sq[n0:n0 + len(pats[f].blocks)], rtol=1e-12)
        k += 1
    assert k > 3 and rep.device["blocks"] == sum(len(p.blocks) for p in pats)


@pytest.mark.parametrize("nframes", [40, 130])
def test_fp64_frame_groups_match_single_frames(gpu, nframes):
    """fp64 mode through the frames API: each group's K1 waits for its own upload
    and its download follows its last iteration launch (the copies overlap the
    kernels). Frame by frame, the bytes of concealing each frame on its own."""
    rng = np.random.default_rng(587)
    H = W = 128
    frames = np.stack([np.clip(smooth_test_image(rng, H) + 0.0, 0, 255).astype(np.uint8) for _ in range(nframes)])
    pats = []
    for f in range(nframes):
        rr = P.gen_losses(800 + f, W // 16, H // 16, 0.12, 16, 16)
        pats.append(P.LossPattern(W, H, 16, 16, [P.Rect(*map(int, (r["row"], r["col"], 16, 16))) for r in rr]))
    cfg = WL.C4.config("fp64")
    out, sq, rep = P.conceal_frames(frames, pats, cfg)
    for f in range(0, nframes, 9):
        one, sq1, _ = P.conceal_frames(frames[f:f + 1], pats[f:f + 1], cfg)
        np.testing.assert_array_equal(one[0], out[f])
        n0 = sum(len(p.blocks) for p in pats[:f])
        np.testing.assert_allclose(sq1, sq[n0:n0 + len(pats[f].blocks)], rtol=1e-12)
    assert rep.device["blocks"] == sum(len(p.blocks) for p in pats)


@pytest.mark.parametrize("tau", [None, 1.0])
def test_fp64_frame_groups_patch_exact_reruns(gpu, tau):
    """Near-tie blocks skip the fast kernel's write-back and are re-run on the
    exact path after their group was downloaded: the frames API copies their
    blocks again. Transpose-symmetric frames (exact ties on the diagonal) and
    guard_tau = 1 (every block re-run): the bytes of one frame at a time."""
    n = 36
    frames, pats = [], []
    for f in range(n):
        a = np.random.default_rng(f).normal(0.0, 12.0, (128, 128))
        x = np.arange(128)
        base = 110 + 40 * np.cos(2 * np.pi * x / 37.0)[:, None] * np.cos(2 * np.pi * x / 37.0)[None, :]
        frames.append(np.clip(np.round(base + a + a.T), 0, 255).astype(np.uint8))
        rr = [(r, r, 16, 16) for r in (16, 48, 80)] + [(16, 80, 16, 16), (96, 32, 16, 16)]
        pats.append(P.LossPattern(128, 128, 16, 16, [P.Rect(*b) for b in rr]))
    frames = np.stack(frames)
    kw = {} if tau is None else {"guard_tau": tau}
    cfg = P.ConcealConfig(gamma=0.5, iterations=80, transform_size=64, rho_hat=0.8, support_width=16, **kw)
    out, sq, rep = P.conceal_frames(frames, pats, cfg)
    assert rep.device["guard_reruns"] > 0 if tau is None else rep.device["guard_reruns"] == 5 * n
    for f in range(0, n, 5):
        one, sq1, _ = P.conceal_frames(frames[f:f + 1], pats[f:f + 1], cfg)
        np.testing.assert_array_equal(one[0], out[f])
        np.testing.assert_allclose(sq1, sq[5 * f:5 * f + 5], rtol=1e-12)


def test_frames_f64_is_the_u8_pipeline_unrounded(gpu):
    """fofse_conceal_frames_f64 runs the u8 frames pipeline (plan, chunks, K2v2r,
    guard, exact near-tie resolution) with unrounded pixels out: rounded like
    write_pgm it gives the u8 call's bytes; the block errors agree."""
    wl = WL.C4
    frames, rects, offs = wl.batch(seed=77, frames=40)
    pats = []
    for f in range(40):
        rr = rects[offs[f]:offs[f + 1]]
        pats.append(P.LossPattern(wl.width, wl.height, 16, 16,
                                  [P.Rect(*map(int, (r["row"], r["col"], 16, 16))) for r in rr]))
    cfg = wl.config("fp32")
    u8, sq8, rep8 = P.conceal_frames(frames, pats, cfg)
    f64, sq64, rep64 = P.conceal_frames(frames.astype(np.float64), pats, cfg)
    np.testing.assert_array_equal(np.clip(np.floor(f64 + 0.5), 0, 255).astype(np.uint8), u8)
    np.testing.assert_allclose(sq64, sq8, rtol=1e-12)
    assert rep64.device["guard_reruns"] == rep8.device["guard_reruns"] > 0


def test_fp32_batch_path_parity_vs_fp64(gpu):
    """The batch path the bench times (40 C4 frames: K2v2r chunks, fp64 head,
    guard, near-tie blocks decided exactly and continued in fp32) vs the fp64
    path on the same batch: every block within 0.5 px, PSNR within 0.05 dB."""
    from paper_2207_01205_b200 import parity as PAR
    import dataclasses
    r = PAR.fp32_vs_fp64(dataclasses.replace(WL.C4, frames=40), 901, per_call=40)
    assert r["blocks"] > 30000 and r["guard_reruns"] > 0
    assert r["blocks_over_0.5"] == 0 and r["max_px"] <= FP32_PX_TOL
    assert r["dpsnr_db"] <= FP32_PSNR_TOL


def test_fused_k1_head_matches_two_kernels(gpu, monkeypatch):
    """K1H (FOFSE_K1H=1: spectra + fp64 head in one kernel, the fp32 hand-off
    straight from the SM; near-tie blocks recompute K1 for the exact
    resolution) against K1f + the K2d head: the same selections up to fp64
    rounding — pixels within fp32 noise — and both within the fp32 bar of
    the fp64 path."""
    from paper_2207_01205_b200 import parity as PAR
    import dataclasses
    wl = dataclasses.replace(WL.C4, frames=32)
    base = PAR.fp32_vs_fp64(wl, 913, per_call=32)
    monkeypatch.setenv("FOFSE_K1H", "1")
    fused = PAR.fp32_vs_fp64(wl, 913, per_call=32)
    for r in (base, fused):
        assert r["blocks_over_0.5"] == 0 and r["dpsnr_db"] <= FP32_PSNR_TOL
    assert abs(fused["guard_reruns"] - base["guard_reruns"]) <= max(3, base["guard_reruns"] // 50)
    assert abs(fused["psnr_fp32_db"] - base["psnr_fp32_db"]) <= 1e-4


@pytest.mark.parametrize("nframes,groups", [(1, 3), (1, 8), (3, 5)])
def test_row_groups_match_one_group(gpu, monkeypatch, nframes, groups):
    """Fewer than 16 frames: the frames' rows are cut into bands (first/last a
    quarter of the others; band uploads overlap iteration, each row range comes
    back once no later band's block writes into it). Forced band counts
    (FOFSE_ROW_GROUPS) give the bytes of one group, including bands without
    losses (the bottom quarter of frame 0 is loss-free)."""
    rng = np.random.default_rng(497 + nframes)
    H, W = 512, 384
    frames = np.stack([np.clip(smooth_test_image(rng, H)[:, :W] + 0.0, 0, 255).astype(np.uint8)
                       for _ in range(nframes)])
    pats = []
    for f in range(nframes):
        rr = P.gen_losses(900 + f, W // 16, H // 16, 0.15, 16, 16)
        rects = [P.Rect(*map(int, (r["row"], r["col"], 16, 16))) for r in rr]
        if f == 0:
            rects = [r for r in rects if r.row < 3 * H // 4]
        pats.append(P.LossPattern(W, H, 16, 16, rects))
    cfg = WL.C4.config("fp32")
    monkeypatch.setenv("FOFSE_ROW_GROUPS", "1")
    one, sq1, rep1 = P.conceal_frames(frames, pats, cfg)
    monkeypatch.setenv("FOFSE_ROW_GROUPS", str(groups))
    out, sq, rep = P.conceal_frames(frames, pats, cfg)
    np.testing.assert_array_equal(one, out)
    np.testing.assert_allclose(sq1, sq, rtol=1e-12)
    assert rep.device["blocks"] == rep1.device["blocks"] == sum(len(p.blocks) for p in pats)


def test_frames_api_batches_large_requests(gpu, monkeypatch):
    """A request above the device-memory budget runs as consecutive batches of
    whole frames (forced here with FOFSE_MAX_BATCH_BLOCKS): same bytes, same
    per-block errors and the same PSNR as one call."""
    rng = np.random.default_rng(491)
    frames = np.stack([np.clip(smooth_test_image(rng, 128), 0, 255).astype(np.uint8) for _ in range(12)])
    pats = []
    for f in range(12):
        rr = P.gen_losses(700 + f, 8, 8, 0.15, 16, 16)
        pats.append(P.LossPattern(128, 128, 16, 16, [P.Rect(*map(int, (r["row"], r["col"], 16, 16))) for r in rr]))
    cfg = WL.C4.config("fp32")
    one, sq1, rep1 = P.conceal_frames(frames, pats, cfg)
    monkeypatch.setenv("FOFSE_MAX_BATCH_BLOCKS", "20")
    many, sqn, repn = P.conceal_frames(frames, pats, cfg)
    np.testing.assert_array_equal(one, many)
    np.testing.assert_allclose(sq1, sqn, rtol=1e-12)
    assert repn.device["blocks"] == rep1.device["blocks"] == sum(len(p.blocks) for p in pats)
    assert repn.psnr_db == pytest.approx(rep1.psnr_db, rel=1e-12)


def test_shards_reassemble_the_full_run(gpu):
    """fofse_conceal_shard_f64: disjoint shards (every block still lost) reproduce
    the single-call result bit for bit — the multi-GPU decomposition."""
    img, pat = WL.C1.frame(seed=12)
    cfg = WL.C1.config()
    full = P.conceal(img.astype(np.float64), pat, cfg).restored
    out = img.astype(np.float64).copy()
    n = len(pat.blocks)
    for first in range(0, n, 37):
        cnt = min(37, n - first)
        r, _ = P.conceal_shard(img.astype(np.float64), pat, first, cnt, cfg)
        for b in pat.blocks[first:first + cnt]:
            out[b.row:b.row + 16, b.col:b.col + 16] = r[b.row:b.row + 16, b.col:b.col + 16]
    np.testing.assert_array_equal(out, full)
