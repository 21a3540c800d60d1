"""Pin the oracle (C restatement of the reference FOFSE path) before trusting it.

1. Golden fixtures produced by the UNMODIFIED reference library
   (tests/golden/make_golden.py): the oracle must reproduce them bit for bit.
2. When the compiled reference (oracle/_ref) is available: live bit-exact
   agreement on fresh seeded cases, including the reference's own FFT-free
   spatial engine as an independent check.
3. The reference's own known-answer tests, re-expressed (engine_spectral_test,
   transform_test, basis_test, grid_test, pipeline_test).
"""
import math
import os

import numpy as np
import pytest

from helpers import MISSING, OUTSIDE, SUPPORT, block_mask, random_grid, random_mask, smooth_test_image

GOLD = os.path.join(os.path.dirname(__file__), "golden", "ref_cases.npz")


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def _blocks(a):
    return [tuple(int(x) for x in r) for r in a]


# ---------------------------------------------------------------- golden ----
def test_golden_pipeline_A(orc, gold):
    img = gold["A_image"].astype(np.float64)
    r = orc.conceal(img, _blocks(gold["A_blocks"]), 16, 16, gamma=0.5, iterations=40, t=64,
                    rho_hat=0.8, support=16, traces=True)
    np.testing.assert_array_equal(r["restored"], gold["A_restored"])
    assert r["psnr_db"] == gold["A_psnr"][0]
    u = np.stack([np.stack([t["u1"], t["u2"]]) for t in r["traces"]])
    np.testing.assert_array_equal(u, gold["A_u"])


def test_golden_borders_neighbours_B(orc, gold):
    img = gold["B_image"].astype(np.float64)
    r = orc.conceal(img, _blocks(gold["B_blocks"]), 12, 16, algorithm=0, iterations=30, t=64,
                    rho_hat=0.8, support=14, traces=True)
    np.testing.assert_array_equal(r["restored"], gold["B_restored"])
    assert r["psnr_db"] == gold["B_psnr"][0]
    np.testing.assert_array_equal([len(t) for t in r["traces"]], gold["B_counts"])
    u = np.concatenate([np.stack([t["u1"], t["u2"]]) for t in r["traces"]], axis=1)
    np.testing.assert_array_equal(u, gold["B_u"])


def test_golden_spectral_engine_C(orc, gold):
    s = orc.init_spectra(gold["C_f"], gold["C_mask"], gold["C_weight"], 16)
    np.testing.assert_array_equal(s.rw, gold["C_rw0"])
    np.testing.assert_array_equal(s.w, gold["C_w"])
    np.testing.assert_array_equal([s.w0, s.weighted_energy, s.initial_energy, s.initial_max],
                                  gold["C_scalars0"])
    rec = orc.fast_iterate(s, 0.3, 25)
    np.testing.assert_array_equal(rec, gold["C_records"])
    np.testing.assert_array_equal(s.rw, gold["C_rw"])
    np.testing.assert_array_equal(s.g, gold["C_g"])
    np.testing.assert_array_equal(orc.synthesize_model(s), gold["C_model"])


def test_golden_fft_boundary_D(orc, gold):
    np.testing.assert_array_equal(orc.dft2d(gold["D_x"]), gold["D_fwd"])
    np.testing.assert_array_equal(orc.dft2d(gold["D_x"], inverse=True), gold["D_inv"])


def test_golden_weights_E(orc, gold):
    np.testing.assert_array_equal(orc.build_isotropic_weight(gold["E_mask"], 0.8), gold["E_weight"])


def test_golden_benchmark_config_F(orc, gold):
    """C1 configuration (T=64, 100 it, rho 0.8, gamma 0.5)."""
    img = gold["F_image"].astype(np.float64)
    bl = _blocks(gold["F_blocks"])
    r = orc.conceal(img, bl, 16, 16, gamma=0.5, iterations=100, t=64, rho_hat=0.8, support=16,
                    traces=True)
    u = np.stack([np.stack([t["u1"], t["u2"]]) for t in r["traces"]])
    np.testing.assert_array_equal(u, gold["F_u"])
    mask = np.zeros(img.shape, bool)
    for (rr, cc, hh, ww) in bl:
        mask[rr:rr + hh, cc:cc + ww] = True
    np.testing.assert_array_equal(r["restored"][mask], gold["F_missing"])
    assert r["psnr_db"] == gold["F_psnr"][0]


# ------------------------------------------------------- live reference ----
@pytest.mark.parametrize("algo,gamma,t,support", [(2, 0.5, 64, 16), (0, 1.0, 64, 16), (1, 0.0, 64, 16),
                                                  (2, 0.3, 32, 8), (2, 0.7, 128, 16)])
def test_oracle_equals_reference_conceal(orc, ref, algo, gamma, t, support):
    rng = np.random.default_rng(7 + t + algo)
    img = smooth_test_image(rng, 192)
    b = 16 if t >= 64 else 8
    blocks = [(support + 2, support + 2, b, b), (100, 40, b, b), (0, 150, b, b), (192 - b, 192 - b, b, b)]
    a = orc.conceal(img, blocks, b, b, algorithm=algo, gamma=gamma, iterations=35, t=t, rho_hat=0.8,
                    support=support, traces=True)
    r = ref.conceal(img, blocks, b, b, algorithm=algo, gamma=gamma, iterations=35, t=t, rho_hat=0.8,
                    support=support, traces=True)
    np.testing.assert_array_equal(a["restored"], r["restored"])
    assert a["psnr_db"] == r["psnr_db"]
    for x, y in zip(a["traces"], r["traces"]):
        np.testing.assert_array_equal(x, y)


def test_oracle_equals_reference_engine(orc, ref):
    rng = np.random.default_rng(31)
    for t, h, w in [(8, 6, 7), (16, 16, 16), (64, 48, 48), (128, 70, 64)]:
        f = random_grid(rng, h, w)
        m = random_mask(rng, h, w)
        wt = ref.build_isotropic_weight(m, 0.85)
        np.testing.assert_array_equal(orc.build_isotropic_weight(m, 0.85), wt)
        a, b = orc.init_spectra(f, m, wt, t), ref.init_spectra(f, m, wt, t)
        np.testing.assert_array_equal(a.rw, b.rw)
        ra, rb = orc.fast_iterate(a, 0.5, 30), ref.fast_iterate(b, 0.5, 30)
        np.testing.assert_array_equal(ra, rb)
        np.testing.assert_array_equal(a.g, b.g)
        ra, rb = orc.fast_iterate_full_od(a, 5), ref.fast_iterate_full_od(b, 5)
        np.testing.assert_array_equal(ra, rb)
        np.testing.assert_array_equal(orc.synthesize_model(a), ref.synthesize_model(b))


def test_spectral_matches_reference_spatial_engine(orc, ref):
    """engine_spectral_test.cpp:225-276 / acceptance #1: the reference's FFT-free
    direct engine selects the same functions; coefficients to 1e-9, model 1e-8."""
    rng = np.random.default_rng(233)
    for t in (8, 16, 32):
        h, w = t - 2, t - 1
        f = random_grid(rng, h, w)
        m = random_mask(rng, h, w)
        model_d, rec_d = ref.spatial_run(f, m, t, 0.8, 20, 1, 1, 0.2)  # max portion, constant gamma
        wt = orc.build_isotropic_weight(m, 0.8)
        s = orc.init_spectra(f, m, wt, t)
        rec = orc.fast_iterate(s, 0.2, 20)
        assert len(rec) == len(rec_d)
        np.testing.assert_array_equal(rec["u1"], rec_d["u1"])
        np.testing.assert_array_equal(rec["u2"], rec_d["u2"])
        for k in ("c_re", "c_im", "p_re", "p_im"):
            assert np.all(np.abs(rec[k] - rec_d[k]) <= 1e-9 * np.maximum(np.abs(rec_d[k]), 1e-300) + 1e-15)
        assert np.abs(orc.synthesize_model(s) - model_d).max() < 1e-8


def test_reference_transform_counts(ref):
    """engine_spectral_test.cpp:162-186: 2 forward at init, none while iterating, 1 inverse."""
    rng = np.random.default_rng(227)
    f = random_grid(rng, 12, 12)
    m = random_mask(rng, 12, 12)
    wt = ref.build_isotropic_weight(m, 0.8)
    f0, i0 = ref.transform_counts()
    s = ref.init_spectra(f, m, wt, 16)
    f1, i1 = ref.transform_counts()
    assert (f1 - f0, i1 - i0) == (2, 0)
    ref.fast_iterate(s, 0.2, 50)
    assert ref.transform_counts() == (f1, i1)
    ref.synthesize_model(s)
    assert ref.transform_counts() == (f1, i1 + 1)


# ------------------------------------------------ reference KATs (oracle) ----
def test_fft_vs_naive_dft(orc):
    """transform_test.cpp:24-32."""
    rng = np.random.default_rng(1)
    x = rng.normal(size=(8, 8)) + 1j * rng.normal(size=(8, 8))
    assert np.abs(orc.dft2d(x) - np.fft.fft2(x)).max() < 1e-9


def test_fft_round_trip_and_hermitian(orc):
    """transform_test.cpp:34-59."""
    rng = np.random.default_rng(2)
    x = rng.normal(size=(16, 16)) + 1j * rng.normal(size=(16, 16))
    y = orc.dft2d(orc.dft2d(x), inverse=True)
    assert np.abs(y - 256 * x).max() < 1e-8
    r = rng.normal(size=(16, 16)).astype(complex)
    X = orc.dft2d(r)
    Xc = np.conj(X[(-np.arange(16)) % 16][:, (-np.arange(16)) % 16])
    assert np.abs(X - Xc).max() < 1e-12


def test_zero_signal_gives_zero_spectra(orc):
    """engine_spectral_test.cpp:65-74 and 298-308."""
    m = np.zeros((8, 8), np.uint8)
    s = orc.init_spectra(np.zeros((8, 8)), m, orc.build_isotropic_weight(m, 0.8), 8)
    assert np.all(s.rw == 0) and s.weighted_energy == 0 and s.initial_max == 0
    rec = orc.fast_iterate(s, 0.5, 10)
    assert s.converged and len(rec) == 0 and s.nu == 0


def test_constant_window(orc):
    """engine_spectral_test.cpp:76-115."""
    c = 2.75
    m = block_mask(6, 6, missing=[(2, 2, 2, 2)])
    w = orc.build_isotropic_weight(m, 0.8)
    s = orc.init_spectra(np.full((6, 6), c), m, w, 8)
    assert np.abs(s.rw - c * s.w).max() < 1e-12 * abs(c) * s.w0
    assert s.w0 == pytest.approx(w.sum(), rel=1e-12)
    assert s.weighted_energy == pytest.approx(c * c * w.sum(), rel=1e-12)
    s = orc.init_spectra(np.full((6, 6), 4.0), m, w, 8)
    before = s.initial_max
    rec = orc.fast_iterate(s, 1.0, 1)
    assert (rec[0]["u1"], rec[0]["u2"]) == (0, 0)
    assert abs(complex(rec[0]["p_re"], rec[0]["p_im"]) - 4.0) < 1e-9
    assert np.abs(s.rw).max() < 1e-9 * before
    np.testing.assert_allclose(orc.synthesize_model(s), 4.0, rtol=1e-9)


def test_energy_bookkeeping_and_parseval(orc):
    """engine_spectral_test.cpp:133-160: tracked energy == spatial replay; Parseval."""
    rng = np.random.default_rng(223)
    f = random_grid(rng, 7, 6)
    m = random_mask(rng, 7, 6)
    w = orc.build_isotropic_weight(m, 0.8)
    s = orc.init_spectra(f, m, w, 8)
    resid = np.where(m == SUPPORT, f, 0.0)
    rows, cols = np.meshgrid(np.arange(7), np.arange(6), indexing="ij")
    for _ in range(20):
        rec = orc.fast_iterate(s, 0.3, 1)
        if len(rec) == 0:
            break
        u1, u2 = int(rec[0]["u1"]), int(rec[0]["u2"])
        c = complex(rec[0]["c_re"], rec[0]["c_im"])
        phi = np.exp(2j * np.pi * (u1 * rows + u2 * cols) / 8)
        self_conj = (u1 == (8 - u1) % 8) and (u2 == (8 - u2) % 8)
        resid = resid - np.where(w > 0, (c.real * phi.real) if self_conj else 2 * (c * phi).real, 0.0)
        assert s.weighted_energy == pytest.approx(float(np.sum(w * resid * resid)), rel=1e-8)
        assert np.sum(np.abs(s.rw) ** 2) / 64 == pytest.approx(float(np.sum((w * resid) ** 2)), rel=1e-8)


def test_weights_known_answers(orc):
    """grid_test.cpp:47-55 and :57-69."""
    w = orc.build_isotropic_weight(np.zeros((5, 5), np.uint8), 0.8)
    assert w[2, 2] == pytest.approx(1.0) and w[2, 4] == pytest.approx(0.64)
    assert w[2, 0] == pytest.approx(0.64) and w[0, 2] == pytest.approx(0.64)
    assert w[1, 1] == pytest.approx(0.8 ** math.sqrt(2.0))
    m = block_mask(48, 48, missing=[(16, 16, 16, 16)], outside=[(0, 0, 48, 4)])
    w = orc.build_isotropic_weight(m, 0.8)
    assert np.all((w > 0) == (m == SUPPORT))
    with pytest.raises(ValueError):
        orc.build_isotropic_weight(np.zeros((4, 4), np.uint8), 1.0)


def test_psnr_known_answer():
    """grid_test.cpp:111-118: single sample with error 16 -> 24.04840395556061 dB."""
    import paper_2207_01205_b200 as P
    a = np.full((4, 4), 10.0)
    b = a.copy()
    b[1, 2] += 16.0
    m = block_mask(4, 4, missing=[(1, 2, 1, 1)])
    db, ident = P.psnr(a, b, m, MISSING)
    assert not ident and db == pytest.approx(24.04840395556061, rel=1e-12)


def test_window_layout(orc, ref):
    """pipeline_test.cpp:92-117: 81 windows of 48x48, 2048 SUPPORT / 256 MISSING,
    first block at (56,56); lost samples stay zero."""
    img = smooth_test_image(np.random.default_rng(401), 512)
    blocks = ref.generate_grid_pattern(512, 512, 16, 48, 81)
    assert len(blocks) == 81 and blocks[0][:2] == (56, 56)
    wins, labs = ref.extract_windows(img, blocks, 16, 16, 16)
    lost = np.zeros((512, 512), np.uint8)
    for (r, c, h, w) in blocks:
        lost[r:r + h, c:c + w] = 1
    for i, bl in enumerate(blocks):
        assert (labs[i] == SUPPORT).sum() == 2048 and (labs[i] == MISSING).sum() == 256
        win, lab = orc.build_window(img, lost, bl, 16)
        np.testing.assert_array_equal(lab, labs[i])
        np.testing.assert_array_equal(win, wins[i])
