"""Generate tests/golden/ref_cases.npz from the UNMODIFIED reference library.

Runs the reference sources compiled from /root/reference (oracle/_ref/
libfse_ref.so: fse::conceal, spectral::init_spectra / fast_iterate /
synthesize_model, build_isotropic_weight, the FFT boundary) on small seeded
inputs and stores inputs + outputs. The fixtures travel with the repo, so the
oracle is pinned to the reference even where /root/reference is absent (the
GPU box). Re-run:  python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from helpers import block_mask, random_grid, random_mask, smooth_test_image  # noqa: E402


def main():
    if not oracle.have_reference():
        oracle.build(ref=True)
    ref = oracle.Reference()
    out = {}

    # A: pipeline case (pipeline_test.cpp:140-169 layout), fofse gamma 0.5
    img = smooth_test_image(np.random.default_rng(419), 96)
    blocks = [(16, 16, 16, 16), (16, 64, 16, 16), (64, 16, 16, 16), (64, 64, 16, 16)]
    r = ref.conceal(img, blocks, 16, 16, gamma=0.5, iterations=40, t=64, rho_hat=0.8, support=16,
                    traces=True)
    out["A_image"] = img.astype(np.uint8)
    out["A_blocks"] = np.array(blocks, np.int32)
    out["A_restored"] = r["restored"]
    out["A_psnr"] = np.array([r["psnr_db"]])
    out["A_u"] = np.stack([np.stack([t["u1"], t["u2"]]) for t in r["traces"]]).astype(np.int16)

    # B: borders + neighbouring losses, rectangular blocks, fse (gamma 1)
    img = smooth_test_image(np.random.default_rng(409), 160)
    blocks = [(0, 0, 12, 16), (0, 24, 12, 16), (20, 10, 12, 16), (148, 144, 12, 16),
              (70, 70, 12, 16), (82, 90, 12, 16), (40, 140, 12, 16)]
    r = ref.conceal(img, blocks, 12, 16, algorithm=oracle.ALGO_FSE, iterations=30, t=64,
                    rho_hat=0.8, support=14, traces=True)
    out["B_image"] = img.astype(np.uint8)
    out["B_blocks"] = np.array(blocks, np.int32)
    out["B_restored"] = r["restored"]
    out["B_psnr"] = np.array([r["psnr_db"]])
    out["B_u"] = [np.stack([t["u1"], t["u2"]]) for t in r["traces"]]
    out["B_u"] = np.concatenate(out["B_u"], axis=1).astype(np.int16)
    out["B_counts"] = np.array([len(t) for t in r["traces"]], np.int32)

    # C: spectral engine, T=16, random window + mask (engine_spectral_test.cpp:225-276 style)
    rng = np.random.default_rng(233)
    f = random_grid(rng, 14, 13)
    m = random_mask(rng, 14, 13)
    w = ref.build_isotropic_weight(m, 0.8)
    s = ref.init_spectra(f, m, w, 16)
    out["C_f"], out["C_mask"], out["C_weight"] = f, m, w
    out["C_rw0"], out["C_w"] = s.rw.copy(), s.w.copy()
    out["C_scalars0"] = np.array([s.w0, s.weighted_energy, s.initial_energy, s.initial_max])
    recs = ref.fast_iterate(s, 0.3, 25)
    out["C_records"] = recs
    out["C_rw"], out["C_g"] = s.rw, s.g
    out["C_model"] = ref.synthesize_model(s)

    # D: FFT boundary (transform.hpp:15-20) on a random complex 8x8 grid
    x = rng.normal(size=(8, 8)) + 1j * rng.normal(size=(8, 8))
    out["D_x"], out["D_fwd"], out["D_inv"] = x, ref.dft2d(x), ref.dft2d(x, inverse=True)

    # E: weights (grid.cpp:75-92) on a 48x48 window with a hole and an outside strip
    mE = block_mask(48, 48, missing=[(16, 16, 16, 16)], outside=[(0, 0, 48, 4)])
    out["E_mask"], out["E_weight"] = mE, ref.build_isotropic_weight(mE, 0.8)

    # F: benchmark configuration C1 (T=64, 100 it, rho 0.8, gamma 0.5) on 8 blocks
    from paper_2207_01205_b200 import workloads as WL
    img, pat = WL.C1.frame(seed=5)
    bl = [tuple(b) for b in pat.blocks[:8]]
    r = ref.conceal(img.astype(np.float64), bl, 16, 16, gamma=0.5, iterations=100, t=64,
                    rho_hat=0.8, support=16, traces=True)
    out["F_image"] = img
    out["F_blocks"] = np.array(bl, np.int32)
    out["F_u"] = np.stack([np.stack([t["u1"], t["u2"]]) for t in r["traces"]]).astype(np.int16)
    mask = np.zeros(img.shape, bool)
    for (rr, cc, hh, ww) in bl:
        mask[rr:rr + hh, cc:cc + ww] = True
    out["F_missing"] = r["restored"][mask]
    out["F_psnr"] = np.array([r["psnr_db"]])

    path = os.path.join(HERE, "ref_cases.npz")
    np.savez_compressed(path, **out)
    print(path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
