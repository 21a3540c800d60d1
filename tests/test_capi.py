"""CPU tests of the C ABI library (no GPU needed): it loads, exports every
symbol include/fofse.h declares, validates exactly like the reference (same
exception class and message), and its host logic (window-mask classes)
reproduces the reference's build_window labels."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2207_01205_b200 as P
from paper_2207_01205_b200 import _capi as capi
from helpers import smooth_test_image

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol(lib):
    header = open(os.path.join(ROOT, "include", "fofse.h")).read()
    declared = set(re.findall(r"\b(fofse_[a-z0-9_]+)\s*\(", header))
    assert declared == set(capi.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.fofse_abi_version() == 3


def test_generator_library_is_separate(lib):
    """The synthetic-input generator lives in libfofse_gen.so (include/fofse_gen.h),
    so generating a workload (the reference arm of bench.py) never maps libfofse.so."""
    header = open(os.path.join(ROOT, "include", "fofse_gen.h")).read()
    declared = set(re.findall(r"\b(fofse_[a-z0-9_]+)\s*\(", header))
    assert declared == set(capi.GEN_EXPORTS)
    g = capi.gen_lib()
    for name in declared:
        assert hasattr(g, name), name
        assert not hasattr(lib, name), name


def test_params_default_match_conceal_config(lib):
    p = capi.default_params()
    # pipeline.hpp:19-33 defaults
    assert (p.algorithm, p.gamma, p.iterations, p.transform_size, p.rho_hat, p.support_width,
            p.threads, p.record_traces) == (capi.ALGO_FOFSE, 0.2, 200, 64, 0.8, 16, 1, 0)
    assert p.precision == capi.PREC_FP64


def test_struct_layouts_match_header(lib):
    assert C.sizeof(capi.Params) == 64
    assert capi.RECORD_DTYPE.itemsize == 72
    assert C.sizeof(capi.Report) == 128


def test_generators_deterministic(lib):
    a = P.gen_image_u8(5, 333, 211)
    b = P.gen_image_u8(5, 333, 211)
    np.testing.assert_array_equal(a, b)
    assert a.std() > 20 and 0 <= a.min() and a.max() <= 255
    assert not np.array_equal(a, P.gen_image_u8(6, 333, 211))


@pytest.mark.parametrize("gw,gh,frac,expect", [(120, 68, 0.25, 2040), (32, 32, 0.10, 102),
                                                (512, 512, 0.20, 52429), (256, 256, 0.05, 3277),
                                                (120, 68, 0.10, 816)])
def test_loss_sampler_counts_and_isolation(lib, gw, gh, frac, expect):
    r = P.gen_losses(9, gw, gh, frac, 16, 16)
    assert len(r) == expect
    cells = set(zip(r["row"] // 16, r["col"] // 16))
    for (a, b) in cells:
        for da in (-1, 0, 1):
            for db in (-1, 0, 1):
                if (da, db) != (0, 0):
                    assert (a + da, b + db) not in cells


def _validate(lib, params, w, h, blocks, bh, bw):
    rects = capi.rects_array(blocks)
    rc = lib.fofse_validate_conceal(C.byref(params), w, h, rects.ctypes.data_as(C.POINTER(capi.Rect_)),
                                    len(rects), bh, bw)
    return rc, lib.fofse_last_error().decode() if rc else ""


def _params(**kw):
    p = capi.default_params()
    for k, v in kw.items():
        setattr(p, k, v)
    return p


BAD = [
    (dict(gamma=0.0), None),
    (dict(gamma=1.5), None),
    (dict(rho_hat=1.0), None),
    (dict(rho_hat=0.0), None),
    (dict(iterations=-1), None),
    (dict(transform_size=0), None),
    (dict(support_width=0), None),
    (dict(threads=0), None),
    (dict(support_width=25), None),  # window 66 > 64
    (dict(algorithm=0, gamma=0.0), "ok"),  # fse ignores gamma
]


@pytest.mark.parametrize("kw,expect", BAD)
def test_config_validation_matches_reference(lib, ref, kw, expect):
    img = smooth_test_image(np.random.default_rng(431), 96)
    blocks = [(16, 16, 16, 16), (64, 64, 16, 16)]
    p = _params(**kw)
    rc, msg = _validate(lib, p, 96, 96, blocks, 16, 16)
    try:
        ref.conceal(img, blocks, 16, 16, algorithm=p.algorithm, gamma=p.gamma, iterations=max(p.iterations, 0) if p.iterations >= 0 else p.iterations,
                    t=p.transform_size, rho_hat=p.rho_hat, support=p.support_width, threads=p.threads)
        rrc, rmsg = 0, ""
    except Exception as e:
        rrc, rmsg = (1 if isinstance(e, ValueError) else 2), str(e)
    assert (rc, msg) == (rrc, rmsg)
    assert (rc == 0) == (expect == "ok")


def test_pattern_validation_matches_reference(lib, ref):
    rng = np.random.default_rng(3)
    img = smooth_test_image(rng, 200)
    cases = [
        [(0, 0, 16, 16), (0, 10, 16, 16)],                       # overlap 0 and 1
        [(0, 0, 16, 16), (40, 40, 16, 16), (190, 0, 16, 16)],    # out of bounds
        [(0, 0, 16, 16), (40, 40, 16, 8)],                       # size mismatch
        [(-1, 0, 16, 16)],
        [(20, 20, 16, 16), (60, 60, 16, 16), (30, 25, 16, 16), (33, 33, 16, 16)],  # 0 and 2 overlap
    ]
    # a long valid list with a late overlap against an early block
    cells = [(r * 20, c * 20, 16, 16) for r in range(9) for c in range(9)]
    cells.append((41, 39, 16, 16))
    cases.append(cells)
    for blocks in cases:
        p = _params(iterations=3)
        rc, msg = _validate(lib, p, 200, 200, blocks, 16, 16)
        with pytest.raises(ValueError) as ei:
            ref.conceal(img, blocks, 16, 16, iterations=3)
        assert rc == 1 and msg == str(ei.value)


def test_large_pattern_validation_matches_reference(lib, ref):
    """Patterns of >= 16384 blocks are validated in parallel (engine.cpp
    validate_pattern): same first failing block and message as the reference's
    in-order scan (pattern.cpp:55-69)."""
    img = np.zeros((1200, 1200))
    grid = [(r * 9, c * 9, 8, 8) for r in range(133) for c in range(133)]
    assert len(grid) >= 16384
    p = _params(iterations=1, transform_size=32, support_width=8)
    assert _validate(lib, p, 1200, 1200, grid, 8, 8) == (0, "")
    mid = len(grid) // 2
    cases = [
        grid + [(4, 4, 8, 8)],                                       # late overlap with block 0
        grid[:mid] + [(grid[5][0] + 3, grid[5][1] + 2, 8, 8)] + grid[mid:] + [(1195, 0, 8, 8)],
        grid[:mid] + [(1195, 0, 8, 8)] + grid[mid:] + [(4, 4, 8, 8)],  # bounds before overlap
        grid[:mid] + [(grid[mid][0] + 1, grid[mid][1] + 1, 8, 8)] + grid[mid:],  # same anchor cell
        grid[:100] + [(0, 0, 8, 4)] + grid[100:],                    # size mismatch
    ]
    for blocks in cases:
        rc, msg = _validate(lib, p, 1200, 1200, blocks, 8, 8)
        with pytest.raises(ValueError) as ei:
            ref.conceal(img, blocks, 8, 8, iterations=1, t=32, support=8)
        assert rc == 1 and msg == str(ei.value)


def _host_plan(lib, blocks_per_frame, w, h, bh, bw, **kw):
    allb = [b for fr in blocks_per_frame for b in fr]
    offs = np.cumsum([0] + [len(f) for f in blocks_per_frame]).astype(np.int64)
    rects = capi.rects_array(allb)
    plan = C.c_void_p()
    p = _params(**kw)
    capi.check(lib.fofse_plan_frames_u8(None, len(blocks_per_frame), w, h,
                                        rects.ctypes.data_as(C.POINTER(capi.Rect_)),
                                        offs.ctypes.data_as(C.POINTER(C.c_int64)), bh, bw,
                                        C.byref(p), C.byref(plan)))
    return plan, allb, offs


def test_plan_classes_reproduce_build_window_labels(lib, orc):
    """Host window classes (geometry keys) == pipeline.cpp:80-112 labels, block by block,
    for isolated grid losses, border blocks and non-isolated off-grid neighbours."""
    w, h = 200, 168
    img = np.zeros((h, w))
    frames = [
        [(0, 0, 12, 16), (0, 24, 12, 16), (20, 10, 12, 16), (156, 184, 12, 16), (70, 70, 12, 16),
         (82, 90, 12, 16), (40, 150, 12, 16), (100, 3, 12, 16)],
        [(r, c, 12, 16) for (r, c) in [(30, 30), (30, 100), (90, 30), (90, 100), (150, 180)]],
    ]
    plan, allb, offs = _host_plan(lib, frames, w, h, 12, 16, support_width=14, transform_size=64)
    try:
        nb, ncls, nsym = C.c_int64(), C.c_int64(), C.c_int64()
        capi.check(lib.fofse_plan_info(plan, C.byref(nb), C.byref(ncls), C.byref(nsym)))
        assert nb.value == len(allb)
        got = np.zeros((40, 44), np.uint8)
        for f, fr in enumerate(frames):
            lost = np.zeros((h, w), np.uint8)
            for (r, c, hh, ww) in fr:
                lost[r:r + hh, c:c + ww] = 1
            for k, b in enumerate(fr):
                capi.check(lib.fofse_plan_block_labels(plan, int(offs[f] + k), capi.ptr(got, C.c_uint8)))
                _, lab = orc.build_window(img, lost, b, 14)
                np.testing.assert_array_equal(got, lab, err_msg=f"frame {f} block {k} {b}")
        # interior isolated blocks share one symmetric class
        assert 1 <= nsym.value < ncls.value <= len(allb)
    finally:
        lib.fofse_plan_destroy(plan)


def test_plan_class_count_for_benchmark_pattern(lib):
    """C2: 2040 isolated losses on 120x68 cells -> interior + edge/corner classes only."""
    r = P.gen_losses(21, 120, 68, 0.25, 16, 16)
    blocks = [tuple(map(int, (x["row"], x["col"], 16, 16))) for x in r]
    plan, _, _ = _host_plan(lib, [blocks], 1920, 1088, 16, 16, gamma=0.5)
    try:
        nb, ncls, nsym = C.c_int64(), C.c_int64(), C.c_int64()
        capi.check(lib.fofse_plan_info(plan, C.byref(nb), C.byref(ncls), C.byref(nsym)))
        assert nb.value == 2040 and ncls.value <= 9 and nsym.value == 1
    finally:
        lib.fofse_plan_destroy(plan)


def test_product_fails_loudly_without_gpu(lib):
    """No CPU fallback: without a usable CUDA device the product raises."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    img = np.zeros((64, 64))
    with pytest.raises(capi.FofseCudaError):
        P.conceal(img, P.LossPattern(64, 64, 16, 16, [P.Rect(16, 16, 16, 16)]), P.ConcealConfig())


def test_python_config_validation_messages():
    for kw, msg in [(dict(gamma=0.0), "config: gamma must lie in (0, 1]"),
                    (dict(rho_hat=1.0), "config: rho_hat must lie in (0, 1)"),
                    (dict(iterations=-2), "config: iterations must be >= 0"),
                    (dict(support_width=0), "config: support width must be >= 1"),
                    (dict(threads=0), "config: thread count must be >= 1")]:
        with pytest.raises(ValueError, match=re.escape(msg)):
            P.ConcealConfig(**kw).validate()
    with pytest.raises(ValueError, match="unknown algorithm 'bogus'"):
        P.parse_algorithm("bogus")
    assert P.series_label(P.ConcealConfig(gamma=0.35)) == "fofse_g0.35"
    assert P.series_label(P.ConcealConfig(algorithm="fse")) == "fse"


def test_psnr_curves_validation_without_gpu():
    """pipeline.cpp:267-270: stride and iteration bounds are checked first."""
    pat = P.LossPattern(64, 64, 16, 16, [])
    with pytest.raises(ValueError, match="stride must be >= 1"):
        P.psnr_vs_iterations(np.zeros((64, 64)), pat, [P.ConcealConfig()], 10, 0)
    with pytest.raises(ValueError, match="iterations must be >= 0"):
        P.psnr_vs_iterations(np.zeros((64, 64)), pat, [P.ConcealConfig()], -1, 5)
    assert P.psnr_vs_iterations(np.zeros((64, 64)), pat, [P.ConcealConfig(gamma=0.5)], 3, 5)[0].label == "fofse_g0.5"
