"""The link-level drop-in (paper_2207_01205_b200/adapter/fse_b200.cpp ->
_lib/libfse_b200.so): one program written only against the reference's headers
(tests/cpp/ref_caller.cpp) linked against the compiled reference (CPU) and
with libfse_b200.so first (GPU). Both must give the reference's results."""
import os
import struct
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "tests", "cpp", "_build")
ADAPTER = os.path.join(ROOT, "paper_2207_01205_b200", "_lib", "libfse_b200.so")
HOT = ["_ZN3fse7concealERKNS_10SampleGridERKNS_11LossPatternERKNS_13ConcealConfigE",
       "_ZN3fse18extrapolate_windowERKNS_10SampleGridERKNS_10RegionMaskERKNS_13ConcealConfigE",
       "_ZN3fse8spectral12init_spectraERKNS_10SampleGridERKNS_10RegionMaskERKNS_11WeightFieldEi",
       "_ZN3fse8spectral12fast_iterateERNS0_8SpectrumEdi",
       "_ZN3fse8spectral20fast_iterate_full_odERNS0_8SpectrumEi",
       "_ZN3fse8spectral16synthesize_modelERKNS0_8SpectrumE"]


def _need(path):
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (build() builds it where the reference headers exist)")
    return path


def _dyn_symbols(path):
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True, check=True).stdout
    defined = {l.split()[-1] for l in out.splitlines() if l.strip()}
    out = subprocess.run(["nm", "-D", "--undefined-only", path], capture_output=True, text=True, check=True).stdout
    undefined = {l.split()[-1] for l in out.splitlines() if l.strip()}
    return defined, undefined


def test_adapter_defines_the_reference_hot_path_symbols():
    defined, undefined = _dyn_symbols(_need(ADAPTER))
    for s in HOT:
        assert s in defined, s
    # stands alone: nothing of the reference library is needed to load it
    assert not [s for s in undefined if s.startswith("_ZN3fse")]
    needed = subprocess.run(["readelf", "-d", _need(os.path.join(BUILD, "ref_caller_gpu"))], capture_output=True,
                            text=True, check=True).stdout
    order = [l.split("[")[1].rstrip("]") for l in needed.splitlines() if "(NEEDED)" in l]
    assert order.index("libfse_b200.so") < order.index("libfse_ref.so")


def _write_input(path, img, blocks, bh=16, bw=16, algo=2, iterations=60, t=64, support=16, gamma=0.5, rho=0.8):
    h, w = img.shape
    with open(path, "wb") as f:
        f.write(struct.pack("9i", w, h, len(blocks), bh, bw, algo, iterations, t, support))
        f.write(struct.pack("2d", gamma, rho))
        for r, c in blocks:
            f.write(struct.pack("2i", r, c))
        f.write(np.ascontiguousarray(img, np.float64).tobytes())


REC = np.dtype([("nu", "<i4"), ("k1", "<i4"), ("k2", "<i4"), ("p_re", "<f8"), ("p_im", "<f8"), ("c_re", "<f8"),
                ("c_im", "<f8"), ("energy", "<f8")])


def _read_output(path, h, w, nblocks, win):
    buf = open(path, "rb").read()
    off = 0

    def take(dt, n):
        nonlocal off
        a = np.frombuffer(buf, dt, n, off)
        off += a.nbytes
        return a

    def trace():
        n, conv = take("<i4", 2)
        return take(REC, int(n)), bool(conv)

    out = {"restored": take("<f8", h * w).reshape(h, w), "psnr": float(take("<f8", 1)[0])}
    out["traces"] = [trace() for _ in range(nblocks)]
    out["win_model"] = take("<f8", win * win)
    out["win_trace"] = trace()
    out["init"] = take("<f8", 3)
    out["eng_trace"] = trace()
    out["eng_model"] = take("<f8", win * win)
    assert off == len(buf)
    return out


def _run(exe, inp, outp):
    r = subprocess.run([exe, inp, outp], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    return outp


def _case():
    from helpers import random_grid
    rng = np.random.default_rng(23)
    img = np.clip(np.round(120 + 60 * random_grid(rng, 160, 192)), 0, 255)
    blocks = [(48, 48), (0, 96), (112, 176), (96, 16)]  # interior + borders
    return img, blocks


def test_reference_caller_cpu_runs(tmp_path):
    exe = _need(os.path.join(BUILD, "ref_caller_cpu"))
    img, blocks = _case()
    inp = str(tmp_path / "in.bin")
    _write_input(inp, img, blocks)
    o = _read_output(_run(exe, inp, str(tmp_path / "cpu.bin")), 160, 192, len(blocks), 48)
    assert all(len(t) == 60 for t, _ in o["traces"]) and o["psnr"] > 10


@pytest.mark.gpu
def test_reference_caller_linked_to_b200_matches_the_reference(gpu, tmp_path):
    cpu = _need(os.path.join(BUILD, "ref_caller_cpu"))
    gpux = _need(os.path.join(BUILD, "ref_caller_gpu"))
    img, blocks = _case()
    inp = str(tmp_path / "in.bin")
    _write_input(inp, img, blocks)
    a = _read_output(_run(cpu, inp, str(tmp_path / "cpu.bin")), 160, 192, len(blocks), 48)
    b = _read_output(_run(gpux, inp, str(tmp_path / "gpu.bin")), 160, 192, len(blocks), 48)
    # image level: same selected-basis sequences, pixels within 1e-9
    for (ta, ca), (tb, cb) in zip(a["traces"], b["traces"]):
        np.testing.assert_array_equal(ta[["k1", "k2"]], tb[["k1", "k2"]])
        assert ca == cb
    assert np.abs(a["restored"] - b["restored"]).max() <= 1e-9
    assert b["psnr"] == pytest.approx(a["psnr"], rel=1e-12)
    # window level
    np.testing.assert_array_equal(a["win_trace"][0][["k1", "k2"]], b["win_trace"][0][["k1", "k2"]])
    assert np.abs(a["win_model"] - b["win_model"]).max() <= 1e-9
    # engine level (K1x + strict kernel): bit-identical spectra and records, resumed in two calls
    np.testing.assert_array_equal(a["init"], b["init"])
    np.testing.assert_array_equal(a["eng_trace"][0], b["eng_trace"][0])
    assert np.abs(a["eng_model"] - b["eng_model"]).max() <= 1e-9
