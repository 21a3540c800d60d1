"""The header-only C++ drop-in (include/fofse_fse.hpp) compiles against the C
ABI and behaves like fse::conceal: same exception classes and messages (CPU),
same results as the oracle (GPU)."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def exe(lib, tmp_path_factory):
    from paper_2207_01205_b200 import _capi
    libdir = os.path.dirname(_capi.LIB_PATH)
    out = str(tmp_path_factory.mktemp("cpp") / "adapter_check")
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "adapter_check.cpp"), "-L", libdir, "-lfofse",
                    "-Wl,-rpath," + libdir, "-o", out], check=True)
    return out


def test_adapter_validation_matches_reference(exe, ref):
    res = subprocess.run([exe, "validate"], capture_output=True, text=True, check=True).stdout.splitlines()
    got = {l.split("|")[0]: l.split("|")[1:] for l in res}
    img = np.round(128 + 90 * np.sin(0.09 * np.arange(96))[:, None] * np.cos(0.07 * np.arange(96))[None, :])
    blocks = [(16, 16, 16, 16), (64, 64, 16, 16)]
    cases = {"gamma0": dict(gamma=0.0), "rho1": dict(rho_hat=1.0), "window": dict(support=25)}
    for name, kw in cases.items():
        with pytest.raises(ValueError) as ei:
            ref.conceal(img, blocks, 16, 16, **kw)
        assert got[name] == ["invalid_argument", str(ei.value)]
    with pytest.raises(ValueError) as ei:
        ref.conceal(img, blocks + [(70, 70, 16, 16)], 16, 16)
    assert got["overlap"] == ["invalid_argument", str(ei.value)]
    assert got["dims"] == ["invalid_argument", "conceal: pattern dimensions do not match the image"]


@pytest.mark.gpu
def test_adapter_conceal_matches_oracle(exe, orc, tmp_path):
    path = str(tmp_path / "restored.bin")
    out = subprocess.run([exe, "conceal", path], capture_output=True, text=True, check=True).stdout
    both = np.fromfile(path, np.float64).reshape(2, 96, 96)
    img, got = both[0], both[1]
    ref = orc.conceal(img, [(16, 16, 16, 16), (64, 64, 16, 16)], 16, 16, gamma=0.5, iterations=60)
    assert np.abs(got - ref["restored"]).max() <= 1e-9
    assert "records=60" in out
