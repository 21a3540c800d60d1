"""The reference-CLI front-end (paper_2207_01205_b200/cli/fofse_cli.cpp, SURVEY §8f
rank 3): flags, output files, fingerprints, number formats and exit codes of
proj/tools/main.cpp, on the GPU path."""
import os
import subprocess

import numpy as np
import pytest

import paper_2207_01205_b200 as P
from paper_2207_01205_b200 import build
from helpers import smooth_test_image


@pytest.fixture(scope="module")
def cli(lib):
    return build.build_cli()


def run(cli, *args, env=None):
    return subprocess.run([cli, *map(str, args)], capture_output=True, text=True, env=env, timeout=300)


def write_pgm(path, img):
    img = np.clip(np.floor(img + 0.5), 0, 255).astype(np.uint8)
    with open(path, "wb") as f:
        f.write(b"P5\n# test image\n%d %d\n255\n" % (img.shape[1], img.shape[0]))
        f.write(img.tobytes())
    return img


def read_pgm(path):
    with open(path, "rb") as f:
        data = f.read()
    assert data.startswith(b"P5\n")
    head = data.split(b"\n", 3)
    w, h = map(int, head[1].split())
    assert head[2] == b"255"
    return np.frombuffer(head[3], np.uint8).reshape(h, w)


def fingerprint(cmd, inp, **kw):
    o = dict(algorithm="fofse", gamma="0.2", iterations=200, fft_size=64, rho_hat="0.8", block=16, support=16,
             spacing=48, count_limit=81, pattern="grid", threads=1, seed=0, stride=5)
    o.update(kw)
    keys = ["algorithm", "gamma", "iterations", "fft_size", "rho_hat", "block", "support", "spacing",
            "count_limit", "pattern", "threads", "seed", "stride"]
    return "# config: command=%s " % cmd + " ".join(f"{k}={o[k]}" for k in keys) + f" input={inp}"


# ---- exit codes and validation (host only) ----
def test_usage_errors_exit_1(cli, tmp_path):
    assert run(cli).returncode == 1
    assert run(cli, "frobnicate", "--input", "x.pgm").returncode == 1
    r = run(cli, "conceal")
    assert r.returncode == 1 and "--input is required" in r.stderr
    assert run(cli, "conceal", "--input", "x.pgm", "--bogus", "1").returncode == 1
    assert run(cli, "conceal", "--input", "x.pgm", "--gamma", "abc").returncode == 1
    r = run(cli, "sweep-gamma", "--input", "x.pgm", "--gammas", "0.5,1.5")
    assert r.returncode == 1 and "gamma must lie in (0, 1]" in r.stderr


def test_runtime_errors_exit_2(cli, tmp_path):
    r = run(cli, "conceal", "--input", tmp_path / "missing.pgm")
    assert r.returncode == 2 and "cannot open" in r.stderr
    bad = tmp_path / "bad.pgm"
    bad.write_bytes(b"P2\n2 2\n255\n0 0 0 0\n")
    r = run(cli, "conceal", "--input", bad)
    assert r.returncode == 2 and "not a binary PGM (P5)" in r.stderr
    trunc = tmp_path / "trunc.pgm"
    trunc.write_bytes(b"P5\n4 4\n255\n\x00\x01")
    assert "truncated PGM raster" in run(cli, "conceal", "--input", trunc).stderr


def test_invalid_config_exits_1_before_any_device_work(cli, tmp_path):
    img = tmp_path / "img.pgm"
    write_pgm(img, np.full((96, 96), 100.0))
    r = run(cli, "conceal", "--input", img, "--rho-hat", "1.5", "--out-dir", tmp_path / "o")
    assert r.returncode == 1 and "rho_hat must lie in (0, 1)" in r.stderr
    r = run(cli, "conceal", "--input", img, "--spacing", "20", "--out-dir", tmp_path / "o")
    assert r.returncode == 1 and "spacing must leave a support frame" in r.stderr


# ---- outputs on the GPU, vs the oracle ----
@pytest.mark.gpu
def test_conceal_outputs_match_the_reference(cli, gpu, ref, tmp_path):
    rng = np.random.default_rng(463)
    img = write_pgm(tmp_path / "scene.pgm", smooth_test_image(rng, 176))
    out = tmp_path / "out"
    r = run(cli, "conceal", "--input", tmp_path / "scene.pgm", "--iterations", 40, "--gamma", 0.5,
            "--out-dir", out)
    assert r.returncode == 0, r.stderr
    blocks = ref.generate_grid_pattern(176, 176, 16, 48, 81)
    exp = ref.conceal(img.astype(np.float64), blocks, 16, 16, gamma=0.5, iterations=40, t=64, rho_hat=0.8,
                      support=16)
    restored = read_pgm(out / "restored.pgm")
    np.testing.assert_array_equal(restored, np.clip(np.floor(exp["restored"] + 0.5), 0, 255).astype(np.uint8))
    damaged = read_pgm(out / "damaged.pgm")
    for (rr, cc, h, w) in blocks:
        assert (damaged[rr:rr + h, cc:cc + w] == 0).all()
    lines = (out / "report.csv").read_text().splitlines()
    assert lines[0] == fingerprint("conceal", tmp_path / "scene.pgm", gamma="0.5", iterations=40)
    assert lines[1] == "image,algorithm,gamma,iterations,psnr_db,sec_per_block"
    f = lines[2].split(",")
    assert f[:4] == ["scene.pgm", "fofse", "0.5", "40"]
    assert f[4] == "%.6f" % exp["psnr_db"]
    assert r.stdout.startswith("blocks=%d psnr_db=%.4f " % (len(blocks), exp["psnr_db"]))


@pytest.mark.gpu
def test_sweep_gamma_curves_match_the_reference(cli, gpu, ref, tmp_path):
    rng = np.random.default_rng(467)
    img = write_pgm(tmp_path / "s.pgm", smooth_test_image(rng, 128))
    pat = tmp_path / "pat.txt"
    blocks = [(16, 16, 16, 16), (16, 80, 16, 16), (80, 48, 16, 16)]
    pat.write_text("# 3 lost blocks\n" + "".join("%d %d %d %d\n" % b for b in blocks))
    out = tmp_path / "o"
    r = run(cli, "sweep-gamma", "--input", tmp_path / "s.pgm", "--gammas", "0.25,0.75", "--iterations", 30,
            "--stride", 10, "--pattern", pat, "--out-dir", out)
    assert r.returncode == 0, r.stderr
    for label, algo, g in [("fofse_g0.25", 2, 0.25), ("fofse_g0.75", 2, 0.75), ("fse", 0, 1.0), ("ofse", 1, 1.0)]:
        lines = (out / f"curve_{label}.csv").read_text().splitlines()
        assert lines[0] == fingerprint("sweep-gamma", tmp_path / "s.pgm", iterations=30, stride=10, pattern=pat)
        assert lines[1] == "iteration,psnr_db"
        pts = [tuple(x.split(",")) for x in lines[2:]]
        assert [int(p[0]) for p in pts] == [10, 20, 30]
        for it, db in pts:
            exp = ref.conceal(img.astype(np.float64), blocks, 16, 16, algorithm=algo, gamma=g, iterations=int(it),
                              t=64, rho_hat=0.8, support=16)
            assert float(db) == pytest.approx(exp["psnr_db"], rel=1e-8), (label, it)
        assert f"series={label} " in r.stdout


@pytest.mark.gpu
def test_extrapolate_writes_model_and_trace(cli, gpu, tmp_path):
    rng = np.random.default_rng(479)
    win = write_pgm(tmp_path / "w.pgm", smooth_test_image(rng, 48))
    out = tmp_path / "o"
    r = run(cli, "extrapolate", "--input", tmp_path / "w.pgm", "--iterations", 25, "--outside", "0,0,4,48",
            "--out-dir", out)
    assert r.returncode == 0, r.stderr
    lab = np.zeros((48, 48), np.uint8)
    lab[16:32, 16:32] = 1
    lab[0:4, :] = 2
    runs = P.extrapolate_windows(win[None].astype(np.float64), lab[None],
                                 P.ConcealConfig(iterations=25, record_traces=True))
    model = read_pgm(out / "extrapolated.pgm")
    np.testing.assert_array_equal(model, np.clip(np.floor(runs[0].model + 0.5), 0, 255).astype(np.uint8))
    lines = (out / "trace.csv").read_text().splitlines()
    assert lines[1] == "nu,u_k1,u_k2,p_abs,c_abs,gamma_effective,weighted_energy"
    rows = [x.split(",") for x in lines[2:]]
    assert len(rows) == 25
    assert [int(x[1]) for x in rows] == list(runs[0].trace["u1"])
    assert r.stdout.startswith("iterations=25 converged=false ")


# ---- JSON config (main.cpp:66-110,274-293): flags beat the file, the file beats defaults ----
def test_dump_config_defaults_and_flag_precedence(cli, tmp_path):
    import json
    r = run(cli, "conceal", "--input", "in.pgm", "--dump-config", "-")
    assert r.returncode == 0, r.stderr
    d = json.loads(r.stdout)
    assert d == {"algorithm": "fofse", "block": 16, "count_limit": 81, "fft_size": 64, "gamma": 0.2,
                 "input": "in.pgm", "iterations": 200, "out_dir": "", "pattern": "", "rho_hat": 0.8, "seed": 0,
                 "spacing": 48, "stride": 5, "support": 16, "threads": 1}
    assert list(d) == sorted(d) and r.stdout.startswith('{\n  "algorithm": "fofse",\n')
    cfg = tmp_path / "c.json"
    cfg.write_text('{"gamma": 0.5, "iterations": 50, "pattern": "p.txt", "seed": 7, "rho_hat": 1e-1}')
    out = tmp_path / "eff.json"
    r = run(cli, "conceal", "--input", "in.pgm", "--config", cfg, "--iterations", "80", "--dump-config", out)
    assert r.returncode == 0, r.stderr
    d = json.loads(out.read_text())
    assert (d["gamma"], d["iterations"], d["pattern"], d["seed"], d["rho_hat"]) == (0.5, 80, "p.txt", 7, 0.1)


def test_config_file_errors(cli, tmp_path):
    bad = tmp_path / "bad.json"
    bad.write_text('{"gamma": 0.5, "colour": 3}')
    r = run(cli, "conceal", "--input", "in.pgm", "--config", bad)
    assert r.returncode == 1 and "unknown key 'colour'" in r.stderr
    bad.write_text('{"gamma": 0.5,,}')
    r = run(cli, "conceal", "--input", "in.pgm", "--config", bad)
    assert r.returncode == 1 and "invalid JSON" in r.stderr
    bad.write_text('[1, 2]')
    r = run(cli, "conceal", "--input", "in.pgm", "--config", bad)
    assert r.returncode == 1 and "config must be a JSON object" in r.stderr
    r = run(cli, "conceal", "--input", "in.pgm", "--config", tmp_path / "nope.json")
    assert r.returncode == 2 and "cannot open config file" in r.stderr


def test_pattern_file_parsing_and_validation(cli, tmp_path):
    """pattern.cpp:55-96: comments and blank lines skipped, short lines rejected with
    the line number, bounds / overlap checked in load order (before any device work)."""
    img = tmp_path / "img.pgm"
    write_pgm(img, np.full((64, 64), 90.0))
    pat = tmp_path / "p.txt"
    pat.write_text("# lost blocks\n\n0 0 16 16\n16 16 16\n")
    r = run(cli, "conceal", "--input", img, "--pattern", pat, "--out-dir", tmp_path / "o")
    assert r.returncode == 2 and f"{pat}:4: expected 'row col height width'" in r.stderr
    pat.write_text("0 0 16 16  # first\n8 8 16 16\n")
    r = run(cli, "conceal", "--input", img, "--pattern", pat, "--out-dir", tmp_path / "o")
    assert r.returncode == 1 and "pattern: blocks 0 and 1 overlap" in r.stderr
    pat.write_text("0 0 16 16\n56 56 16 16\n")
    r = run(cli, "conceal", "--input", img, "--pattern", pat, "--out-dir", tmp_path / "o")
    assert r.returncode == 1 and "pattern: block 1 exceeds image bounds" in r.stderr
    pat.write_text("0 0 16 16\n32 32 8 8\n")
    r = run(cli, "conceal", "--input", img, "--pattern", pat, "--out-dir", tmp_path / "o")
    assert r.returncode == 1 and "pattern: blocks must share one size" in r.stderr
