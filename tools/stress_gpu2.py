"""Randomised GPU stress, second sweep (not a unit test): blocks at arbitrary
(non grid-aligned) positions, rectangular blocks, non-square images, generic
transform sizes (36, 40, 96), the DCT basis (vs the compiled reference when
oracle/_ref is present), and the frames API with frame groups (>= 16 frames,
u8 and f64, both precisions) against the image path frame by frame.

usage: python tools/stress_gpu2.py [cases] [seed]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle  # test infrastructure (the checker)
import paper_2207_01205_b200 as P


def image(rng, h, w):
    y, x = np.mgrid[0:h, 0:w]
    f = 110 + 45 * np.cos(2 * np.pi * x / rng.uniform(15, 80) + rng.uniform(0, 6)) * np.sin(
        2 * np.pi * y / rng.uniform(15, 80)) + 25 * (y > rng.integers(0, h)) + rng.normal(0, 2.5, (h, w))
    return np.clip(np.round(f), 0, 255)


def random_blocks(rng, h, w, bh, bw, n):
    """n non-overlapping blocks at arbitrary positions (rejection sampling)."""
    taken = np.zeros((h, w), bool)
    out = []
    for _ in range(20 * n):
        if len(out) == n:
            break
        r, c = int(rng.integers(0, h - bh + 1)), int(rng.integers(0, w - bw + 1))
        if taken[r:r + bh, c:c + bw].any():
            continue
        taken[r:r + bh, c:c + bw] = True
        out.append((r, c, bh, bw))
    return out


def main(cases=80, seed=3):
    rng = np.random.default_rng(seed)
    orc = oracle.Oracle()
    ref = oracle.Reference() if oracle.have_reference() else None
    fails, worst = [], {"f64": 0.0, "f32": 0.0, "dct": 0.0, "frames": 0.0}
    for c in range(cases):
        kind = rng.choice(["free", "free", "generic", "dct", "frames"])
        try:
            if kind == "frames":
                t, b, s = 64, 16, 16
                nf = int(rng.integers(16, 40))
                h, w = int(rng.choice([96, 128, 160])), int(rng.choice([128, 192]))
                frames = np.stack([image(rng, h, w) for _ in range(nf)])
                pats = [P.LossPattern(w, h, b, b, [P.Rect(*x) for x in random_blocks(rng, h, w, b, b,
                                                                                     int(rng.integers(1, 8)))])
                        for _ in range(nf)]
                prec = str(rng.choice(["fp32", "fp64"]))
                cfg = P.ConcealConfig(gamma=0.5, iterations=int(rng.choice([30, 120])), transform_size=t,
                                      support_width=s, precision=prec)
                u8, _, _ = P.conceal_frames(frames.astype(np.uint8), pats, cfg)
                f64, _, _ = P.conceal_frames(frames, pats, cfg)
                d = 0.0
                # u8 = the same pipeline rounded (fp32: the image path may take another kernel
                # form, so its fp32 noise may flip a rounding: compared unrounded)
                if not np.array_equal(np.clip(np.floor(f64 + 0.5), 0, 255).astype(np.uint8), u8):
                    d = 1.0
                for f in range(0, nf, 5):
                    one = P.conceal(frames[f], pats[f], cfg).restored
                    d = max(d, float(np.abs(f64[f] - one).max()))
                worst["frames"] = max(worst["frames"], d)
                bad = d > (1e-9 if prec == "fp64" else 0.05)
                print(f"case {c:3d} frames {nf} x {h}x{w} {prec}: batch vs image {d:.2e}{'  <-- FAIL' if bad else ''}",
                      flush=True)
                if bad:
                    fails.append((c, kind, d))
                continue
            if kind == "generic":
                t = int(rng.choice([36, 40, 96]))
                b = int(rng.choice([8, 12, 16]))
                s = max(2, (t - b) // 2 - int(rng.integers(0, 3)))
                bh = bw = b
            else:
                t = int(rng.choice([16, 32, 64, 128]))
                s = {16: 4, 32: 8, 64: 16, 128: 16}[t]
                bh = int(rng.choice([b for b in (4, 8, 16, 32, 64) if b + 2 * s <= t]))
                bw = int(rng.choice([b for b in (4, 8, 16, 32, 64) if b + 2 * s <= t]))
            h, w = int(rng.integers(3, 9)) * max(bh, 16), int(rng.integers(3, 9)) * max(bw, 16)
            img = image(rng, h, w)
            blocks = random_blocks(rng, h, w, bh, bw, int(rng.integers(1, 14)))
            pat = P.LossPattern(w, h, bh, bw, [P.Rect(*x) for x in blocks])
            its = int(rng.choice([5, 40, 120]))
            kw = dict(gamma=float(rng.choice([0.3, 0.5])), iterations=its, transform_size=t,
                      rho_hat=float(rng.choice([0.75, 0.85])), support_width=s)
            if kind == "dct":
                if ref is None:
                    continue
                kw["transform_size"] = t = int(rng.choice([16, 32]))
                kw["support_width"] = s = {16: 4, 32: 8}[t]
                bh = bw = 8
                blocks = random_blocks(rng, h, w, 8, 8, int(rng.integers(1, 8)))
                pat = P.LossPattern(w, h, 8, 8, [P.Rect(*x) for x in blocks])
                out = P.conceal(img, pat, P.ConcealConfig(basis="dct2d", **kw))
                r = ref.conceal(img, blocks, 8, 8, gamma=kw["gamma"], iterations=its, t=t, rho_hat=kw["rho_hat"],
                                support=s, basis=1)
                d = float(np.abs(out.restored - r["restored"]).max())
                worst["dct"] = max(worst["dct"], d)
                bad = d > 1e-9
                print(f"case {c:3d} dct T={t} {h}x{w} blocks={len(blocks)} I={its}: vs reference {d:.2e}"
                      f"{'  <-- FAIL' if bad else ''}", flush=True)
                if bad:
                    fails.append((c, kind, d))
                continue
            o64 = P.conceal(img, pat, P.ConcealConfig(**kw))
            r = orc.conceal(img, blocks, bh, bw, gamma=kw["gamma"], iterations=its, t=t, rho_hat=kw["rho_hat"],
                            support=s)
            d64 = float(np.abs(o64.restored - r["restored"]).max())
            d32 = 0.0
            if kind != "generic":
                o32 = P.conceal(img, pat, P.ConcealConfig(precision="fp32", **kw))
                d32 = float(np.abs(o32.restored - o64.restored).max())
            worst["f64"], worst["f32"] = max(worst["f64"], d64), max(worst["f32"], d32)
            bad = d64 > 1e-9 or d32 > 0.5
            print(f"case {c:3d} {kind:7s} T={t:3d} blk={bh}x{bw} S={s} {h}x{w} blocks={len(blocks)} I={its}: "
                  f"fp64-oracle {d64:.2e} fp32-fp64 {d32:.3f}{'  <-- FAIL' if bad else ''}", flush=True)
            if bad:
                fails.append((c, kind, t, bh, bw, d64, d32))
        except Exception as e:
            fails.append((c, kind, repr(e)[:160]))
            print(f"case {c:3d} {kind}: EXCEPTION {repr(e)[:160]}", flush=True)
    print(f"worst: {worst}; failures: {len(fails)}")
    for f in fails:
        print("FAIL", f)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 80, int(sys.argv[2]) if len(sys.argv) > 2 else 3)
