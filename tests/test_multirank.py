"""Multi-rank sharding + final gather on CPU (gloo, world_size 2). The per-shard
compute is the oracle here (no GPU in this container); on the B200 box the same
code path runs fofse_conceal_shard_f64 per rank over NCCL."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch.distributed as dist

    import oracle
    import paper_2207_01205_b200 as P
    from paper_2207_01205_b200.distributed import conceal_sharded, shard_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(5)
        img = np.clip(np.round(128 + 60 * np.sin(0.1 * np.arange(160))[:, None] *
                               np.cos(0.08 * np.arange(160))[None, :] + rng.uniform(-4, 4, (160, 160))), 0, 255)
        blocks = [(16, 16, 16, 16), (16, 80, 16, 16), (64, 40, 16, 16), (112, 112, 16, 16), (0, 144, 16, 16)]
        pat = P.LossPattern(160, 160, 16, 16, [P.Rect(*b) for b in blocks])
        orc = oracle.Oracle()
        seen = []

        def compute(im, p, first, count, cfg):  # oracle stands in for the GPU shard
            seen.append((first, count))
            return orc.conceal(im, [tuple(b) for b in p.blocks], 16, 16, gamma=cfg.gamma,
                               iterations=cfg.iterations, t=64, rho_hat=0.8, support=16)["restored"]

        cfg = P.ConcealConfig(gamma=0.5, iterations=20)
        res = conceal_sharded(img, pat, cfg, compute=compute)
        b, e = shard_range(5, world, rank)
        assert seen == [(b, e - b)]
        if rank == 0:
            full = orc.conceal(img, blocks, 16, 16, gamma=0.5, iterations=20, t=64, rho_hat=0.8, support=16)
            out, db, ident = res
            q.put((np.array_equal(out, full["restored"]), abs(db - full["psnr_db"]) < 1e-9, ident))
        else:
            assert res is None
    finally:
        dist.destroy_process_group()


def test_shard_range_covers_all():
    from paper_2207_01205_b200.distributed import shard_range
    for n in (0, 1, 5, 102, 2040):
        for w in (1, 2, 3, 8):
            got = [shard_range(n, w, r) for r in range(w)]
            idx = [i for b, e in got for i in range(b, e)]
            assert idx == list(range(n))


def test_two_rank_gloo_gather_matches_single_run(oracle_mod):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    same, psnr_ok, ident = q.get(timeout=5)
    assert same and psnr_ok and not ident
