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
            full = orc.conceal(im, [tuple(b) for b in p.blocks], 16, 16, gamma=cfg.gamma,
                               iterations=cfg.iterations, t=64, rho_hat=0.8, support=16)["restored"]
            return np.stack([full[b.row:b.row + 16, b.col:b.col + 16] for b in p.blocks[first:first + count]])

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


def _frames_worker(rank, world, port, q):
    """Frame shards of one batch in shared host memory: each rank writes its
    restored frames into its own region; rank 0 then sees the whole batch."""
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_2207_01205_b200 import _capi as capi
    from paper_2207_01205_b200.distributed import SharedHost, conceal_frames_sharded, shard_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nf, h, w = 5, 48, 64
        shm_in, shm_out = SharedHost(nf * h * w), SharedHost(nf * h * w)
        fin = shm_in.array((nf, h, w), np.uint8)
        fout = shm_out.array((nf, h, w), np.uint8)
        if rank == 0:
            fin[:] = (np.arange(nf * h * w) % 251).reshape(nf, h, w)
            fout[:] = 0
        dist.barrier()
        offs = np.array([0, 2, 3, 3, 5, 6], np.int64)
        rects = np.zeros(6, capi.RECT_DTYPE)
        rects["row"] = [0, 16, 32, 0, 16, 32]
        rects["col"] = [0, 16, 32, 48, 0, 16]
        rects["height"] = rects["width"] = 16
        calls = []

        def call(f0, f1, a, b, r, o):  # stands in for fofse_conceal_frames_u8
            calls.append((f0, f1, len(r), o.tolist()))
            b[:] = a
            for f in range(f1 - f0):
                for k in range(o[f], o[f + 1]):
                    b[f, r["row"][k]:r["row"][k] + 16, r["col"][k]:r["col"][k] + 16] = 255 - (f0 + f)

        f0, f1 = conceal_frames_sharded(None, fin, fout, rects, offs, (16, 16), None, world, rank, call=call)
        assert (f0, f1) == shard_range(nf, world, rank)
        assert calls and calls[0][2] == offs[f1] - offs[f0] and calls[0][3][0] == 0
        dist.barrier()
        if rank == 0:
            ref = fin.copy()
            for f in range(nf):
                for k in range(offs[f], offs[f + 1]):
                    ref[f, rects["row"][k]:rects["row"][k] + 16, rects["col"][k]:rects["col"][k] + 16] = 255 - f
            q.put(bool(np.array_equal(fout, ref)))
        dist.barrier()
        del fin, fout
        shm_in.close()
        shm_out.close()
    finally:
        dist.destroy_process_group()


def test_two_rank_frame_shards_gather_in_shared_host_memory():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_frames_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5)


def test_scatter_tiles_vectorised():
    import paper_2207_01205_b200 as P
    from paper_2207_01205_b200.distributed import scatter_tiles
    img = np.zeros((40, 40))
    pat = P.LossPattern(40, 40, 8, 8, [P.Rect(0, 0, 8, 8), P.Rect(16, 24, 8, 8)])
    tiles = np.stack([np.full((8, 8), 3.0), np.arange(64.0).reshape(8, 8)])
    out = scatter_tiles(img, pat, tiles)
    assert (out[:8, :8] == 3).all() and np.array_equal(out[16:24, 24:32], tiles[1])
    assert out.sum() == 3 * 64 + tiles[1].sum()


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
