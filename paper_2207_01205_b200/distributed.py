"""Multi-GPU concealment: shard lost blocks across ranks, gather at the end.

Blocks are independent (pipeline_test.cpp:213-222), so the only
inter-GPU traffic is the final gather of the concealed B x B tiles. One process
per GPU; torch.distributed (NCCL over NVLink on the B200 box, gloo in the CPU
tests) is plumbing only.

  shard_range(n, world, rank)   contiguous block-index shard (ceil(n / world))
  conceal_sharded(...)          per-rank fofse_conceal_shard_f64 + gather to rank 0
"""
from __future__ import annotations

import numpy as np

from .fse import ConcealConfig, LossPattern, conceal_shard


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [begin, end) of n units for `rank` of `world` (ceil split)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    per = -(-n // world)
    b = min(n, rank * per)
    return b, min(n, b + per)


def conceal_sharded(image: np.ndarray, pattern: LossPattern, config: ConcealConfig | None = None,
                    group=None, device: int | None = None, compute=None):
    """Rank r conceals blocks shard_range(n, world, r) (every block of the
    pattern stays lost, exactly as in a single-GPU run); rank 0 gathers the
    tiles and returns (restored image, psnr_db, identical) like fse::conceal
    (pipeline.cpp:205-262). Other ranks return None.
    compute(image, pattern, first, count, config) -> restored image defaults to
    the GPU shard entry point on `device`."""
    import torch
    import torch.distributed as dist

    config = config or ConcealConfig()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = len(pattern.blocks)
    b0, b1 = shard_range(n, world, rank)
    bh, bw = pattern.block_height, pattern.block_width
    image = np.ascontiguousarray(image, np.float64)
    if compute is None:
        dev = device if device is not None else 0
        compute = lambda im, p, f, c, cfg: conceal_shard(im, p, f, c, cfg, device=dev)[0]  # noqa: E731
    restored = compute(image, pattern, b0, b1 - b0, config)
    per = -(-n // world) if n else 1
    send = torch.zeros((per, bh, bw), dtype=torch.float64)
    for i, blk in enumerate(pattern.blocks[b0:b1]):
        send[i] = torch.from_numpy(np.ascontiguousarray(restored[blk.row:blk.row + bh, blk.col:blk.col + bw]))
    if dist.get_backend(group) == "nccl":
        send = send.cuda()
    if rank != 0:
        dist.gather(send, None, dst=0, group=group)
        return None
    recv = [torch.zeros_like(send) for _ in range(world)]
    dist.gather(send, recv, dst=0, group=group)
    out = image.copy()
    for r in range(world):
        rb0, rb1 = shard_range(n, world, r)
        t = recv[r].cpu().numpy()
        for i in range(rb1 - rb0):
            blk = pattern.blocks[rb0 + i]
            out[blk.row:blk.row + bh, blk.col:blk.col + bw] = t[i]
    lost = np.zeros(image.shape, bool)
    for blk in pattern.blocks:
        lost[blk.row:blk.row + bh, blk.col:blk.col + bw] = True
    if n == 0:
        return out, 0.0, True
    d = image[lost] - out[lost]  # psnr over MISSING samples (grid.cpp:103-121)
    sq = float(np.sum(d * d))
    if sq == 0.0:
        return out, 0.0, True
    return out, 10.0 * np.log10(255.0 ** 2 / (sq / int(lost.sum()))), False
