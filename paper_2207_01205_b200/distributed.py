"""Multi-GPU concealment: shard lost blocks (or whole frames) across ranks, one
final gather. Replaces the reference's parallel_blocks worker threads
(pipeline.cpp:136-162): blocks are independent (pipeline_test.cpp:213-222,
SURVEY §8e), so the only inter-GPU traffic is the gather of the concealed
B x B tiles. One process per GPU; torch.distributed (NCCL over NVLink on the
B200 box, gloo in the CPU tests) is plumbing only.

  shard_range(n, world, rank)   contiguous [begin, end) share of n units
  conceal_sharded(...)          one image, blocks sharded by index: each rank
                                conceals its shard, the tiles are packed on the
                                device (fofse_conceal_shard_tiles_f64) and
                                gathered to rank 0 in ONE collective
  SharedHost                    a POSIX shared-memory host buffer all local ranks
                                map (pinned with cudaHostRegister)
  conceal_frames_sharded(...)   video batch, whole frames per rank: every rank
                                runs fofse_conceal_frames_u8 on its frames of a
                                SharedHost batch; the D2H of each rank lands in
                                its disjoint region, so the gather is the
                                transfers themselves (no extra copy)
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _capi as capi
from .fse import ConcealConfig, LossPattern


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [begin, end) of n units for `rank` of `world` (ceil split)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    per = -(-n // world)
    b = min(n, rank * per)
    return b, min(n, b + per)


def local_device() -> int:
    """The GPU of this rank: LOCAL_RANK (torchrun), else the current device."""
    if "LOCAL_RANK" in os.environ:
        return int(os.environ["LOCAL_RANK"])
    import torch
    return torch.cuda.current_device() if torch.cuda.is_available() else 0


def shard_tiles(image: np.ndarray, pattern: LossPattern, first: int, count: int, config: ConcealConfig,
                out_ptr: int, on_device: bool, device: int):
    """Conceal blocks[first:first+count] of `image` (every block of the pattern
    stays lost) and write their tiles (count, bh, bw) f64 to out_ptr."""
    image = np.ascontiguousarray(image, np.float64)
    h, w = image.shape
    rects = capi.rects_array(pattern.blocks)
    rep = capi.Report()
    capi.check(capi.lib().fofse_conceal_shard_tiles_f64(
        capi.context(device).handle, capi.ptr(image), w, h, rects.ctypes.data_as(C.POINTER(capi.Rect_)),
        C.c_int64(len(rects)), C.c_int64(int(first)), C.c_int64(int(count)), pattern.block_height,
        pattern.block_width, C.byref(config.params()), C.cast(C.c_void_p(out_ptr), C.POINTER(C.c_double)),
        int(bool(on_device)), C.byref(rep)))
    return rep


def scatter_tiles(image: np.ndarray, pattern: LossPattern, tiles: np.ndarray) -> np.ndarray:
    """image with the (n, bh, bw) tiles written at the pattern's blocks (vectorised)."""
    out = np.array(image, np.float64, copy=True)
    n = len(pattern.blocks)
    if n == 0:
        return out
    bh, bw = pattern.block_height, pattern.block_width
    rc = np.array([(b.row, b.col) for b in pattern.blocks], np.int64)
    rows = rc[:, 0, None, None] + np.arange(bh)[None, :, None]
    cols = rc[:, 1, None, None] + np.arange(bw)[None, None, :]
    out[rows, cols] = tiles[:n]
    return out


def _psnr_missing(image: np.ndarray, out: np.ndarray, pattern: LossPattern):
    """PSNR over MISSING samples (grid.cpp:103-121; blocks are disjoint)."""
    n = len(pattern.blocks)
    if n == 0:
        return 0.0, True
    bh, bw = pattern.block_height, pattern.block_width
    rc = np.array([(b.row, b.col) for b in pattern.blocks], np.int64)
    rows = rc[:, 0, None, None] + np.arange(bh)[None, :, None]
    cols = rc[:, 1, None, None] + np.arange(bw)[None, None, :]
    d = image[rows, cols] - out[rows, cols]
    sq = float(np.sum(d * d))
    if sq == 0.0:
        return 0.0, True
    return 10.0 * np.log10(255.0 ** 2 / (sq / d.size)), False


def conceal_sharded(image: np.ndarray, pattern: LossPattern, config: ConcealConfig | None = None,
                    group=None, device: int | None = None, compute=None):
    """Rank r conceals blocks shard_range(n, world, r) (every block of the
    pattern stays lost, exactly as in a single-GPU run); the tiles are packed
    on the device and gathered to rank 0 in one collective; rank 0 returns
    (restored image, psnr_db, identical) like fse::conceal (pipeline.cpp:205-262).
    Other ranks return None.

    compute(image, pattern, first, count, config) -> (count, bh, bw) tiles
    replaces the GPU shard (CPU tests)."""
    import torch
    import torch.distributed as dist

    config = config or ConcealConfig()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = len(pattern.blocks)
    b0, b1 = shard_range(n, world, rank)
    bh, bw = pattern.block_height, pattern.block_width
    image = np.ascontiguousarray(image, np.float64)
    per = max(-(-n // world), 1)
    nccl = dist.get_backend(group) == "nccl"
    if compute is None:
        dev = local_device() if device is None else device
        send = torch.zeros((per, bh, bw), dtype=torch.float64,
                           device=torch.device("cuda", dev) if nccl else "cpu")
        if b1 > b0:
            shard_tiles(image, pattern, b0, b1 - b0, config, send.data_ptr(), nccl, dev)
    else:
        send = torch.zeros((per, bh, bw), dtype=torch.float64)
        if b1 > b0:
            send[: b1 - b0] = torch.from_numpy(np.ascontiguousarray(compute(image, pattern, b0, b1 - b0, config)))
        if nccl:
            send = send.cuda(local_device() if device is None else device)
    if rank != 0:
        dist.gather(send, None, dst=0, group=group)
        return None
    recv = [torch.empty_like(send) for _ in range(world)]
    dist.gather(send, recv, dst=0, group=group)
    tiles = torch.cat([recv[r][: shard_range(n, world, r)[1] - shard_range(n, world, r)[0]]
                       for r in range(world)]).cpu().numpy()
    out = scatter_tiles(image, pattern, tiles)
    db, ident = _psnr_missing(image, out, pattern)
    return out, db, ident


class SharedHost:
    """A host buffer every local rank maps (POSIX shared memory). Rank 0
    creates it and broadcasts its name; `pin(nbytes_offset, nbytes)` page-locks
    a range in this process (cudaHostRegister) so copies to and from it are
    DMA transfers. The frames API then reads each rank's frames from, and
    writes each rank's restored frames into, disjoint regions of the one
    buffer: after a barrier the caller sees the whole batch."""

    def __init__(self, nbytes: int, group=None):
        import torch.distributed as dist
        from multiprocessing import shared_memory

        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        name = [None]
        if self.rank == 0:
            self.shm = shared_memory.SharedMemory(create=True, size=max(int(nbytes), 1))
            name[0] = self.shm.name
        if dist.is_initialized():
            dist.broadcast_object_list(name, src=0, group=group)
        if self.rank != 0:
            self.shm = shared_memory.SharedMemory(name=name[0])
            try:  # the creator owns the segment's lifetime
                from multiprocessing import resource_tracker
                resource_tracker.unregister(self.shm._name, "shared_memory")
            except Exception:
                pass
        self.nbytes = int(nbytes)
        self._pinned = []

    def array(self, shape, dtype, offset: int = 0) -> np.ndarray:
        return np.ndarray(shape, dtype=dtype, buffer=self.shm.buf, offset=offset)

    def address(self, offset: int = 0) -> int:
        return C.addressof(C.c_char.from_buffer(self.shm.buf, offset))

    def pin(self, offset: int, nbytes: int):
        import torch
        if nbytes <= 0:
            return
        rc = torch._C._cudart.cudaHostRegister(self.address(offset), nbytes, 0)
        if int(rc) != 0:
            raise capi.FofseCudaError(f"cudaHostRegister failed ({int(rc)})")
        self._pinned.append(self.address(offset))

    def close(self):
        import torch
        for p in self._pinned:
            torch._C._cudart.cudaHostUnregister(p)
        self._pinned = []
        try:
            self.shm.close()
            if self.rank == 0:
                self.shm.unlink()
        except Exception:
            pass


def conceal_frames_sharded(ctx, frames_in: np.ndarray, frames_out: np.ndarray, rects: np.ndarray,
                           offsets: np.ndarray, block: tuple[int, int], params, world: int, rank: int,
                           block_sq: np.ndarray | None = None, report=None, call=None):
    """Rank `rank` conceals frames shard_range(F, world, rank) of the batch:
    frames_in / frames_out are (F, H, W) u8 views of shared host memory,
    rects / offsets the whole batch's blocks (frame f owns rects[offsets[f]:
    offsets[f+1]]). Each rank's restored frames land in its own region of
    frames_out — the gather. Returns (f0, f1). `call` replaces the GPU call
    (CPU tests): call(f0, f1, in_slice, out_slice, rects_slice, offs_slice)."""
    nf, h, w = frames_in.shape
    f0, f1 = shard_range(nf, world, rank)
    if f1 <= f0:
        return f0, f1
    r0, r1 = int(offsets[f0]), int(offsets[f1])
    sub_rects = np.ascontiguousarray(rects[r0:r1])
    sub_offs = np.ascontiguousarray(offsets[f0:f1 + 1] - offsets[f0], dtype=np.int64)
    if call is not None:
        call(f0, f1, frames_in[f0:f1], frames_out[f0:f1], sub_rects, sub_offs)
        return f0, f1
    rep = report if report is not None else capi.Report()
    sq = None if block_sq is None else block_sq[r0:r1]
    capi.check(capi.lib().fofse_conceal_frames_u8(
        ctx.handle, C.cast(frames_in[f0:f1].ctypes.data, C.POINTER(C.c_uint8)), f1 - f0, w, h,
        sub_rects.ctypes.data_as(C.POINTER(capi.Rect_)), capi.ptr(sub_offs, C.c_int64), block[0], block[1],
        C.byref(params), C.cast(frames_out[f0:f1].ctypes.data, C.POINTER(C.c_uint8)),
        None if sq is None else capi.ptr(sq), C.byref(rep)))
    return f0, f1
