#!/usr/bin/env python3
"""FOFSE block-concealment benchmark (BASELINE.json metric: lost blocks
extrapolated per second at 16x16 blocks, 64^2 FFT, 200 iterations).

Workload: BASELINE config C4 — ONE batch of 256 synthetic 1920x1088 frames,
10 % isolated 16x16 losses per frame (208,896 blocks), rho 0.8, gamma 0.5, 200
iterations, fp32 fast mode. Under torchrun the batch is sharded by frame
across the ranks (strong scaling): rank r conceals frames
shard_range(256, N, r); there is no data-path collective, the final gather is
each rank's D2H into its region of the caller's shared host batch.

  value : blocks/s with the frames resident in HBM (plan/execute, kernels only)
  e2e   : blocks/s through the public C ABI call with pinned HOST buffers
          (H2D frames + host prep + kernels + D2H restored frames every step)
  parity: fp32 vs the fp64 path over every frame of rank 0 (outside the timed
          regions): max |px|, blocks above 0.5 px, |dPSNR| (north_star fp32 bar)
  detail.fp64: the same batch and harness in fp64 (the reference's precision)

`--impl reference` runs the reference's own CPU implementation (the
unmodified reference sources compiled as oracle/_ref, fse::conceal with all
host threads) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "lost blocks extrapolated/sec (16x16, 64^2 FFT, 200 it) and % of SMEM/FP roofline"
UNIT = "blocks/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="C4")
    ap.add_argument("--frames", type=int, default=None, help="frames of the batch (default: config)")
    ap.add_argument("--precision", default=None)
    ap.add_argument("--seed", type=int, default=2207)
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU baseline sample budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--parity-frames", type=int, default=None, help="parity over the first n frames (default all)")
    ap.add_argument("--no-fp64", action="store_true", help="skip the fp64 (reference precision) detail")
    # diagnostics only (not the BASELINE configuration): guard threshold / fp64 head overrides
    ap.add_argument("--guard-tau", type=float, default=None)
    ap.add_argument("--fp64-head", type=int, default=None)
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
# clocks sampled during the timed region (B200_PROFILING.md "clocks" line)
# ---------------------------------------------------------------------------
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.25)
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                p = [x.strip() for x in line.split(",")]
                if len(p) < 9:
                    continue
                try:
                    s, m = float(p[1]), float(p[2])
                except ValueError:
                    continue
                sm.append(s)
                mx = max(mx, m)
                for n, v in zip(names, p[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
        except Exception:
            pass
        busy = [s for s in sm if s > 0.5 * mx] if mx else sm
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU reference arm
# ---------------------------------------------------------------------------
def cpu_reference_rate(wl, seed, budget_s, threads):
    """Reference fse::conceal (oracle/_ref) on whole frames until ~budget_s."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle  # checker / CPU baseline only

    kind = "reference"
    if oracle.have_reference():
        impl = oracle.Reference()
    else:
        impl, kind = oracle.Oracle(), "port"
        threads = 1
    cfg = wl.config("fp64")
    blocks_done, secs, frames = 0, 0.0, 0
    f = 0
    while (frames == 0 or secs < budget_s) and f < max(wl.frames, 1) * 4:
        img, pat = wl.frame(seed + 100000, f)
        t0 = time.perf_counter()
        impl.conceal(img.astype(np.float64), [tuple(b) for b in pat.blocks], wl.block, wl.block,
                     gamma=cfg.gamma, iterations=cfg.iterations, t=cfg.transform_size,
                     rho_hat=cfg.rho_hat, support=cfg.support_width, threads=threads)
        secs += time.perf_counter() - t0
        blocks_done += len(pat.blocks)
        frames += 1
        f += 1
    return {"value": blocks_done / secs, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"{frames} frame(s) of {wl.name} = {blocks_done} blocks, fse::conceal fp64, "
                      f"{threads} threads, {secs:.1f} s"}


def cpu_reference_1thread(wl, seed, nblocks=160):
    """One host thread, the first `nblocks` lost blocks of one frame (SURVEY §8d
    asks for a 1-thread figure beside the all-core baseline)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle  # checker / CPU baseline only

    impl = oracle.Reference() if oracle.have_reference() else oracle.Oracle()
    cfg = wl.config("fp64")
    img, pat = wl.frame(seed + 100000, 0)
    blocks = [tuple(b) for b in pat.blocks[:nblocks]]
    t0 = time.perf_counter()
    impl.conceal(img.astype(np.float64), blocks, wl.block, wl.block, gamma=cfg.gamma,
                 iterations=cfg.iterations, t=cfg.transform_size, rho_hat=cfg.rho_hat,
                 support=cfg.support_width, threads=1)
    secs = time.perf_counter() - t0
    return {"value": len(blocks) / secs, "unit": UNIT, "cores": 1,
            "sample": f"{len(blocks)} blocks of one {wl.name} frame, 1 thread, {secs:.1f} s"}


def run_reference_arm(args, wl):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_reference_rate(wl, args.seed, 0.0, threads)  # one frame each
    vals = []
    base = None
    for _ in range(args.steps):
        base = cpu_reference_rate(wl, args.seed, args.cpu_seconds / max(args.steps, 1), threads)
        vals.append(base["value"])
    value = statistics.mean(vals)
    from paper_2207_01205_b200 import _capi as capi  # generator library only (libfofse_gen.so)
    total_blocks = sum(len(capi.gen_losses(args.seed + f, wl.width // wl.block, wl.height // wl.block,
                                           wl.loss_frac, wl.block, wl.block)) for f in range(wl.frames))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator, SURVEY §8d)",
        "config": config_dict(wl, total_blocks),
        "cpu_baseline": dict(base, value=value),
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def timed_steps(fn, steps, stream, barrier):
    """K calls of fn bracketed by a barrier + synchronize on both sides; CUDA
    events on the launching stream; returns (ms per step, per-call results)."""
    import torch
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    ev0.record(stream)
    out = [fn() for _ in range(steps)]
    ev1.record(stream)
    barrier()
    return ev0.elapsed_time(ev1) / steps, out


def main():
    args = parse()
    from paper_2207_01205_b200 import workloads as WL

    wl = WL.ALL[args.workload]
    if args.frames is not None:
        import dataclasses
        wl = dataclasses.replace(wl, frames=args.frames)
    if args.impl == "reference":
        run_reference_arm(args, wl)
        return

    import torch

    world, rank, local = dist_env()
    backend = os.environ.get("FOFSE_DIST_BACKEND", "nccl")  # gloo: functional runs of N ranks on one GPU
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    if backend != "nccl":
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    import paper_2207_01205_b200 as P
    from paper_2207_01205_b200 import _capi as capi
    from paper_2207_01205_b200 import build as native
    from paper_2207_01205_b200 import distributed as D

    if not os.path.exists(capi.LIB_PATH):
        native.build()
    L = capi.lib()
    prec = args.precision or wl.precision
    cfg = wl.config(prec)
    if args.guard_tau is not None:
        cfg.guard_tau = args.guard_tau
    if args.fp64_head is not None:
        cfg.fp64_head = args.fp64_head
    params = cfg.params()

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    # ---- inputs: ONE batch (BASELINE C4), whole frames sharded across ranks (strong scaling) ----
    nf_all = wl.frames
    f0, f1 = D.shard_range(nf_all, world, rank)
    nf = f1 - f0
    t0 = time.time()
    shm_in = shm_out = None
    if world > 1:
        # the caller's batch lives in shared host memory: every rank uploads its
        # frames from it and downloads its restored frames into its own region
        fb = wl.height * wl.width
        shm_in, shm_out = D.SharedHost(nf_all * fb), D.SharedHost(nf_all * fb)
        h_all_in = shm_in.array((nf_all, wl.height, wl.width), np.uint8)
        h_all_out = shm_out.array((nf_all, wl.height, wl.width), np.uint8)
        frames_np, rects, offs = wl.batch(args.seed, frames=nf, first=f0, out=h_all_in[f0:f1])
    else:
        frames_np, rects, offs = wl.batch(args.seed, frames=nf, first=f0)
    gen_s = time.time() - t0
    n_blocks = int(offs[-1])
    fbytes = frames_np.nbytes

    ctx = capi.Context(local)
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)
    rects_c = rects.ctypes.data_as(C.POINTER(capi.Rect_))

    def device_arm(prm):
        """plan once, execute K times on frames resident in HBM"""
        plan = C.c_void_p()
        capi.check(L.fofse_plan_frames_u8(ctx.handle, nf, wl.width, wl.height, rects_c, capi.ptr(offs, C.c_int64),
                                          wl.block, wl.block, C.byref(prm), C.byref(plan)))
        d_frames = torch.from_numpy(frames_np).to(dev)
        d_sq = torch.zeros(max(n_blocks, 1), dtype=torch.float64, device=dev)

        def execute():
            r = capi.Report()
            capi.check(L.fofse_plan_execute_device(plan, C.c_void_p(d_frames.data_ptr()), capi.ptr_dev(d_sq),
                                                   C.byref(r)))
            return r

        first = None
        for i in range(args.warmup):
            r = execute()
            first = first or r
        torch.cuda.synchronize()
        ms, reps = timed_steps(execute, args.steps, stream, barrier)
        L.fofse_plan_destroy(plan)
        del d_frames, d_sq
        return ms, reps, first

    # ---- end-to-end: the public frames call with HOST buffers (H2D + host prep +
    # kernels + D2H every step); at N > 1 each rank's D2H lands in its region of
    # the shared output batch — the gather ----
    if world > 1:
        h_in, h_out = h_all_in, h_all_out
        shm_in.pin(f0 * fbytes // max(nf, 1) if nf else 0, fbytes)
        shm_out.pin(f0 * fbytes // max(nf, 1) if nf else 0, fbytes)
        rects_all = offs_all = None
    else:
        h_in_t = torch.from_numpy(frames_np).pin_memory()
        h_out_t = torch.empty_like(h_in_t).pin_memory()
        h_in, h_out = h_in_t.numpy(), h_out_t.numpy()
    h_sq = np.zeros(max(n_blocks, 1), np.float64)

    def e2e_arm(prm):
        rep = capi.Report()

        def call():
            if nf == 0:
                return rep
            capi.check(L.fofse_conceal_frames_u8(
                ctx.handle, C.cast(h_in[f0:f1].ctypes.data if world > 1 else h_in.ctypes.data, C.POINTER(C.c_uint8)),
                nf, wl.width, wl.height, rects_c, capi.ptr(offs, C.c_int64), wl.block, wl.block, C.byref(prm),
                C.cast(h_out[f0:f1].ctypes.data if world > 1 else h_out.ctypes.data, C.POINTER(C.c_uint8)),
                capi.ptr(h_sq), C.byref(rep)))
            return capi.Report.from_buffer_copy(rep)

        for _ in range(max(1, min(args.warmup, 2))):
            call()
        psnr = rep.psnr_db
        wall = []

        def step():
            t = time.perf_counter()
            r = call()
            wall.append((time.perf_counter() - t) * 1e3)
            return r

        ms, reps = timed_steps(step, args.steps, stream, barrier)
        return ms, reps, psnr, wall

    with ClockSampler(local) as clk:
        ms, reps, first = device_arm(params)
    clocks = clk.summary()
    e2e_ms, e2e_reps, e2e_psnr, e2e_wall = e2e_arm(params)

    # ---- reference precision (fp64) on the same batch and harness ----
    f64 = None
    if prec == "fp32" and not args.no_fp64:
        p64 = wl.config("fp64").params()
        ms64, reps64, _ = device_arm(p64)
        e2e64, _, _, _ = e2e_arm(p64)
        f64 = [ms64, e2e64, statistics.mean(r.total_ms for r in reps64) if reps64 else 0.0]

    def mean(xs):
        xs = list(xs)
        return statistics.mean(xs) if xs else 0.0

    # ---- max over ranks ----
    vals = [ms, e2e_ms, mean(r.iterate_ms for r in reps), mean(r.real_iterate_ms for r in reps),
            mean(r.k1_ms for r in reps)] + (f64[:2] if f64 else [0.0, 0.0])
    t = torch.tensor(vals, dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
    nb = torch.tensor([float(n_blocks)], dtype=torch.float64, device=t.device)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(nb)
    total_blocks = int(nb.item())
    ms, e2e_ms, k2_avg, real_avg, k1_avg, ms64, e2e64 = (float(x) for x in t.tolist())
    launches = sum(r.kernel_launches for r in reps)
    real_blocks = reps[-1].real_blocks if reps else 0
    head = reps[-1].fp64_head if reps else 0

    # ---- fp32 parity vs the fp64 path on this rank's frames (outside the timed regions) ----
    parity = None
    if rank == 0 and prec == "fp32" and not args.no_parity:
        from paper_2207_01205_b200 import parity as PAR
        try:
            pf = nf if args.parity_frames is None else min(nf, args.parity_frames)
            import dataclasses
            pc = wl.config("fp32")
            pc.guard_tau, pc.fp64_head = params.guard_tau, params.fp64_head
            pr = PAR.fp32_vs_fp64(dataclasses.replace(wl, frames=pf), args.seed + f0, cfg32=pc, device=local,
                                  per_call=64)
            parity = {"frames": pr["frames"], "blocks": pr["blocks"], "max_px": pr["max_px"],
                      "blocks_over_0.5": pr["blocks_over_0.5"], "dpsnr_db": pr["dpsnr_db"],
                      "max_frame_dpsnr_db": pr["max_frame_dpsnr_db"], "guard_reruns": pr["guard_reruns"],
                      "bar": "max |px| <= 0.5 and |dPSNR| <= 0.05 dB vs the fp64 path (oracle-pinned)",
                      "pass": pr["blocks_over_0.5"] == 0 and pr["dpsnr_db"] <= 0.05,
                      "how": "every frame concealed through the timed batch path (fofse_conceal_frames_f64: "
                             "same plan, chunk pipeline and kernels as the u8 frames API, unrounded pixels out), "
                             "64 frames per call, in fp32 (the timed params) and fp64; pixels compared block by block"}
        except Exception as e:  # reported, never fatal
            parity = {"error": str(e)}

    if rank == 0:
        H = wl.transform_size ** 2 // 2 + 2
        s = 4 if prec == "fp32" else 8
        its = wl.iterations - (head if prec == "fp32" else 0)
        if prec == "fp32" and real_avg > 0:
            alg_bytes = 4 * s * H * its * real_blocks
            achieved = alg_bytes / (real_avg * 1e-3) / 1e9
        else:
            alg_bytes = 4 * s * H * wl.iterations * n_blocks
            achieved = alg_bytes / (k2_avg * 1e-3) / 1e9
        peaks = load_peaks()
        for kind, key in ((0, "smem_gbs"), (3, "dfma_tflops")):
            try:  # live, same box
                peaks[key] = capi.microbench(local, kind)
            except Exception:
                pass
        peak = peaks.get("smem_gbs")
        T = wl.transform_size
        k32 = (f"fofse::k2v2h_kernel<{T}>" if T == 128
               else f"fofse::k2v2r_kernel<{T}>" + (" or k2v2h_kernel<64> (jobs of about one wave)" if T == 64 and n_blocks < 8192 else ""))
        kname = (f"{k32} (fp32 rotated-frame iterate + fused synthesis)" if prec == "fp32"
                 else f"fofse::k2d_kernel<{T}> / k2_kernel (fp64 iterate + fused synthesis)")
        roof = {"bound": "smem", "kernel": kname,
                "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if peak else None,
                "traffic": (peaks["dram_per_unit"][wl.name] * its * (real_blocks if prec == "fp32" else n_blocks)
                            if wl.name in peaks.get("dram_per_unit", {}) and prec == "fp32" else None),
                "per_unit": f"4*s*H = {4 * s * H} B per block-iteration (s={s}, H={H}); "
                            f"{its} {prec} iterations x {real_blocks if prec == 'fp32' else n_blocks} blocks per step",
                "peak_source": "measured live by fofse_microbench(kind=0): conflict-free LDS.64, 148 SMs",
                "traffic_source": "ncu --set full dram__bytes_read.sum + dram__bytes_write.sum of this kernel, per "
                                  "block-iteration x the units of one step (profiles/peaks.json)",
                "note": "the iteration kernel is bound by on-chip shared-memory bandwidth / issue, not by HBM or "
                        "tensor cores (GEMM-free: shifted complex updates + argmax)",
                "timing": "summed CUDA-event durations of the kernel's launches on its stream; where the pipeline "
                          "runs other kernels beside it (C5: the previous chunk's guard re-runs and the next "
                          "chunk's preparation) the SMs are shared and this understates the kernel's own rate"}
        # K1: window gather + weighted forward FFT in fp64 (2.5 T^2 log2(T^2)
        # flops per block for the real-input 2-D FFT + 3 per window sample for w f and w f^2)
        if prec == "fp32" and k1_avg > 0:
            Lw = wl.window
            k1_flops = 2.5 * T * T * math.log2(T * T) + 3 * Lw * Lw
            k1_ach = k1_flops * real_blocks / (k1_avg * 1e-3) / 1e12
            k1_name = ("fofse::k1p_kernel (persistent register FFT, cp.async-staged windows, fp64)"
                       if T == 64 and wl.window <= 48 else
                       f"fofse::k1f_kernel<{T}> (register FFT, fp64)" if T <= 64 else "fofse::k1w_kernel")
            roof["k1"] = {"kernel": k1_name,
                          "bound": "fp64", "achieved": k1_ach, "peak": peaks.get("dfma_tflops"), "unit": "TFLOP/s",
                          "frac": k1_ach / peaks["dfma_tflops"] if peaks.get("dfma_tflops") else None,
                          "per_unit": f"{k1_flops:.0f} flop per block x {real_blocks} blocks",
                          "ms_per_step": k1_avg,
                          "peak_source": "measured live by fofse_microbench(kind=3): DFMA, 148 SMs",
                          "timing": "CUDA events around K1 inside the concurrent chunk pipeline (it shares the SMs "
                                    "with the border chunks and guard re-runs): a lower bound of its own rate; "
                                    "K1 alone, serialised under ncu: profiles/r02_launches_C4.txt; issue / shared-memory / barrier "
                                    "bound, not DFMA (profiles/r02_ncu_k1p_full.txt)"}
            roof["k3"] = {"kernel": "fused into the iteration kernel's epilogue (sparse synthesis of the B x B hole "
                                    "from <= 2I records + clamp + write-back); no separate launch — its time is "
                                    "inside the K2 figure above, its share is in profiles/r02_k3_share.txt"}
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            try:
                cpu = cpu_reference_rate(wl, args.seed, args.cpu_seconds, os.cpu_count() or 1)
                cpu["one_thread"] = cpu_reference_1thread(wl, args.seed)
            except Exception as e:  # baseline is reported, never required
                cpu = {"error": str(e)}
        detail = {"k2_ms": k2_avg, "k1_ms": k1_avg, "init_ms": mean(r.init_ms for r in reps),
                  "guard_reruns_per_step": mean(r.guard_reruns for r in reps),
                  "psnr_db": first.psnr_db if first else None, "e2e_psnr_db": e2e_psnr,
                  "classes": first.classes if first else None, "input_gen_s": gen_s,
                  "real_blocks": real_blocks, "real_iterate_ms": real_avg, "fp64_head": head,
                  "frames_rank0": [f0, f1],
                  # library-side device span (first to last event of run_job) and host wall
                  # time per e2e call: the gap is host preparation + transfers
                  "device_total_ms": mean(r.total_ms for r in reps),
                  "e2e_device_total_ms": mean(r.total_ms for r in e2e_reps), "e2e_wall_ms": mean(e2e_wall)}
        if f64:
            detail["fp64"] = {"value": total_blocks / (ms64 * 1e-3), "unit": UNIT, "ms_per_step": ms64,
                              "e2e": {"value": total_blocks / (e2e64 * 1e-3), "unit": UNIT},
                              "note": "the same batch and harness in fp64 (the reference's precision; same "
                                      "selected-basis sequence as the oracle)"}
        line = {
            "metric": METRIC, "value": total_blocks / (ms * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32" if prec == "fp32" else "f64",
            "data": "synthetic (seeded generator, SURVEY §8d; see DESIGN.md)",
            "config": config_dict(wl, total_blocks),
            "e2e": {"value": total_blocks / (e2e_ms * 1e-3), "unit": UNIT,
                    "h2d_bytes_per_step": nf_all * wl.width * wl.height + rects.nbytes * 0 + 16 * total_blocks
                                          + 8 * (nf_all + 1),
                    "d2h_bytes_per_step": nf_all * wl.width * wl.height + 8 * total_blocks,
                    "note": "whole-job bytes: frames + block rects + frame offsets in, restored frames + per-block "
                            "squared errors out" + ("; each rank's D2H lands in its region of the shared host "
                                                    "batch (the gather)" if world > 1 else "")},
            "roofline": roof,
            "cpu_baseline": cpu,
            "parity": parity,
            "clocks": clocks,
            "gpu_launches": launches,
            "parallelism": f"{world} rank(s), whole frames sharded by index ({nf} frames on rank 0), "
                           f"no data-path collective; final gather = D2H into disjoint host regions",
            "detail": detail,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        del h_in, h_out, h_all_in, h_all_out, frames_np
        import torch.distributed as dist
        dist.barrier()
        shm_in.close()
        shm_out.close()
        dist.destroy_process_group()


def config_dict(wl, total_blocks):
    """The workload, identical for both arms (the driver compares them)."""
    return {"workload": wl.name,
            "description": f"{wl.frames} frame(s) of {wl.width}x{wl.height}, {wl.loss_frac:.0%} isolated "
                           f"{wl.block}x{wl.block} losses",
            "frames": wl.frames, "blocks": total_blocks, "width": wl.width, "height": wl.height,
            "block": wl.block, "support": wl.support, "transform_size": wl.transform_size,
            "iterations": wl.iterations, "rho_hat": wl.rho_hat, "gamma": wl.gamma, "loss_frac": wl.loss_frac,
            "l2": "inputs (frames + spectra) larger than L2; no flush needed"}


def load_peaks():
    out = {}
    try:
        with open(os.path.join(ROOT, "profiles", "peaks.json")) as f:
            p = json.load(f)
        out["smem_gbs"] = p.get("smem_gbs")
        out["smem_source"] = p.get("source")
        out["dram_per_unit"] = p.get("dram_bytes_per_block_iteration", {})
    except Exception:
        pass
    return out


if __name__ == "__main__":
    main()
