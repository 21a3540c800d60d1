#!/usr/bin/env python3
"""FOFSE block-concealment benchmark (BASELINE.json metric: lost blocks
extrapolated per second at 16x16 blocks, 64^2 FFT, 200 iterations).

Workload (N=1): BASELINE config C4 — 256 synthetic 1920x1088 frames, 10 %
isolated 16x16 losses per frame (~209k blocks), rho 0.8, gamma 0.5, 200
iterations, fp32 fast mode. Under torchrun each rank processes its own C4
batch (frames seeded per rank): weak scaling, no data-path collective.

  value : blocks/s with the frames resident in HBM (plan/execute, kernels only)
  e2e   : blocks/s through the public C ABI call with pinned HOST buffers
          (H2D frames + host prep + kernels + D2H restored frames every step)

`--impl reference` runs the reference's own CPU implementation (the
unmodified reference sources compiled as oracle/_ref, fse::conceal with all
host threads) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
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
    ap.add_argument("--frames", type=int, default=None, help="frames per rank (default: config)")
    ap.add_argument("--precision", default=None)
    ap.add_argument("--seed", type=int, default=2207)
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU baseline sample budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
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
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl.name, "frames_per_rank": wl.frames, "width": wl.width,
                   "height": wl.height, "block": wl.block, "transform_size": wl.transform_size,
                   "iterations": wl.iterations, "loss_frac": wl.loss_frac},
        "cpu_baseline": dict(base, value=value),
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
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
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    import paper_2207_01205_b200 as P
    from paper_2207_01205_b200 import _capi as capi
    from paper_2207_01205_b200 import build as native

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

    # ---- inputs for this rank (weak scaling: own frames per rank) ----
    seed = args.seed + rank * 1000003
    t0 = time.time()
    frames_np, rects, offs = wl.batch(seed)
    gen_s = time.time() - t0
    nf = frames_np.shape[0]
    n_blocks = int(offs[-1])
    fbytes = frames_np.nbytes

    ctx = capi.Context(local)
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)

    # ---- device-resident value: plan once, execute K times ----
    plan = C.c_void_p()
    capi.check(L.fofse_plan_frames_u8(ctx.handle, nf, wl.width, wl.height,
                                      rects.ctypes.data_as(C.POINTER(capi.Rect_)),
                                      capi.ptr(offs, C.c_int64), wl.block, wl.block, C.byref(params),
                                      C.byref(plan)))
    d_frames = torch.from_numpy(frames_np).to(dev)
    d_sq = torch.zeros(max(n_blocks, 1), dtype=torch.float64, device=dev)
    rep = capi.Report()

    def execute():
        capi.check(L.fofse_plan_execute_device(plan, C.c_void_p(d_frames.data_ptr()),
                                               capi.ptr_dev(d_sq), C.byref(rep)))
        return rep

    first = None
    for i in range(args.warmup):
        r = execute()
        if i == 0:
            first = capi.Report.from_buffer_copy(r)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k2_ms, init_ms, launches, reruns, real_ms, real_blocks, head = [], [], 0, 0, [], 0, 0
    dev_total, e2e_total, e2e_wall = [], [], []
    barrier()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            r = execute()
            k2_ms.append(r.iterate_ms)
            init_ms.append(r.init_ms)
            dev_total.append(r.total_ms)
            real_ms.append(r.real_iterate_ms)
            real_blocks, head = r.real_blocks, r.fp64_head
            launches += r.kernel_launches
            reruns += r.guard_reruns
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    clocks = clk.summary()

    # ---- end-to-end through the public C ABI with pinned host buffers ----
    h_in = torch.from_numpy(frames_np).pin_memory()
    h_out = torch.empty_like(h_in).pin_memory()
    h_sq = np.zeros(max(n_blocks, 1), np.float64)
    rects_c = rects.ctypes.data_as(C.POINTER(capi.Rect_))

    def e2e_call():
        capi.check(L.fofse_conceal_frames_u8(
            ctx.handle, C.cast(h_in.data_ptr(), C.POINTER(C.c_uint8)), nf, wl.width, wl.height,
            rects_c, capi.ptr(offs, C.c_int64), wl.block, wl.block, C.byref(params),
            C.cast(h_out.data_ptr(), C.POINTER(C.c_uint8)), capi.ptr(h_sq), C.byref(rep)))

    for _ in range(max(1, min(args.warmup, 2))):
        e2e_call()
    e2e_psnr = rep.psnr_db
    barrier()
    ev0.record(stream)
    for _ in range(args.steps):
        t0 = time.perf_counter()
        e2e_call()
        e2e_wall.append((time.perf_counter() - t0) * 1e3)
        e2e_total.append(rep.total_ms)
    ev1.record(stream)
    barrier()
    e2e_ms = ev0.elapsed_time(ev1) / args.steps

    # ---- max over ranks ----
    t = torch.tensor([ms, e2e_ms, statistics.mean(k2_ms), statistics.mean(real_ms)], dtype=torch.float64,
                     device=dev)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        nb = torch.tensor([n_blocks], dtype=torch.float64, device=dev)
        dist.all_reduce(nb)
        total_blocks = int(nb.item())
    else:
        total_blocks = n_blocks
    ms, e2e_ms, k2_avg, real_avg = (float(x) for x in t.tolist())

    if rank == 0:
        # roofline of the dominant kernel, the real-path iteration K2v2 (SMEM
        # bytes = 4 s H per block-iteration): its algorithmic bytes over the summed
        # durations of its launches (CUDA events on the launching stream, in the library)
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
        try:  # live, same box: LDS.64 bandwidth (the W gathers of K2 are LDS.64 / LDS.32)
            peaks["smem_gbs"] = capi.microbench(local, 0)
            peaks["smem_source"] = "measured live by fofse_microbench(kind=0): conflict-free LDS.64, 148 SMs"
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
                "frac": (achieved / peak) if peak else None, "traffic": peaks.get("k2_dram_bytes"),
                "per_unit": f"4*s*H = {4 * s * H} B per block-iteration (s={s}, H={H}); "
                            f"{its} fp32 iterations x {real_blocks if prec == 'fp32' else n_blocks} blocks per step",
                "peak_source": peaks.get("smem_source"),
                "note": "the iteration kernel is bound by on-chip shared-memory bandwidth / issue, not by HBM or "
                        "tensor cores (GEMM-free: shifted complex updates + argmax); hbm_check shows its DRAM share"}
        try:  # HBM side of the same kernel: ncu DRAM bytes of one chunk launch, scaled to the step
            with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
                hbm_peak = json.load(f).get("hbm_gbs")
        except Exception:
            hbm_peak = None
        tr = peaks.get("k2_dram_bytes")
        if prec == "fp32" and tr and real_avg > 0 and hbm_peak:
            hbm = tr * (real_blocks / 24906.0) / (real_avg * 1e-3) / 1e9
            roof["hbm_check"] = {"achieved": hbm, "peak": hbm_peak, "unit": "GB/s", "frac": hbm / hbm_peak,
                                 "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            try:
                cpu = cpu_reference_rate(wl, args.seed, args.cpu_seconds, os.cpu_count() or 1)
                cpu["one_thread"] = cpu_reference_1thread(wl, args.seed)
            except Exception as e:  # baseline is reported, never required
                cpu = {"error": str(e)}
        line = {
            "metric": METRIC, "value": total_blocks / (ms * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32" if prec == "fp32" else "f64",
            "data": "synthetic (seeded generator, SURVEY §8d; see DESIGN.md)",
            "config": {"workload": f"{wl.name}: {nf} frames/rank of {wl.width}x{wl.height}, "
                                   f"{wl.loss_frac:.0%} isolated {wl.block}x{wl.block} losses",
                       "frames_per_rank": nf, "blocks_per_rank": n_blocks, "transform_size": wl.transform_size,
                       "iterations": wl.iterations, "rho_hat": wl.rho_hat, "gamma": wl.gamma,
                       "precision": prec, "parallelism": f"blocks sharded by frame, {world} rank(s)",
                       "l2": "inputs (frames + spectra) larger than L2; no flush needed"},
            "e2e": {"value": total_blocks / (e2e_ms * 1e-3), "unit": UNIT,
                    "h2d_bytes_per_step": fbytes + rects.nbytes + offs.nbytes,
                    "d2h_bytes_per_step": fbytes + 8 * n_blocks},
            "roofline": roof,
            "cpu_baseline": cpu,
            "clocks": clocks,
            "gpu_launches": launches,
            "detail": {"k2_ms": k2_avg, "init_ms": statistics.mean(init_ms), "guard_reruns_per_step": reruns / args.steps,
                       "psnr_db": first.psnr_db if first else None, "e2e_psnr_db": e2e_psnr,
                       "classes": first.classes if first else None, "input_gen_s": gen_s,
                       "real_blocks": real_blocks, "real_iterate_ms": real_avg, "fp64_head": head,
                       # library-side device span (first to last event of run_job) and host wall
                       # time per e2e call: the gap is host preparation + transfers
                       "device_total_ms": statistics.mean(dev_total), "e2e_device_total_ms": statistics.mean(e2e_total),
                       "e2e_wall_ms": statistics.mean(e2e_wall)},
        }
        print(json.dumps(line), flush=True)
    L.fofse_plan_destroy(plan)
    ctx.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def load_peaks():
    out = {}
    try:
        with open(os.path.join(ROOT, "profiles", "peaks.json")) as f:
            p = json.load(f)
        out["smem_gbs"] = p.get("smem_gbs")
        out["smem_source"] = p.get("source")
        out["k2_dram_bytes"] = p.get("k2_dram_bytes_per_launch")
    except Exception:
        pass
    return out


if __name__ == "__main__":
    main()
