#!/usr/bin/env python
"""Benchmark of the optimisation hot path (BASELINE.json metric): iterations/s
of one full step -- raster fwd, ASM fwd, loss, ASM bwd, raster bwd, Adan --
at 1080p RGB (cfg2: 1920x1080, C=3, N=200k, L=1, pad 2), plus its HBM
roofline fraction.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N = 1: the graph-captured cfg2 step on one B200.
N > 1: one rank per GPU (launched by torchrun, or by bench.py itself when
WORLD_SIZE is unset), and by default the SAME cfg2 scene split over the ranks
as row slabs (strong scaling): the 2D FFTs are distributed with four transposes
per step, stored by the FFT kernels straight into the peers' receive buffers
over NVLink, plus an NCCL all-reduce of the gradients (--shard slabs
--exchange put).  --shard planes (cfg3, 8 planes), channels and replicas are
the other decompositions.  Fewer visible GPUs than N is an error.
Timing: CUDA events on the trainer's stream around exactly K steps, barrier +
synchronize on both sides, max over ranks.  The step's working set (~0.45 GB)
exceeds the 126 MB L2, so no explicit flush is used.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "optimisation iters/sec (raster+ASM fwd+bwd) at 1080p RGB; % of HBM roofline"
UNIT = "iters/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=400)
    p.add_argument("--warmup", type=int, default=20)
    p.add_argument("--impl", choices=("ours", "reference"), default="ours")
    p.add_argument("--workload", default="cfg2")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--e2e-steps", type=int, default=50)
    p.add_argument("--profile-steps", type=int, default=10)
    p.add_argument("--scenes", type=int, default=64, help="cfg5: scenes in the batch (split over ranks)")
    p.add_argument("--scene-sample", type=int, default=2,
                   help="cfg5: scenes this rank actually runs (a bounded sample of its share; 0 = all)")
    p.add_argument("--train-steps", type=int, default=2000, help="cfg5: optimisation steps per scene")
    p.add_argument("--poh-steps", type=int, default=600, help="cfg5: random-POH conversion steps per scene")
    p.add_argument("--exchange", choices=("nccl", "put"), default="put",
                   help="--shard slabs: transposes as NCCL all_to_all_single, or as peer-put stores into "
                        "the peers' IPC-mapped receive buffers with device-flag synchronisation")
    p.add_argument("--virtual-ranks", type=int, default=0,
                   help="--shard slabs on ONE GPU: R slab trainers stepped in lock-step with the "
                        "all-to-alls done as device copies (parallel.LocalSlabGroup); reports the "
                        "decomposition's compute per rank, no interconnect")
    p.add_argument("--native", action="store_true",
                   help="sharded modes: run the whole sharded step inside the library over its own NCCL "
                        "communicator (hs_trainer_sharded_step) instead of torch.distributed collectives")
    p.add_argument("--trained-steps", type=int, default=1000,
                   help="N=1: also time the step after this many optimisation steps (trained state: "
                        "moved/rescaled Gaussians, a different pair count); 0 = off")
    p.add_argument("--shard", choices=("replicas", "channels", "planes", "slabs"), default=None,
                   help="N>1: replicas = one scene per GPU (weak scaling, no collective); "
                        "channels = the wavelengths of one scene split over ranks (<= C ranks), "
                        "planes = the depth planes of one scene (cfg3) split over ranks; both "
                        "all-reduce gradients over NCCL (strong scaling); slabs = the canvas rows "
                        "and spectrum columns of one scene (cfg4) split over ranks: four NCCL "
                        "all-to-all transposes + the gradient all-reduce per step.  Default: replicas "
                        "at N=1 (a single unsharded scene), slabs at N>1")
    a = p.parse_args()
    if a.shard is None:
        a.shard = "slabs" if a.gpus > 1 else "replicas"
    return a


def self_launch(args):
    """`python bench.py --gpus N` without torchrun: re-launch as N ranks
    (torch.distributed.run, 127.0.0.1 rendezvous) after checking the GPUs."""
    import socket

    import torch

    have = torch.cuda.device_count()
    if args.impl == "ours" and have < args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {have}\n")
        raise SystemExit(2)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # the NCCL init lines show the rank count and the transport
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    raise SystemExit(subprocess.call(cmd, env=env))


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def algorithmic_bytes(cfg, pairs):
    """B = C(13 + 12L) A + L H W + 592 N + 24 K, A = 8 H W."""
    h, w, c, L, n = cfg["height"], cfg["width"], cfg["channels"], cfg["planes"], cfg["count"]
    A = 8.0 * h * w
    return c * (13 + 12 * L) * A + L * h * w + 592.0 * n + 24.0 * pairs


def kernel_bytes(cfg, pairs):
    """Algorithmic bytes per launch of each kernel slot (A = 8HW per channel)."""
    h, w, c, L, n = cfg["height"], cfg["width"], cfg["channels"], cfg["planes"], cfg["count"]
    A = 8.0 * h * w
    P = (6 + 2 * c) * n
    return {
        "binning": 4.0 * P + 64.0 * n + 3 * 16.0 * pairs,  # params in, records out, keys w/r x2 passes
        "raster_fwd": c * A + 8.0 * pairs + (48.0 + 16 * c) * n,
        "rows_fwd": c * (A + 2 * A),
        "cols_fwd": c * (2 * A + 2 * L * A),
        "rows_inv": c * (2 * L * A + L * A),
        "loss_ssim": c * (L * A + 0.5 * A + L * A) + L * h * w,
        "rows_fwd_bwd": c * (L * A + 2 * L * A),
        "cols_bwd": c * (2 * L * A + 2 * A),
        "rows_inv_bwd": c * (2 * A + A),
        "raster_bwd": c * A + (48.0 + 16 * c + 16 + 4 * (6 + 2 * c)) * n + 4.0 * P,
        "adan": 44.0 * P,
    }


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "50",
                 "-i", str(self.device)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.12)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_reference_run(wl, gset32, max_seconds, threads, min_steps=1, max_steps=3, warmup=0):
    """Times the reference's own CPU implementation (oracle/_ref = the reference
    sources compiled here) on the same inputs, in the order of
    pipeline.cpp:253-297.  Returns (seconds per step, steps timed, stage ms)."""
    from oracle import ref  # checker / baseline only

    cfg = wl["cfg"]
    c, h, w = cfg["channels"], cfg["height"], cfg["width"]
    ref.set_thread_count(threads)
    rs = ref.GaussianSet(cfg["count"], c, *[np.ascontiguousarray(gset32[k]) for k in ref.GROUPS])
    target = wl["target"].astype(np.float32).astype(np.float64)
    tr = ref.Trainer(rs, w, h, target, wl["depth"], cfg["planes"], 3e-3, cfg["dz"],
                     ref.PropagationSpec(tuple(wl["wavelengths"])), total_steps=max_steps + warmup + 1)
    for _ in range(warmup):
        tr.step()
    times = []
    t_all = time.perf_counter()
    while len(times) < max_steps:
        t0 = time.perf_counter()
        tr.step()
        times.append(time.perf_counter() - t0)
        if len(times) >= min_steps and time.perf_counter() - t_all + times[-1] > max_seconds:
            break
    st = tr.stage_ms() / max(len(times) + warmup, 1)
    names = ("raster_fwd", "propagate_multi", "training_loss_grad", "propagate_multi_backward",
             "rasterize_backward", "adan", "total")
    return float(np.mean(times)), len(times), dict(zip(names, [round(float(x), 2) for x in st]))


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    return "unknown"


def fft_speed():
    """The FFT under the reference arm: oracle/fftw_shim.cpp (FFTW3 is not in the
    image) against numpy's pocketfft, both fp64 on one core, at the cfg2 padded
    grid 2160 x 3840: ms per forward + inverse 2D transform pair.  The shim is
    timed through the reference's single-plane propagate(), i.e. its two FFTs
    plus pad / transfer / crop."""
    from oracle import ref

    h, w = 1080, 1920
    rng = np.random.default_rng(0)
    re, im = rng.standard_normal((1, h, w)), rng.standard_normal((1, h, w))
    ref.set_thread_count(1)
    ref.propagate(re, im, ref.PropagationSpec((532e-9,)), 3e-3)  # plan / warm
    t0 = time.perf_counter()
    ref.propagate(re, im, ref.PropagationSpec((532e-9,)), 3e-3)
    shim = (time.perf_counter() - t0) * 1e3
    z = (rng.standard_normal((2 * h, 2 * w)) + 1j * rng.standard_normal((2 * h, 2 * w)))
    np.fft.ifft2(np.fft.fft2(z))
    t0 = time.perf_counter()
    np.fft.ifft2(np.fft.fft2(z))
    pocket = (time.perf_counter() - t0) * 1e3
    # the shim's own forward + backward 2D transform through its FFTW3 entry points
    import ctypes as C
    L = ref.lib()
    L.fftw_plan_dft_2d.restype = C.c_void_p
    L.fftw_plan_dft_2d.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_uint]
    L.fftw_execute.argtypes = [C.c_void_p]
    L.fftw_destroy_plan.argtypes = [C.c_void_p]
    buf = np.ascontiguousarray(z)
    ptr = buf.ctypes.data
    pf = L.fftw_plan_dft_2d(2 * h, 2 * w, ptr, ptr, -1, 64)
    pb = L.fftw_plan_dft_2d(2 * h, 2 * w, ptr, ptr, 1, 64)
    L.fftw_execute(pf)
    t0 = time.perf_counter()
    L.fftw_execute(pf)
    L.fftw_execute(pb)
    shim_pair = (time.perf_counter() - t0) * 1e3
    L.fftw_destroy_plan(pf)
    L.fftw_destroy_plan(pb)
    return {"fft": "oracle/fftw_shim.cpp (FFTW3 API, mixed-radix Stockham + Bluestein, fp64); FFTW3 "
                   "itself is absent from the image",
            "grid": "2160x3840 complex128", "shim_propagate_ms_1core": round(shim, 1),
            "shim_fft2_ifft2_ms_1core": round(shim_pair, 1),
            "numpy_pocketfft_fft2_ifft2_ms_1core": round(pocket, 1)}


def cpu_baseline(wl, gset32):
    """The reference's own fp64 step (oracle/_ref) on this box's host cores:
    set_thread_count(nproc) (the reported value) and set_thread_count(1), with
    the CPU model and the FFT used (BASELINE.md CPU-baseline plan)."""
    nproc = os.cpu_count() or 1
    sec, k, st = cpu_reference_run(wl, gset32, 30.0, nproc, 1, 3, 0)
    sec1, k1, st1 = cpu_reference_run(wl, gset32, 20.0, 1, 1, 1, 0)
    fft = fft_speed()
    return {"value": 1.0 / sec, "unit": UNIT, "cores": nproc, "kind": "reference",
            "sample": f"{k} full cfg2 step(s) through the reference's fp64 C++ (oracle/_ref), "
                      f"set_thread_count({nproc}); only its rasterizer is threaded",
            "stages_ms": st, "cpu_model": cpu_model(),
            "single_thread": {"value": 1.0 / sec1, "unit": UNIT, "cores": 1, "steps": k1, "stages_ms": st1},
            "fft": fft, "fft_adjusted_estimate": fft_adjusted(st, fft, wl["cfg"]["channels"], wl["cfg"]["planes"])}


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return
    from paper_2511_15022_b200 import synthetic as S
    from oracle import ref

    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libholoref.so not built"}))
        return
    wl = S.workload(args.workload)
    gset32 = {k: np.asarray(v, np.float32).astype(np.float64) for k, v in wl["gaussians"].items()}
    threads = os.cpu_count() or 1
    budget = 150.0
    k_cap = max(1, min(args.steps, 3))
    w_cap = 1 if args.warmup > 0 else 0
    sec, k, stages = cpu_reference_run(wl, gset32, budget, threads, 1, k_cap, w_cap)
    v = 1.0 / sec
    cfg = wl["cfg"]
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": k, "warmup": w_cap, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_of(args.workload, cfg, world),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"{k} full step(s) after {w_cap} warm-up of {args.workload} through the "
                                   f"reference's own fp64 C++ (oracle/_ref, FFTW3 API shim), "
                                   f"set_thread_count({threads}); steps capped to stay within minutes",
                         "stages_ms": stages, "cpu_model": cpu_model()},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    fft = fft_speed()
    line["cpu_baseline"]["fft"] = fft
    line["cpu_baseline"]["fft_adjusted_estimate"] = fft_adjusted(stages, fft, cfg["channels"], cfg["planes"])
    print(json.dumps(line))


def fft_adjusted(stages, fft, C, L):
    """What the reference step would take if its 2D FFTs ran at numpy-pocketfft
    speed instead of the shim's (an ESTIMATE, not a measurement): the step's
    2C(L + 1) FFT2s (propagate_multi: one forward FFT per channel and one inverse
    per plane, propagate_multi_backward the adjoint, propagation.cpp:189-243)
    charged at the measured pocketfft instead of the shim time per transform.
    An FFTW build of the reference would be faster still."""
    shim, pocket = fft.get("shim_fft2_ifft2_ms_1core", 0.0), fft.get("numpy_pocketfft_fft2_ifft2_ms_1core", 0.0)
    if "total" not in stages or shim <= 0 or pocket <= 0:
        return None
    n_fft = 2 * C * (L + 1)
    total = stages["total"] - n_fft * 0.5 * (shim - pocket)
    return {"value": 1e3 / total, "unit": UNIT, "ms_per_step": round(total, 1), "fft2_per_step": n_fft,
            "note": "estimate: the step's FFT2s charged at pocketfft speed; not measured"}


def config_of(name, cfg, world, shard="replicas"):
    par = {"replicas": f"replicas x{world} (one scene per GPU, no collective)",
           "channels": f"wavelength shards x{world} (one scene; NCCL all-reduce of the 6N geometry gradients)",
           "planes": f"plane shards x{world} (one scene; NCCL all-reduce of the gradient buffer)",
           "slabs": f"row slabs x{world} (one scene; 4 FFT transposes as peer-put NVLink stores or NCCL "
                    "all-to-all + gradient all-reduce)",
           }[shard]
    seed = "init_gaussians(seed 42+rank)" if shard == "replicas" else "init_gaussians(seed 42)"
    return {"workload": f"{name}: {cfg['width']}x{cfg['height']} x{cfg['channels']} wavelengths, "
                        f"{cfg['count']} Gaussians, {cfg['planes']} plane(s), pad 2, {seed}",
            "width": cfg["width"], "height": cfg["height"], "channels": cfg["channels"],
            "gaussians": cfg["count"], "planes": cfg["planes"], "pad_factor": 2, "parallelism": par,
            "l2": "no flush: per-step working set ~0.45 GB > 126 MB L2"}


def run_sharded(args):
    """--shard channels|planes: one scene split over the ranks with a real
    gradient exchange (parallel.ChannelShardedStep / ShardedStep); eager steps
    (the NCCL all-reduce sits between the trainer's two halves), timed with CUDA
    events on the trainer stream, max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2511_15022_b200 import holo, parallel as P, synthetic as S

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    wl = S.workload(args.workload, scene=0)
    cfg = wl["cfg"]
    C_, h, w, n, L = cfg["channels"], cfg["height"], cfg["width"], cfg["count"], cfg["planes"]
    g32 = {k: np.asarray(v, np.float32).astype(np.float64) for k, v in wl["gaussians"].items()}
    total = args.warmup + args.steps + max(1, min(args.e2e_steps, 20)) + 2
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        if args.shard == "channels":
            if world > C_:
                raise SystemExit(f"--shard channels needs <= {C_} ranks")
            b, e = P.channel_shard(C_, rank, world)
            gs = P.slice_channels(g32, n, C_, b, e)
            tr = holo.Trainer(holo.GaussianSet(n, e - b, **gs), w, h,
                              holo.RealField(e - b, h, w, wl["target"][b:e].astype(np.float32).astype(np.float64)),
                              wl["masks"], wl["distances"], holo.PropagationSpec(tuple(wl["wavelengths"][b:e])),
                              total_steps=total, channels_total=C_)
            step = P.ChannelShardedStep(tr, n, e - b, C_, h, w, L)
        elif args.shard == "slabs":
            def mk(r, R):
                t = holo.Trainer(holo.GaussianSet(n, C_, **g32), w, h,
                                 holo.RealField(C_, h, w, wl["target"].astype(np.float32).astype(np.float64)),
                                 wl["masks"], wl["distances"], holo.PropagationSpec(tuple(wl["wavelengths"])),
                                 total_steps=total)
                t.set_row_slab(r, R)
                return t
            if args.virtual_ranks > 1 and world == 1:
                trs = [mk(r, args.virtual_ranks) for r in range(args.virtual_ranks)]
                tr = trs[0]
                step = P.LocalSlabGroup(trs, C_, h, w, L, put=args.exchange == "put")
            else:
                tr = mk(rank, world)
                step = P.SlabShardedStep(tr, C_, h, w, L, exchange=args.exchange)
        else:
            tr = holo.Trainer(holo.GaussianSet(n, C_, **g32), w, h,
                              holo.RealField(C_, h, w, wl["target"].astype(np.float32).astype(np.float64)),
                              wl["masks"], wl["distances"], holo.PropagationSpec(tuple(wl["wavelengths"])),
                              total_steps=total, plane_range=P.plane_shard(L, rank, world))
            step = P.ShardedStep(tr, C_, h, w, L)
        if args.native and not (args.shard == "slabs" and args.virtual_ranks > 1 and world == 1):
            step = P.NativeShardedStep(tr)  # (slab peer buffers were mapped by SlabShardedStep above)
        for _ in range(args.warmup):
            loss = step.step()
        stream.synchronize()
        sampler = ClockSampler(local)
        sampler.start()
        time.sleep(0.3)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        l0 = holo.kernel_launch_count()
        for i in range(args.steps):
            loss = step.step(with_loss=i + 1 == args.steps)  # the loss (a host sync) on the last step only
        e1.record(stream)
        e1.synchronize()
        torch.cuda.synchronize()
        launches = holo.kernel_launch_count() - l0
        if world > 1:
            dist.barrier()
        clocks = sampler.stop()
        ms = e0.elapsed_time(e1) / args.steps

        # e2e through the public API with host-resident parameters: per step the
        # H2D of this rank's parameters from pinned memory, the sharded step
        # (exchanges + all-reduce), the loss read (a sync) and the D2H of the
        # updated parameters.
        host = torch.empty(tr.param_count, dtype=torch.float32, pin_memory=True)
        host.copy_(tr.params_tensor())
        dev = tr.params_tensor()
        e2e_steps = max(1, min(args.e2e_steps, 20))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            dev.copy_(host, non_blocking=True)
            loss = step.step(with_loss=True)
            host.copy_(dev, non_blocking=True)
        torch.cuda.synchronize()
        e2e_s = (time.perf_counter() - t0) / e2e_steps
    if world > 1:
        t = torch.tensor([ms, e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, e2e_s = float(t[0]), float(t[1])
    if rank == 0:
        peak, peak_src = peaks()
        B = algorithmic_bytes(cfg, tr.last_loss()[1])
        line = {
            "metric": METRIC, "value": 1e3 / ms, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
            "config": config_of(args.workload, cfg, world, args.shard),
            "step_roofline": {"bound": "hbm", "achieved": B / (ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                              "frac": B / (ms * 1e-3) / 1e9 / peak / world, "peak_source": peak_src,
                              "note": "whole-job algorithmic bytes over world x peak"},
            "roofline": {"bound": "hbm", "kernel": "whole step (sharded)", "achieved": B / (ms * 1e-3) / 1e9 / world,
                         "peak": peak, "unit": "GB/s", "frac": B / (ms * 1e-3) / 1e9 / peak / world, "traffic": None,
                         "peak_source": peak_src,
                         "note": "per GPU: the step's algorithmic bytes (SURVEY 8d) / world / ms_per_step"},
            "e2e": {"value": 1.0 / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 4 * tr.param_count,
                    "d2h_bytes_per_step": 4 * tr.param_count + 16,
                    "path": "per rank and step: H2D of its parameters (pinned), the sharded step, the loss "
                            "read and the D2H of the updated parameters; max over ranks"},
            "gpu_launches": int(launches), "clocks": clocks, "loss": loss,
            "timing": ("slab steps: stages 0-4 as one CUDA graph (peer-put, device-flag sync), NCCL "
                       "all-reduce of the gradients, Adan; " if args.shard == "slabs" and args.exchange == "put"
                       else "eager steps (NCCL all-reduce between forward_backward and apply_update); ")
                      + "loss (a host sync) on the last timed step only; CUDA events on the trainer stream, "
                        "max over ranks",
        }
        if args.shard == "slabs" and args.virtual_ranks > 1 and world == 1:
            R = args.virtual_ranks
            line["virtual_ranks"] = {
                "ranks": R, "ms_all_ranks_one_gpu": ms, "ms_per_rank_compute": ms / R,
                "note": "R slab trainers on one GPU, exchanges as device copies: ms/R is the "
                        "per-rank compute of an R-GPU run without the interconnect time"}
            line["value"] = None
            line["metric"] = METRIC + " (virtual ranks: decomposition check, not a throughput)"
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_cfg5(args):
    """cfg5: a batch of 1080p RGB scenes (L = 2), each optimised
    for --train-steps iterations, rasterised, DPAC-encoded (smooth POH) and
    converted to a random POH (--poh-steps); scenes are split over the ranks
    (replicas, no collective).  Reports scenes/s for the whole batch from the
    measured per-scene device time of a bounded sample (--scene-sample)."""
    import ctypes as C
    import torch
    import torch.distributed as dist

    from paper_2511_15022_b200 import _lib, holo, synthetic as S

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    mine = list(range(rank, args.scenes, world))
    run = mine if args.scene_sample <= 0 else mine[:args.scene_sample]
    lib = _lib.load()
    phase_ms = {"train": 0.0, "raster": 0.0, "dpac": 0.0, "random_poh": 0.0}
    host_ms = 0.0  # initial random phase raster (host mt19937_64, like the reference)
    stream = torch.cuda.Stream()
    launches0 = holo.kernel_launch_count()
    with torch.cuda.stream(stream):
        for i in run:
            wl = S.workload("cfg5", scene=i)
            cfg = wl["cfg"]
            c, h, w, n, L = cfg["channels"], cfg["height"], cfg["width"], cfg["count"], cfg["planes"]
            g32 = {k: np.asarray(v, np.float32).astype(np.float64) for k, v in wl["gaussians"].items()}
            spec = holo.PropagationSpec(tuple(wl["wavelengths"]))
            tr = holo.Trainer(holo.GaussianSet(n, c, **g32), w, h,
                              holo.RealField(c, h, w, wl["target"].astype(np.float32).astype(np.float64)),
                              wl["masks"], wl["distances"], spec, total_steps=args.train_steps)
            tr.use_graph(True)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
            stream.synchronize()
            ev[0].record(stream)
            for _ in range(args.train_steps):
                tr.step(sync_loss=False)
            ev[1].record(stream)
            # the initial random-POH phase raster is drawn on the host (mt19937_64,
            # like the reference) while the queued training steps run
            h0 = time.perf_counter()
            phase_h = holo.random_phase(i, c * h * w).astype(np.float32)
            host_ms += (time.perf_counter() - h0) * 1e3
            field = holo.rasterize_forward_device(tr.params_tensor(), n, c, w, h)
            ev[2].record(stream)
            smooth = torch.empty((c, h, w), dtype=torch.float32, device=field.device)
            holo.check(lib.hs_dpac_encode(holo.ctx_handle(), holo._ptr(field), c, h, w, 0, holo._ptr(smooth)))
            ev[3].record(stream)
            phase = torch.from_numpy(phase_h).to(field.device)
            d = (C.c_double * L)(*wl["distances"])
            tgt = np.ascontiguousarray(wl["target"], dtype=np.float32)
            msk = np.ascontiguousarray(wl["masks"], dtype=np.uint8)
            pc = holo.hs_poh_config(c, h, w, L, C.cast(d, C.POINTER(C.c_double)), spec.c_struct(),
                                    tgt.ctypes.data_as(C.POINTER(C.c_float)), msk.ctypes.data_as(C.POINTER(C.c_uint8)),
                                    int(args.poh_steps), 0.1, 0.01, 2.5e-3)
            holo.check(lib.hs_convert_random_poh_field(holo.ctx_handle(), C.byref(pc), holo._ptr(field),
                                                       holo._ptr(phase), None))
            ev[4].record(stream)
            ev[4].synchronize()
            for k, (a, b) in zip(phase_ms, zip(ev[:-1], ev[1:])):
                phase_ms[k] += a.elapsed_time(b)
            del tr
    launches = holo.kernel_launch_count() - launches0
    per_scene = sum(phase_ms.values()) / max(1, len(run))  # device timeline ev0 -> ev4 (host gaps included)
    total_ms = per_scene * len(mine)  # this rank's share of the batch
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t[0])
    if rank == 0:
        line = {
            "metric": "cfg5 conversion batch: scenes/s (train + raster + DPAC + random POH per scene)",
            "value": args.scenes / (total_ms * 1e-3), "unit": "scenes/s", "n_gpus": world,
            "higher_is_better": True, "scaling": "weak" if world == 1 else "strong", "dtype": "fp32",
            "data": "synthetic", "vs_baseline": None,
            "config": {"workload": f"cfg5: {args.scenes} scenes of 1920x1080 x3, {S.CONFIGS['cfg5']['count']} "
                                   f"Gaussians, 2 planes, {args.train_steps} train steps + {args.poh_steps} "
                                   "random-POH steps per scene",
                       "parallelism": f"replicas x{world} (scenes split over ranks, no collective)",
                       "sample": f"{len(run)} of this rank's {len(mine)} scenes timed; the batch time is "
                                 "the per-scene device time x the rank's share (max over ranks)"},
            "ms_per_scene": per_scene,
            "phase_ms_per_scene": {**{k: v / max(1, len(run)) for k, v in phase_ms.items()},
                                   "random_phase_init_host_overlapped": host_ms / max(1, len(run))},
            "gpu_launches": int(launches),
        }
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    rank, world, _ = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        self_launch(args)
    if world != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}\n")
        raise SystemExit(2)
    if args.impl == "reference":
        run_reference(args)
        return
    if args.workload == "cfg5" and args.shard == "replicas":
        run_cfg5(args)
        return
    if args.shard != "replicas":
        run_sharded(args)
        return
    import torch
    import torch.distributed as dist

    from paper_2511_15022_b200 import holo, synthetic as S

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    wl = S.workload(args.workload, scene=rank)
    cfg = wl["cfg"]
    c, h, w, n, L = cfg["channels"], cfg["height"], cfg["width"], cfg["count"], cfg["planes"]
    gset32 = {k: np.asarray(v, np.float32).astype(np.float64) for k, v in wl["gaussians"].items()}
    gs = holo.GaussianSet(n, c, **gset32)
    target = holo.RealField(c, h, w, wl["target"].astype(np.float32).astype(np.float64))
    spec = holo.PropagationSpec(tuple(wl["wavelengths"]))
    trained_extra = max(0, args.trained_steps - args.warmup - args.steps) if args.trained_steps > 0 else 0
    total = args.warmup + args.steps + trained_extra + (args.steps if args.trained_steps > 0 else 0) \
        + 2 * args.e2e_steps + args.profile_steps + args.steps + 11
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        tr = holo.Trainer(gs, w, h, target, wl["masks"], wl["distances"], spec, total_steps=total)
        tr.use_graph(True)
        for _ in range(args.warmup):
            tr.step(sync_loss=False)
        tr.last_loss()  # surfaces any error of the warm-up
        stream.synchronize()
        sampler = ClockSampler(local)
        sampler.start()
        time.sleep(0.3)  # let the sampler attach before the timed region
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            tr.step(sync_loss=False)
        e1.record(stream)
        e1.synchronize()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        clocks = sampler.stop()
        ms = e0.elapsed_time(e1) / args.steps
        loss, pairs = tr.last_loss()
        # per-step distribution (median and p10/p90): the same
        # graph step, K more times, an event pair around each launch
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        for a0, a1 in evs:
            a0.record(stream)
            tr.step(sync_loss=False)
            a1.record(stream)
        torch.cuda.synchronize()
        per = np.array([a0.elapsed_time(a1) for a0, a1 in evs])
        dist_ms = {"median": float(np.median(per)), "p10": float(np.percentile(per, 10)),
                   "p90": float(np.percentile(per, 90)), "n": len(per)}

        trained = None
        if args.trained_steps > 0:
            # the same step after `trained_steps` optimisation steps: Gaussians moved,
            # rescaled and re-weighted, a different pair count and tile balance
            for _ in range(trained_extra):
                tr.step(sync_loss=False)
            tr.last_loss()
            torch.cuda.synchronize()
            t0e, t1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0e.record(stream)
            for _ in range(args.steps):
                tr.step(sync_loss=False)
            t1e.record(stream)
            t1e.synchronize()
            tms = t0e.elapsed_time(t1e) / args.steps
            tloss, tpairs = tr.last_loss()
            trained = {"after_steps": args.warmup + args.steps + trained_extra, "value": world * 1e3 / tms,
                       "ms_per_step": tms, "pairs": tpairs, "loss": tloss,
                       "step_roofline_frac": algorithmic_bytes(cfg, tpairs) / (tms * 1e-3) / 1e9 / peaks()[0]}

        # e2e through the public API with a host-resident GaussianSet (like the
        # reference loop): per step H2D params from pinned memory, the step,
        # D2H of the updated params and the loss (hs_trainer_step_host).
        P = tr.param_count
        host = torch.empty(P, dtype=torch.float32, pin_memory=True)
        host.copy_(torch.from_numpy(tr.params()))
        for _ in range(3):  # warm-up (captures the host-step graph)
            tr.step_host(host, host)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            tr.step_host(host, host)
        torch.cuda.synchronize()
        e2e_single_s = (time.perf_counter() - t0) / args.e2e_steps
        # the training loop as one call (hs_trainer_run_host): every step still
        # uploads all parameters from and downloads them back into the pinned
        # host buffer; the copies of consecutive steps overlap
        tr.run_host(host, 3)  # warm-up (captures the run graphs)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tr.run_host(host, args.e2e_steps)
        torch.cuda.synchronize()
        e2e_s = (time.perf_counter() - t0) / args.e2e_steps

        # kernels per step: one eager step (every kernel a counted launch)
        tr.use_graph(False)
        l0 = holo.kernel_launch_count()
        tr.step(sync_loss=False)
        per_step_launches = holo.kernel_launch_count() - l0
        # per-stage profile: graph-replayed steps whose graph also holds an event
        # record at every stage boundary (the same kernels, no host enqueue gaps)
        tr.use_graph(True)
        tr.set_profiling(True)
        stages = {}
        for i in range(args.profile_steps):
            tr.step(sync_loss=False)
            for k, v in tr.stage_ms().items():
                stages.setdefault(k, []).append(v)
        stage_ms = {k: float(np.median(v)) for k, v in stages.items()}

    if world > 1:
        t = torch.tensor([ms, e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, e2e_s = float(t[0]), float(t[1])
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    peak, peak_src = peaks()
    kb = kernel_bytes(cfg, pairs)
    kern = {k: v for k, v in stage_ms.items() if k in kb}
    dom = max(kern, key=kern.get)
    dom_gbs = kb[dom] / (kern[dom] * 1e-3) / 1e9
    B = algorithmic_bytes(cfg, pairs)
    step_gbs = B / (ms * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            tj = json.load(f)
        if tj.get("workload", "cfg2") == args.workload:  # profiled on this workload only
            traffic = tj.get(dom)
    line = {
        "metric": METRIC, "value": world * 1e3 / ms, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
        "config": config_of(args.workload, cfg, world),
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": dom_gbs, "peak": peak, "unit": "GB/s",
                     "frac": dom_gbs / peak, "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": kb[dom], "ms_per_launch": kern[dom],
                     "note": "the rasterizer, SSIM and FFT kernels are instruction-issue bound (ncu issue-active "
                             "44-71%, profiles/r02_ncu_summary_v7.md), not HBM bound: the HBM fraction "
                             "measures bytes, not the binding resource (DESIGN.md section 3)"},
        "step_roofline": {"bound": "hbm", "achieved": step_gbs, "peak": peak, "unit": "GB/s",
                          "frac": step_gbs / peak, "algorithmic_bytes_per_step": B,
                          "formula": "C(13+12L)8HW + LHW + 592N + 24K (SURVEY §8d)"},
        "step_ms_dist": dist_ms,
        "stages_ms": {k: round(v, 4) for k, v in stage_ms.items()},
        "e2e": {"value": world / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 4 * P,
                "d2h_bytes_per_step": 4 * P + 12,
                "path": "hs_trainer_run_host over --e2e-steps steps, wall clock: every step H2D of all params "
                        "from the pinned host buffer, the graph step, D2H of the updated params into it (+ the "
                        "step's loss and flag words); step k's amplitude/phase D2H overlaps step k+1's "
                        "geometry H2D and projection",
                "single_call": {"value": world / e2e_single_s, "unit": UNIT,
                                "path": "hs_trainer_step_host per step (H2D, graph step, D2H, one sync each)"}},
        "gpu_launches": int(round(per_step_launches * args.steps)),
        "clocks": clocks, "loss": loss, "pairs": pairs,
    }
    if trained:
        line["trained"] = trained
    if world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(wl, gset32)
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                                    "sample": f"unavailable: {e}"}
    print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
