#!/usr/bin/env python
"""bench.py -- RayGauss hot path on B200 (BASELINE.json metric: Mrays/s forward and
forward+backward, 800x800 Blender-like, at 1/2/4/8 B200, and % of roofline).

Headline `value`: Mrays/s of one C1/C2 training step (BVH rebuild + forward +
L1 loss gradient + backward + finalize + NCCL all-reduce of the per-Gaussian
gradients for N > 1) on the Blender-like scene (300k Gaussians, SH degree 3 +
7 SG lobes), one 800x800 view per rank per step (weak scaling: rank r renders
view r, so N = 8 is the C2 step of BASELINE.json configs[2]).

Also reported on the same line:
  fwd       C1 forward-only Mrays/s (the paper's inference metric; BVH built once),
            the view's 16x16 tiles interleaved over the N ranks (strong scaling);
  configs   C3 Mip-NeRF360-like (2M Gaussians, 1245x825) forward and training step,
            and C4 stress (5M Gaussians, 1920x1080) forward, tiles interleaved over
            the ranks, gradients all-reduced (864 MB at C3);
  roofline  §8(d) for the dominant kernel of the headline step:
            t_roof = max(FP32 / (148*128*f), MUFU / (148*16*f), bytes / HBM, RED / R_red)
            from the kernel's own counters and §8(d)'s unit costs, frac = t_roof / t_measured,
            at the logged SM clock and at 1965 MHz;
  cpu_baseline  the oracle on a bounded stratified sample, 1 core and nproc processes.

Contract: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
prints ONE JSON line on rank 0.  Device timing with CUDA events over exactly K
steps bracketed by barrier + synchronize, max over ranks.  For N > 1 without a
torchrun environment the script re-launches itself under torch.distributed.run.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import platform
import socket
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Mrays/s fwd and fwd+bwd (800x800 Blender-like) at 1/2/4/8 B200; % of roofline"
PAPER_FPS = 25.0   # P:25, P:358 (RTX 4090, 800x800): context only
TILE = 16          # interleaved tile sharding

# --- SURVEY.md §8(d) cost model: (FP32 instructions, MUFU ops) per unit ------
# eval = one (sample, Gaussian) contribution, pair = one (ray, Gaussian) set-up
# (deg 3 + 7 SG), samp = one composited sample; the backward adds 27 float4
# reductions per pair.  FMA = 1 FP32 instruction.
UNITS = {"fwd": {"eval": (9, 1), "pair": (190, 10), "samp": (12, 2)},
         "bwd": {"eval": (25, 1), "pair": (400, 10), "samp": (12, 2)}}
RED_PER_PAIR = 27
RECORD_BYTES = 432      # per Gaussian input record at C1-C4 (§8(a))
RAY_BYTES = 28          # rays in and out


def load_json(*parts):
    try:
        return json.load(open(os.path.join(ROOT, *parts)))
    except (OSError, ValueError):
        return {}


def hbm_peak():
    p = load_json("MEASURED_PEAKS.json")
    if p.get("hbm_gbs"):
        return float(p["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (of measured)"
    return 6650.0, "B200_PROFILING.md fallback 6.65 TB/s (of fallback)"


def roofline_8d(stats, which, t_ms, mhz, n_gauss, red_gops=None):
    """t_roof = max(FP32/(148*128*f), MUFU/(148*16*f), bytes/HBM, RED/R_red);
    frac = t_roof / t_measured.  Counts come from the kernel's counters (identical to
    the oracle's definitions for evals and samples; pairs = set-ups)."""
    u = UNITS[which]
    n = {"eval": stats["evals"], "pair": stats["pairs"], "samp": stats["samples"]}
    fp32 = sum(n[k] * u[k][0] for k in n)
    mufu = sum(n[k] * u[k][1] for k in n)
    nbytes = min(n_gauss, stats["pairs"]) * RECORD_BYTES + RAY_BYTES * stats["rays"]
    reds = RED_PER_PAIR * stats["pairs"] if which == "bwd" else 0
    hbm, hbm_src = hbm_peak()
    t = t_ms * 1e-3

    def terms(f_mhz):
        f = f_mhz * 1e6
        out = {"fp32": fp32 / (148 * 128 * f), "mufu": mufu / (148 * 16 * f),
               "hbm": nbytes / (hbm * 1e9)}
        if reds and red_gops:
            out["red"] = reds / (red_gops * 1e9)
        return out
    tl = terms(mhz)
    bound = max(tl, key=tl.get)
    t_roof = tl[bound]
    peak = {"fp32": 148 * 128 * mhz * 1e6 / 1e12, "mufu": 148 * 16 * mhz * 1e6 / 1e12,
            "hbm": hbm, "red": red_gops}[bound]
    work = {"fp32": fp32 / 1e12, "mufu": mufu / 1e12, "hbm": nbytes / 1e9, "red": reds / 1e9}[bound]
    unit = {"fp32": "T FP32 instr/s", "mufu": "T MUFU op/s", "hbm": "GB/s", "red": "G float4 RED/s"}[bound]
    t1965 = terms(1965.0)
    return {
        "bound": "alu" if bound in ("fp32", "mufu") else bound,
        "pipe": bound, "achieved": work / t, "peak": peak, "unit": unit,
        "frac": t_roof / t, "frac_at_1965mhz": max(t1965.values()) / t,
        "t_roof_ms": 1e3 * t_roof, "t_measured_ms": t_ms, "sm_mhz": mhz,
        "terms_ms": {k: 1e3 * v for k, v in tl.items()},
        "work": {"fp32_instr": fp32, "mufu": mufu, "bytes": nbytes, "red_f32x4": reds,
                 "evals": n["eval"], "pairs": n["pair"], "samples": n["samp"]},
        "peak_source": ("148 SM x 128 FP32 lanes (MUFU 16/SM) x SM clock, B200_PROFILING.md "
                        "counts; " + hbm_src + "; RED: tools/microbench.cu "
                        "(profiles/r1/microbench.json)"),
    }


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms (B200_PROFILING.md)."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_id: str | None):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        cmd = ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "200"]
        if gpu_id:
            cmd += ["-i", gpu_id]
        try:
            self.p = subprocess.Popen(cmd, stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
        self.f.flush()
        rows = []
        for line in open(self.f.name):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower() == "active"})
        loaded = [s for s in sm if s > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def stratified(cam, step):
    import numpy as np
    ys, xs = np.meshgrid(np.arange(step // 2, cam.height, step), np.arange(step // 2, cam.width, step),
                         indexing="ij")
    return (ys * cam.width + xs).reshape(-1)


def oracle_step(sc, p, cam, target_rgb, idx, bvh=None):
    """One oracle pass over the rays `idx` of the view: BVH build (unless given),
    forward, L1 gradient, backward (the same path, single-threaded C, fp64 values)."""
    import numpy as np
    from oracle import oracle as O
    o_all, d_all = O.camera_rays(cam)
    o, d = o_all[idx], d_all[idx]
    t0 = time.perf_counter()
    b = bvh if bvh is not None else O.BVH(sc, p)
    r = O.render(sc, p, o, d, mode=2, bvh=b)
    gr = np.sign(r["rgb"] - target_rgb[idx]) / (3.0 * len(idx))
    O.backward(sc, p, o, d, gr, mode=2, bvh=b)
    return len(idx), time.perf_counter() - t0


def _oracle_worker(args):
    """one of nproc independent oracle processes (disjoint ray subsets)"""
    import numpy as np
    from oracle import oracle as O
    from paper_2408_03356_b200 import synth
    part, parts, step_px = args
    wl = synth.workload("blender")
    sc, cam, p = wl.scene, wl.cameras[0], wl.params
    idx = stratified(cam, step_px)[part::parts]
    tgt = np.full((cam.n_rays, 3), 0.5)
    t0 = time.perf_counter()
    b = O.BVH(sc, p)
    n, s = oracle_step(sc, p, cam, tgt, idx, bvh=b)
    return n, time.perf_counter() - t0


def oracle_parallel(step_px=4):
    """nproc independent oracle processes on disjoint subsets of the same stratified
    sample (each builds its own BVH): whole-host Mrays/s (SURVEY §8(d) oracle timing)."""
    import multiprocessing as mp
    nproc = os.cpu_count() or 1
    t0 = time.perf_counter()
    with mp.get_context("spawn").Pool(nproc) as pool:
        res = pool.map(_oracle_worker, [(k, nproc, step_px) for k in range(nproc)])
    wall = time.perf_counter() - t0
    rays = sum(r[0] for r in res)
    return {"value": rays / wall / 1e6, "unit": "Mrays/s", "cores": nproc, "kind": "oracle",
            "sample": f"{rays} stratified rays (every {step_px}th pixel) of the C1 800x800 view split "
                      f"over {nproc} processes (each: own BVH build + fwd + L1 grad + bwd), "
                      f"{wall:.1f} s wall incl. process start"}


def perturbed(sc, seed=77):
    import numpy as np
    rng = np.random.default_rng(seed)
    q = sc.copy()
    q.mean += rng.normal(0.0, 0.002, size=q.mean.shape).astype(np.float32)
    q.sh[:, 0, :] *= rng.uniform(0.9, 1.1, size=(q.n, 1)).astype(np.float32)
    return q


# ----------------------------------------------------------------------------
def run_reference(args):
    """--impl reference: the oracle (CPU) timed on bounded samples of the same
    workload, rank 0 only (the other ranks exit 0 without work)."""
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return 0
    import numpy as np
    from paper_2408_03356_b200 import synth
    from oracle import oracle as O
    O.build()
    wl = synth.workload("blender_train", views=8)
    sc, cam, p = wl.scene, wl.cameras[0], wl.params
    step_px = 16
    idx = stratified(cam, step_px)
    o_all, d_all = O.camera_rays(cam)
    tgt = np.zeros((cam.n_rays, 3))
    tgt[idx] = O.render(perturbed(sc), p, o_all[idx], d_all[idx], mode=2)["rgb"]
    for _ in range(args.warmup):
        oracle_step(sc, p, cam, tgt, idx)
    tot_rays, tot_s = 0, 0.0
    for _ in range(args.steps):
        n, s = oracle_step(sc, p, cam, tgt, idx)
        tot_rays += n
        tot_s += s
    v = tot_rays / tot_s / 1e6
    sample = (f"1/{step_px * step_px} stratified pixels ({n} rays) of the 800x800 view per step: "
              "oracle BVH build + forward + L1 grad + backward, 1 core")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "Mrays/s",
            "n_gpus": args.gpus, "hardware": "1 host CPU core (n_gpus echoes the launch)",
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tot_s / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C1 Blender-like training step (300k Gaussians, SH3+7SG, 800x800 view)",
                       "global_batch": n, "seq_len": None, "parallelism": "cpu1"},
            "cpu_baseline": {"value": v, "unit": "Mrays/s", "cores": 1, "kind": "oracle",
                             "sample": sample, "cpu": cpu_model(), "nproc": os.cpu_count()},
            "e2e": {"value": v, "unit": "Mrays/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------
class Ctx:
    """per-rank plumbing shared by the measurements"""

    def __init__(self):
        import torch
        import torch.distributed as dist
        from paper_2408_03356_b200 import dist as rgd
        self.torch, self.dist = torch, dist
        self.rank, self.world, self.local = rgd.init()
        torch.cuda.set_device(self.local)
        self.dev = torch.device("cuda", self.local)
        self.stream = torch.cuda.current_stream()

    def ev(self):
        return self.torch.cuda.Event(enable_timing=True)

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max_over_ranks(self, x):
        if self.world > 1:
            t = self.torch.tensor([x], dtype=self.torch.float64, device=self.dev)
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
            return float(t.item())
        return x

    def timed(self, fn, steps, warmup):
        """device ms per call: W untimed calls, then exactly `steps` calls bracketed by
        barrier + synchronize on both sides, CUDA events on the launch stream, max over ranks"""
        torch = self.torch
        for _ in range(warmup):
            fn()
        self.barrier(); torch.cuda.synchronize()
        a, b = self.ev(), self.ev()
        a.record(self.stream)
        for _ in range(steps):
            fn()
        b.record(self.stream)
        torch.cuda.synchronize(); self.barrier()
        return self.max_over_ranks(a.elapsed_time(b) / steps)


def tile_camera(cam, ctx):
    """this rank's interleaved 16x16 tiles of the view (rg_camera.tile)"""
    return dataclasses.replace(cam, tile=TILE, shard=ctx.rank, shards=ctx.world)


def measure_config(ctx, name, args, train, red_gops, ppr):
    """forward (and training step) Mrays/s of one view of `name`, tiles interleaved over
    the ranks; counters from one instrumented untimed pass; roofline per §8(d)."""
    torch = ctx.torch
    from paper_2408_03356_b200 import dist as rgd
    from paper_2408_03356_b200 import rg, synth
    t_setup = time.perf_counter()
    wl = synth.workload(name)
    sc, p = wl.scene, wl.params
    cam_full = wl.cameras[0]
    cam = tile_camera(cam_full, ctx)
    sample = args.stress_sample if name == "stress" else 1
    if sample > 1:
        # C4 costs ~4 min per frame (every slab truncated to K, ~360k node visits per ray):
        # a stratified sample, every `sample`-th 16x16 square, a different one per rank
        cam = dataclasses.replace(cam_full, tile=TILE, shard=(ctx.rank * 7) % sample, shards=sample)
    R = cam.n_rays
    rays_timed = R * ctx.world if sample > 1 else cam_full.n_rays
    cfg = rg.Config.of(p)
    g = rg.Gaussians.from_scene(sc, device=ctx.dev)
    bws = rg.bvh_workspace(g)
    bvh = rg.build_bvh(g, cfg, ws=bws, check=True)
    fo = dict(rgb=torch.empty(R, 3, device=ctx.dev), T=torch.empty(R, device=ctx.dev),
              replay=torch.empty(R, dtype=torch.int32, device=ctx.dev))
    out = {"workload": wl.notes, "rays_per_frame": cam_full.n_rays, "rays_timed": rays_timed,
           "gaussians": sc.n,
           "parallelism": f"{TILE}x{TILE} tiles interleaved over {ctx.world} rank(s)",
           "steps": args.cfg_steps, "warmup": args.cfg_warmup}
    if sample > 1:
        out["sample"] = (f"every {sample}th {TILE}x{TILE} square of the frame per rank "
                         f"({R} rays per rank), forward only")
    st_f = rg.new_stats(ctx.dev)
    rg.render_forward(g, bvh, cfg, camera=cam, out=fo, stats=st_f)
    torch.cuda.synchronize()
    sf = rg.stats_dict(st_f)
    ms = ctx.timed(lambda: rg.render_forward(g, bvh, cfg, camera=cam, out=fo),
                   args.cfg_steps, args.cfg_warmup)
    mhz = args.mhz or 1965.0
    out["fwd"] = {"value": rays_timed / (ms * 1e-3) / 1e6, "unit": "Mrays/s", "ms": ms,
                  "fps": 1e3 / ms if sample == 1 else None,
                  "frame_s_extrapolated": cam_full.n_rays / (rays_timed / (ms * 1e-3)), "counters": sf,
                  "roofline": roofline_8d(sf, "fwd", ms, mhz, sc.n)}
    if train:
        gws = rg.backward_workspace(g)
        gb = rgd.GradBuffer.like(g)
        drgb = torch.empty(R, 3, device=ctx.dev)
        flog = rg.new_log(R, device=ctx.dev, pairs_per_ray=ppr)
        loss = torch.zeros(1, device=ctx.dev)
        gp = rg.Gaussians.from_scene(perturbed(sc), device=ctx.dev)
        tgt = rg.render_forward(gp, rg.build_bvh(gp, cfg), cfg, camera=cam)["rgb"].clone()
        del gp
        scale = 1.0 / (3.0 * cam_full.n_rays)
        marks = {}

        def step(mark=False):
            ev = [ctx.ev() for _ in range(4)] if mark else None
            if mark: ev[0].record(ctx.stream)
            bv = rg.build_bvh(g, cfg, ws=bws)
            f = rg.render_forward(g, bv, cfg, camera=cam, out=fo, log=flog)
            if mark: ev[1].record(ctx.stream)
            loss.zero_()
            rg.l1_loss_grad(f["rgb"], tgt, scale, d_rgb=drgb, loss=loss)
            gb.zero_()
            rg.render_backward(g, bv, cfg, f, drgb, camera=cam, grads=gb.views, ws=gws)
            if mark: ev[2].record(ctx.stream)
            gb.all_reduce()
            if mark:
                ev[3].record(ctx.stream)
                marks.setdefault("ev", []).append(ev)
        st_b = rg.new_stats(ctx.dev)
        f = rg.render_forward(g, bvh, cfg, camera=cam, out=fo, log=flog)
        rg.l1_loss_grad(f["rgb"], tgt, scale, d_rgb=drgb, loss=loss)
        rg.render_backward(g, bvh, cfg, f, drgb, camera=cam, grads=gb.views, ws=gws, stats=st_b)
        torch.cuda.synchronize()
        sb = rg.stats_dict(st_b)
        ms_t = ctx.timed(lambda: step(True), args.cfg_steps, args.cfg_warmup)
        evs = marks["ev"][-args.cfg_steps:]
        stages = {k: statistics.mean(e[i].elapsed_time(e[i + 1]) for e in evs)
                  for i, k in enumerate(("build_fwd", "loss_bwd", "allreduce"))}
        out["train"] = {"value": cam_full.n_rays / (ms_t * 1e-3) / 1e6, "unit": "Mrays/s",
                        "ms": ms_t, "stages_ms": stages, "counters_bwd": sb,
                        "allreduce_bytes": gb.nbytes, "fetch_log_pairs_per_ray": ppr,
                        "roofline_bwd": roofline_8d(sb, "bwd", stages["loss_bwd"], mhz, sc.n,
                                                    red_gops)}
    out["setup_s"] = time.perf_counter() - t_setup
    return out


def run_ours(args):
    import numpy as np
    import torch

    from paper_2408_03356_b200 import dist as rgd
    from paper_2408_03356_b200 import rg, synth

    ctx = Ctx()
    rank, world, dev, stream = ctx.rank, ctx.world, ctx.dev, ctx.stream
    wl = synth.workload("blender_train", views=8)
    sc, p = wl.scene, wl.params
    cam = wl.cameras[rank % len(wl.cameras)]
    R = cam.n_rays
    cfg = rg.Config.of(p)
    g = rg.Gaussians.from_scene(sc, device=dev)
    bws = rg.bvh_workspace(g)
    gws = rg.backward_workspace(g)
    gb = rgd.GradBuffer.like(g)
    fo = dict(rgb=torch.empty(R, 3, device=dev), T=torch.empty(R, device=dev),
              replay=torch.empty(R, dtype=torch.int32, device=dev))
    drgb = torch.empty(R, 3, device=dev)
    flog = rg.new_log(R, device=dev)
    loss = torch.zeros(1, device=dev)
    # target image: the same view of a seeded perturbation of the scene (setup)
    gp = rg.Gaussians.from_scene(perturbed(sc), device=dev)
    tgt = rg.render_forward(gp, rg.build_bvh(gp, cfg), cfg, camera=cam)["rgb"].clone()
    tgt_host = tgt.cpu().pin_memory()
    tgt_dev = torch.empty_like(tgt)
    loss_host = torch.zeros(1).pin_memory()
    del gp
    scale = 1.0 / (3.0 * R)
    ev = ctx.ev
    stage_ms = {k: 0.0 for k in ("build", "forward", "loss", "backward", "allreduce")}

    def step(target, marks=None):
        if marks is not None:
            marks[0].record(stream)
        bvh = rg.build_bvh(g, cfg, ws=bws)
        if marks is not None:
            marks[1].record(stream)
        f = rg.render_forward(g, bvh, cfg, camera=cam, out=fo, log=flog)
        if marks is not None:
            marks[2].record(stream)
        loss.zero_()
        rg.l1_loss_grad(f["rgb"], target, scale, d_rgb=drgb, loss=loss)
        gb.zero_()
        if marks is not None:
            marks[3].record(stream)
        rg.render_backward(g, bvh, cfg, f, drgb, camera=cam, grads=gb.views, ws=gws)
        if marks is not None:
            marks[4].record(stream)
        gb.all_reduce()
        if marks is not None:
            marks[5].record(stream)

    tgt_dev.copy_(tgt)
    for _ in range(args.warmup):
        step(tgt_dev)
    torch.cuda.synchronize()
    # counters for the roofline's algorithmic work (one instrumented step, untimed)
    st_f, st_b = rg.new_stats(dev), rg.new_stats(dev)
    bvh = rg.build_bvh(g, cfg, ws=bws, check=True)
    f = rg.render_forward(g, bvh, cfg, camera=cam, out=fo, stats=st_f, log=flog)
    rg.l1_loss_grad(f["rgb"], tgt_dev, scale, d_rgb=drgb, loss=loss)
    gb.zero_()
    rg.render_backward(g, bvh, cfg, f, drgb, camera=cam, grads=gb.views, ws=gws, stats=st_b)
    torch.cuda.synchronize()
    sf, sb = rg.stats_dict(st_f), rg.stats_dict(st_b)
    gpu_id = None
    try:
        gpu_id = "GPU-" + str(torch.cuda.get_device_properties(dev).uuid)
    except Exception:  # noqa: BLE001
        gpu_id = str(ctx.local)
    clocks = ClockSampler(gpu_id)
    # ---- timed: K training steps (device time, events on the launch stream)
    marks = [[ev() for _ in range(6)] for _ in range(args.steps)]
    ctx.barrier(); torch.cuda.synchronize()
    l0 = rg.kernel_launches()
    e0, e1 = ev(), ev()
    e0.record(stream)
    for k in range(args.steps):
        step(tgt_dev, marks[k])
    e1.record(stream)
    torch.cuda.synchronize(); ctx.barrier()
    launches = rg.kernel_launches() - l0
    ms = ctx.max_over_ranks(e0.elapsed_time(e1) / args.steps)
    for m in marks:
        for i, key in enumerate(stage_ms):
            stage_ms[key] += m[i].elapsed_time(m[i + 1]) / args.steps
    # ---- end to end through the public API with host buffers
    for _ in range(args.warmup):
        tgt_dev.copy_(tgt_host, non_blocking=True); step(tgt_dev); loss_host.copy_(loss, non_blocking=True)
    ctx.barrier(); torch.cuda.synchronize()
    e4, e5 = ev(), ev()
    e4.record(stream)
    for _ in range(args.steps):
        tgt_dev.copy_(tgt_host, non_blocking=True)
        step(tgt_dev)
        loss_host.copy_(loss, non_blocking=True)
    e5.record(stream)
    torch.cuda.synchronize(); ctx.barrier()
    e2e_ms = ctx.max_over_ranks(e4.elapsed_time(e5) / args.steps)
    clk = clocks.stop()
    mhz = clk.get("sm_mhz") or 1965.0
    args.mhz = mhz
    # ---- C1 forward only (inference: BVH built once), tiles interleaved over the ranks
    cam1 = synth.workload("blender").cameras[0]
    camt = tile_camera(cam1, ctx)
    fo_t = dict(rgb=torch.empty(camt.n_rays, 3, device=dev), T=torch.empty(camt.n_rays, device=dev),
                replay=torch.empty(camt.n_rays, dtype=torch.int32, device=dev))
    bvh = rg.build_bvh(g, cfg, ws=bws)
    fwd_ms = ctx.timed(lambda: rg.render_forward(g, bvh, cfg, camera=camt, out=fo_t),
                       args.steps, args.warmup)
    build_ms = ctx.timed(lambda: rg.build_bvh(g, cfg, ws=bws), args.steps, args.warmup)
    next_rows = {} if args.quick else next_section(ctx, args, g, sc, p, cfg, cam, wl, bws, gws, gb,
                                                   fo, flog, tgt_dev, fwd_ms, R)
    # ---- C3 / C4, tiles interleaved over the ranks
    mb = load_json("profiles", "r1", "microbench.json")
    configs = {}
    for name in [c for c in args.configs.split(",") if c]:
        try:
            configs[name] = measure_config(ctx, name, args, train=(name == "mip"),
                                           red_gops=mb.get("red_f32x4_gops"), ppr=args.mip_ppr)
        except Exception as e:  # noqa: BLE001 -- report, keep the headline line
            configs[name] = {"error": f"{type(e).__name__}: {e}"}
        torch.cuda.empty_cache()

    if rank != 0:
        if world > 1:
            ctx.dist.destroy_process_group()
        return 0
    total_rays = world * R
    value = total_rays / (ms * 1e-3) / 1e6
    dom = "backward" if stage_ms["backward"] >= stage_ms["forward"] else "forward"
    roof = roofline_8d(sb if dom == "backward" else sf, "bwd" if dom == "backward" else "fwd",
                       stage_ms[dom], mhz, sc.n, mb.get("red_f32x4_gops"))
    roof["kernel"] = f"k_render<{'true' if dom == 'backward' else 'false'}, 8, false, 0> ({dom})"
    roof["traffic"] = load_json("profiles", "r2", "ncu_traffic.json").get(dom)
    roof["other"] = roofline_8d(sf if dom == "backward" else sb, "fwd" if dom == "backward" else "bwd",
                                stage_ms["forward" if dom == "backward" else "backward"], mhz, sc.n,
                                mb.get("red_f32x4_gops"))
    line = {
        "metric": METRIC, "value": value, "unit": "Mrays/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": "C1 Blender-like training step: 300k Gaussians SH3+7SG, 800x800 view per rank "
                               "(build + fwd + L1 grad + bwd + finalize + grad all-reduce)",
                   "global_batch": total_rays, "seq_len": None, "parallelism": f"dp{world}",
                   "l2": "per-step working set (fetch-log arena ~720 MB, params 130 MB, grad buffers 270 MB) > 126 MB L2; no flush"},
        "fwd": {"value": cam1.n_rays / (fwd_ms * 1e-3) / 1e6, "unit": "Mrays/s", "ms": fwd_ms,
                "fps": 1e3 / fwd_ms, "paper_fps_rtx4090": PAPER_FPS,
                "parallelism": f"{TILE}x{TILE} tiles interleaved over {world} rank(s)",
                "build_ms": build_ms},
        "stages_ms": stage_ms,
        "configs": configs,
        "next": next_rows,
        "e2e": {"value": total_rays / (e2e_ms * 1e-3) / 1e6, "unit": "Mrays/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": int(tgt_host.numel() * 4), "d2h_bytes_per_step": 4},
        "gpu_launches": int(launches),
        "roofline": roof,
        "counters": {"fwd": sf, "bwd": sb},
        "clocks": clk,
    }
    if world == 1 and not args.no_cpu_baseline:
        from oracle import oracle as O
        O.build()
        tgt_np = tgt.cpu().numpy().astype(np.float64)
        idx = stratified(cam, 4)
        n, s = oracle_step(sc, p, cam, tgt_np, idx)
        cb = {"value": n / s / 1e6, "unit": "Mrays/s", "cores": 1, "kind": "oracle",
              "sample": f"{n} stratified rays (every 4th pixel) of the 800x800 view: "
                        f"oracle BVH build + fwd + L1 grad + bwd, {s:.1f} s",
              "cpu": cpu_model(), "nproc": os.cpu_count(),
              "full_frame_s_extrapolated": R / (n / s)}
        if not args.quick:
            try:
                par = oracle_parallel(4)
                par["full_frame_s_extrapolated"] = R / (par["value"] * 1e6)
                cb["all_cores"] = par
            except Exception as e:  # noqa: BLE001
                cb["all_cores"] = {"error": f"{type(e).__name__}: {e}"}
        line["cpu_baseline"] = cb
    print(json.dumps(line), flush=True)
    if world > 1:
        ctx.dist.destroy_process_group()
    return 0


def next_section(ctx, args, g, sc, p, cfg, cam, wl, bws, gws, gb, fo, flog, tgt_dev, fwd_ms, R):
    """SURVEY §8(f) NEXT rows, each timed alone on the C1 workload"""
    import torch

    from paper_2408_03356_b200 import rg
    dev = ctx.dev

    def timed(fn):
        return ctx.timed(fn, args.steps, args.warmup)
    bvh = rg.build_bvh(g, cfg, ws=bws)
    refit_ms = timed(lambda: rg.refit_bvh(bvh, g, cfg))
    ga = rg.Gaussians(*[t.clone() for t in g.tensors()], sh_degree=g.sh_degree, sg_count=g.sg_count)
    opt = rg.Adam(ga)
    adam_ms = timed(lambda: opt.step(gb.views, it=0))
    n_el = sum(int(t.numel()) for t in g.tensors())
    adam_bytes = 32 * n_el          # read raw, m, v, grad; write raw, m, v, activated (fp32)
    ssim_d = torch.empty(R, 3, device=dev)
    ssim_ws = torch.empty(int(rg.lib().rg_dssim_workspace_bytes(cam.width, cam.height)) // 4,
                          device=dev)
    ssim_loss = torch.zeros(1, device=dev)
    ssim_ms = timed(lambda: rg.l1_dssim_loss_grad(fo["rgb"], tgt_dev, cam.width, cam.height,
                                                  d_rgb=ssim_d, loss=ssim_loss, ws=ssim_ws))
    hbm, _ = hbm_peak()

    def full_iteration():     # one Alg. 3 iteration on its own scene copy
        bv = rg.build_bvh(ga, cfg, ws=bws)
        f_ = rg.render_forward(ga, bv, cfg, camera=cam, out=fo, log=flog)
        ssim_loss.zero_()
        rg.l1_dssim_loss_grad(f_["rgb"], tgt_dev, cam.width, cam.height, d_rgb=ssim_d,
                              loss=ssim_loss, ws=ssim_ws)
        gb.zero_()
        rg.render_backward(ga, bv, cfg, f_, ssim_d, camera=cam, grads=gb.views, ws=gws)
        opt.step(gb.views, it=0)
    iter_ms = timed(full_iteration)
    bvh = rg.build_bvh(g, cfg, ws=bws)
    cam4 = dataclasses.replace(cam, spp=4)
    fo4 = dict(rgb=torch.empty(4 * R, 3, device=dev), T=torch.empty(4 * R, device=dev),
               replay=torch.empty(4 * R, dtype=torch.int32, device=dev))
    fwd4_ms = timed(lambda: rg.render_forward(g, bvh, cfg, camera=cam4, out=fo4))
    fwd1_ms = timed(lambda: rg.render_forward(g, bvh, cfg, camera=cam, out=fo))
    mix_o, mix_d = [], []
    for c in wl.cameras:
        o_, d_ = rg.camera_rays(c, device=dev)
        mix_o.append(o_); mix_d.append(d_)
    perm = torch.randperm(len(wl.cameras) * R, device=dev,
                          generator=torch.Generator(device=dev).manual_seed(7))[:R]
    mo, md = torch.cat(mix_o)[perm].contiguous(), torch.cat(mix_d)[perm].contiguous()
    del mix_o, mix_d
    mix_ms = timed(lambda: rg.render_forward(g, bvh, cfg, rays=(mo, md), out=fo))
    dstats = rg.DensityStats(g.n, dev)
    dstats.accumulate(gb.views["mean"])
    dz = torch.randn(g.n, 2, 3, device=dev, generator=torch.Generator(device=dev).manual_seed(3))
    dens_out = {}

    def dens_step():
        g3, _ = rg.densify(ga, dstats, 5e-5, 1.3, p.sigma_eps, z=dz, adam=opt)
        dens_out["n"] = g3.n
        opt.scene = ga
    dens_ms = timed(dens_step)
    return {
        "alg3_iteration_ms": iter_ms,
        "refit_bvh_ms": refit_ms,
        "adam": {"ms": adam_ms, "elements": n_el, "bytes": adam_bytes,
                 "achieved_gbs": adam_bytes / (adam_ms * 1e-3) / 1e9, "peak_gbs": hbm,
                 "frac": adam_bytes / (adam_ms * 1e-3) / 1e9 / hbm, "bound": "hbm"},
        "l1_dssim_ms": ssim_ms,
        "raygauss4x": {"fwd_ms": fwd4_ms, "rays": 4 * R, "cost_vs_1x": fwd4_ms / fwd1_ms,
                       "paper": "about 3x (P:775)"},
        "densify": {"ms": dens_ms, "n_in": g.n, "n_out": dens_out.get("n"),
                    "what": "accumulate + plan + apply (params, raw, m, v), grad_eps 5e-5"},
        "uncorrelated_rays": {"fwd_ms": mix_ms, "rays": R, "mrays_s": R / (mix_ms * 1e-3) / 1e6,
                              "what": "random sample of the rays of the 8 training views, shuffled"},
    }


def relaunch_distributed(n, script=None, argv=None):
    """python bench.py --gpus N (no torchrun environment): re-run under torch.distributed.run
    (one process per GPU, rendezvous on 127.0.0.1 at a free port)"""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(script or __file__), *(sys.argv[1:] if argv is None else argv)]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--configs", default="mip,stress",
                    help="extra SURVEY §8 configs to measure (mip = C3, stress = C4)")
    ap.add_argument("--stress-sample", type=int, default=64,
                    help="C4: time every n-th 16x16 square of the frame (1 = full frame)")
    ap.add_argument("--cfg-steps", type=int, default=3)
    ap.add_argument("--cfg-warmup", type=int, default=3)
    ap.add_argument("--mip-ppr", type=int, default=320,
                    help="fetch-log budget (pairs per ray) of the C3 training step")
    ap.add_argument("--quick", action="store_true", help="skip the NEXT rows and the parallel oracle")
    args = ap.parse_args()
    args.mhz = None
    if args.warmup < 3:
        args.warmup = 3
    if args.cfg_warmup < 3:
        args.cfg_warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_distributed(args.gpus)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
