#!/usr/bin/env python
"""bench.py -- RayGauss hot path on B200: Mrays/s of one training step
(BVH rebuild + forward + L1 loss gradient + backward + finalize [+ NCCL
all-reduce of the per-Gaussian gradients for N > 1]) on the Blender-like C1
scene (300k Gaussians, SH degree 3 + 7 SG lobes, 800x800 rays per rank and
step; BASELINE.json configs[1]/[2]).  Weak scaling: each rank renders and
backprops its own 800x800 view (view = rank, azimuths 45 deg apart, so N = 8
is the C2 training step), gradients are summed across ranks.

Contract (task statement / DESIGN.md §7):
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
prints ONE JSON line on rank 0.  Device timing with CUDA events over exactly
K steps bracketed by barrier + synchronize, max over ranks.  Also reported:
forward-only Mrays/s (paper's inference metric), end-to-end (host target
image in, host loss out), per-stage ms, roofline of the dominant kernel, the
oracle CPU baseline, SM clocks sampled during the timed region.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Mrays/s fwd and fwd+bwd (800x800 Blender-like) at 1/2/4/8 B200; % of roofline"
PAPER_FPS = 25.0   # P:25, P:358 (RTX 4090, 800x800): context only

# --- algorithmic ALU work per unit, deg 3 + 7 SG -------------
# flops count an FMA as 2; MUFU ops (ex2/lg2/rcp-class SFU) counted apart and
# weighted by the FP32:SFU throughput ratio (128*2 : 16 = 16) in the roofline.
def unit_costs(deg, lobes):
    nc = (deg + 1) ** 2
    sh_basis = {0: 0, 1: 3, 2: 18, 3: 45}[deg]
    pair_f = 120 + sh_basis + 6 * nc + 16 * lobes          # interval + offset + exponent + colour
    pair_m = 2 + lobes
    return dict(
        fwd=dict(eval_f=12, eval_m=1, pair_f=pair_f, pair_m=pair_m, samp_f=25, samp_m=2),
        bwd=dict(eval_f=12 + 26, eval_m=2, pair_f=pair_f + 130 + sh_basis + 6 * nc + 20 * lobes,
                 pair_m=pair_m + lobes, samp_f=50, samp_m=2),
    )


def alu_work(stats, c, which):
    k = c[which]
    f = stats["evals"] * k["eval_f"] + stats["pairs"] * k["pair_f"] + stats["samples"] * k["samp_f"]
    m = stats["evals"] * k["eval_m"] + stats["pairs"] * k["pair_m"] + stats["samples"] * k["samp_m"]
    return f, m


def _ncu_traffic(stage):
    """DRAM bytes per launch of the dominant kernel from the committed ncu
    capture (profiles/r1/ncu_traffic.json); None when absent."""
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r1", "ncu_traffic.json")
    try:
        return json.load(open(p)).get(stage)
    except (OSError, ValueError):
        return None


def _microbench():
    """Measured FFMA / MUFU / RED rates (tools/microbench.cu, profiles/r1/microbench.json)."""
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r1", "microbench.json")
    try:
        return json.load(open(p))
    except (OSError, ValueError):
        return {}


def red_ops(stats, deg, lobes):
    """float4 reductions the backward scatter issues: 4 geometry + the appearance
    chunks (3 * pad4(nc) / 4 + 2 * lobes) per pair (upper bound: pairs whose
    moments are all zero are skipped)."""
    nc = (deg + 1) ** 2
    return stats["pairs"] * (4 + 3 * ((nc + 3) // 4) + 2 * lobes)


def peaks(sm_mhz):
    sms = 148
    fp32 = sms * 128 * 2 * sm_mhz * 1e6      # FLOP/s
    mufu = sms * 16 * sm_mhz * 1e6           # SFU op/s
    return fp32, mufu


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


def oracle_step(sc, p, cam, target_rgb, step_px):
    """One oracle pass over a stratified ray sample: BVH build, forward,
    L1 gradient, backward (the same path, single-threaded C, fp64 values)."""
    import numpy as np
    from oracle import oracle as O
    idx = stratified(cam, step_px)
    o_all, d_all = O.camera_rays(cam)
    o, d = o_all[idx], d_all[idx]
    t0 = time.perf_counter()
    b = O.BVH(sc, p)
    r = O.render(sc, p, o, d, mode=2, bvh=b)
    gr = np.sign(r["rgb"] - target_rgb[idx]) / (3.0 * len(idx))
    O.backward(sc, p, o, d, gr, mode=2, bvh=b)
    return len(idx), time.perf_counter() - t0


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
    workload, rank 0 only."""
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
    # targets only where the sample looks (the oracle renders ~3k rays/s)
    idx = stratified(cam, step_px)
    o_all, d_all = O.camera_rays(cam)
    tgt = np.zeros((cam.n_rays, 3))
    tgt[idx] = O.render(perturbed(sc), p, o_all[idx], d_all[idx], mode=2)["rgb"]
    for _ in range(args.warmup):
        oracle_step(sc, p, cam, tgt, step_px)
    tot_rays, tot_s = 0, 0.0
    for _ in range(args.steps):
        n, s = oracle_step(sc, p, cam, tgt, step_px)
        tot_rays += n
        tot_s += s
    v = tot_rays / tot_s / 1e6
    sample = f"1/{step_px * step_px} stratified pixels ({n} rays) of the 800x800 view per step: oracle BVH build + forward + L1 grad + backward"
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "Mrays/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tot_s / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C1 Blender-like training step (300k Gaussians, SH3+7SG, 800x800 view)",
                       "global_batch": n, "seq_len": None, "parallelism": "cpu1"},
            "cpu_baseline": {"value": v, "unit": "Mrays/s", "cores": 1, "kind": "oracle",
                             "sample": sample, "cpu": cpu_model(), "nproc": os.cpu_count()},
            "e2e": {"value": v, "unit": "Mrays/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2408_03356_b200 import dist as rgd
    from paper_2408_03356_b200 import rg, synth

    rank, world, local = rgd.init()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
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
    stream = torch.cuda.current_stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
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

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world > 1:
            t = torch.tensor([x], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())
        return x

    tgt_dev.copy_(tgt)
    for _ in range(args.warmup):
        step(tgt_dev)
    torch.cuda.synchronize()
    # counters for the roofline's algorithmic work (one instrumented step, untimed)
    st_f, st_b = rg.new_stats(dev), rg.new_stats(dev)
    bvh = rg.build_bvh(g, cfg, ws=bws)
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
        gpu_id = str(local)
    clocks = ClockSampler(gpu_id)
    # ---- timed: K training steps (device time, events on the launch stream)
    marks = [[ev() for _ in range(6)] for _ in range(args.steps)]
    barrier(); torch.cuda.synchronize()
    l0 = rg.kernel_launches()
    e0, e1 = ev(), ev()
    e0.record(stream)
    for k in range(args.steps):
        step(tgt_dev, marks[k])
    e1.record(stream)
    torch.cuda.synchronize(); barrier()
    launches = rg.kernel_launches() - l0
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    for m in marks:
        for i, key in enumerate(stage_ms):
            stage_ms[key] += m[i].elapsed_time(m[i + 1]) / args.steps
    # ---- forward only (inference: BVH built once, outside the timed region)
    bvh = rg.build_bvh(g, cfg, ws=bws)
    for _ in range(args.warmup):
        rg.render_forward(g, bvh, cfg, camera=cam, out=fo)
    barrier(); torch.cuda.synchronize()
    e2, e3 = ev(), ev()
    e2.record(stream)
    for _ in range(args.steps):
        rg.render_forward(g, bvh, cfg, camera=cam, out=fo)
    e3.record(stream)
    torch.cuda.synchronize(); barrier()
    fwd_ms = max_over_ranks(e2.elapsed_time(e3) / args.steps)
    # ---- UpdateBVH by refit (rg_refit_bvh): reported beside the
    # rebuild the step uses (the paper rebuilds after every step)
    for _ in range(args.warmup):
        rg.refit_bvh(bvh, g, cfg)
    torch.cuda.synchronize()
    e6, e7 = ev(), ev()
    e6.record(stream)
    for _ in range(args.steps):
        rg.refit_bvh(bvh, g, cfg)
    e7.record(stream)
    torch.cuda.synchronize()
    refit_ms = max_over_ranks(e6.elapsed_time(e7) / args.steps)
    # ---- the other NEXT-1 kernels, each timed alone on the same workload
    def timed(fn):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        a, b_ = ev(), ev()
        a.record(stream)
        for _ in range(args.steps):
            fn()
        b_.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b_) / args.steps
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
    hbm = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                      "MEASURED_PEAKS.json"))).get("hbm_gbs", 6547.8) \
        if os.path.exists(os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                       "MEASURED_PEAKS.json")) else 6547.8
    # one full optimisation iteration of Alg. 3: UpdateBVH (rebuild),
    # RayCast, Loss (L1 + D-SSIM), backward, AdamOptim -- on its own scene copy
    def full_iteration():
        bv = rg.build_bvh(ga, cfg, ws=bws)
        f_ = rg.render_forward(ga, bv, cfg, camera=cam, out=fo, log=flog)
        ssim_loss.zero_()
        rg.l1_dssim_loss_grad(f_["rgb"], tgt_dev, cam.width, cam.height, d_rgb=ssim_d,
                              loss=ssim_loss, ws=ssim_ws)
        gb.zero_()
        rg.render_backward(ga, bv, cfg, f_, ssim_d, camera=cam, grads=gb.views, ws=gws)
        opt.step(gb.views, it=0)
    iter_ms = timed(full_iteration)
    # NEXT-2: RayGauss4x (P:775, 4 rays per pixel) and uncorrelated ray batches
    # mixing the 8 training views, forward only, BVH built once
    import dataclasses
    bvh = rg.build_bvh(g, cfg, ws=bws)
    cam4 = dataclasses.replace(cam, spp=4)
    fo4 = dict(rgb=torch.empty(4 * R, 3, device=dev), T=torch.empty(4 * R, device=dev),
               replay=torch.empty(4 * R, dtype=torch.int32, device=dev))
    fwd4_ms = timed(lambda: rg.render_forward(g, bvh, cfg, camera=cam4, out=fo4))
    mix_o, mix_d = [], []
    for c in wl.cameras:
        o_, d_ = rg.camera_rays(c, device=dev)
        mix_o.append(o_); mix_d.append(d_)
    perm = torch.randperm(len(wl.cameras) * R, device=dev,
                          generator=torch.Generator(device=dev).manual_seed(7))[:R]
    mo, md = torch.cat(mix_o)[perm].contiguous(), torch.cat(mix_d)[perm].contiguous()
    del mix_o, mix_d
    mix_ms = timed(lambda: rg.render_forward(g, bvh, cfg, rays=(mo, md), out=fo))
    # NEXT-4: one adaptive-density-control step (statistic of this step's dL/dmu,
    # plan, apply to the parameters and the Adam state), grad_eps of P:644 (Blender)
    dstats = rg.DensityStats(g.n, dev)
    dstats.accumulate(gb.views["mean"])
    dz = torch.randn(g.n, 2, 3, device=dev, generator=torch.Generator(device=dev).manual_seed(3))
    dens_out = {}

    def dens_step():
        g3, act3 = rg.densify(ga, dstats, 5e-5, 1.3, p.sigma_eps, z=dz, adam=opt)
        dens_out["n"] = g3.n
        opt.scene = ga
    dens_ms = timed(dens_step)
    next_rows = {
        "alg3_iteration_ms": iter_ms,
        "refit_bvh_ms": refit_ms,
        "adam": {"ms": adam_ms, "elements": n_el, "bytes": adam_bytes,
                 "achieved_gbs": adam_bytes / (adam_ms * 1e-3) / 1e9, "peak_gbs": hbm,
                 "frac": adam_bytes / (adam_ms * 1e-3) / 1e9 / hbm, "bound": "hbm"},
        "l1_dssim_ms": ssim_ms,
        "raygauss4x": {"fwd_ms": fwd4_ms, "rays": 4 * R, "cost_vs_1x": fwd4_ms / fwd_ms,
                       "paper": "about 3x (P:775)"},
        "densify": {"ms": dens_ms, "n_in": g.n, "n_out": dens_out.get("n"),
                    "what": "accumulate + plan + apply (params, raw, m, v), grad_eps 5e-5"},
        "uncorrelated_rays": {"fwd_ms": mix_ms, "rays": R,
                              "mrays_s": R / (mix_ms * 1e-3) / 1e6,
                              "what": "random sample of the rays of the 8 training views, shuffled"},
    }
    # ---- end to end through the public API with host buffers
    for _ in range(args.warmup):
        tgt_dev.copy_(tgt_host, non_blocking=True); step(tgt_dev); loss_host.copy_(loss, non_blocking=True)
    barrier(); torch.cuda.synchronize()
    e4, e5 = ev(), ev()
    e4.record(stream)
    for _ in range(args.steps):
        tgt_dev.copy_(tgt_host, non_blocking=True)
        step(tgt_dev)
        loss_host.copy_(loss, non_blocking=True)
    e5.record(stream)
    torch.cuda.synchronize(); barrier()
    e2e_ms = max_over_ranks(e4.elapsed_time(e5) / args.steps)
    clk = clocks.stop()

    if rank != 0:
        return 0
    total_rays = world * R
    value = total_rays / (ms * 1e-3) / 1e6
    # roofline of the dominant kernel (largest stage)
    costs = unit_costs(sc.sh_degree, sc.sg_count)
    mhz = clk.get("sm_max_mhz") or 1965.0
    pf, pm = peaks(mhz)
    dom = "backward" if stage_ms["backward"] >= stage_ms["forward"] else "forward"
    flops, mufu = alu_work(sb if dom == "backward" else sf, costs, "bwd" if dom == "backward" else "fwd")
    t_dom = stage_ms[dom] * 1e-3
    achieved = (flops + 16.0 * mufu) / t_dom / 1e12
    # the backward's second bound: float4 reductions into the gradient rows (L2 RED rate)
    mb = _microbench()
    red_line = None
    if dom == "backward" and mb.get("red_f32x4_gops"):
        ops = red_ops(sb, sc.sh_degree, sc.sg_count)
        ach = ops / t_dom / 1e9
        red_line = {"ops": int(ops), "achieved_gops": ach, "peak_gops": mb["red_f32x4_gops"],
                    "frac": ach / mb["red_f32x4_gops"], "unit": "G float4 RED/s",
                    "peak_source": "tools/microbench.cu (profiles/r1/microbench.json)"}
    peak = pf / 1e12
    line = {
        "metric": METRIC, "value": value, "unit": "Mrays/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": "C1 Blender-like training step: 300k Gaussians SH3+7SG, 800x800 view per rank "
                               "(build + fwd + L1 grad + bwd + finalize + grad all-reduce)",
                   "global_batch": total_rays, "seq_len": None, "parallelism": f"dp{world}",
                   "l2": "per-step working set (fetch-log arena ~720 MB, params 130 MB, grad buffers 270 MB) > 126 MB L2; no flush"},
        "fwd": {"value": world * R / (fwd_ms * 1e-3) / 1e6, "unit": "Mrays/s", "ms": fwd_ms,
                "fps_per_gpu": 1e3 / fwd_ms, "paper_fps_rtx4090": PAPER_FPS},
        "stages_ms": stage_ms,
        "next": next_rows,
        "e2e": {"value": total_rays / (e2e_ms * 1e-3) / 1e6, "unit": "Mrays/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": int(tgt_host.numel() * 4), "d2h_bytes_per_step": 4},
        "gpu_launches": int(launches),
        "roofline": {"bound": "alu", "kernel": f"k_render<{'true' if dom == 'backward' else 'false'}> ({dom})",
                     "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                     "traffic": _ncu_traffic(dom),
                     "work": {"flops": flops, "mufu": mufu, "mufu_weight": 16, "sm_mhz_for_peak": mhz},
                     "peak_source": "148 SM x 128 FP32 lanes x 2 x sm_max_mhz (B200_PROFILING.md counts); MUFU 16/SM/clk",
                     "measured_ffma_tflops": mb.get("ffma_tflops"),
                     "red": red_line},
        "counters": {"fwd": sf, "bwd": sb},
        "clocks": clk,
    }
    if world == 1 and not args.no_cpu_baseline:
        from oracle import oracle as O
        O.build()
        tgt_np = tgt.cpu().numpy().astype(np.float64)
        n, s = oracle_step(sc, p, cam, tgt_np, 4)
        line["cpu_baseline"] = {"value": n / s / 1e6, "unit": "Mrays/s", "cores": 1, "kind": "oracle",
                                "sample": f"{n} stratified rays (every 4th pixel) of the 800x800 view: "
                                          f"oracle BVH build + fwd + L1 grad + bwd, {s:.1f} s",
                                "cpu": cpu_model(), "nproc": os.cpu_count()}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
