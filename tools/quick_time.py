"""Quick timing of build / forward / backward on one workload (dev tool).

usage: quick_time.py [name] [--nostats] [--ppr PAIRS] [--rect x0 y0 x1 y1] [--iters N] [--nobwd]
  --ppr   fetch-log budget (pairs per ray, rg_fetch_log_bytes)
  --rect  render only a pixel rectangle of the view (e.g. a crop of C4)
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2408_03356_b200 import rg, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("name", nargs="?", default="blender")
ap.add_argument("--nostats", action="store_true")
ap.add_argument("--ppr", type=int, default=0)
ap.add_argument("--rect", type=int, nargs=4, default=None)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--nobwd", action="store_true")
ap.add_argument("--lc", type=int, default=None, help="rg_config.list_capacity override")
a = ap.parse_args()
wl = synth.workload(a.name)
sc, cam, p = wl.scene, wl.cameras[0], wl.params
if a.rect:
    cam.rect = tuple(a.rect)
g = rg.Gaussians.from_scene(sc)
cfg = rg.Config.of(p)
if a.lc is not None:
    cfg.list_capacity = a.lc


def ev():
    return torch.cuda.Event(enable_timing=True)


lg = rg.new_log(cam.n_rays, pairs_per_ray=a.ppr)
st = rg.new_stats()
for it in range(a.iters):
    st.zero_()
    e0, e1, e2, e3 = ev(), ev(), ev(), ev()
    e0.record(); b = rg.build_bvh(g, cfg); e1.record()
    f = rg.render_forward(g, b, cfg, camera=cam, stats=None if a.nostats else st, log=lg,
                          check=False)
    e2.record()
    if not a.nobwd:
        up = torch.full_like(f["rgb"], 1.0 / f["rgb"].numel())
        rg.render_backward(g, b, cfg, f, up, camera=cam)
    e3.record()
    torch.cuda.synchronize()
    n = cam.n_rays
    print(f"{a.name} it{it}: rays {n} build {e0.elapsed_time(e1):.3f} ms  fwd {e1.elapsed_time(e2):.3f} ms "
          f"({n/e1.elapsed_time(e2)/1e3:.2f} Mrays/s)  bwd {e2.elapsed_time(e3):.3f} ms", flush=True)
if not a.nostats:
    print(rg.stats_dict(st))
    hdr = lg[:16].view(torch.int64).cpu().tolist()
    print(f"fetch log: pair slots used beyond the per-ray blocks {hdr[0]}, window samples {hdr[1]}")
