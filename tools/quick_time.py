"""Quick timing of build / forward / backward on the C1 workload (dev tool)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2408_03356_b200 import rg, synth
nostats = "--nostats" in sys.argv
sys.argv = [a for a in sys.argv if a != "--nostats"]
name = sys.argv[1] if len(sys.argv) > 1 else "blender"
wl = synth.workload(name)
sc, cam, p = wl.scene, wl.cameras[0], wl.params
g = rg.Gaussians.from_scene(sc)
cfg = rg.Config.of(p)
def ev(): return torch.cuda.Event(enable_timing=True)
lg = rg.new_log(cam.n_rays)
for it in range(3):
    st = rg.new_stats()
    e0, e1, e2, e3 = ev(), ev(), ev(), ev()
    e0.record(); b = rg.build_bvh(g, cfg); e1.record()
    f = rg.render_forward(g, b, cfg, camera=cam, stats=None if nostats else st, log=lg); e2.record()
    up = torch.full_like(f["rgb"], 1.0 / f["rgb"].numel())
    gr = rg.render_backward(g, b, cfg, f, up, camera=cam); e3.record()
    torch.cuda.synchronize()
    n = cam.n_rays
    print(f"{name} it{it}: build {e0.elapsed_time(e1):.3f} ms  fwd {e1.elapsed_time(e2):.3f} ms "
          f"({n/e1.elapsed_time(e2)/1e3:.1f} Mrays/s)  bwd {e2.elapsed_time(e3):.3f} ms", flush=True)
e4, e5 = ev(), ev()
e4.record(); rg.refit_bvh(b, g, cfg); e5.record(); torch.cuda.synchronize()
print(f"refit {e4.elapsed_time(e5):.3f} ms")
print(rg.stats_dict(st))
