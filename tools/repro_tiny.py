import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2408_03356_b200 import rg, synth
wl = synth.workload("tiny")
sc, cam, p = wl.scene, wl.cameras[0], wl.params
g = rg.Gaussians.from_scene(sc)
cfg = rg.Config.of(p)
b = rg.build_bvh(g, cfg); torch.cuda.synchronize(); print("build ok", flush=True)
f = rg.render_forward(g, b, cfg, camera=cam); torch.cuda.synchronize(); print("fwd ok", flush=True)
o, d = rg.camera_rays(cam)
f = rg.render_forward(g, b, cfg, rays=(o, d), debug=(64, 512)); torch.cuda.synchronize(); print("fwd dbg ok", flush=True)
