"""dev tool: first per-slab hit-set difference GPU vs oracle on sampled C4 rays"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
from paper_2408_03356_b200 import rg, synth
from oracle import oracle as O
from test_gpu_parity import _scene, _sampled
O.build()
wl = _scene("stress"); sc, cam, p = wl.scene, wl.cameras[0], wl.params
o, d = _sampled(cam, 24, 5)
g = rg.Gaussians.from_scene(sc); cfg = rg.Config.of(p); b = rg.build_bvh(g, cfg)
st = rg.new_stats()
out = rg.render_forward(g, b, cfg, rays=(torch.from_numpy(o).cuda(), torch.from_numpy(d).cuda()), stats=st, debug=(24, 300000))
torch.cuda.synchronize()
ref = O.render(sc, p, o, d, mode=2, dump_cap=300000)
cnts = out["debug_counts"].cpu().numpy(); recs = out["debug_records"].cpu().numpy()
print(rg.stats_dict(st))
for r in range(24):
    gr = recs[r, :cnts[r]]; rr = ref["dump"][r]
    if len(gr) == len(rr) and np.array_equal(gr, rr):
        continue
    n = min(len(gr), len(rr)); i = 0
    while i < n and np.array_equal(gr[i], rr[i]): i += 1
    print("ray", r, "gpu", len(gr), "ref", len(rr), "first diff at", i, "gpu", gr[i:i+4].tolist(), "ref", rr[i:i+4].tolist())
    s = rr[i][0] if i < len(rr) else gr[i][0]
    gs = set(int(x) for x in gr[gr[:, 0] == s][:, 1]); rs = set(int(x) for x in rr[rr[:, 0] == s][:, 1])
    print("   slab", s, "missing", sorted(rs - gs)[:8], "extra", sorted(gs - rs)[:8], "sizes", len(gs), len(rs))
