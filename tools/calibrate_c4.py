"""C4 calibration with the oracle (SURVEY.md §8(d) rule, dev tool): on 1,000
stratified rays of the 1920x1080 stress view, the mean per-slab hit set before
truncation must be >= 2K and the median termination depth >= 0.2 units.

The untruncated per-slab sets are those of an oracle render with
hit_capacity = 4096 (never reached), read from its per-slab dump; the
termination depth is (s_end + 1) * B * dt of the K = 512 render (the
workload's).  Runs the oracle in nproc processes (each builds its own BVH).
Writes profiles/r2/c4_calibration.json.

usage: python tools/calibrate_c4.py [n_rays]
"""
import json
import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def work(args):
    import numpy as np
    from oracle import oracle as O
    from paper_2408_03356_b200 import synth
    part, parts, n_rays = args
    wl = synth.workload("stress")
    sc, cam, p = wl.scene, wl.cameras[0], wl.params
    o_all, d_all = O.camera_rays(cam)
    idx = np.linspace(0, len(o_all) - 1, n_rays).astype(np.int64)[part::parts]
    o, d = o_all[idx], d_all[idx]
    b = O.BVH(sc, p)
    big = p.replace(hit_capacity=4096)
    r_big = O.render(sc, big, o, d, mode=2, bvh=b, dump_cap=400_000)
    r = O.render(sc, p, o, d, mode=2, bvh=b)
    sizes = []
    for dump in r_big["dump"]:
        if len(dump):
            _, counts = np.unique(dump[:, 0], return_counts=True)
            sizes.extend(counts.tolist())
    depth = [(s + 1) * p.slab_samples * p.dt for s in r["s_term"] if s >= 0]
    return sizes, depth, len(idx), int((r["s_term"] < 0).sum())


def main():
    import numpy as np
    n_rays = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
    nproc = os.cpu_count() or 1
    t0 = time.time()
    with mp.get_context("spawn").Pool(nproc) as pool:
        res = pool.map(work, [(k, nproc, n_rays) for k in range(nproc)])
    sizes = np.concatenate([np.asarray(r[0]) for r in res])
    depth = np.concatenate([np.asarray(r[1]) for r in res])
    out = {"rays": int(sum(r[2] for r in res)), "rays_not_terminated": int(sum(r[3] for r in res)),
           "slabs": int(len(sizes)), "mean_slab_set_untruncated": float(sizes.mean()),
           "median_slab_set_untruncated": float(np.median(sizes)),
           "K": 512, "mean_ge_2K": bool(sizes.mean() >= 1024),
           "median_termination_depth": float(np.median(depth)) if len(depth) else None,
           "depth_ge_0.2": bool(len(depth) and np.median(depth) >= 0.2),
           "how": "oracle (mode 2) on evenly spaced pixels of the C4 view; untruncated sets from a "
                  "K = 4096 render's per-slab dump; depth = (s_end + 1) B dt of the K = 512 render",
           "seconds": time.time() - t0, "processes": nproc}
    os.makedirs(os.path.join(ROOT, "profiles", "r2"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "profiles", "r2", "c4_calibration.json"), "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
