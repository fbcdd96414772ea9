"""World-size-N check of the multi-rank plumbing bench.py uses (run under
torch.distributed.run; gloo on CPU): every rank builds its interleaved 16x16
tile camera of the C1 and C3 views (rg_camera.tile/shard/shards), the C-ABI's
host-side rg_camera_ray_count agrees with the binding's slot count, and the
ranks' slots cover every pixel exactly once (all-reduced coverage counts)."""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2408_03356_b200 import dist as rgd  # noqa: E402
from paper_2408_03356_b200 import rg, synth  # noqa: E402


def main():
    rank, world, _ = rgd.init("gloo")
    for cam in (synth.orbit_camera(4.0311, 15.0, 30.0, 800, 800, synth.BLENDER_FX),
                synth.orbit_camera(3.0, 10.0, 0.0, 1245, 825, 1078.2, height_offset=0.6)):
        c = dataclasses.replace(cam, tile=16, shard=rank, shards=world)
        assert rg.camera_ray_count(c) == c.n_rays, (rg.camera_ray_count(c), c.n_rays)
        pix = c.slot_pixels()
        cnt = torch.zeros(cam.width * cam.height, dtype=torch.int64)
        cnt[torch.from_numpy(pix[pix >= 0])] += 1
        if world > 1:
            dist.all_reduce(cnt)
        assert int(cnt.min()) == 1 and int(cnt.max()) == 1
        n = torch.tensor([int((pix >= 0).sum())])
        if world > 1:
            dist.all_reduce(n)
        assert int(n) == cam.width * cam.height
    print(f"rank {rank}/{world} ok", flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
