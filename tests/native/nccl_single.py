"""One-rank NCCL run of shard.run_sharded with the exchange path forced on:
every collective of the multi-GPU pipeline (all_reduce of the order
histogram, all_to_all_single of capture records and face histories,
all_to_all_single gather of the image lists, all_reduce of the pulse
histograms) runs through NCCL on device tensors, and the result must equal
the plain single-GPU pipeline.  Invoked by tests/test_gpu_shard.py."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1811_05784_b200 import roomray as rr  # noqa: E402
from paper_1811_05784_b200 import scenes, shard  # noqa: E402


def main():
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    s = scenes.config3()  # 5 receivers, open scene
    tree = rr.AccelTree(rr.TriangleMesh(s.vertices, s.faces, s.absorption))
    src = rr.SourceConfig(s.source, 200_000)
    recv = [rr.Receiver(*r) for r in s.receivers]
    cfg = rr.TraceConfig(max_iterations=s.max_iterations, max_range=s.max_range)
    kw = dict(air=rr.AirModel(), options=rr.ClusterOptions(1e-6, True), sample_rate=48000.0, length=48000)
    a = shard.run_sharded(tree, src, recv, cfg, exchange=False, **kw)
    b = shard.run_sharded(tree, src, recv, cfg, exchange=True, **kw)
    h = shard.run_sharded(tree, src, recv, cfg, exchange=True, host=True, **kw)  # pinned host results
    total = 0
    for r in range(len(recv)):
        for f in a.images[r].__dataclass_fields__:
            x, y = getattr(a.images[r], f).cpu().numpy(), getattr(b.images[r], f).cpu().numpy()
            assert np.array_equal(x, y), (r, f)
            z = getattr(h.images[r], f)
            assert not z.is_cuda and np.array_equal(x, z.numpy()), (r, f)
        assert torch.equal(a.band_ir[r], b.band_ir[r]), r
        assert torch.equal(a.band_ir[r].cpu(), h.band_ir[r]), r
        total += len(a.images[r])
    assert total > 20, total
    dist.destroy_process_group()
    print(f"nccl single-rank exchange ok: {total} images over {len(recv)} receivers")


if __name__ == "__main__":
    main()
