"""One C2 end-to-end step through the C ABI (scene from host arrays ->
reference + SAH trees -> trace -> image sources -> IR -> fetch), for ncu
launch lists (development tool)."""
import sys

sys.path.insert(0, '.')
import torch  # noqa: E402

from paper_1811_05784_b200 import roomray as rr, scenes, shard  # noqa: E402

s = scenes.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]()
L = int(round(s.ir_seconds * s.sample_rate))
for i in range(2):
    tree = rr.AccelTree(rr.TriangleMesh(s.vertices, s.faces, s.absorption))
    res = shard.run_sharded(tree, rr.SourceConfig(s.source, s.ray_count), [rr.Receiver(*r) for r in s.receivers],
                            rr.TraceConfig(max_iterations=s.max_iterations, max_range=s.max_range),
                            air=rr.AirModel(), options=rr.ClusterOptions(1e-6, True), sample_rate=s.sample_rate,
                            length=L)
    torch.cuda.synchronize()
    print(f"step {i}: {len(res.images[0])} images", file=sys.stderr)
