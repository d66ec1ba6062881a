import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_1811_05784_b200 import Context, TriangleMesh, scenes
from paper_1811_05784_b200 import roomray as rr
s = scenes.config5()
ctx = Context(0)
m = TriangleMesh(s.vertices, s.faces, s.absorption)
for i in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    tree = rr.AccelTree(m, ctx)
    torch.cuda.synchronize(); print("scene create %.2f ms" % ((time.perf_counter() - t) * 1e3), file=sys.stderr)
    del tree
