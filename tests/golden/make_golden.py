"""Regenerate the golden fixtures from the reference itself.

Runs the UNMODIFIED reference sources (oracle/_ref/libroomray_ref.so, built
by `make -C oracle ref` against the from-scratch Eigen subset) on small
seeded cases and stores inputs + outputs as .npz files next to this script.
Needs /root/reference (this container); the fixtures are committed so the
tests can check the oracle restatement and the GPU path anywhere.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1811_05784_b200 import scenes  # noqa: E402

CONCRETE = [0.36, 0.36, 0.44, 0.31, 0.29, 0.39, 0.25, 0.25]
PODIUM = [0.4, 0.4, 0.3, 0.2, 0.17, 0.15, 0.1, 0.1]
AIR = np.array([1.0, 20.0, 50.0, 101.325])


def save(name, **arrays):
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **arrays)
    print("wrote", name, {k: getattr(v, "shape", v) for k, v in arrays.items()})


def tree_case(ref, name, v, f, a):
    a = np.zeros((int(f[:, 3].max()) + 1, 8)) if len(a) <= f[:, 3].max() else a
    t = ref.scene(oracle.Mesh(v, f, a)).tree()
    save(name, vertices=v, faces=f, absorption=a, left=t.left, right=t.right, face=t.face, lo=t.lo, hi=t.hi,
         root=np.int32(t.root), depth=np.int32(t.depth))


def hit_case(ref, name, v, f, a, o, d):
    sc = ref.scene(oracle.Mesh(v, f, a))
    face, delta, point = sc.nearest_hit(o, d)
    bface, bdelta, _ = sc.nearest_hit(o, d, brute=True)
    save(name, vertices=v, faces=f, absorption=a, origins=o, dirs=d, face=face, delta=delta, point=point,
         brute_face=bface, brute_delta=bdelta)


def trace_case(ref, name, v, f, a, src, n, recv, radius, max_it, max_range, merge):
    sc = ref.scene(oracle.Mesh(v, f, a))
    cap, st = sc.trace(src, n, recv, radius, max_it, max_range, 1)
    im = sc.image_sources(cap, n, AIR, recv, 1e-6, merge)
    save(name, vertices=v, faces=f, absorption=a, source=np.array(src, float), ray_count=np.int64(n),
         receiver=np.array(recv, float), radius=np.float64(radius), max_iterations=np.int32(max_it),
         max_range=np.float64(max_range), merge=np.int32(merge), dirs=ref.fibonacci(n),
         iterations=np.int32(st.iterations), truncated=np.int32(st.truncated), escaped=np.int64(st.escaped),
         out_of_range=np.int64(st.out_of_range), resolved_max_range=np.float64(st.max_range),
         cap_ray=cap.ray, cap_point=cap.point, cap_dir=cap.dir, cap_path=cap.path, cap_mult=cap.mult,
         cap_hist_off=cap.hist_off, cap_hist=cap.hist,
         img_pos=im.pos, img_dist=im.dist, img_energy=im.energy, img_mult=im.mult, img_count=im.ray_count,
         img_order=im.order, img_has_proj=im.has_proj, img_proj=im.proj, img_path_off=im.path_off,
         img_path=im.path)


def main():
    oracle.build(ref=True)
    ref = oracle.Ref()
    # trees: reference generators + seeded soups
    v, f = ref.mesh_gen("box", (5, 4, 3))
    tree_case(ref, "tree_box", v, f, np.zeros((1, 8)))
    v, f = ref.mesh_gen("tetra", level=12)
    tree_case(ref, "tree_tetra4096", v, f, np.zeros((1, 8)))
    v, f, a = scenes.random_soup(5150, 777, 10.0, 0.5)
    tree_case(ref, "tree_soup777", v, f, a)
    beads = []
    for x in (0.0, 10.0, 20.0, 30.0):
        beads += [[x, 0, 0], [x + 0.1, 0, 0], [x, 0.1, 0]]
    tree_case(ref, "tree_beads", np.array(beads), np.array([[3 * i, 3 * i + 1, 3 * i + 2, 0] for i in range(4)]),
              np.zeros((1, 8)))
    # closest hit (acceptance criterion 5 shape)
    v, f, a = scenes.random_soup(424243, 1000, 10.0, 0.4)
    o, d = scenes.random_rays(424250, 4000, 0.0, 10.0)
    hit_case(ref, "hit_soup1000", v, f, a, o, d)
    v, f = ref.mesh_gen("icosphere", level=3)
    o, d = scenes.random_rays(77, 2000, -0.5, 0.5)
    hit_case(ref, "hit_icosphere3", v, f, np.zeros((1, 8)), o, d)
    # traces + image sources
    v, f, a = scenes.box_scene((5, 4, 3), per_wall=[CONCRETE, PODIUM] * 3)
    trace_case(ref, "trace_shoebox_fixture", v, f, a, (4, 2, 1.7), 20000, (2, 2, 1.7), 0.2, 1000, 0.0, 1)
    s = scenes.config1()
    trace_case(ref, "trace_c1", s.vertices, s.faces, s.absorption, s.source, s.ray_count, s.receivers[0][0],
               s.receivers[0][1], s.max_iterations, s.max_range, 1)
    v, f, a = scenes.box_scene((10, 10, 10))
    trace_case(ref, "trace_source_in_receiver", v, f, a, (5, 5, 5), 16, (5, 5, 5), 0.5, 1, 100.0, 0)
    # IR synthesis (1023 taps, per band and broadband)
    dist = scenes.uniform(11, 400, 1.0, 40.0)
    energy = 10.0 ** scenes.uniform(12, 400 * 8, -8.0, 0.0).reshape(400, 8)
    bands = np.stack([ref.synthesize(dist, energy, 343.0, 48000.0, 1 << b) for b in range(8)])
    full = ref.synthesize(dist, energy, 343.0, 48000.0, 0xFF)
    kern = np.stack([ref.band_filter(b, 44100.0) for b in range(8)])
    save("rir_small", dist=dist, energy=energy, band_ir=bands, broadband=full, kernels_44100=kern)
    # air absorption
    betas = {f"beta_{t}_{h}": ref.air_beta(np.array([1.0, t, h, 101.325])) for t, h in [(20, 50), (20, 70), (10, 30)]}
    save("air", alpha_1k_20_70=np.float64(ref.air_alpha(np.array([1.0, 20, 70, 101.325]), 1000.0)),
         alpha_8k_20_50=np.float64(ref.air_alpha(np.array([1.0, 20, 50, 101.325]), 8000.0)), **betas)
    # shoebox lattice oracle (shoebox.cpp:43-116) for the fixture box
    pos, dist, order, energy = ref.lattice((5, 4, 3), np.array([CONCRETE, PODIUM] * 3), (4, 2, 1.7), (2, 2, 1.7),
                                           60.0, 0.2, AIR)
    save("lattice_shoebox", pos=pos, dist=dist, order=order, energy=energy)


if __name__ == "__main__":
    main()
