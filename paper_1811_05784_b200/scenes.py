"""Seeded synthetic scenes for the BASELINE.json configurations.

The reference ships only a 12-triangle box generator (mesh_gen.cpp:9-33) and
no meshes for these configs (the paper's theatre mesh is unavailable,
SPEC.md:15), so every scene here is generated deterministically from a seed.
The RNG is splitmix64 (no libstdc++ distributions, so the GPU path, the
oracle and any other tool read identical bytes).  Each generator returns a
``Scene`` (mesh arrays + source / receivers / trace settings).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

MASK64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(seed: int, n: int) -> np.ndarray:
    """n outputs of splitmix64 starting from `seed` (uint64)."""
    with np.errstate(over="ignore"):
        idx = np.arange(1, n + 1, dtype=np.uint64)
        z = np.uint64(seed) + idx * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def uniform(seed: int, n: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
    """n doubles in [lo, hi) from the top 53 bits of splitmix64."""
    u = (splitmix64(seed, n) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    return lo + (hi - lo) * u


@dataclass
class Scene:
    name: str
    vertices: np.ndarray
    faces: np.ndarray
    absorption: np.ndarray
    source: tuple
    receivers: list  # [(center, radius)]
    ray_count: int
    max_iterations: int
    max_range: float
    sample_rate: float
    ir_seconds: float
    speed_of_sound: float = 343.0
    seed: int = 0
    notes: str = ""

    @property
    def n_faces(self) -> int:
        return len(self.faces)


def _grid_wall(axis: int, value: float, u_axis: int, v_axis: int, u_len: float, v_len: float, nu: int, nv: int,
               material: int, vbase: int):
    """Quad grid on the plane x[axis] = value: nu x nv quads, 2 triangles each.
    Coordinates u_i = u_len * i / nu (identical on shared edges of adjacent
    walls, so the box is closed at the coordinate level)."""
    iu = np.arange(nu + 1)
    iv = np.arange(nv + 1)
    U, V = np.meshgrid(u_len * iu / nu, v_len * iv / nv, indexing="ij")
    verts = np.zeros((nu + 1, nv + 1, 3))
    verts[..., axis] = value
    verts[..., u_axis] = U
    verts[..., v_axis] = V
    vid = np.arange((nu + 1) * (nv + 1)).reshape(nu + 1, nv + 1) + vbase
    a = vid[:-1, :-1].reshape(-1)
    b = vid[1:, :-1].reshape(-1)
    c = vid[1:, 1:].reshape(-1)
    d = vid[:-1, 1:].reshape(-1)
    m = np.full(a.shape, material)
    faces = np.stack([np.stack([a, b, c, m], 1), np.stack([a, c, d, m], 1)], 1).reshape(-1, 4)
    return verts.reshape(-1, 3), faces


def gridded_shoebox(dims, grids, materials):
    """Box [0,Lx]x[0,Ly]x[0,Lz] with walls x0,x1,y0,y1,z0,z1 (order of
    make_box_mesh, mesh_gen.cpp:26-31) split into quad grids.
    grids[w] = (nu, nv) along the wall's two in-plane axes (ascending)."""
    Lx, Ly, Lz = dims
    L = (Lx, Ly, Lz)
    walls = [(0, 0.0), (0, Lx), (1, 0.0), (1, Ly), (2, 0.0), (2, Lz)]
    V, F = [], []
    vbase = 0
    for w, (axis, value) in enumerate(walls):
        ua, va = [k for k in range(3) if k != axis]
        nu, nv = grids[w]
        v, f = _grid_wall(axis, value, ua, va, L[ua], L[va], nu, nv, materials[w], vbase)
        V.append(v)
        F.append(f)
        vbase += len(v)
    return np.concatenate(V), np.concatenate(F).astype(np.int32)


def config1() -> Scene:
    """C1: shoebox 8x6x3 m, 1 200 triangles, alpha 0.1 in all bands,
    10^4 rays, 20 reflections, 1 s IR at 44.1 kHz."""
    v, f = gridded_shoebox((8.0, 6.0, 3.0), [(10, 10)] * 6, [0] * 6)
    alpha = np.full((1, 8), 0.1)
    return Scene("c1_shoebox_1200", v, f, alpha, (2.0, 3.0, 1.5), [((6.0, 2.0, 1.2), 0.5)], 10_000, 20, 343.0,
                 44100.0, 1.0, notes="max_range = c * 1 s (explicit on both sides)")


def config2(seed: int = 20240611) -> Scene:
    """C2: same room, walls gridded to exactly 100 000 triangles, per-wall
    per-octave alpha ~ U[0.02, 0.4) from splitmix64(seed), 10^6 rays,
    50 reflections, 2 s IR at 48 kHz."""
    # x-walls (6x3 m): 85x40 quads; y-walls (8x3): 80x30; z-walls (8x6): 160x120
    grids = [(85, 40), (85, 40), (80, 30), (80, 30), (160, 120), (160, 120)]
    v, f = gridded_shoebox((8.0, 6.0, 3.0), grids, list(range(6)))
    assert len(f) == 100_000
    alpha = uniform(seed, 48, 0.02, 0.4).reshape(6, 8)
    return Scene("c2_shoebox_100k", v, f, alpha, (2.0, 3.0, 1.5), [((6.0, 2.0, 1.2), 0.5)], 1_000_000, 50, 686.0,
                 48000.0, 2.0, seed=seed, notes="max_range = c * 2 s")


def box_scene(dims=(5.0, 4.0, 3.0), absorption=None, per_wall=None) -> tuple:
    """make_box_mesh (mesh_gen.cpp:9-33): 12 triangles, one material per wall."""
    Lx, Ly, Lz = dims
    v = np.array([[0, 0, 0], [Lx, 0, 0], [Lx, Ly, 0], [0, Ly, 0], [0, 0, Lz], [Lx, 0, Lz], [Lx, Ly, Lz],
                  [0, Ly, Lz]], dtype=np.float64)
    quads = [(0, 4, 7, 3), (1, 2, 6, 5), (0, 1, 5, 4), (3, 7, 6, 2), (0, 3, 2, 1), (4, 5, 6, 7)]
    f = []
    for w, (a, b, c, d) in enumerate(quads):
        f.append((a, b, c, w))
        f.append((a, c, d, w))
    if per_wall is not None:
        alpha = np.asarray(per_wall, np.float64).reshape(6, 8)
    else:
        a = np.zeros(8) if absorption is None else np.broadcast_to(np.asarray(absorption, np.float64), (8,))
        alpha = np.tile(a, (6, 1))
    return v, np.array(f, np.int32), alpha


def random_soup(seed: int, n_faces: int, extent: float = 10.0, face_size: float = 0.4):
    """Triangle soup: centres U[0, extent)^3, vertices centre + U[-s, s)^3
    (the shape of tests/test_support.hpp:38-58, seeded splitmix64)."""
    r = uniform(seed, n_faces * 12).reshape(n_faces, 12)
    c = r[:, :3] * extent
    off = (r[:, 3:].reshape(n_faces, 3, 3) * 2.0 - 1.0) * face_size
    v = (c[:, None, :] + off).reshape(-1, 3)
    f = np.stack([np.arange(n_faces) * 3, np.arange(n_faces) * 3 + 1, np.arange(n_faces) * 3 + 2,
                  np.zeros(n_faces, int)], 1).astype(np.int32)
    e1 = v[f[:, 1]] - v[f[:, 0]]
    e2 = v[f[:, 2]] - v[f[:, 0]]
    area = 0.5 * np.linalg.norm(np.cross(e1, e2), axis=1)
    keep = area > 1e-9
    f = f[keep]
    f[:, :3] = np.arange(len(f) * 3).reshape(-1, 3)
    v = v.reshape(n_faces, 3, 3)[keep].reshape(-1, 3)
    return v, f, np.zeros((1, 8))


def random_rays(seed: int, n: int, lo: float, hi: float):
    """Origins U[lo, hi)^3 and unit directions (normalised Gaussians via
    Box-Muller on splitmix64 uniforms)."""
    u = uniform(seed, n * 9).reshape(n, 9)
    o = lo + (hi - lo) * u[:, :3]
    r = np.sqrt(-2.0 * np.log(1.0 - u[:, 3:6]))
    g = r * np.cos(2.0 * np.pi * u[:, 6:9])
    g /= np.linalg.norm(g, axis=1, keepdims=True)
    return o, g


CONFIGS = {"c1": config1, "c2": config2}
