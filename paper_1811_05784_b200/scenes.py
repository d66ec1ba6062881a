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


# ---------------------------------------------------------------- mesh builder
class _MeshBuilder:
    """Accumulates vertices / triangles (a, b, c, material)."""

    def __init__(self):
        self.V, self.F, self.nv = [], [], 0

    def add(self, verts, faces):
        verts = np.asarray(verts, np.float64).reshape(-1, 3)
        faces = np.asarray(faces, np.int64).reshape(-1, 4).copy()
        faces[:, :3] += self.nv
        self.V.append(verts)
        self.F.append(faces)
        self.nv += len(verts)

    def grid(self, P, material):
        """Quad grid over the point array P (nu+1, nv+1, 3): 2 triangles per cell."""
        nu, nv = P.shape[0] - 1, P.shape[1] - 1
        vid = np.arange((nu + 1) * (nv + 1)).reshape(nu + 1, nv + 1)
        a, b, c, d = vid[:-1, :-1].ravel(), vid[1:, :-1].ravel(), vid[1:, 1:].ravel(), vid[:-1, 1:].ravel()
        m = np.full(a.shape, material)
        f = np.stack([np.stack([a, b, c, m], 1), np.stack([a, c, d, m], 1)], 1).reshape(-1, 4)
        self.add(P.reshape(-1, 3), f)

    def count(self):
        return sum(len(f) for f in self.F)

    def arrays(self):
        return np.concatenate(self.V), np.concatenate(self.F).astype(np.int32)


def _icosphere(level: int):
    """Unit icosphere: icosahedron, `level` midpoint subdivisions projected
    on the sphere (20 * 4^level faces)."""
    t = (1.0 + 5 ** 0.5) / 2.0
    v = np.array([[-1, t, 0], [1, t, 0], [-1, -t, 0], [1, -t, 0], [0, -1, t], [0, 1, t], [0, -1, -t], [0, 1, -t],
                  [t, 0, -1], [t, 0, 1], [-t, 0, -1], [-t, 0, 1]], np.float64)
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    f = np.array([[0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11], [1, 5, 9], [5, 11, 4], [11, 10, 2],
                  [10, 7, 6], [7, 1, 8], [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8], [3, 8, 9], [4, 9, 5],
                  [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1]], np.int64)
    for _ in range(level):
        e = np.concatenate([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]])
        key = np.sort(e, 1)
        uniq, inv = np.unique(key[:, 0] * len(v) + key[:, 1], return_inverse=True)
        a, b = uniq // len(v), uniq % len(v)
        mid = v[a] + v[b]
        mid /= np.linalg.norm(mid, axis=1, keepdims=True)
        m = inv.reshape(3, -1).T + len(v)  # midpoints of edges (01, 12, 20)
        v = np.concatenate([v, mid])
        f = np.concatenate([np.stack([f[:, 0], m[:, 0], m[:, 2]], 1), np.stack([f[:, 1], m[:, 1], m[:, 0]], 1),
                            np.stack([f[:, 2], m[:, 2], m[:, 1]], 1), m])
    return v, f


def _rotation(u3):
    """Uniform random rotation from three uniforms (Shoemake quaternions)."""
    u1, u2, u3_ = u3
    q = np.array([np.sqrt(1 - u1) * np.sin(2 * np.pi * u2), np.sqrt(1 - u1) * np.cos(2 * np.pi * u2),
                  np.sqrt(u1) * np.sin(2 * np.pi * u3_), np.sqrt(u1) * np.cos(2 * np.pi * u3_)])
    x, y, z, w = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                     [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                     [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])


def _box_surface(n: int):
    """Unit cube [-1,1]^3, every face an n x n quad grid (12 n^2 faces)."""
    t = np.linspace(-1.0, 1.0, n + 1)
    V, F, base = [], [], 0
    for axis in range(3):
        for side in (-1.0, 1.0):
            ua, va = [k for k in range(3) if k != axis]
            U, W = np.meshgrid(t, t, indexing="ij")
            P = np.zeros((n + 1, n + 1, 3))
            P[..., axis] = side
            P[..., ua] = U
            P[..., va] = W
            vid = np.arange((n + 1) ** 2).reshape(n + 1, n + 1) + base
            a, b, c, d = vid[:-1, :-1].ravel(), vid[1:, :-1].ravel(), vid[1:, 1:].ravel(), vid[:-1, 1:].ravel()
            F.append(np.stack([np.stack([a, b, c], 1), np.stack([a, c, d], 1)], 1).reshape(-1, 3))
            V.append(P.reshape(-1, 3))
            base += (n + 1) ** 2
    return np.concatenate(V), np.concatenate(F)


def _shoebox_grid_for(dims, n_tri):
    """Per-wall quad grids of a [0,Lx]x[0,Ly]x[0,Lz] box with exactly n_tri
    triangles: cells of about equal area, the remainder absorbed by the
    floor's column count (n_tri must be even)."""
    assert n_tri % 2 == 0
    Lx, Ly, Lz = dims
    quads = n_tri // 2
    area = 2 * (Ly * Lz + Lx * Lz + Lx * Ly)
    h = (area / quads) ** 0.5
    walls = [(Ly, Lz), (Ly, Lz), (Lx, Lz), (Lx, Lz), (Lx, Ly), (Lx, Ly)]
    grids = [(max(1, round(a / h)), max(1, round(b / h))) for a, b in walls]
    used = sum(u * v for u, v in grids[:4]) + grids[5][0] * grids[5][1]
    rest = quads - used  # floor (wall 4) gets the rest: nu x nv with nu*nv == rest
    nv = grids[4][1]
    while rest % nv:
        nv -= 1
    grids[4] = (rest // nv, nv)
    return grids


def subdivided_tetrahedron(log2_faces: int):
    """The paper's complexity fixture (the reference's
    make_subdivided_tetrahedron, mesh_gen.cpp:111-153, restated): a regular
    tetrahedron inscribed in the unit sphere, 4-way flat midpoint subdivision
    to 4^q faces, plus one longest-edge bisection pass for odd exponents, so
    exactly 2^log2_faces faces.  Returns (vertices, faces, absorption=0)."""
    if log2_faces < 2:
        raise ValueError("need log2_faces >= 2 (a tetrahedron has 4 faces)")
    s = 1.0 / 3.0 ** 0.5
    v = [(s, s, s), (s, -s, -s), (-s, s, -s), (-s, -s, s)]
    f = [(0, 1, 2), (0, 3, 1), (0, 2, 3), (1, 3, 2)]
    V = np.array(v, np.float64)
    F = np.array(f, np.int64)
    for _ in range((log2_faces - 2) // 2):
        e = np.concatenate([F[:, [0, 1]], F[:, [1, 2]], F[:, [2, 0]]])
        key = np.sort(e, 1)
        uniq, inv = np.unique(key[:, 0] * len(V) + key[:, 1], return_inverse=True)
        a, b = uniq // len(V), uniq % len(V)
        mid = 0.5 * (V[a] + V[b])
        m = inv.reshape(3, -1).T + len(V)  # midpoints of edges (ab, bc, ca)
        V = np.concatenate([V, mid])
        F = np.concatenate([np.stack([F[:, 0], m[:, 0], m[:, 2]], 1), np.stack([m[:, 0], F[:, 1], m[:, 1]], 1),
                            np.stack([m[:, 2], m[:, 1], F[:, 2]], 1), m])
    if log2_faces % 2 == 1:
        a, b, c = F[:, 0], F[:, 1], F[:, 2]
        lab = np.linalg.norm(V[a] - V[b], axis=1)
        lbc = np.linalg.norm(V[b] - V[c], axis=1)
        lca = np.linalg.norm(V[c] - V[a], axis=1)
        u, w, x = a.copy(), b.copy(), c.copy()  # split edge (u, w), apex x
        sel_bc = (lbc >= lab) & (lbc >= lca)
        sel_ca = ~sel_bc & (lca >= lab) & (lca >= lbc)
        u[sel_bc], w[sel_bc], x[sel_bc] = b[sel_bc], c[sel_bc], a[sel_bc]
        u[sel_ca], w[sel_ca], x[sel_ca] = c[sel_ca], a[sel_ca], b[sel_ca]
        key = np.sort(np.stack([u, w], 1), 1)
        uniq, inv = np.unique(key[:, 0] * len(V) + key[:, 1], return_inverse=True)
        mid = 0.5 * (V[uniq // len(V)] + V[uniq % len(V)])
        mi = inv + len(V)
        V = np.concatenate([V, mid])
        F = np.concatenate([np.stack([u, mi, x], 1), np.stack([mi, w, x], 1)])
    assert len(F) == 1 << log2_faces
    return V, np.c_[F, np.zeros(len(F), np.int64)].astype(np.int32), np.zeros((1, 8))


def config3(seed: int = 20240612) -> Scene:
    """C3: procedural open-air semicircular amphitheatre, exactly 436 000
    triangles: 100 m diameter cavea of 40 tiers (0.4 m rise, 0.8 m tread)
    around an 18 m orchestra, a 35 m back wall with 200 arched niches (two
    bands of 100), a stage platform and a row of 60 24-facet columns.
    Materials: stone (tiers, wall, niches, columns) alpha ~ U[0.02, 0.05),
    ground (orchestra, stage) alpha ~ U[0.1, 0.3) per octave.  No roof:
    escaping rays die (tracer.cpp:46-49).  10^6 rays, 30 reflections,
    5 receivers of radius 1 m on the tiers."""
    STONE, GROUND = 0, 1
    A = 800          # angular segments of the cavea (theta in [0, pi])
    R0, NT, TREAD, RISE = 18.0, 40, 0.8, 0.4
    mb = _MeshBuilder()
    th = np.linspace(0.0, np.pi, A + 1)
    ct, st = np.cos(th), np.sin(th)

    def ring(r, z):
        return np.stack([r * ct, r * st, np.full_like(th, z)], 1)

    # orchestra: centre fan + polar grid out to R0 (ground)
    r_in0 = 1.0
    centre = np.array([[0.0, 0.0, 0.0]])
    fan = np.stack([np.zeros(A, np.int64), np.arange(1, A + 1), np.arange(2, A + 2), np.full(A, GROUND)], 1)
    mb.add(np.concatenate([centre, ring(r_in0, 0.0)]), fan)
    radii = np.linspace(r_in0, R0, 21)
    mb.grid(np.stack([ring(r, 0.0) for r in radii], 1), GROUND)
    # tiers: riser (2 rows) then tread (3 radial rows) per step
    for i in range(NT):
        r = R0 + TREAD * i
        z0, z1 = RISE * i, RISE * (i + 1)
        mb.grid(np.stack([ring(r, z) for z in np.linspace(z0, z1, 3)], 1), STONE)
        mb.grid(np.stack([ring(rr, z1) for rr in np.linspace(r, r + TREAD, 4)], 1), STONE)
    # back wall at R1 from the top tread to 35 m, 200 cells x 38 rows of
    # 0.5 m; niche regions (1 cell x 4 rows) in two bands, every other cell
    R1, ZW0, ZW1 = R0 + TREAD * NT, RISE * NT, 35.0
    AW, NR = 200, 38
    thw = np.linspace(0.0, np.pi, AW + 1)
    zw = np.linspace(ZW0, ZW1, NR + 1)
    band_rows = [(6, 10), (22, 26)]
    niche_cell = np.zeros((AW, NR), bool)
    for r0, r1 in band_rows:
        niche_cell[1::2, r0:r1] = True
    for j in range(AW):
        c0 = np.array([R1 * np.cos(thw[j]), R1 * np.sin(thw[j])])
        c1 = np.array([R1 * np.cos(thw[j + 1]), R1 * np.sin(thw[j + 1])])
        rows = [k for k in range(NR) if not niche_cell[j, k]]
        # plain cells: vertical runs of non-niche rows as one grid column
        runs, k = [], 0
        while k < NR:
            if niche_cell[j, k]:
                k += 1
                continue
            k1 = k
            while k1 < NR and not niche_cell[j, k1]:
                k1 += 1
            runs.append((k, k1))
            k = k1
        for k0, k1 in runs:
            P = np.zeros((2, k1 - k0 + 1, 3))
            P[0, :, :2], P[1, :, :2] = c0, c1
            P[:, :, 2] = zw[k0:k1 + 1]
            mb.grid(P, STONE)
        for r0, r1 in band_rows:
            if niche_cell[j, r0]:
                _niche(mb, c0, c1, zw[r0], zw[r1], STONE)
        del rows
    # stage platform in front of the orchestra (y < 0), and 60 columns
    n_cols, col_r, col_h, facets = 60, 0.35, 8.0, 24
    phi = np.linspace(0.0, 2 * np.pi, facets + 1)[:-1]
    for k in range(n_cols):
        cx, cy = -44.25 + 1.5 * k, -12.0
        bot = np.stack([cx + col_r * np.cos(phi), cy + col_r * np.sin(phi), np.zeros(facets)], 1)
        top = bot.copy()
        top[:, 2] = col_h
        V = np.concatenate([bot, top, [[cx, cy, 0.0], [cx, cy, col_h]]])
        i = np.arange(facets)
        j = (i + 1) % facets
        side = np.concatenate([np.stack([i, j, j + facets], 1), np.stack([i, j + facets, i + facets], 1)])
        capb = np.stack([np.full(facets, 2 * facets), j, i], 1)
        capt = np.stack([np.full(facets, 2 * facets + 1), i + facets, j + facets], 1)
        f = np.concatenate([side, capb, capt])
        mb.add(V, np.c_[f, np.full(len(f), STONE)])
    # stage: x in [-50, 50], y in [-20, 0]; its grid takes the remaining count
    target = 436_000
    rest = target - mb.count()
    assert rest > 0 and rest % 2 == 0, rest
    quads = rest // 2
    ny = 10
    while quads % ny:
        ny -= 1
    nx = quads // ny
    X, Y = np.meshgrid(np.linspace(-50.0, 50.0, nx + 1), np.linspace(-20.0, 0.0, ny + 1), indexing="ij")
    mb.grid(np.stack([X, Y, np.zeros_like(X)], 2), GROUND)
    v, f = mb.arrays()
    assert len(f) == target, len(f)
    alpha = np.stack([uniform(seed, 8, 0.02, 0.05), uniform(seed + 1, 8, 0.1, 0.3)])
    recv = []
    for tier, ang in ((5, 0.5), (15, 0.25), (25, 0.75), (35, 0.5), (10, 0.15)):
        r = R0 + TREAD * tier + 0.4
        recv.append(((r * np.cos(np.pi * ang), r * np.sin(np.pi * ang), RISE * (tier + 1) + 1.2), 1.0))
    return Scene("c3_amphitheatre_436k", v, f, alpha, (0.0, -4.0, 1.7), recv, 1_000_000, 30, 500.0, 48000.0, 2.0,
                 seed=seed, notes="open air; 5 receivers r = 1 m; max_range 500 m")


def _niche(mb, c0, c1, za, zb, material, depth=1.0, k_arch=8):
    """Arched recess in the wall cell between the vertical edges at c0, c1
    (xy) and heights za..zb: the cell face around the opening (stitched ring),
    the opening's reveal (sides) and the recessed back face."""
    W, H = float(np.linalg.norm(c1 - c0)), zb - za
    ex = np.array([*(c1 - c0) / W, 0.0])
    out = np.array([c0[0] + c1[0], c0[1] + c1[1], 0.0])
    out /= np.linalg.norm(out)  # outward (away from the cavea)
    base = np.array([c0[0], c0[1], za])

    def to3(u, v, d=0.0):
        return base + u * ex + np.array([0, 0, 1.0]) * v + d * out

    hw, yb, ys = 0.3 * W, 0.15 * H, 0.85 * H - 0.3 * W  # half width, sill, spring
    cu = 0.5 * W
    opening = [(cu - hw, yb), (cu + hw, yb), (cu + hw, ys)]
    for q in range(1, k_arch):
        a = np.pi * q / k_arch
        opening.append((cu + hw * np.cos(a), ys + hw * np.sin(a)))
    opening.append((cu - hw, ys))
    opening = np.array(opening)
    ctr = np.array([cu, 0.5 * (yb + ys)])
    # sample angles: opening vertices + outer corners, sorted
    corners = np.array([(0.0, 0.0), (W, 0.0), (W, H), (0.0, H)])
    angs = np.unique(np.round(np.concatenate([np.arctan2(*(opening - ctr).T[::-1]),
                                              np.arctan2(*(corners - ctr).T[::-1])]), 12))

    def hit_convex(poly, a):
        d = np.array([np.cos(a), np.sin(a)])
        best = np.inf
        for i in range(len(poly)):
            p, q = poly[i], poly[(i + 1) % len(poly)]
            e = q - p
            den = d[0] * (-e[1]) - d[1] * (-e[0])
            if abs(den) < 1e-15:
                continue
            w = p - ctr
            t = (w[0] * (-e[1]) - w[1] * (-e[0])) / den
            s = (d[0] * w[1] - d[1] * w[0]) / den
            if t > 0 and -1e-12 <= s <= 1 + 1e-12:
                best = min(best, t)
        return ctr + best * d

    inner = np.array([hit_convex(opening, a) for a in angs])
    outer = np.array([hit_convex(corners, a) for a in angs])
    M = len(angs)
    V = np.concatenate([[to3(*p) for p in inner], [to3(*p) for p in outer], [to3(*p, depth) for p in inner],
                        [to3(*ctr, depth)]])
    i = np.arange(M)
    j = (i + 1) % M
    ring = np.concatenate([np.stack([i, M + i, M + j], 1), np.stack([i, M + j, j], 1)])
    reveal = np.concatenate([np.stack([i, j, 2 * M + j], 1), np.stack([i, 2 * M + j, 2 * M + i], 1)])
    back = np.stack([np.full(M, 3 * M), 2 * M + j, 2 * M + i], 1)
    f = np.concatenate([ring, reveal, back])
    mb.add(V, np.c_[f, np.full(len(f), material)])


def config4(seed: int = 20240613) -> dict:
    """C4 (IR synthesis only): 2 000 000 image sources uniform in a 50 m
    cube, receiver at the cube centre, 8-band energies log-uniform in
    [1e-8, 1], distance |x - x_m|, t = d / 343; 3 s at 48 kHz, 8 FIR octave
    filters of 2 048 taps."""
    n = 2_000_000
    pos = uniform(seed, 3 * n, 0.0, 50.0).reshape(n, 3)
    recv = np.array([25.0, 25.0, 25.0])
    d = np.sqrt(((pos - recv) ** 2).sum(1))
    energy = 10.0 ** uniform(seed + 1, 8 * n, -8.0, 0.0).reshape(n, 8)
    return dict(name="c4_ir_2M", position=pos, receiver=recv, distance=d, energy=energy, speed_of_sound=343.0,
                sample_rate=48000.0, seconds=3.0, taps=2048)


def config5(seed: int = 20240614) -> Scene:
    """C5 (stress): shoebox 30 x 20 x 12 m holding 500 seeded, randomly
    rotated scatterers — 250 icospheres (level 4, 5 120 faces) and 250 boxes
    (12 x 12 quads per side, 1 728 faces), radius 0.3-0.8 m, kept clear of the
    source and receiver — walls gridded so the total is exactly 2 000 000
    triangles; per-octave alpha from seed (walls U[0.02, 0.3), scatterers
    U[0.05, 0.5)); 8 * 10^6 rays, 100 reflections."""
    dims = (30.0, 20.0, 12.0)
    src = np.array([7.0, 10.0, 4.0])
    rcv = np.array([22.0, 8.0, 5.0])
    ico_v, ico_f = _icosphere(4)
    box_v, box_f = _box_surface(12)
    mb = _MeshBuilder()
    u = uniform(seed, 500 * 8).reshape(500, 8)
    k = 0
    placed = 0
    while placed < 500:
        if k >= len(u):
            u = np.concatenate([u, uniform(seed + 7 + k, 500 * 8).reshape(500, 8)])
        r = 0.3 + 0.5 * u[k, 3]
        c = np.array([r + 0.05 + (dims[0] - 2 * r - 0.1) * u[k, 0], r + 0.05 + (dims[1] - 2 * r - 0.1) * u[k, 1],
                      r + 0.05 + (dims[2] - 2 * r - 0.1) * u[k, 2]])
        rot = _rotation(u[k, 4:7])
        k += 1
        if np.linalg.norm(c - src) < r * 1.8 + 1.0 or np.linalg.norm(c - rcv) < r * 1.8 + 1.0:
            continue
        is_ico = placed < 250
        bv, bf = (ico_v, ico_f) if is_ico else (box_v, box_f)
        scale = r if is_ico else r / np.sqrt(3.0)
        mb.add(c + scale * (bv @ rot.T), np.c_[bf, np.full(len(bf), 6 + placed % 2)])
        placed += 1
    n_scat = mb.count()
    grids = _shoebox_grid_for(dims, 2_000_000 - n_scat)
    wv, wf = gridded_shoebox(dims, grids, list(range(6)))
    mb.add(wv, wf)
    v, f = mb.arrays()
    assert len(f) == 2_000_000, len(f)
    alpha = np.concatenate([uniform(seed + 1, 48, 0.02, 0.3).reshape(6, 8),
                            uniform(seed + 2, 16, 0.05, 0.5).reshape(2, 8)])
    return Scene("c5_scatter_2M", v, f, alpha, tuple(src), [(tuple(rcv), 0.5)], 8_000_000, 100, 3430.0, 48000.0,
                 10.0, seed=seed, notes="500 scatterers; max_range = c * 10 s")


CONFIGS = {"c1": config1, "c2": config2, "c3": config3, "c5": config5}
