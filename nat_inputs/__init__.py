"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no kernels, quadrature, sampling,
solves or radiation).  It only produces input arrays:

* closed, outward-oriented, welded triangle meshes shaped like the paper's scenes
  (spheres for the analytic pins, a thick bowl for the modal object, a bowl on a
  slab for the NAT scene sweep; SURVEY.md §8(d) "Configs as concrete synthetic
  inputs", "construct the scene and obtain its surface triangle mesh");
* per-triangle Neumann data ("the Neumann condition remains unchanged
  for each triangle");
* wavenumbers of the configs (c = 343 m/s).

Every generator is a pure function of its arguments (and a seed where random).
Meshes are returned as ``Mesh(v=(V,3) float64, t=(N,3) int32)``; ``soa()`` gives the
``[3][V]`` / ``[3][N]`` structure-of-arrays layout the C ABI takes.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

SEED = 20250606           # seed of every config
SPEED_OF_SOUND = 343.0    # m/s (the paper never states c)


@dataclasses.dataclass
class Mesh:
    v: np.ndarray  # (V, 3) float64 vertex coordinates, metres
    t: np.ndarray  # (N, 3) int32 vertex indices, CCW seen from outside

    @property
    def n_vert(self) -> int:
        return int(self.v.shape[0])

    @property
    def n_tri(self) -> int:
        return int(self.t.shape[0])

    def soa(self):
        """(vxyz [3][V] float64 contiguous, tri [3][N] int32 contiguous)."""
        return (np.ascontiguousarray(self.v.T, dtype=np.float64),
                np.ascontiguousarray(self.t.T, dtype=np.int32))


# ----------------------------------------------------------------------------------
# helpers (input construction only)
# ----------------------------------------------------------------------------------

def _tri_raw_normals(v, t):
    a = v[t[:, 1]] - v[t[:, 0]]
    b = v[t[:, 2]] - v[t[:, 0]]
    return np.cross(a, b)


def _orient_star(v, t, centre):
    """Flip triangles of a star-shaped (about ``centre``) surface to face outward."""
    e = _tri_raw_normals(v, t)
    c = v[t].mean(axis=1) - centre
    flip = np.einsum("ij,ij->i", e, c) < 0
    t = t.copy()
    t[flip] = t[flip][:, [0, 2, 1]]
    return t


def signed_volume(mesh: Mesh) -> float:
    v, t = mesh.v, mesh.t
    return float(np.einsum("ij,ij->i", v[t[:, 0]], np.cross(v[t[:, 1]], v[t[:, 2]])).sum() / 6.0)


def check_closed_oriented(mesh: Mesh) -> None:
    """Every directed edge appears once and its reverse once (closed, consistent)."""
    t = mesh.t.astype(np.int64)
    e = np.concatenate([t[:, [0, 1]], t[:, [1, 2]], t[:, [2, 0]]])
    key = e[:, 0] * mesh.n_vert + e[:, 1]
    rkey = e[:, 1] * mesh.n_vert + e[:, 0]
    if np.unique(key).size != key.size:
        raise ValueError("duplicate directed edge: inconsistent orientation")
    if not np.array_equal(np.sort(key), np.sort(rkey)):
        raise ValueError("open mesh: a directed edge has no reverse")
    if signed_volume(mesh) <= 0:
        raise ValueError("mesh is inward-oriented")


def mesh_concat(*meshes: Mesh) -> Mesh:
    vs, ts, off = [], [], 0
    for m in meshes:
        vs.append(m.v)
        ts.append(m.t + off)
        off += m.n_vert
    return Mesh(np.concatenate(vs), np.concatenate(ts).astype(np.int32))


def mesh_transform(m: Mesh, scale: float = 1.0, shift=(0.0, 0.0, 0.0)) -> Mesh:
    return Mesh(m.v * scale + np.asarray(shift, dtype=np.float64), m.t.copy())


# ----------------------------------------------------------------------------------
# meshes
# ----------------------------------------------------------------------------------

def icosphere(level: int, radius: float = 1.0) -> Mesh:
    """Regular icosahedron, edge-midpoint subdivided ``level`` times, every new vertex
    projected to the sphere; welded.  L3: 1280 tri / 642 vert; L5: 20480 / 10242."""
    phi = (1.0 + math.sqrt(5.0)) / 2.0
    base = []
    for s1 in (-1.0, 1.0):
        for s2 in (-1.0, 1.0):
            base += [(0.0, s1, s2 * phi), (s1, s2 * phi, 0.0), (s2 * phi, 0.0, s1)]
    v = np.array(base, dtype=np.float64)
    # faces = triangles of the edge graph (edge length 2)
    d = np.linalg.norm(v[:, None, :] - v[None, :, :], axis=2)
    adj = np.abs(d - 2.0) < 1e-9
    faces = [(i, j, k) for i in range(12) for j in range(i + 1, 12) for k in range(j + 1, 12)
             if adj[i, j] and adj[j, k] and adj[i, k]]
    assert len(faces) == 20
    v = v / np.linalg.norm(v, axis=1, keepdims=True)
    t = _orient_star(v, np.array(faces, dtype=np.int64), np.zeros(3))
    verts = [tuple(x) for x in v]
    for _ in range(level):
        cache = {}
        nt = []

        def mid(a, b):
            key = (a, b) if a < b else (b, a)
            if key not in cache:
                p = (np.asarray(verts[a]) + np.asarray(verts[b])) * 0.5
                p = p / np.linalg.norm(p)
                cache[key] = len(verts)
                verts.append(tuple(p))
            return cache[key]

        for a, b, c in t:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            nt += [(a, ab, ca), (ab, b, bc), (ca, bc, c), (ab, bc, ca)]
        t = np.array(nt, dtype=np.int64)
    v = np.array(verts, dtype=np.float64) * radius
    return Mesh(v, t.astype(np.int32))


def _lattice_surface(coords_x, coords_y, coords_z, centre):
    """Closed surface of the box lattice coords_x × coords_y × coords_z (boundary
    points only, welded by integer index), each boundary quad split along its
    (i,j)-(i+1,j+1) diagonal, oriented outward about ``centre`` (convex)."""
    nx, ny, nz = len(coords_x) - 1, len(coords_y) - 1, len(coords_z) - 1
    index = {}
    verts = []

    def vid(a, b, c):
        key = (a, b, c)
        if key not in index:
            index[key] = len(verts)
            verts.append((coords_x[a], coords_y[b], coords_z[c]))
        return index[key]

    tris = []
    dims = (nx, ny, nz)
    for axis in range(3):
        u_ax, w_ax = [a for a in range(3) if a != axis]
        for side in (0, dims[axis]):
            for i in range(dims[u_ax]):
                for j in range(dims[w_ax]):
                    def p(ii, jj):
                        idx = [0, 0, 0]
                        idx[axis] = side
                        idx[u_ax] = ii
                        idx[w_ax] = jj
                        return vid(*idx)
                    q00, q10, q11, q01 = p(i, j), p(i + 1, j), p(i + 1, j + 1), p(i, j + 1)
                    tris.append((q00, q10, q11))
                    tris.append((q00, q11, q01))
    v = np.array(verts, dtype=np.float64)
    t = _orient_star(v, np.array(tris, dtype=np.int64), np.asarray(centre, dtype=np.float64))
    return v, t.astype(np.int32)


def cubed_sphere(n: int, radius: float = 1.0) -> Mesh:
    """Equiangular cubed sphere: per face (xi, eta) = -pi/4 + (i, j)(pi/2)/n, point =
    normalise(1, tan xi, tan eta) on each face; welded (V = 6n^2 + 2), quads split along
    the (i,j)-(i+1,j+1) diagonal.  n = 129 gives 199,692 triangles (config C5)."""
    tg = np.tan(-math.pi / 4 + np.arange(n + 1) * (math.pi / 2) / n)
    tg[0], tg[-1] = -1.0, 1.0
    v, t = _lattice_surface(tg, tg, tg, (0.0, 0.0, 0.0))
    v = v / np.linalg.norm(v, axis=1, keepdims=True) * radius
    t = _orient_star(v, t, np.zeros(3)).astype(np.int32)
    return Mesh(v, t)


def slab(lx: float, ly: float, lz: float, nx: int, ny: int, nz: int,
         centre=(0.0, 0.0, 0.0)) -> Mesh:
    """Closed box [-lx/2, lx/2] x [-ly/2, ly/2] x [-lz/2, lz/2] + centre, faces gridded."""
    c = np.asarray(centre, dtype=np.float64)
    xs = c[0] + np.linspace(-lx / 2, lx / 2, nx + 1)
    ys = c[1] + np.linspace(-ly / 2, ly / 2, ny + 1)
    zs = c[2] + np.linspace(-lz / 2, lz / 2, nz + 1)
    v, t = _lattice_surface(xs, ys, zs, c)
    return Mesh(v, t)


def bowl(n_az: int = 256, n_psi: int = 48, n_rim: int = 2,
         r_out: float = 1.0, r_in: float = 0.9) -> Mesh:
    """Closed thick hemispherical shell ("bowl"), opening up, rim at z = 0.

    Surface of revolution of the closed profile: outer arc radius r_out from the bottom
    pole (0, -r_out) to the rim (r_out, 0); flat rim annulus z = 0 from rho = r_out to
    r_in; inner arc radius r_in back down to the inner pole (0, -r_in).  Triangles:
    n_az * (2(2 n_psi - 1) + 2 n_rim)  (49,664 for 256/48/2; 12,544 for 128/24/2)."""
    prof = [(0.0, -r_out)]
    for k in range(1, n_psi + 1):
        psi = (math.pi / 2) * k / n_psi
        prof.append((r_out * math.sin(psi), -r_out * math.cos(psi)))
    for k in range(1, n_rim + 1):
        prof.append((r_out + (r_in - r_out) * k / n_rim, 0.0))
    for k in range(n_psi - 1, -1, -1):
        psi = (math.pi / 2) * k / n_psi
        prof.append((r_in * math.sin(psi), -r_in * math.cos(psi)))
    prof[-1] = (0.0, -r_in)
    K = len(prof) - 1
    verts = [(0.0, 0.0, prof[0][1])]
    ring = {}
    for k in range(1, K):
        ring[k] = len(verts)
        rho, z = prof[k]
        for a in range(n_az):
            ph = 2 * math.pi * a / n_az
            verts.append((rho * math.cos(ph), rho * math.sin(ph), z))
    top = len(verts)
    verts.append((0.0, 0.0, prof[K][1]))
    tris = []
    for a in range(n_az):
        b = (a + 1) % n_az
        tris.append((0, ring[1] + b, ring[1] + a))
        for k in range(1, K - 1):
            p00, p01 = ring[k] + a, ring[k] + b
            p10, p11 = ring[k + 1] + a, ring[k + 1] + b
            tris.append((p00, p01, p11))
            tris.append((p00, p11, p10))
        tris.append((ring[K - 1] + a, ring[K - 1] + b, top))
    m = Mesh(np.array(verts, dtype=np.float64), np.array(tris, dtype=np.int32))
    if signed_volume(m) < 0:
        m = Mesh(m.v, m.t[:, [0, 2, 1]].copy())
    return m


# ----------------------------------------------------------------------------------
# Neumann data (per triangle, complex; modes are real-valued)
# ----------------------------------------------------------------------------------

def tri_centroid_direction(mesh: Mesh, origin=(0.0, 0.0, 0.0)) -> np.ndarray:
    c = mesh.v[mesh.t].mean(axis=1) - np.asarray(origin, dtype=np.float64)
    return c / np.linalg.norm(c, axis=1, keepdims=True)


def neumann_constant(mesh: Mesh, g: complex = 1.0) -> np.ndarray:
    """Pulsating body: dp/dn = g on every triangle (C1)."""
    return np.full(mesh.n_tri, g, dtype=np.complex128)


def neumann_rigid_z(mesh: Mesh, g0: float = 1.0) -> np.ndarray:
    """Rigid oscillation along z: dp/dn = g0 * (z_hat . n_t) with n_t the unit normal of
    the flat triangle (C2, C5 oscillating-sphere dipole)."""
    e = _tri_raw_normals(mesh.v, mesh.t)
    n = e / np.linalg.norm(e, axis=1, keepdims=True)
    return (g0 * n[:, 2]).astype(np.complex128)


def real_sph_harm_list(n: int):
    """(l, q) in order (0,0), (1,-1), (1,0), (1,1), (2,-2), ... (first n)."""
    out = []
    l = 0
    while len(out) < n:
        for q in range(-l, l + 1):
            out.append((l, q))
            if len(out) == n:
                break
        l += 1
    return out


def neumann_harmonics(mesh: Mesh, n_modes: int, origin=(0.0, 0.0, 0.0),
                      tri_mask=None) -> np.ndarray:
    """Synthetic smooth mode shapes: g_{m,t} = Y_{l,q}(c_hat_t), the real spherical
    harmonics in order (0,0),(1,-1),(1,0),(1,1),..., each normalised to max|g| = 1
    (SURVEY.md §8(c-9) #20).  Triangles outside ``tri_mask`` get 0 (passive objects,
    PAPER.md l.191).  Returns [n_modes][N] complex128."""
    from scipy.special import sph_harm_y
    d = tri_centroid_direction(mesh, origin)
    theta = np.arccos(np.clip(d[:, 2], -1.0, 1.0))  # polar
    phi = np.arctan2(d[:, 1], d[:, 0])              # azimuth
    out = np.zeros((n_modes, mesh.n_tri), dtype=np.complex128)
    for m, (l, q) in enumerate(real_sph_harm_list(n_modes)):
        y = sph_harm_y(l, abs(q), theta, phi)
        if q < 0:
            val = math.sqrt(2.0) * y.imag
        elif q == 0:
            val = y.real
        else:
            val = math.sqrt(2.0) * y.real
        if tri_mask is not None:
            val = np.where(tri_mask, val, 0.0)
        mx = np.max(np.abs(val))
        out[m] = val / mx if mx > 0 else val
    return out


# ----------------------------------------------------------------------------------
# configs
# ----------------------------------------------------------------------------------

def c3_wavenumbers(n_modes: int = 32, a: float = 1.0) -> np.ndarray:
    """k_m a = 0.5 + 7.5 m / 31 (C3)."""
    return (0.5 + 7.5 * np.arange(n_modes) / 31.0) / a


C4_HEIGHTS = np.linspace(0.005, 0.30, 8)        # bowl bottom above slab top, m
C4_DIAMETERS = np.linspace(0.10, 0.20, 8)       # outer diameter, m
C4_EOVERRHO = np.geomspace(7.8e6, 2.6e7, 8)     # E/rho


def c4_geometry(i: int, n_az: int = 128, n_psi: int = 24, n_rim: int = 2):
    """C4 geometry i = 8*i_h + i_D: bowl of outer diameter D whose bottom sits h above a
    passive closed slab 0.4 x 0.4 x 0.02 m (top face at z = 0).  Returns (mesh, g
    [8][N] complex (first 8 harmonics on the bowl, 0 on the slab), bowl diameter D)."""
    i_h, i_d = divmod(i, 8)
    h, D = float(C4_HEIGHTS[i_h]), float(C4_DIAMETERS[i_d])
    b = mesh_transform(bowl(n_az, n_psi, n_rim), scale=D / 2, shift=(0.0, 0.0, h + D / 2))
    s = slab(0.4, 0.4, 0.02, 40, 40, 2, centre=(0.0, 0.0, -0.01))
    m = mesh_concat(b, s)
    mask = np.zeros(m.n_tri, dtype=bool)
    mask[: b.n_tri] = True
    g = neumann_harmonics(m, 8, origin=(0.0, 0.0, h + D / 2), tri_mask=mask)
    return m, g, D


def c4_wavenumbers(D: float) -> np.ndarray:
    """64 wavenumbers of one geometry: index 8*i_material + m,
    f = 400 (m+1) sqrt((E/rho)/7.8e6) (0.1/D) Hz, k = 2 pi f / 343."""
    out = []
    for er in C4_EOVERRHO:
        for m in range(8):
            f = 400.0 * (m + 1) * math.sqrt(er / 7.8e6) * (0.1 / D)
            out.append(2 * math.pi * f / SPEED_OF_SOUND)
    return np.array(out)


def random_points_in_shell(n: int, r_lo: float, r_hi: float, seed: int) -> np.ndarray:
    """(n, 3) points uniform in volume in the shell r_lo <= r <= r_hi (test inputs only)."""
    rng = np.random.default_rng(seed)
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    r = (r_lo ** 3 + (r_hi ** 3 - r_lo ** 3) * rng.random(n)) ** (1.0 / 3.0)
    return d * r[:, None]


def random_complex(shape, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.normal(size=shape) + 1j * rng.normal(size=shape)


# ----------------------------------------------------------------------------------
# NEXT-4 neural field: seeded parameters and training samples (inputs only)
# ----------------------------------------------------------------------------------

def nf_init_params(shapes, seed: int, grid_scale: float = 1e-4) -> np.ndarray:
    """Flat float32 parameter vector for the given block shapes (grid tables [rows][4]
    first, then per layer W [out][in], b [out]): grid features U(-grid_scale, grid_scale)
    (instant-NGP's small init), W Xavier-uniform, b = 0."""
    rng = np.random.default_rng(seed)
    parts = []
    for shp in shapes:
        shp = tuple(shp)
        if len(shp) == 2 and shp[1] == 4:          # feature table
            parts.append(rng.uniform(-grid_scale, grid_scale, size=shp))
        elif len(shp) == 2:                        # W [out][in]
            lim = math.sqrt(6.0 / (shp[0] + shp[1]))
            parts.append(rng.uniform(-lim, lim, size=shp))
        else:                                      # bias
            parts.append(np.zeros(shp))
    return np.concatenate([p.reshape(-1) for p in parts]).astype(np.float32)


def nf_samples(n: int, n_v: int, seed: int) -> np.ndarray:
    """n training inputs [n][3 + n_v] uniform in [0, 1) (normalised theta, phi, r and the
    condition variables)."""
    return np.random.default_rng(seed).random((n, 3 + n_v)).astype(np.float32)
