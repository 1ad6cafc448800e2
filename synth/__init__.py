"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no element matrices, no
assembly, no load integration, no solver).  It only describes grids and draws
the per-element material fields, initial fields and random test vectors that
both sides take as *inputs*.  Neither ``oracle/`` nor the CUDA package is
imported here, and this module imports neither of them.

Grid convention (§4.1 "Mesh Geometry"):
node (i, j, k) has linear index ``i + (nx+1)*(j + (ny+1)*k)`` (x fastest) and
element (ex, ey, ez) has index ``ex + nx*(ey + ny*ez)`` ("six in the first
cube, then ... in the x direction ... then the next slice in z"; here
one trilinear hexahedron per cube, reading R1).

Material constants are the paper's verbatim values (§5.1):
mild steel rhoC = 3.724e6, k = 4.9e8; iron(III) oxide rhoC = 1.65e6, k = 4e6.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Tuple

import numpy as np

# P:271 (§5.1): "rho C = 3.724e6 ... x3 <= 5, 1.65e6 ... x3 > 5; k = 4.9e8 ..., 4e6 ..."
STEEL = (3.724e6, 4.9e8)   # (c = rhoC, k)
OXIDE = (1.65e6, 4.0e6)

# 10 W laser in the unit system of the paper's rho C and k: those are SI values
# read in (g, mm, s) units (J/(m^3 K) == g/(mm s^2 K)), where 1 W = 1e9 g mm^2 s^-3.
# (reading R12.)
BEAM_POWER = 10.0 * 1e9

# face ids used by both sides: bit f of a Dirichlet mask / the ``face`` argument
FACE_XM, FACE_XP, FACE_YM, FACE_YP, FACE_ZM, FACE_ZP = range(6)


@dataclass(frozen=True)
class Grid:
    """Structured voxel grid: ``ne`` elements per axis, spacing ``h``, min corner ``origin``."""
    ne: Tuple[int, int, int]
    h: Tuple[float, float, float]
    origin: Tuple[float, float, float] = (0.0, 0.0, 0.0)

    @property
    def nn(self) -> Tuple[int, int, int]:
        return (self.ne[0] + 1, self.ne[1] + 1, self.ne[2] + 1)

    @property
    def n_nodes(self) -> int:
        a, b, c = self.nn
        return a * b * c

    @property
    def n_elems(self) -> int:
        return self.ne[0] * self.ne[1] * self.ne[2]

    def node_coords(self):
        """(x, y, z) of every node, each of shape (nz+1, ny+1, nx+1) (C order == linear index)."""
        nx, ny, nz = self.nn
        z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
        return (self.origin[0] + x * self.h[0], self.origin[1] + y * self.h[1],
                self.origin[2] + z * self.h[2])

    def elem_centroids(self):
        """(x, y, z) of every element centroid, each of shape (nz, ny, nx)."""
        nx, ny, nz = self.ne
        z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
        return (self.origin[0] + (x + 0.5) * self.h[0], self.origin[1] + (y + 0.5) * self.h[1],
                self.origin[2] + (z + 0.5) * self.h[2])


@dataclass
class Problem:
    """One transient workload: grid, per-element fields, BCs, time stepping and solver options."""
    name: str
    grid: Grid
    k: np.ndarray                      # per-element conductivity, float64, len n_elems
    c: np.ndarray                      # per-element capacity rhoC, float64, len n_elems
    u0: np.ndarray                     # initial nodal field, float64, len n_nodes
    theta: float
    dt: float
    nsteps: int
    rtol: float = 1e-12
    max_iter: int = 10000
    replace_every: int = 50            # Alg. 1 line 9
    flux_face: int = FACE_ZM           # face carrying the flux load ("f = 1 on x3 = 0")
    flux_const: float = 0.0            # constant flux f on that face
    beam: Optional[Tuple[float, float, float, float]] = None   # (P, sigma, cx, cy) Gaussian beam
    dirichlet_bits: int = 0            # bit f set -> face f is Dirichlet (extension, DESIGN R3)
    dirichlet_values: Tuple[float, ...] = (0.0,) * 6
    extra: dict = field(default_factory=dict)


# ----------------------------------------------------------------------------------------------
# material fields (element-centroid rule, reading R2)


def two_layer(grid: Grid, z_split: float, below=STEEL, above=OXIDE):
    """Laminate of P:270-272: material ``below`` where centroid z <= z_split, else ``above``."""
    _, _, zc = grid.elem_centroids()
    lower = (zc <= z_split).ravel()
    c = np.where(lower, below[0], above[0]).astype(np.float64)
    k = np.where(lower, below[1], above[1]).astype(np.float64)
    return k, c


def inclusion_ids(grid: Grid, seed: int = 0, frac: float = 0.20, rmin_h: float = 2.0,
                  rmax_h: float = 8.0) -> np.ndarray:
    """Random spherical inclusions (SURVEY §8(d) C3/C4 recipe).

    Spheres with radius U[rmin_h*h, rmax_h*h] and centre U(domain) are drawn from
    ``default_rng(seed)`` and added one at a time until the fraction of elements whose
    centroid lies inside any sphere reaches ``frac``.  Returns uint8 ids (1 = inclusion),
    shape (nz, ny, nx).
    """
    rng = np.random.default_rng(seed)
    nx, ny, nz = grid.ne
    hx, hy, hz = grid.h
    hmin = min(grid.h)
    L = (nx * hx, ny * hy, nz * hz)
    ids = np.zeros((nz, ny, nx), dtype=np.uint8)
    target = int(np.ceil(frac * grid.n_elems))
    count = 0
    while count < target:
        r = rng.uniform(rmin_h * hmin, rmax_h * hmin)
        cx, cy, cz = rng.uniform(0.0, L[0]), rng.uniform(0.0, L[1]), rng.uniform(0.0, L[2])
        # element index range whose centroids may fall inside the sphere
        lo = [max(0, int(np.floor((cc - r) / hh - 0.5))) for cc, hh in zip((cx, cy, cz), grid.h)]
        hi = [min(n, int(np.ceil((cc + r) / hh - 0.5)) + 1) for cc, hh, n in zip((cx, cy, cz), grid.h, grid.ne)]
        if any(h_ <= l_ for l_, h_ in zip(lo, hi)):
            continue
        xs = (np.arange(lo[0], hi[0]) + 0.5) * hx - cx
        ys = (np.arange(lo[1], hi[1]) + 0.5) * hy - cy
        zs = (np.arange(lo[2], hi[2]) + 0.5) * hz - cz
        inside = (zs[:, None, None] ** 2 + ys[None, :, None] ** 2 + xs[None, None, :] ** 2) <= r * r
        box = ids[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]]
        new = inside & (box == 0)
        count += int(new.sum())
        box[new] = 1
    return ids


def ids_to_fields(ids: np.ndarray, materials=(STEEL, OXIDE)):
    """Map material ids to flat float64 (k, c) element arrays."""
    cs = np.array([m[0] for m in materials], dtype=np.float64)
    ks = np.array([m[1] for m in materials], dtype=np.float64)
    flat = ids.ravel()
    return ks[flat], cs[flat]


def corrosion_ids(grid: Grid, depth: float, H: float, z_rear: float) -> np.ndarray:
    """Parabolic corrosion region anchored at the rear face (Fig. 6; DESIGN R13).

    An element is oxide (id 1) iff its centroid satisfies |y| <= H and
    (z_rear - z) <= depth * (1 - (y/H)^2); constant in x.
    """
    _, yc, zc = grid.elem_centroids()
    d_rear = z_rear - zc
    inside = (np.abs(yc) <= H) & (d_rear <= depth * (1.0 - (yc / H) ** 2))
    return inside.astype(np.uint8)


def lognormal_perturbation(n: int, seed: int, sigma: float = 0.1) -> np.ndarray:
    """Multiplicative per-element factor exp(sigma * N(0,1)) (C5 perturbed conductivity)."""
    return np.exp(sigma * np.random.default_rng(seed).standard_normal(n))


def random_vector(n: int, seed: int) -> np.ndarray:
    return np.random.default_rng(seed).standard_normal(n)


def random_fields(grid: Grid, seed: int, contrast: float = 122.5):
    """Independent log-uniform k and c per element (spans the paper's 122x k contrast)."""
    rng = np.random.default_rng(seed)
    k = np.exp(rng.uniform(0.0, np.log(contrast), grid.n_elems))
    c = np.exp(rng.uniform(0.0, np.log(2.3), grid.n_elems))
    return k, c


# ----------------------------------------------------------------------------------------------
# the five BASELINE.json configurations


def c1() -> Problem:
    """8x8x8 unit cube, two materials, backward Euler, 10 steps, tol 1e-12."""
    g = Grid((8, 8, 8), (0.125, 0.125, 0.125))
    k, c = two_layer(g, 0.5)
    return Problem("c1", g, k, c, np.zeros(g.n_nodes), theta=1.0, dt=0.01, nsteps=10,
                   rtol=1e-12, flux_face=FACE_ZM, flux_const=1.0)


def c2() -> Problem:
    """64x4x4 bar, k = c = 1, Dirichlet 0 at x = 0, 1, u0 = sin(pi x), CN, 200 steps."""
    h = 1.0 / 64
    g = Grid((64, 4, 4), (h, h, h))
    x, _, _ = g.node_coords()
    u0 = np.sin(np.pi * x).ravel()
    ones = np.ones(g.n_elems)
    return Problem("c2", g, ones.copy(), ones.copy(), u0, theta=0.5, dt=5e-4, nsteps=200,
                   rtol=1e-12, flux_const=0.0,
                   dirichlet_bits=(1 << FACE_XM) | (1 << FACE_XP))


def c3(n_nodes_axis: int = 100, nsteps: int = 300, seed: int = 0) -> Problem:
    """~1M DoF (100^3 nodes) cube, h = 0.2 mm, 20% spherical oxide inclusions, CN dt = 0.01."""
    n = n_nodes_axis - 1
    g = Grid((n, n, n), (0.2, 0.2, 0.2))
    ids = inclusion_ids(g, seed=seed)
    k, c = ids_to_fields(ids)
    return Problem("c3", g, k, c, np.zeros(g.n_nodes), theta=0.5, dt=0.01, nsteps=nsteps,
                   rtol=1e-12, flux_face=FACE_ZM, flux_const=1.0,
                   extra={"ids": ids.ravel().copy(), "materials": (STEEL, OXIDE)})


def c4_grid(n_nodes_axis: int = 512) -> Grid:
    n = n_nodes_axis - 1
    return Grid((n, n, n), (0.2, 0.2, 0.2))


def c5_grid(n_nodes_axis: int = 100) -> Grid:
    """Plate [-15,15]^2 x [0,12.7] mm with 99^3 elements (P:357 plate, 12.7 mm thick)."""
    n = n_nodes_axis - 1
    return Grid((n, n, n), (30.0 / n, 30.0 / n, 12.7 / n), (-15.0, -15.0, 0.0))


def c5_depths(nsims: int, seed: int = 1, thickness: float = 12.7) -> np.ndarray:
    return np.random.default_rng(seed).uniform(0.0, thickness, nsims)


def c5(j: int, depth: Optional[float] = None, n_nodes_axis: int = 100, nsteps: int = 300,
       perturb: bool = True) -> Problem:
    """Forward simulation j of the corrosion inverse problem."""
    g = c5_grid(n_nodes_axis)
    if depth is None:
        depth = float(c5_depths(j + 1)[j])
    ids = corrosion_ids(g, depth, H=15.0, z_rear=12.7)
    k, c = ids_to_fields(ids)
    if perturb:
        k = k * lognormal_perturbation(g.n_elems, seed=2 + j)
    return Problem(f"c5[{j}]", g, k, c, np.zeros(g.n_nodes), theta=0.5, dt=10.0 / nsteps,
                   nsteps=nsteps, rtol=1e-12, flux_face=FACE_ZM, flux_const=0.0,
                   beam=(BEAM_POWER, 2.0, 0.0, 0.0), extra={"depth": depth})


def laminate(s: int) -> Problem:
    """§5.1 laminate [-15,15]^2 x [0,10] with C = (30s, 30s, 10s) cubes."""
    h = 1.0 / s
    g = Grid((30 * s, 30 * s, 10 * s), (h, h, h), (-15.0, -15.0, 0.0))
    k, c = two_layer(g, 5.0)
    return Problem(f"laminate{s}", g, k, c, np.zeros(g.n_nodes), theta=0.5, dt=0.01,
                   nsteps=50, rtol=1e-6, flux_face=FACE_ZM, flux_const=1.0)
