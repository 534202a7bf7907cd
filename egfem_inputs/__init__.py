"""Seeded synthetic inputs shared by the CPU oracle and the CUDA path.

This module holds NO arithmetic of the EGFEM method (no basis functions, no
quadrature, no integrals, no contractions).  It only produces the data both
sides consume: structured simplicial meshes, DOF numberings (cell -> global DOF
tables), the seeded nodal vectors ``u`` of BASELINE.json's five configs, and
the config registry.  Conventions follow SURVEY.md §8(c) C.1 (mesh, numbering)
and §8(d) D.1 / C.13 (random inputs); DESIGN.md §3 restates them.

Paper anchors: meshes are n-dimensional simplicial partitions Ω_h
(§2.1); the trial space is P1 "linear finite elements in all of
the examples" (§5); W_h is P0 (L584, §5.5 p-Laplace) or W = V
(L99, §3.1 GFEM recovered).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

# Space family codes (must match include/egfem.h egfem_family and oracle/).
P0, P1, P2, QUAD = 0, 1, 2, 3
# Form codes (include/egfem.h egfem_form).
FORM_CONV_K, FORM_CONV_J, FORM_PLAP, FORM_MASS3, FORM_CONV_I = 0, 1, 2, 3, 4
# Interp kinds (include/egfem.h egfem_interp_kind).
INTERP_IDENTITY, INTERP_SQUARE, INTERP_GRADPOW_P0, INTERP_P1_TO_P2_SQUARE = 0, 1, 2, 3
INTERP_MINSURF_P0, INTERP_RECIPROCAL = 4, 5
# Jacobian modes.
JAC_PICARD, JAC_NEWTON = 0, 1


@dataclasses.dataclass
class Mesh:
    """Simplicial mesh: ``coords`` (n_vertices, dim) f64, ``cells`` (n_cells, dim+1) int32."""
    dim: int
    coords: np.ndarray
    cells: np.ndarray

    @property
    def n_vertices(self) -> int:
        return int(self.coords.shape[0])

    @property
    def n_cells(self) -> int:
        return int(self.cells.shape[0])


@dataclasses.dataclass
class Space:
    """A DOF numbering: family code, DOF count, (n_cells, n_local) int32 table, DOF coordinates."""
    family: int
    n_dofs: int
    cell_dofs: np.ndarray
    dof_coords: Optional[np.ndarray] = None

    @property
    def n_local(self) -> int:
        return int(self.cell_dofs.shape[1])


# --------------------------------------------------------------------------- meshes
def mesh_interval(n: int) -> Mesh:
    """1D: x_i = i/n, cell e = [e, e+1] with local order (left, right)."""
    x = (np.arange(n + 1, dtype=np.float64) / n).reshape(-1, 1)
    e = np.arange(n, dtype=np.int32)
    cells = np.stack([e, e + 1], axis=1).astype(np.int32)
    return Mesh(1, x, cells)


def mesh_square(n: int) -> Mesh:
    """2D unit square, n×n cells, each split along the bottom-left→top-right diagonal.

    Node (ix,iy) -> id iy*(n+1)+ix, coords (ix/n, iy/n).  Cell c = cy*n+cx gives
    triangles 2c = (v00, v10, v11) and 2c+1 = (v00, v11, v01), both CCW.
    """
    m = n + 1
    iy, ix = np.meshgrid(np.arange(m), np.arange(m), indexing="ij")
    coords = np.stack([ix.ravel() / n, iy.ravel() / n], axis=1).astype(np.float64)
    cy, cx = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    cx = cx.ravel().astype(np.int64)
    cy = cy.ravel().astype(np.int64)
    v00 = cy * m + cx
    v10 = v00 + 1
    v01 = v00 + m
    v11 = v01 + 1
    cells = np.empty((2 * n * n, 3), dtype=np.int32)
    cells[0::2] = np.stack([v00, v10, v11], axis=1)
    cells[1::2] = np.stack([v00, v11, v01], axis=1)
    return Mesh(2, coords, cells)


# Kuhn permutations of (x, y, z) in lexicographic order: xyz, xzy, yxz, yzx, zxy, zyx.
KUHN_PERMS = ((0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0))


def mesh_cube(n: int) -> Mesh:
    """3D unit cube, n³ cubes, 6 Kuhn tetrahedra per cube.

    Node id (iz*(n+1)+iy)*(n+1)+ix.  Cube c = (cz*n+cy)*n+cx.  Tet 6c+t follows
    permutation σ_t: v0 = base, v1 = v0+e_σ0, v2 = v1+e_σ1, v3 = base+(1,1,1).
    """
    m = n + 1
    iz, iy, ix = np.meshgrid(np.arange(m), np.arange(m), np.arange(m), indexing="ij")
    coords = np.stack([ix.ravel() / n, iy.ravel() / n, iz.ravel() / n], axis=1).astype(np.float64)
    cz, cy, cx = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    base = ((cz.ravel().astype(np.int64) * m + cy.ravel()) * m + cx.ravel())
    stride = (1, m, m * m)
    cells = np.empty((6 * n ** 3, 4), dtype=np.int32)
    for t, perm in enumerate(KUHN_PERMS):
        v1 = base + stride[perm[0]]
        v2 = v1 + stride[perm[1]]
        v3 = base + (1 + m + m * m)
        cells[t::6] = np.stack([base, v1, v2, v3], axis=1)
    return Mesh(3, coords, cells)


# --------------------------------------------------------------------------- spaces
def space_p1(mesh: Mesh) -> Space:
    return Space(P1, mesh.n_vertices, mesh.cells.copy(), mesh.coords)


def space_p0(mesh: Mesh) -> Space:
    cd = np.arange(mesh.n_cells, dtype=np.int32).reshape(-1, 1)
    return Space(P0, mesh.n_cells, cd, None)


def space_quad(mesh: Mesh, nq: int) -> Space:
    """The quadrature-embedded space I_k: N_q DOFs per cell numbered
    K·N_q + ℓ (N_f = N_q·N_el, L139).  Only the count is an input; each side (GPU builder,
    oracle) uses its own rule with N_q points (2D: 1, 3, 6; 3D: 1, 4)."""
    cd = np.arange(mesh.n_cells * nq, dtype=np.int32).reshape(-1, nq)
    return Space(QUAD, mesh.n_cells * nq, cd, None)


def space_p2_square(n: int) -> Space:
    """P2 on mesh_square(n) with lattice numbering on the (2n+1)² grid.

    DOF (a,b) -> id b*(2n+1)+a at (a/2n, b/2n).  Local order (v0, v1, v2, m01, m12, m20)
    matching the triangle vertex order of mesh_square.
    """
    L = 2 * n + 1
    cy, cx = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    ax = 2 * cx.ravel().astype(np.int64)
    by = 2 * cy.ravel().astype(np.int64)

    def lid(a, b):
        return b * L + a

    cd = np.empty((2 * n * n, 6), dtype=np.int32)
    # lower triangle: v00 (ax,by), v10 (ax+2,by), v11 (ax+2,by+2)
    cd[0::2] = np.stack([lid(ax, by), lid(ax + 2, by), lid(ax + 2, by + 2),
                         lid(ax + 1, by), lid(ax + 2, by + 1), lid(ax + 1, by + 1)], axis=1)
    # upper triangle: v00 (ax,by), v11 (ax+2,by+2), v01 (ax,by+2)
    cd[1::2] = np.stack([lid(ax, by), lid(ax + 2, by + 2), lid(ax, by + 2),
                         lid(ax + 1, by + 1), lid(ax + 1, by + 2), lid(ax, by + 1)], axis=1)
    bb, aa = np.meshgrid(np.arange(L), np.arange(L), indexing="ij")
    dof_coords = np.stack([aa.ravel() / (2 * n), bb.ravel() / (2 * n)], axis=1).astype(np.float64)
    return Space(P2, L * L, cd, dof_coords)


# --------------------------------------------------------------------------- configs
@dataclasses.dataclass
class Problem:
    """One BASELINE.json config, fully materialised (mesh, V, W, form, u)."""
    name: str
    mesh: Mesh
    V: Space
    W: Space
    form: int
    interp: int
    p: float
    dtypes: tuple
    u: np.ndarray            # (N_u,) or (B, N_u) for batched
    batch: int = 0
    description: str = ""

    @property
    def n_u(self) -> int:
        return self.V.n_dofs

    @property
    def n_f(self) -> int:
        return self.W.n_dofs


def _u_cfg1(x):
    rng = np.random.default_rng(0)
    return np.sin(np.pi * x[:, 0]) + 0.1 * rng.standard_normal(x.shape[0])


def _u_cfg2(x):
    rng = np.random.default_rng(1)
    return np.sin(np.pi * x[:, 0]) * np.sin(np.pi * x[:, 1]) + 0.05 * rng.standard_normal(x.shape[0])


def _u_cfg3(x):
    rng = np.random.default_rng(2)
    return (x[:, 0] * (1 - x[:, 0]) * x[:, 1] * (1 - x[:, 1])
            + 0.01 * rng.uniform(-1.0, 1.0, x.shape[0]))


def _u_cfg4(x):
    rng = np.random.default_rng(3)
    return (np.sin(np.pi * x[:, 0]) * np.sin(np.pi * x[:, 1]) * np.sin(np.pi * x[:, 2])
            + 0.01 * rng.standard_normal(x.shape[0]))


def _u_cfg5(x, batch):
    rng = np.random.default_rng(4)
    Z = rng.standard_normal((batch, x.shape[0]))
    U = np.empty((batch, x.shape[0]), dtype=np.float64)
    for p in range(batch):
        a, b = 1 + p % 4, 1 + (p // 4) % 4
        U[p] = np.sin(a * np.pi * x[:, 0]) * np.sin(b * np.pi * x[:, 1]) + 0.05 * Z[p]
    return U


def _u_paper_bc(x, seed):
    """x1 x2 (x1 + x2) (the exact solution of PAPER.md §5.4 L521 / §5.6) + 0.01·N(0,1)."""
    rng = np.random.default_rng(seed)
    return x[:, 0] * x[:, 1] * (x[:, 0] + x[:, 1]) + 0.01 * rng.standard_normal(x.shape[0])


# Full BASELINE.json sizes; "small" variants use the same recipe at a size the
# oracle finishes in seconds but that still spans many kernel tiles.
FULL_N = {"cfg1": 256, "cfg2": 512, "cfg3": 1024, "cfg4": 128, "cfg5": 256,
          "minsurf2d": 1024, "minsurf3d": 64, "biochem_p1": 512, "biochem_p0": 512,
          "quadratic_i4": 512, "biochem_i2": 512, "plap_i1": 1024, "plap3d_i2": 32, "gfem2d": 512}
SMALL_N = {"cfg1": 256, "cfg2": 40, "cfg3": 48, "cfg4": 10, "cfg5": 24,
           "minsurf2d": 40, "minsurf3d": 8, "biochem_p1": 32, "biochem_p0": 32,
           "quadratic_i4": 24, "biochem_i2": 32, "plap_i1": 40, "plap3d_i2": 5, "gfem2d": 40}
CONFIG_NAMES = ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5")
# SURVEY §8(f) F1 pointwise kinds (not BASELINE configs): minimal surface a = (1+|∇u|²)^{-1/2}
# with P0 W (§5.6) and the biochemical c̃ = σ/(k+u), σ = 1 = k, on the
# trilinear mass tensor M_c̃ with W = P1 (GFEM) or P0 (§5.4).
# F2 quadrature-embedded W = I_k (Case 3): the §5.1 quadratic term M:(u⊗w),
# w = u² at the points of the 6-point rule (I_4, Table 1's "EGFEM (I4)", L492); the biochemical
# term on I_2 (3 points, L541–550); the p-Laplace K_a on I_1 (centroid, L143–149, L616) and on the
# 4-point tetrahedral I_2 (3D).
# F3 bilinear GFEM form: the paper's Burgers N^f_ik = ∫ η_k (∂x+∂y)φ_i with f = u² at the nodes
# (PAPER.md L402–409), on cfg2's mesh and u; its tensor is the paper's N (CONV_I, L400).
EXTRA_NAMES = ("minsurf2d", "minsurf3d", "biochem_p1", "biochem_p0", "quadratic_i4", "biochem_i2", "plap_i1",
               "plap3d_i2", "gfem2d")


def make_problem(name: str, n: Optional[int] = None, batch: Optional[int] = None) -> Problem:
    """Materialise BASELINE.json config ``name`` (cfg1..cfg5), optionally at mesh size ``n``."""
    if n is None:
        n = FULL_N[name]
    if name == "cfg1":
        mesh = mesh_interval(n)
        V = space_p1(mesh)
        return Problem(name, mesh, V, V, FORM_CONV_K, INTERP_IDENTITY, 0.0, ("f64",),
                       _u_cfg1(mesh.coords), description=f"1D Burgers P1, n={n}")
    if name == "cfg2":
        mesh = mesh_square(n)
        V = space_p1(mesh)
        return Problem(name, mesh, V, V, FORM_CONV_J, INTERP_IDENTITY, 0.0, ("f64",),
                       _u_cfg2(mesh.coords), description=f"2D Burgers P1, {n}x{n}")
    if name == "cfg3":
        mesh = mesh_square(n)
        return Problem(name, mesh, space_p1(mesh), space_p0(mesh), FORM_PLAP, INTERP_GRADPOW_P0,
                       4.0, ("f64",), _u_cfg3(mesh.coords), description=f"2D p-Laplace p=4, {n}x{n}")
    if name == "cfg4":
        mesh = mesh_cube(n)
        return Problem(name, mesh, space_p1(mesh), space_p0(mesh), FORM_PLAP, INTERP_GRADPOW_P0,
                       3.0, ("f64", "f32"), _u_cfg4(mesh.coords), description=f"3D p-Laplace p=3, {n}^3x6")
    if name == "cfg5":
        if batch is None:
            batch = 256
        mesh = mesh_square(n)
        V = space_p2_square(n)
        return Problem(name, mesh, V, V, FORM_CONV_J, INTERP_IDENTITY, 0.0, ("f64",),
                       _u_cfg5(V.dof_coords, batch), batch=batch,
                       description=f"batched 2D Burgers P2, {n}x{n}, B={batch}")
    if name == "minsurf2d":
        mesh = mesh_square(n)
        return Problem(name, mesh, space_p1(mesh), space_p0(mesh), FORM_PLAP, INTERP_MINSURF_P0, 0.0,
                       ("f64",), _u_paper_bc(mesh.coords, 6), description=f"2D minimal surface P1/P0, {n}x{n}")
    if name == "minsurf3d":
        mesh = mesh_cube(n)
        return Problem(name, mesh, space_p1(mesh), space_p0(mesh), FORM_PLAP, INTERP_MINSURF_P0, 0.0,
                       ("f64",), _u_paper_bc(mesh.coords, 7), description=f"3D minimal surface P1/P0, {n}^3x6")
    if name in ("biochem_p1", "biochem_p0"):
        mesh = mesh_square(n)
        V = space_p1(mesh)
        W = V if name == "biochem_p1" else space_p0(mesh)
        return Problem(name, mesh, V, W, FORM_MASS3, INTERP_RECIPROCAL, 1.0, ("f64",),
                       _u_paper_bc(mesh.coords, 8), description=f"2D biochemical sigma/(k+u), W={name[-2:]}, {n}x{n}")
    if name == "quadratic_i4":
        mesh = mesh_square(n)
        return Problem(name, mesh, space_p1(mesh), space_quad(mesh, 6), FORM_MASS3, INTERP_SQUARE, 0.0, ("f64",),
                       _u_paper_bc(mesh.coords, 9), description=f"2D quadratic u^2 on I4 (6-pt), {n}x{n}")
    if name == "biochem_i2":
        mesh = mesh_square(n)
        return Problem(name, mesh, space_p1(mesh), space_quad(mesh, 3), FORM_MASS3, INTERP_RECIPROCAL, 1.0,
                       ("f64",), _u_paper_bc(mesh.coords, 10), description=f"2D biochemical on I2 (3-pt), {n}x{n}")
    if name == "plap_i1":
        mesh = mesh_square(n)
        return Problem(name, mesh, space_p1(mesh), space_quad(mesh, 1), FORM_PLAP, INTERP_GRADPOW_P0, 4.0,
                       ("f64",), _u_cfg3(mesh.coords), description=f"2D p-Laplace p=4 on I1 (centroid), {n}x{n}")
    if name == "plap3d_i2":
        mesh = mesh_cube(n)
        return Problem(name, mesh, space_p1(mesh), space_quad(mesh, 4), FORM_PLAP, INTERP_GRADPOW_P0, 3.0,
                       ("f64",), _u_cfg4(mesh.coords), description=f"3D p-Laplace p=3 on I2 (4-pt), {n}^3x6")
    if name == "gfem2d":
        mesh = mesh_square(n)
        V = space_p1(mesh)
        return Problem(name, mesh, V, V, FORM_CONV_I, INTERP_SQUARE, 0.0, ("f64",), _u_cfg2(mesh.coords),
                       description=f"2D Burgers GFEM N^f f, f = u^2, {n}x{n}")
    raise KeyError(name)


def random_vector(n: int, seed: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """Generic seeded test vector (uniform)."""
    return np.random.default_rng(seed).uniform(lo, hi, n)
