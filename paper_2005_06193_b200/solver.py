"""Online Picard iteration of the EGFEM (§4 Example L235–270, §5).

For a problem of the form

    ν K u + T:(u ⊗ w(u)) = d,    u = g on the Dirichlet boundary,

with K the P1 stiffness matrix (∫ ∇φ_i·∇φ_j), T an EGFEM trilinear tensor of the nonlinear term
(e.g. the biochemical M_c̃ of PAPER.md L533 with c̃ = 1/(k+u)) and w = interp(u), each Picard
iteration (lag the coefficients, solve the linear system, update them) is

    w^n = interp(u^n)                 egfem_interp                     (hot path step 1)
    A^n = ν K + T·w^n                 egfem_jacobian(PICARD)            (hot path step 3)
    A^n u^{n+1} = d  (Dirichlet rows and columns eliminated), Jacobi-preconditioned CG whose
    matrix-vector products are egfem_csr_spmv; stop when ‖u^{n+1} − u^n‖_∞ ≤ tol (L304: O(1e-12)).

Every matrix and vector lives on the device; the tensor work runs in libegfem.so's kernels.
The CG vector updates (dot, axpy) and the Dirichlet masks are torch elementwise ops — the
solver is the paper's online loop around the hot path, not part of it (the
linear solve is a separate cost).  The source d is assembled as M d_h (the nodal interpolant of
the source times the mass matrix M = (MASS3 tensor)·₂1, egfem_bilinear_build), the GFEM
treatment of a known function, which keeps the P1 error O(h²).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import (F64, FORM_MASS3, FORM_PLAP, INTERP_IDENTITY, JAC_PICARD, Tensor, egfem_bilinear_build,
               egfem_csr_spmv, egfem_interp, egfem_jacobian, egfem_tensor_build)


@dataclass
class SolveResult:
    u: np.ndarray
    iterations: int
    converged: bool
    increments: list
    cg_iterations: list


class PicardEGFEM:
    """ν K u + T:(u ⊗ w(u)) = d with Dirichlet data, on P1 V (mesh, V: egfem_inputs-style objects).

    T must share V's CSR pattern (any trilinear tensor with V = P1 on the same mesh does:
    the pattern is the union of element cliques)."""

    def __init__(self, mesh, V, T: Tensor, kind: int, p: float, nu: float = 1.0, device: int = 0):
        import torch
        self.torch = torch
        self.dev = torch.device("cuda", device)
        self.T, self.kind, self.p, self.nu = T, kind, p, nu
        self.mesh, self.V = mesh, V
        import egfem_inputs as I  # structured mesh / space generators (no EGFEM arithmetic)
        W0 = I.space_p0(mesh)
        # K = T_plap·1 with P0 coefficient 1 (∫_K 1 ∇φ_i·∇φ_j summed over cells: the stiffness)
        self._tk = egfem_tensor_build(mesh, V, W0, FORM_PLAP, dtype=F64, device=device)
        # M = (MASS3 with W = V)·₂1 (mass matrix, for the source term)
        self._tm = egfem_tensor_build(mesh, V, V, FORM_MASS3, dtype=F64, device=device)
        rp, col = T.export(values=False)["csr_row_ptr"], T.export(values=False)["csr_col"]
        for other in (self._tk, self._tm):
            ex = other.export(values=False)
            if not (np.array_equal(ex["csr_row_ptr"], rp) and np.array_equal(ex["csr_col"], col)):
                raise ValueError("T does not share the P1 CSR pattern of the mesh")
        n = T.n_u
        self.n = n
        f64 = torch.float64
        ones_w = torch.ones(self._tk.n_f, dtype=f64, device=self.dev)
        self.K = torch.empty(T.nnz_csr, dtype=f64, device=self.dev)
        egfem_jacobian(self._tk, JAC_PICARD, INTERP_IDENTITY, 0.0, None, ones_w, None, self.K)
        self.M = torch.empty(T.nnz_csr, dtype=f64, device=self.dev)
        egfem_bilinear_build(self._tm, self.M)
        # Dirichlet masks on the CSR slots: boundary = vertices on ∂[0,1]^d
        x = mesh.coords
        bnd = np.any((x <= 1e-12) | (x >= 1 - 1e-12), axis=1)
        rows = np.repeat(np.arange(n), np.diff(rp))
        bi, bj = bnd[rows], bnd[col]
        self.bnd = torch.tensor(bnd, device=self.dev)
        self.keep = torch.tensor((~bi & ~bj).astype(np.float64), device=self.dev)
        self.lift = torch.tensor((~bi & bj).astype(np.float64), device=self.dev)
        self.dbnd = torch.tensor((bi & (rows == col)).astype(np.float64), device=self.dev)

    def source(self, d_nodal: np.ndarray):
        """d = M d_h on the device (GFEM interpolation of a known source)."""
        torch = self.torch
        dn = torch.tensor(d_nodal, dtype=torch.float64, device=self.dev)
        out = torch.empty_like(dn)
        egfem_csr_spmv(self._tm, self.M, dn, out)
        return out

    def _cg(self, A, b, x0, tol, maxit):
        """Jacobi-preconditioned CG on the SPD eliminated matrix A (values on the CSR pattern)."""
        torch = self.torch
        rp = self.T
        diag = self._diag(A)
        x = x0.clone()
        Ax = torch.empty_like(b)
        egfem_csr_spmv(rp, A, x, Ax)
        r = b - Ax
        z = r / diag
        pvec = z.clone()
        rz = torch.dot(r, z)
        bnorm = torch.linalg.vector_norm(b).item() or 1.0
        Ap = torch.empty_like(b)
        it = 0
        for it in range(1, maxit + 1):
            egfem_csr_spmv(rp, A, pvec, Ap)
            alpha = rz / torch.dot(pvec, Ap)
            x += alpha * pvec
            r -= alpha * Ap
            if torch.linalg.vector_norm(r).item() <= tol * bnorm:
                break
            z = r / diag
            rz_new = torch.dot(r, z)
            pvec = z + (rz_new / rz) * pvec
            rz = rz_new
        return x, it

    def _diag(self, A):
        ex = getattr(self, "_diag_slots", None)
        if ex is None:
            e = self.T.export(values=False)
            rows = np.repeat(np.arange(self.n), np.diff(e["csr_row_ptr"]))
            self._diag_slots = self.torch.tensor(np.nonzero(rows == e["csr_col"])[0], device=self.dev)
        return A[self._diag_slots]

    def solve(self, d_vec, g_nodal: np.ndarray, u0: np.ndarray | None = None, tol: float = 1e-12,
              maxit: int = 100, cg_tol: float = 1e-14, cg_maxit: int = 5000) -> SolveResult:
        torch = self.torch
        T = self.T
        g = torch.tensor(g_nodal, dtype=torch.float64, device=self.dev)  # only its boundary values are used
        u = torch.zeros_like(g) if u0 is None else torch.tensor(u0, dtype=torch.float64, device=self.dev)
        u = torch.where(self.bnd, g, u)
        w = torch.empty(T.n_f, dtype=torch.float64, device=self.dev)
        TA = torch.empty(T.nnz_csr, dtype=torch.float64, device=self.dev)
        lift_rhs = torch.empty_like(u)
        incs, cgits = [], []
        converged = False
        for n in range(1, maxit + 1):
            egfem_interp(T, self.kind, self.p, u, w)                                   # w^n = f(u^n)
            egfem_jacobian(T, JAC_PICARD, self.kind, self.p, None, w, None, TA)        # T·w^n
            A = self.nu * self.K + TA
            egfem_csr_spmv(T, A * self.lift, g, lift_rhs)                             # Σ_{j∈Γ} A_ij g_j
            b = torch.where(self.bnd, g, d_vec - lift_rhs)
            Ae = A * self.keep + self.dbnd
            u_new, it = self._cg(Ae, b, u, cg_tol, cg_maxit)
            inc = torch.max(torch.abs(u_new - u)).item()
            u = u_new
            incs.append(inc)
            cgits.append(it)
            if inc <= tol:
                converged = True
                break
        return SolveResult(u.cpu().numpy(), n, converged, incs, cgits)


def biochemical_problem(n: int, device: int = 0, W: str = "P1"):
    """PAPER.md §5.4 (L516–535): −Δu + σ u/(k+u) = d on [0,1]², σ = 1 = k, exact solution
    u = x1 x2 (x1 + x2) (L521), so d = −(2x1 + 2x2) + u/(1+u).  EGFEM: K u + M_c̃:(u ⊗ c̃) = d with
    c̃ = 1/(k+u) interpolated onto W (P1: GFEM nodes; P0: centroids).  Returns (solver, d, g, u_exact)."""
    import egfem_inputs as I  # the structured mesh / space generators (no EGFEM arithmetic)
    mesh = I.mesh_square(n)
    V = I.space_p1(mesh)
    Wsp = V if W == "P1" else I.space_p0(mesh)
    T = egfem_tensor_build(mesh, V, Wsp, FORM_MASS3, dtype=F64, device=device)
    x = mesh.coords
    ue = x[:, 0] * x[:, 1] * (x[:, 0] + x[:, 1])
    d_nodal = -(2 * x[:, 0] + 2 * x[:, 1]) + ue / (1.0 + ue)
    from . import INTERP_RECIPROCAL
    s = PicardEGFEM(mesh, V, T, INTERP_RECIPROCAL, 1.0, nu=1.0, device=device)
    return s, s.source(d_nodal), ue
