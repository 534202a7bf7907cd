"""Online Picard and Newton iterations of the EGFEM (§4, §5).

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

from . import (F64, FORM_MASS3, FORM_PLAP, INTERP_IDENTITY, JAC_NEWTON, JAC_PICARD, Tensor, egfem_apply,
               egfem_bilinear_build, egfem_csr_spmv, egfem_interp, egfem_jacobian, egfem_tensor_build)


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


# ----------------------------------------------------------------------------- Newton (F4)
@dataclass
class NewtonResult:
    u: np.ndarray
    iterations: int
    converged: bool
    status: str                 # "converged" | "diverged" | "maxit" | "krylov"
    residuals: list             # ‖F(u^n)‖₂ over the free rows, before each step
    increments: list            # ‖δ^n‖_∞
    damping: list               # step length taken (1 = full Newton step)
    krylov_iterations: list


class NewtonEGFEM(PicardEGFEM):
    """Newton's method for ν K u + T:(u ⊗ w(u)) = d with Dirichlet data.

    Per iteration, on the device:
        w = interp(u) with D_u w                    egfem_interp (+ chain)          (step 1)
        F = ν K u + T:(u ⊗ w) − d                   egfem_apply + CSR SpMV           (step 2)
        J = ν K + T·w + (T·₂u)·D_u w                egfem_jacobian(NEWTON)           (step 3)
        J δ = −F on the free rows (Dirichlet rows / columns eliminated, δ = 0 on Γ),
        right-Jacobi-preconditioned restarted GMRES whose products are egfem_csr_spmv
        u ← u + λ δ with λ = 1, halved while ‖F(u + λδ)‖ does not decrease (backtracking;
        PAPER.md L296 leaves damping open — reading F4 in DESIGN.md)
    The reduced Jacobian is the Schur complement of the paper's block Jacobian D_z F̃ (L290) once
    the identity blocks of the intermediate variables are eliminated (reading C10); it needs
    no integration, only the precomputed tensor and the pointwise D_u w (L292).  Stops when
    ‖δ‖_∞ ≤ tol (L304: O(1e-12)); reports "diverged" when ‖F‖ becomes non-finite or exceeds
    `div_factor`·‖F(u⁰)‖, or the line search fails."""

    def __init__(self, mesh, V, T: Tensor, kind: int, p: float, nu: float = 1.0, device: int = 0,
                 cell_wise: bool | None = None):
        super().__init__(mesh, V, T, kind, p, nu=nu, device=device)
        torch = self.torch
        # cell-wise W (P0 / QUAD) carries D_u w as chain rows (include/egfem.h egfem_interp)
        cell_wise = (T.n_f != T.n_u) if cell_wise is None else cell_wise
        self.chain = (torch.empty(T.n_f * (mesh.dim + 1), dtype=torch.float64, device=self.dev)
                      if cell_wise else None)
        self.free = (~self.bnd).to(torch.float64)

    def residual(self, u, d_vec, w):
        """F(u) = ν K u + T:(u ⊗ w(u)) − d (w from egfem_interp of u); zero on the Dirichlet rows."""
        torch = self.torch
        egfem_interp(self.T, self.kind, self.p, u, w, self.chain)
        r = torch.empty_like(u)
        egfem_apply(self.T, u, w, r)
        if self.nu != 0.0:
            ku = torch.empty_like(u)
            egfem_csr_spmv(self.T, self.K, u, ku)
            r = r + self.nu * ku
        return (r - d_vec) * self.free

    def _gmres(self, A, b, tol, restart, maxit):
        """Right-Jacobi-preconditioned restarted GMRES(m) for A x = b (A on the CSR pattern,
        eliminated).  Arnoldi with classical Gram-Schmidt twice, Givens rotations."""
        torch = self.torch
        dinv = 1.0 / self._diag(A)
        n = b.numel()
        x = torch.zeros_like(b)
        bnorm = torch.linalg.vector_norm(b).item()
        if bnorm == 0.0:
            return x, 0, True
        total = 0
        Av = torch.empty_like(b)
        while total < maxit:
            egfem_csr_spmv(self.T, A, x, Av)
            r = b - Av
            beta = torch.linalg.vector_norm(r).item()
            if beta <= tol * bnorm:
                return x, total, True
            m = min(restart, maxit - total)
            Vb = torch.empty((m + 1, n), dtype=b.dtype, device=b.device)
            Hm = np.zeros((m + 1, m))
            Vb[0] = r / beta
            cs, sn = np.zeros(m), np.zeros(m)
            g = np.zeros(m + 1)
            g[0] = beta
            k_done = 0
            for k in range(m):
                egfem_csr_spmv(self.T, A, Vb[k] * dinv, Av)
                wv = Av.clone()
                for _ in range(2):  # CGS2
                    h = Vb[:k + 1] @ wv
                    wv -= h @ Vb[:k + 1]
                    Hm[:k + 1, k] += h.cpu().numpy()
                hn = torch.linalg.vector_norm(wv).item()
                Hm[k + 1, k] = hn
                if hn > 0:
                    Vb[k + 1] = wv / hn
                for i in range(k):  # apply the previous rotations to column k
                    t0 = cs[i] * Hm[i, k] + sn[i] * Hm[i + 1, k]
                    Hm[i + 1, k] = -sn[i] * Hm[i, k] + cs[i] * Hm[i + 1, k]
                    Hm[i, k] = t0
                den = np.hypot(Hm[k, k], Hm[k + 1, k])
                cs[k], sn[k] = (1.0, 0.0) if den == 0 else (Hm[k, k] / den, Hm[k + 1, k] / den)
                Hm[k, k] = cs[k] * Hm[k, k] + sn[k] * Hm[k + 1, k]
                Hm[k + 1, k] = 0.0
                g[k + 1] = -sn[k] * g[k]
                g[k] = cs[k] * g[k]
                total += 1
                k_done = k + 1
                if abs(g[k + 1]) <= tol * bnorm or hn == 0:
                    break
            y = np.linalg.solve(np.triu(Hm[:k_done, :k_done]), g[:k_done]) if k_done else np.zeros(0)
            yt = torch.tensor(y, dtype=b.dtype, device=b.device)
            x += (yt @ Vb[:k_done]) * dinv
            if abs(g[k_done]) <= tol * bnorm:
                egfem_csr_spmv(self.T, A, x, Av)
                return x, total, bool(torch.linalg.vector_norm(b - Av).item() <= 10 * tol * bnorm)
        return x, total, False

    def solve(self, d_vec, g_nodal: np.ndarray, u0: np.ndarray | None = None, tol: float = 1e-12,
              maxit: int = 50, krylov_tol: float = 1e-13, restart: int = 60, krylov_maxit: int = 3000,
              div_factor: float = 1e6, max_halvings: int = 30, damping: bool = True,
              initial: str = "laplace") -> NewtonResult:
        """u0: initial guess (its boundary values are replaced by g); None and initial="laplace":
        the solution of K u = d with the same Dirichlet data (the p = 2 / a ≡ 1 problem — the
        degenerate p-Laplacian has a singular Jacobian at ∇u = 0, so u0 = 0 cannot start it);
        initial="zero": u0 = 0 in the interior."""
        torch = self.torch
        T = self.T
        g = torch.tensor(g_nodal, dtype=torch.float64, device=self.dev)
        if u0 is not None:
            u = torch.tensor(u0, dtype=torch.float64, device=self.dev)
        elif initial == "laplace":
            lift = torch.empty_like(g)
            egfem_csr_spmv(T, self.K * self.lift, g, lift)
            b = torch.where(self.bnd, g, d_vec - lift)
            u, _ = self._cg(self.K * self.keep + self.dbnd, b, torch.where(self.bnd, g, torch.zeros_like(g)),
                            1e-14, 20000)
        else:
            u = torch.zeros_like(g)
        u = torch.where(self.bnd, g, u)
        w = torch.empty(T.n_f, dtype=torch.float64, device=self.dev)
        J = torch.empty(T.nnz_csr, dtype=torch.float64, device=self.dev)
        F = self.residual(u, d_vec, w)
        f0 = torch.linalg.vector_norm(F).item()
        res, incs, lams, kits = [f0], [], [], []
        status = "maxit"
        if not np.isfinite(f0):
            return NewtonResult(u.cpu().numpy(), 0, False, "diverged", res, incs, lams, kits)
        for n in range(1, maxit + 1):
            # J at u (the last residual evaluated w and the chain at u)
            egfem_jacobian(T, JAC_NEWTON, self.kind, self.p, u, w, self.chain, J)
            A = J + self.nu * self.K if self.nu != 0.0 else J
            Ae = A * self.keep + self.dbnd
            delta, it, ok = self._gmres(Ae, -F, krylov_tol, restart, krylov_maxit)
            kits.append(it)
            if not ok:
                status = "krylov"
                break
            fn = res[-1]
            lam = 1.0
            for _ in range(max_halvings + 1):
                u_try = u + lam * delta
                F_try = self.residual(u_try, d_vec, w)
                f_try = torch.linalg.vector_norm(F_try).item()
                if not damping or (np.isfinite(f_try) and (f_try < fn or f_try <= 1e-12 * f0)):
                    break
                lam *= 0.5
            else:
                status = "diverged"
                break
            inc = lam * torch.max(torch.abs(delta)).item()
            u, F = u_try, F_try
            res.append(f_try)
            incs.append(inc)
            lams.append(lam)
            if not np.isfinite(f_try) or f_try > div_factor * max(f0, 1e-300):
                status = "diverged"
                break
            if inc <= tol:
                status = "converged"
                break
        return NewtonResult(u.cpu().numpy(), len(incs), status == "converged", status, res, incs, lams, kits)


def _square_source(name: str, x: np.ndarray, p: float = 4.0) -> np.ndarray:
    """Manufactured sources on the unit square for u = x1 x2 (x1 + x2):
    g = ∇u = (2 x1 x2 + x2², x1² + 2 x1 x2), H = ∇²u = [[2 x2, 2(x1+x2)], [2(x1+x2), 2 x1]].
      minsurf:  d = −∇·(g / √(1+|g|²)) = −Δu/√s + gᵀHg / s^{3/2},  s = 1 + |g|²   (L600–605)
      plap:     d = −∇·(|g|^{p−2} g) = −|g|^{p−2} Δu − (p−2)|g|^{p−4} gᵀHg          (L568–574)"""
    x1, x2 = x[:, 0], x[:, 1]
    g1, g2 = 2 * x1 * x2 + x2 ** 2, x1 ** 2 + 2 * x1 * x2
    h11, h12, h22 = 2 * x2, 2 * (x1 + x2), 2 * x1
    lap = h11 + h22
    gHg = g1 * g1 * h11 + 2 * g1 * g2 * h12 + g2 * g2 * h22
    gg = g1 * g1 + g2 * g2
    if name == "minsurf":
        s = 1.0 + gg
        return -lap / np.sqrt(s) + gHg / s ** 1.5
    gn = np.sqrt(gg)
    with np.errstate(divide="ignore", invalid="ignore"):
        t = np.where(gg > 0, (p - 2) * gn ** (p - 4) * gHg, 0.0)
    return -(gn ** (p - 2)) * lap - t


def quasilinear_problem(name: str, n: int, p: float | None = 4.0, device: int = 0):
    """PAPER.md §5.5 / §5.6 on the unit square with the manufactured solution u = x1 x2 (x1+x2)
    (the paper's §5.6 boundary data, L601; §5.5's disk solution needs a curved mesh, so the
    p-Laplace source is manufactured the same way): T = K_a (PLAP, W = P0), a = |∇u|^{p−2}
    (GRADPOW_P0) or (1+|∇u|²)^{−1/2} (MINSURF_P0), ν = 0, d = M d_h.  Returns (solver, d, u_exact)."""
    import egfem_inputs as I
    from . import INTERP_GRADPOW_P0, INTERP_MINSURF_P0
    mesh = I.mesh_square(n)
    V = I.space_p1(mesh)
    T = egfem_tensor_build(mesh, V, I.space_p0(mesh), FORM_PLAP, dtype=F64, device=device)
    x = mesh.coords
    ue = x[:, 0] * x[:, 1] * (x[:, 0] + x[:, 1])
    kind = INTERP_MINSURF_P0 if name == "minsurf" else INTERP_GRADPOW_P0
    p = 4.0 if p is None else float(p)  # ignored by MINSURF_P0
    s = NewtonEGFEM(mesh, V, T, kind, p, nu=0.0, device=device)
    return s, s.source(_square_source(name, x, p)), ue


def biochemical_newton(n: int, device: int = 0, W: str = "P1"):
    """The §5.4 biochemical problem (see biochemical_problem) solved by Newton."""
    import egfem_inputs as I
    from . import INTERP_RECIPROCAL
    mesh = I.mesh_square(n)
    V = I.space_p1(mesh)
    Wsp = V if W == "P1" else I.space_p0(mesh)
    T = egfem_tensor_build(mesh, V, Wsp, FORM_MASS3, dtype=F64, device=device)
    x = mesh.coords
    ue = x[:, 0] * x[:, 1] * (x[:, 0] + x[:, 1])
    d_nodal = -(2 * x[:, 0] + 2 * x[:, 1]) + ue / (1.0 + ue)
    s = NewtonEGFEM(mesh, V, T, INTERP_RECIPROCAL, 1.0, nu=1.0, device=device)
    return s, s.source(d_nodal), ue
