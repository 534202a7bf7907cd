"""F4: Newton's method of PAPER.md §4 (L272–292) around the GPU hot path — the
reduced Jacobian J = ν K + T·w + (T·₂u)·D_u w from egfem_jacobian(NEWTON), solved by GMRES on
egfem_csr_spmv — on the biochemical (§5.4), minimal-surface (§5.6) and p-Laplace (§5.5)
problems with the manufactured solution x1 x2 (x1 + x2).

Checked against (a) the same Newton iteration run on the CPU oracle's tensors with a direct
sparse solve (scipy), iterate for iterate (undamped); (b) quadratic convergence of the
increments; (c) the manufactured solution: the P1 error falls like h²; (d) divergence is
reported, not raised."""
import numpy as np
import pytest

import egfem_inputs as I

pytestmark = pytest.mark.gpu

CASES = [("biochem", "P1", None), ("biochem", "P0", None), ("minsurf", None, None), ("plap", None, 3.0),
         ("plap", None, 4.0)]


@pytest.fixture(scope="module")
def eg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    import paper_2005_06193_b200 as eg
    return eg


def _gpu_problem(name, W, p, n):
    from paper_2005_06193_b200 import solver
    if name == "biochem":
        return solver.biochemical_newton(n, W=W)
    return solver.quasilinear_problem(name, n, p=p)


def _start(ue, x):
    """A shared initial guess for the iterate-for-iterate comparison: 0.8 u_exact + a smooth bump
    (non-degenerate gradients everywhere, so the p-Laplace Jacobian is regular)."""
    return 0.8 * ue + 0.05 * np.sin(np.pi * x[:, 0]) * np.sin(np.pi * x[:, 1])


def _reference_newton(name, W, p, n, iters):
    """CPU reference, written out plainly: the oracle's tensors (T, stiffness K = PLAP·1), the exact
    P1 mass matrix, F = νKu + T:(u⊗w(u)) − M d_h, J = νK + oracle Newton Jacobian, Dirichlet rows and
    columns eliminated, scipy spsolve, undamped steps."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spl

    import oracle
    from oracle import brute
    from paper_2005_06193_b200.solver import _square_source
    mesh = I.mesh_square(n)
    V = I.space_p1(mesh)
    x = mesh.coords
    ue = x[:, 0] * x[:, 1] * (x[:, 0] + x[:, 1])
    M = brute.bilinear_matrix(mesh, V, "v", "v")
    if name == "biochem":
        Wsp = V if W == "P1" else I.space_p0(mesh)
        T = oracle.OracleTensor(mesh, V, Wsp, I.FORM_MASS3)
        kind, pk, nu = I.INTERP_RECIPROCAL, 1.0, 1.0
        d = M @ (-(2 * x[:, 0] + 2 * x[:, 1]) + ue / (1.0 + ue))
    else:
        T = oracle.OracleTensor(mesh, V, I.space_p0(mesh), I.FORM_PLAP)
        kind = I.INTERP_MINSURF_P0 if name == "minsurf" else I.INTERP_GRADPOW_P0
        pk, nu = (p if p else 0.0), 0.0
        d = M @ _square_source(name, x, p or 4.0)
    Tk = oracle.OracleTensor(mesh, V, I.space_p0(mesh), I.FORM_PLAP)
    ex = T.export()
    rows = np.repeat(np.arange(T.n_u), np.diff(ex["csr_row_ptr"]))
    col = ex["csr_col"]
    Kv = Tk.jacobian(I.JAC_PICARD, I.INTERP_IDENTITY, 0.0, np.zeros(T.n_u), np.ones(Tk.n_f))
    K = sp.csr_matrix((Kv, (rows, col)), shape=(T.n_u, T.n_u))
    bnd = np.any((x <= 1e-12) | (x >= 1 - 1e-12), axis=1)
    u = np.where(bnd, ue, _start(ue, x))
    out = []
    for _ in range(iters):
        w = T.interp(kind, pk, u)
        F = nu * (K @ u) + T.apply(u, w) - d
        F[bnd] = 0.0
        J = sp.csr_matrix((T.jacobian(I.JAC_NEWTON, kind, pk, u, w), (rows, col)), shape=(T.n_u, T.n_u)) + nu * K
        J = J.tolil()
        J[bnd, :] = 0
        J[:, bnd] = 0
        J[bnd, bnd] = 1.0
        u = u + spl.spsolve(J.tocsr(), -F)
        out.append(u.copy())
    return out


@pytest.mark.parametrize("name,W,p", CASES)
def test_newton_matches_cpu_reference(eg, name, W, p):
    n = 8
    s, d, ue = _gpu_problem(name, W, p, n)
    x = s.mesh.coords
    res = s.solve(d, ue, u0=_start(ue, x), maxit=4, tol=0.0, damping=False, krylov_tol=1e-15)
    ref = _reference_newton(name, W, p, n, 4)
    assert res.iterations == 4, res.status
    assert np.abs(res.u - ref[-1]).max() <= 1e-9 * max(1.0, np.abs(ref[-1]).max())


@pytest.mark.parametrize("name,W,p", CASES)
def test_newton_converges_quadratically(eg, name, W, p):
    """PAPER.md L304 stopping rule ‖Δu‖ ≤ 1e-12; Newton's increments fall quadratically:
    inc_{k+1} ≤ C inc_k² once in the basin (checked on the last steps above round-off)."""
    s, d, ue = _gpu_problem(name, W, p, 16)
    res = s.solve(d, ue, tol=1e-12)
    assert res.converged, (res.status, res.increments)
    assert res.iterations <= 25, res.increments  # p = 4 starts far from the Laplace guess (15 steps)
    inc = [x for x in res.increments if x > 1e-13]
    quad = [b / a ** 2 for a, b in zip(inc, inc[1:]) if a < 1e-2]
    assert quad and max(quad) < 1e3, res.increments


@pytest.mark.parametrize("name,p", [("minsurf", None), ("plap", 4.0)])
def test_newton_manufactured_second_order(eg, name, p):
    """The EGFEM-P0 solution of the quasilinear problems converges to the manufactured solution
    like h² in the nodal max norm (§5.5–5.6: EGFEM-P0 = SGA for these, L616)."""
    errs = []
    for n in (8, 16, 32):
        s, d, ue = _gpu_problem(name, None, p, n)
        res = s.solve(d, ue, tol=1e-12)
        assert res.converged, res.status
        errs.append(np.abs(res.u - ue).max())
    assert errs[0] / errs[1] > 3.0 and errs[1] / errs[2] > 3.0, errs


def test_newton_divergence_is_reported(eg):
    """A non-finite residual (a NaN source) and an undamped start across the pole of σ/(k+u)
    end with status "diverged" instead of an exception or a silent result."""
    import torch
    s, d, ue = _gpu_problem("biochem", "P1", None, 8)
    bad = d.clone()
    bad[5] = float("nan")
    res = s.solve(bad, ue, maxit=5)
    assert not res.converged and res.status == "diverged"
    s, d, ue = _gpu_problem("biochem", "P1", None, 8)
    res = s.solve(d * 1e6, ue, u0=np.full_like(ue, -0.999), maxit=30, damping=False, div_factor=1e3)
    assert not res.converged and res.status in ("diverged", "maxit", "krylov")
