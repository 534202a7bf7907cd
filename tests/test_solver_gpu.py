"""F4: the online Picard loop of PAPER.md §4 (L235–270) around the GPU hot path,
on the biochemical problem of §5.4 (−Δu + u/(1+u) = d, exact solution x1 x2 (x1+x2), L516–535).

Checked against (a) the same Picard iteration run on the CPU oracle's tensors with a direct
sparse solve (scipy), iterate for iterate, and (b) the manufactured solution: the P1 error
falls like h² under refinement."""
import numpy as np
import pytest

import egfem_inputs as I

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    import paper_2005_06193_b200 as eg
    return eg


def _reference_picard(n, W, iters):
    """CPU reference: the oracle's MASS3 tensor, stiffness = PLAP·1, mass = exact P1 mass matrix,
    Dirichlet elimination, scipy spsolve — PAPER.md L259–266 written out plainly."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spl

    import oracle
    from oracle import brute
    mesh = I.mesh_square(n)
    V = I.space_p1(mesh)
    Wsp = V if W == "P1" else I.space_p0(mesh)
    T = oracle.OracleTensor(mesh, V, Wsp, I.FORM_MASS3)
    Tk = oracle.OracleTensor(mesh, V, I.space_p0(mesh), I.FORM_PLAP)
    ex = T.export()
    rows = np.repeat(np.arange(T.n_u), np.diff(ex["csr_row_ptr"]))
    col = ex["csr_col"]
    Kv = Tk.jacobian(I.JAC_PICARD, I.INTERP_IDENTITY, 0.0, np.zeros(T.n_u), np.ones(Tk.n_f))
    M = brute.bilinear_matrix(mesh, V, "v", "v")
    x = mesh.coords
    ue = x[:, 0] * x[:, 1] * (x[:, 0] + x[:, 1])
    d = M @ (-(2 * x[:, 0] + 2 * x[:, 1]) + ue / (1.0 + ue))
    bnd = np.any((x <= 1e-12) | (x >= 1 - 1e-12), axis=1)
    u = np.where(bnd, ue, 0.0)
    out = []
    for _ in range(iters):
        w = T.interp(I.INTERP_RECIPROCAL, 1.0, u)
        A = sp.csr_matrix((Kv + T.jacobian(I.JAC_PICARD, I.INTERP_RECIPROCAL, 1.0, u, w), (rows, col)),
                          shape=(T.n_u, T.n_u)).tolil()
        b = d.copy()
        A = A.tocsr()
        b -= A[:, bnd] @ ue[bnd]
        A = A.tolil()
        A[bnd, :] = 0
        A[:, bnd] = 0
        A[bnd, bnd] = 1.0
        b[bnd] = ue[bnd]
        u = spl.spsolve(A.tocsr(), b)
        out.append(u.copy())
    return out, ue


@pytest.mark.parametrize("W", ["P1", "P0"])
def test_picard_matches_cpu_reference(eg, W):
    from paper_2005_06193_b200.solver import biochemical_problem
    n = 8
    s, d, ue = biochemical_problem(n, W=W)
    res = s.solve(d, ue, maxit=4, tol=0.0, cg_tol=1e-15)
    ref, _ = _reference_picard(n, W, 4)
    assert np.abs(res.u - ref[-1]).max() < 1e-10


def test_picard_converges_at_second_order(eg):
    """iterate to an increment of O(1e-12); the nodal error vs the manufactured
    solution decreases like h² (P1; the GFEM c̃ and the interpolated source are O(h²) too)."""
    from paper_2005_06193_b200.solver import biochemical_problem
    errs = []
    for n in (8, 16, 32):
        s, d, ue = biochemical_problem(n)
        res = s.solve(d, ue, tol=1e-12, maxit=60)
        assert res.converged, res.increments[-3:]
        assert res.iterations < 30
        errs.append(np.abs(res.u - ue).max())
    assert errs[0] / errs[1] > 3.0 and errs[1] / errs[2] > 3.0, errs
