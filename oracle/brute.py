"""Independent dense brute force for tiny meshes — TEST INFRASTRUCTURE ONLY.

A second, deliberately different route to the same objects as the C++ oracle,
used to pin it (tests/test_oracle_*.py):

* basis functions are polynomials in barycentric coordinates (dict monomial →
  coefficient) and integrals are EXACT, via ∫_K λ^α dx = |K| d! α! / (|α|+d)!
  (no quadrature rule), or a caller-given rule evaluated on the polynomials;
* geometry comes from inverting the (d+1)×(d+1) matrix [[1…1],[x_0…x_d]]
  (λ_a(x) = c_a + ∇λ_a·x) instead of the oracle's edge-matrix adjugate;
* T is a dense numpy array T[N_u, N_u, N_f]; contractions use einsum;
* SGA residuals (no tensor) integrate the nonlinear integrand directly
  (PAPER.md L61–69 eq. (nonlinear_terms)).
"""
from __future__ import annotations

import itertools
from math import factorial

import numpy as np

P0, P1, P2 = 0, 1, 2
FORM_CONV_K, FORM_CONV_J, FORM_PLAP, FORM_MASS3, FORM_CONV_I = 0, 1, 2, 3, 4


# ------------------------------------------------------------------ polynomials
def pmul(p, q):
    out = {}
    for a, ca in p.items():
        for b, cb in q.items():
            e = tuple(x + y for x, y in zip(a, b))
            out[e] = out.get(e, 0.0) + ca * cb
    return out


def padd(p, q, s=1.0):
    out = dict(p)
    for b, cb in q.items():
        out[b] = out.get(b, 0.0) + s * cb
    return out


def pscale(p, s):
    return {e: c * s for e, c in p.items()}


def pderiv_lam(p, b):
    """∂p/∂λ_b."""
    out = {}
    for e, c in p.items():
        if e[b] > 0:
            f = list(e)
            f[b] -= 1
            out[tuple(f)] = out.get(tuple(f), 0.0) + c * e[b]
    return out


def pint(p, vol, d):
    """Exact ∫_K p(λ) dx = Σ c_α |K| d! Π α_a! / (|α|+d)!."""
    s = 0.0
    for e, c in p.items():
        num = factorial(d)
        for x in e:
            num *= factorial(x)
        s += c * vol * num / factorial(sum(e) + d)
    return s


def peval(p, lam):
    s = 0.0
    for e, c in p.items():
        t = c
        for x, l in zip(e, lam):
            t *= l ** x
        s += t
    return s


def mono(d, **kw):
    e = [0] * (d + 1)
    for k, v in kw.items():
        e[int(k[1:])] += v
    return {tuple(e): 1.0}


def lam_poly(d, a):
    e = [0] * (d + 1)
    e[a] = 1
    return {tuple(e): 1.0}


def local_basis(family, d):
    """Polynomials of the local basis in barycentric coordinates."""
    if family == P0:
        return [{tuple([0] * (d + 1)): 1.0}]
    if family == P1:
        return [lam_poly(d, a) for a in range(d + 1)]
    if family == P2 and d == 2:
        out = []
        for a in range(3):
            la = lam_poly(d, a)
            out.append(padd(pscale(pmul(la, la), 2.0), la, -1.0))
        for a, b in ((0, 1), (1, 2), (2, 0)):
            out.append(pscale(pmul(lam_poly(d, a), lam_poly(d, b)), 4.0))
        return out
    raise ValueError("unsupported family")


def geometry(xs):
    """xs: (d+1, d) vertex coords → (G[a, x] = ∂λ_a/∂x, |K|) via the barycentric system."""
    d = xs.shape[1]
    M = np.ones((d + 1, d + 1))
    M[1:, :] = xs.T  # column a = (1, x_a)
    # λ = M^{-1} (1, x): row a of M^{-1} = (c_a, ∇λ_a)
    Minv = np.linalg.inv(M)
    G = Minv[:, 1:]
    vol = abs(np.linalg.det(M)) / factorial(d)
    return G, vol


def grad_poly(p, G, x):
    """∂p/∂x_x = Σ_b ∂p/∂λ_b · ∂λ_b/∂x_x."""
    out = {}
    for b in range(G.shape[0]):
        out = padd(out, pscale(pderiv_lam(p, b), G[b, x]))
    return out


def _slot(op, phi, G, d):
    if op == "v":
        return phi
    if op == "dx":
        return grad_poly(phi, G, 0)
    if op == "dxdy":
        q = grad_poly(phi, G, 0)
        if d >= 2:
            q = padd(q, grad_poly(phi, G, 1))
        return q
    raise ValueError(op)


FORM_OPS = {FORM_CONV_K: ("v", "v", "dx"), FORM_CONV_J: ("v", "dxdy", "v"),
            FORM_MASS3: ("v", "v", "v"), FORM_CONV_I: ("dxdy", "v", "v")}


def local_tensor(form, d, xs, vfam, wfam, quad=None):
    G, vol = geometry(xs)
    phis = local_basis(vfam, d)
    etas = local_basis(wfam, d)
    nA, nC = len(phis), len(etas)
    Tl = np.zeros((nA, nA, nC))

    def integ(p):
        if quad is None:
            return pint(p, vol, d)
        bary, w = quad
        return vol * sum(wq * peval(p, lam) for lam, wq in zip(bary, w))

    for a, b, c in itertools.product(range(nA), range(nA), range(nC)):
        if form == FORM_PLAP:
            ab = {}
            for x in range(d):
                ab = padd(ab, pmul(grad_poly(phis[a], G, x), grad_poly(phis[b], G, x)))
            Tl[a, b, c] = integ(pmul(ab, etas[c]))
        else:
            oa, ob, oc = FORM_OPS[form]
            Tl[a, b, c] = integ(pmul(pmul(_slot(oa, phis[a], G, d), _slot(ob, phis[b], G, d)),
                                     _slot(oc, etas[c], G, d)))
    return Tl


def dense_tensor(mesh, V, W, form, quad=None):
    """Dense T[N_u, N_u, N_f] = Σ_K scatter(local_tensor)."""
    d = mesh.dim
    T = np.zeros((V.n_dofs, V.n_dofs, W.n_dofs))
    for K in range(mesh.n_cells):
        xs = mesh.coords[mesh.cells[K]]
        Tl = local_tensor(form, d, xs, V.family, W.family, quad)
        I = V.cell_dofs[K]
        Wd = W.cell_dofs[K]
        for a, b, c in itertools.product(range(len(I)), range(len(I)), range(len(Wd))):
            T[I[a], I[b], Wd[c]] += Tl[a, b, c]
    return T


def dense_from_canonical(ex, n_u, n_f):
    T = np.zeros((n_u, n_u, n_f))
    rp = ex["t_row_ptr"]
    for i in range(n_u):
        for e in range(rp[i], rp[i + 1]):
            T[i, ex["t_j"][e], ex["t_k"][e]] = ex["t_val"][e]
    return T


def bilinear_matrix(mesh, V, opA, opB):
    """Exact ∫ (opA φ_i)(opB φ_j) (or ∇φ_i·∇φ_j for opA == 'grad')."""
    d = mesh.dim
    A = np.zeros((V.n_dofs, V.n_dofs))
    phis = local_basis(V.family, d)
    for K in range(mesh.n_cells):
        G, vol = geometry(mesh.coords[mesh.cells[K]])
        I = V.cell_dofs[K]
        for a in range(len(I)):
            for b in range(len(I)):
                if opA == "grad":
                    p = {}
                    for x in range(d):
                        p = padd(p, pmul(grad_poly(phis[a], G, x), grad_poly(phis[b], G, x)))
                else:
                    p = pmul(_slot(opA, phis[a], G, d), _slot(opB, phis[b], G, d))
                A[I[a], I[b]] += pint(p, vol, d)
    return A


# ------------------------------------------------------------------ SGA residuals
def sga_plap(mesh, u, p):
    """SGA p-Laplace residual K(a,u)u, a = ‖∇u_h‖^{p-2}."""
    d = mesh.dim
    r = np.zeros(mesh.n_vertices)
    for K in range(mesh.n_cells):
        I = mesh.cells[K]
        G, vol = geometry(mesh.coords[I])
        g = G.T @ u[I]
        a = np.linalg.norm(g) ** (p - 2)
        r[I] += vol * a * (G @ g)
    return r


def sga_minsurf(mesh, u):
    """SGA minimal-surface residual K(a,u)u, a = (1 + ‖∇u_h‖²)^{-1/2}: with P1
    u_h the coefficient is constant on each cell, so this is exact (and equals EGFEM-P0, L616)."""
    r = np.zeros(mesh.n_vertices)
    for K in range(mesh.n_cells):
        I = mesh.cells[K]
        G, vol = geometry(mesh.coords[I])
        g = G.T @ u[I]
        r[I] += vol * (G @ g) / np.sqrt(1.0 + g @ g)
    return r


def tensor_free_reciprocal(mesh, u, k, w_family):
    """r_i = ∫ φ_i u_h c̃_h with c̃ = 1/(k + u) interpolated onto W, by exact
    polynomial integration, no tensor: W = P1 → c̃_h = Σ_v c̃(u_v) φ_v (GFEM); W = P0 → c̃_h|_K =
    c̃(u_h(centroid of K))."""
    d = mesh.dim
    r = np.zeros(mesh.n_vertices)
    phis = local_basis(P1, d)
    for K in range(mesh.n_cells):
        I = mesh.cells[K]
        G, vol = geometry(mesh.coords[I])
        uh = {}
        for a in range(d + 1):
            uh = padd(uh, pscale(phis[a], u[I[a]]))
        if w_family == "P1":
            ch = {}
            for a in range(d + 1):
                ch = padd(ch, pscale(phis[a], 1.0 / (k + u[I[a]])))
        else:
            ch = pscale(mono(d), 1.0 / (k + peval(uh, [1.0 / (d + 1)] * (d + 1))))
        f = pmul(uh, ch)
        for a in range(d + 1):
            r[I[a]] += pint(pmul(phis[a], f), vol, d)
    return r


def sga_rule_mass(mesh, u, f, bary, weights):
    """SGA of the term ∫ φ_i u f(u) with a quadrature rule: Σ_K Σ_ℓ w_ℓ|K| φ_i(x_ℓ)
    u_h(x_ℓ) f(u_h(x_ℓ)) — what EGFEM with W = I_k must reproduce exactly (Case 3, L133–139)."""
    d = mesh.dim
    r = np.zeros(mesh.n_vertices)
    bary = np.asarray(bary, dtype=np.float64).reshape(len(weights), d + 1)
    for K in range(mesh.n_cells):
        I = mesh.cells[K]
        _, vol = geometry(mesh.coords[I])
        for lam, wq in zip(bary, weights):
            uh = lam @ u[I]
            r[I] += wq * vol * lam * uh * f(uh)
    return r


def sga_cubic_mass(mesh, u):
    """r_i = ∫ φ_i u_h³ dx exactly (Case-1 target, PAPER.md L338 / L456)."""
    d = mesh.dim
    r = np.zeros(mesh.n_vertices)
    phis = local_basis(P1, d)
    for K in range(mesh.n_cells):
        I = mesh.cells[K]
        G, vol = geometry(mesh.coords[I])
        uh = {}
        for a in range(d + 1):
            uh = padd(uh, pscale(phis[a], u[I[a]]))
        u3 = pmul(pmul(uh, uh), uh)
        for a in range(d + 1):
            r[I[a]] += pint(pmul(phis[a], u3), vol, d)
    return r


def sga_burgers(mesh, V, u, w, variant):
    """Tensor-free Burgers residuals by exact integration of the nonlinear integrand:
    variant 'K': ∫ φ_i u_h ∂x w_h  (cfg1);  'J': ∫ φ_i w_h (∂x+∂y) u_h  (cfg2, cfg5 exact)."""
    d = mesh.dim
    r = np.zeros(V.n_dofs)
    phis = local_basis(V.family, d)
    for K in range(mesh.n_cells):
        G, vol = geometry(mesh.coords[mesh.cells[K]])
        I = V.cell_dofs[K]
        uh, wh = {}, {}
        for a in range(len(I)):
            uh = padd(uh, pscale(phis[a], u[I[a]]))
            wh = padd(wh, pscale(phis[a], w[I[a]]))
        if variant == "K":
            f = pmul(uh, _slot("dx", wh, G, d))
        else:
            f = pmul(wh, _slot("dxdy", uh, G, d))
        for a in range(len(I)):
            r[I[a]] += pint(pmul(phis[a], f), vol, d)
    return r
