"""Pins of the CPU oracle against things other than itself (-m "not gpu").

Each test cites the passage it checks.  Pins used:
  * closed forms derived by hand (element tensors, 1D stencils);
  * an independent dense brute force with EXACT polynomial integration
    (oracle/brute.py) on tiny, also jittered (unstructured) meshes;
  * invariants: partition of unity, symmetry, integration by parts, Σr = 0,
    bilinearity, Euler homogeneity, contraction consistency;
  * central finite differences of r(u) for the Newton Jacobian;
  * SGA (no tensor) residuals where EGFEM is exact (Case 1, P0 for p-Laplace);
  * printed sizes of PAPER.md Table 1 (tests/golden/table1_sizes.json).
"""
import json
import os

import numpy as np
import pytest

import egfem_inputs as I
from oracle import brute
from helpers import rel_l2

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SIX_PT = (0.445948490915965, 0.2233815896780118, 0.091576213509770549, 0.10995174365532154)


def six_point_rule():
    bary, w = [], []
    a1, w1, a2, w2 = SIX_PT
    for a, ww in ((a1, w1), (a2, w2)):
        b = 1 - 2 * a
        for p in ((b, a, a), (a, b, a), (a, a, b)):
            bary.append(p)
            w.append(ww)
    return np.array(bary), np.array(w)


def jitter(mesh, amp, seed):
    """Perturb interior vertices (unstructured geometry, same topology)."""
    rng = np.random.default_rng(seed)
    x = mesh.coords.copy()
    inner = np.all((x > 1e-12) & (x < 1 - 1e-12), axis=1)
    n = round(1 / np.max(np.diff(np.unique(x[:, 0]))))
    x[inner] += amp / n * rng.uniform(-1, 1, (inner.sum(), mesh.dim))
    return I.Mesh(mesh.dim, x, mesh.cells)


def dense(T):
    return brute.dense_from_canonical(T.export(), T.n_u, T.n_f)


# ----------------------------------------------------------------------------- sizes
def test_config_sizes_match_baseline_text():
    """BASELINE.json configs: node and element counts quoted in the config text."""
    want = {"cfg1": (257, 256), "cfg2": (263169, 524288), "cfg3": (1050625, 2097152),
            "cfg4": (2146689, 12582912), "cfg5": (263169, 131072)}
    for name, (nu, nel) in want.items():
        pr = I.make_problem(name, batch=1)
        assert (pr.n_u, pr.mesh.n_cells) == (nu, nel), name
    assert I.make_problem("cfg3").n_f == 2097152
    assert I.make_problem("cfg4").n_f == 12582912


def test_table1_sizes_golden():
    """PAPER.md Table 1 'Size' column (L490-L495): P1 and P2 spaces on the 64×64 mesh."""
    g = json.load(open(os.path.join(GOLD, "table1_sizes.json")))
    m = I.mesh_square(g["n"])
    n_p1 = I.space_p1(m).n_dofs
    n_p2 = I.space_p2_square(g["n"]).n_dofs
    sizes = {r["model"]: r["size"] for r in g["rows"]}
    assert n_p1 == sizes["SGA"] == 4225
    assert m.n_cells == 8192
    assert n_p1 + n_p1 == sizes["GFEM"]
    assert n_p1 + n_p2 == sizes["EGFEM (P2)"]
    assert n_p1 + 6 * m.n_cells == sizes["EGFEM (I4)"]  # 6-point rule per cell (L139)


def closed_form_counts(name, n):
    if name == "cfg1":
        N = n + 1
        return 7 * N - 6, 3 * N - 2
    if name in ("cfg2", "cfg3"):
        N, Nel, E = (n + 1) ** 2, 2 * n * n, 3 * n * n + 2 * n
        nnz = N + 6 * E + 6 * Nel if name == "cfg2" else 9 * Nel
        return nnz, N + 2 * E
    if name == "cfg4":
        N, Nel = (n + 1) ** 3, 6 * n ** 3
        E = 3 * n * (n + 1) ** 2 + 3 * n * n * (n + 1) + n ** 3
        return 16 * Nel, N + 2 * E
    if name == "cfg5":
        N, Nel, E = (2 * n + 1) ** 2, 2 * n * n, 3 * n * n + 2 * n
        Eint = E - 4 * n
        S2, S3 = 15 * Nel - 3 * Eint, 20 * Nel - Eint
        return N + 6 * S2 + 6 * S3, N + 2 * S2


@pytest.mark.parametrize("name,n", [("cfg1", 7), ("cfg1", 256), ("cfg2", 5), ("cfg3", 6), ("cfg4", 2),
                                    ("cfg4", 3), ("cfg5", 3), ("cfg5", 4)])
def test_counts_closed_form(oracle_mod, name, n):
    """Structural pattern (reading C7/C8): nnz(T) and nnz(CSR) vs closed-form counts."""
    pr = I.make_problem(name, n=n, batch=1)
    T = oracle_mod.OracleTensor(pr.mesh, pr.V, pr.W, pr.form)
    assert (T.nnz, T.nnz_csr) == closed_form_counts(name, n)


def test_counts_full_size_formula():
    """SURVEY §8(a) size table at BASELINE sizes (the closed forms are pinned above)."""
    want = {"cfg1": (1793, 769), "cfg2": (8133633, 1838081), "cfg3": (18874368, 7346177),
            "cfg4": (201326592, 31802497), "cfg5": (23081985, 3018753)}
    for name, v in want.items():
        assert closed_form_counts(name, I.FULL_N[name]) == v


def test_full_size_cfg2_counts(oracle_mod):
    pr = I.make_problem("cfg2")
    T = oracle_mod.OracleTensor(pr.mesh, pr.V, pr.W, pr.form)
    assert (T.nnz, T.nnz_csr) == (8133633, 1838081)


# ----------------------------------------------------------------------------- element closed forms
def test_conv_k_1d_closed_form(oracle_mod):
    """cfg1 T_ijk = ∫ φ_i φ_j ∂x φ_k (BASELINE cfg1): element value s_c (1+δ_ab)/6, s = (−1, +1)."""
    n = 6
    pr = I.make_problem("cfg1", n=n)
    D = dense(oracle_mod.OracleTensor(pr.mesh, pr.V, pr.W, pr.form))
    E = np.zeros_like(D)
    s = (-1.0, 1.0)
    for e in range(n):
        v = (e, e + 1)
        for a in range(2):
            for b in range(2):
                for c in range(2):
                    E[v[a], v[b], v[c]] += s[c] * (1 + (a == b)) / 6
    assert np.abs(D - E).max() < 1e-15


def test_plap_2d_closed_form(oracle_mod):
    """cfg3 T_ijK = |K| ∇φ_i·∇φ_j (PAPER.md L253 with P0 ψ_K): h-independent element matrices."""
    n = 4
    pr = I.make_problem("cfg3", n=n)
    D = dense(oracle_mod.OracleTensor(pr.mesh, pr.V, pr.W, pr.form))
    lower = 0.5 * np.array([[1, -1, 0], [-1, 2, -1], [0, -1, 1]])
    upper = 0.5 * np.array([[1, 0, -1], [0, 1, -1], [-1, -1, 2]])
    E = np.zeros_like(D)
    for K in range(pr.mesh.n_cells):
        v = pr.mesh.cells[K]
        E[np.ix_(v, v, [K])] += (lower if K % 2 == 0 else upper)[:, :, None]
    assert np.abs(D - E).max() < 1e-15


def test_plap_3d_kuhn_closed_form(oracle_mod):
    """cfg4: Kuhn tet of a path v0→v3: |K|∇λ_a·∇λ_b = (h/6)·tridiag(−1, [1,2,2,1], −1)."""
    n = 2
    h = 1.0 / n
    pr = I.make_problem("cfg4", n=n)
    D = dense(oracle_mod.OracleTensor(pr.mesh, pr.V, pr.W, pr.form))
    Lp = (h / 6) * np.array([[1, -1, 0, 0], [-1, 2, -1, 0], [0, -1, 2, -1], [0, 0, -1, 1]])
    E = np.zeros_like(D)
    for K in range(pr.mesh.n_cells):
        v = pr.mesh.cells[K]
        E[np.ix_(v, v, [K])] += Lp[:, :, None]
    assert np.abs(D - E).max() < 1e-15


def test_conv_j_p1_closed_form(oracle_mod):
    """cfg2 T_ijk = ∫ φ_i φ_k (∂x+∂y)φ_j: (∂x+∂y)λ_b · |K|(1+δ_ac)/12 per element."""
    n = 3
    h = 1.0 / n
    pr = I.make_problem("cfg2", n=n)
    D = dense(oracle_mod.OracleTensor(pr.mesh, pr.V, pr.W, pr.form))
    # (∂x+∂y)λ_b for lower (v00,v10,v11): (-1, 0, 1)/h ; upper (v00,v11,v01): (-1, 1, 0)/h
    dl = {0: np.array([-1, 0, 1]) / h, 1: np.array([-1, 1, 0]) / h}
    area = h * h / 2
    E = np.zeros_like(D)
    for K in range(pr.mesh.n_cells):
        v = pr.mesh.cells[K]
        for a in range(3):
            for b in range(3):
                for c in range(3):
                    E[v[a], v[b], v[c]] += dl[K % 2][b] * area * (1 + (a == c)) / 12
    assert np.abs(D - E).max() < 1e-15


# ----------------------------------------------------------------------------- brute force (exact integration)
@pytest.mark.parametrize("case", ["conv_k_1d", "conv_j_p1", "conv_i_p1", "plap_2d", "plap_3d", "mass3_p1p1p2",
                                  "mass3_p1p1p1", "conv_j_p1_jitter", "plap_2d_jitter", "plap_3d_jitter",
                                  "mass3_jitter", "mass3_3d", "mass3_3d_jitter", "mass3_3d_p0", "conv_j_3d_jitter"])
def test_oracle_vs_dense_brute_force(oracle_mod, case):
    """Oracle element loop + canonicalisation vs an independent dense build with exact integration."""
    if case == "conv_k_1d":
        m = I.mesh_interval(5); V = W = I.space_p1(m); form = I.FORM_CONV_K
    elif case.startswith("conv_j_p1"):
        m = I.mesh_square(3); form = I.FORM_CONV_J
    elif case == "conv_i_p1":
        m = I.mesh_square(3); form = I.FORM_CONV_I
    elif case.startswith("plap_2d"):
        m = I.mesh_square(3); form = I.FORM_PLAP
    elif case.startswith("plap_3d"):
        m = I.mesh_cube(2); form = I.FORM_PLAP
    elif case.startswith("mass3_3d"):  # the trilinear mass M, degree 3 in 3D
        m = I.mesh_cube(2); form = I.FORM_MASS3
    elif case == "conv_j_3d_jitter":
        m = I.mesh_cube(2); form = I.FORM_CONV_J
    elif case.startswith("mass3"):
        m = I.mesh_square(2); form = I.FORM_MASS3
    if case.endswith("jitter"):
        m = jitter(m, 0.2, 7)
    if case != "conv_k_1d":
        V = I.space_p1(m)
        if case.startswith("plap") or case == "mass3_3d_p0":
            W = I.space_p0(m)
        elif case in ("mass3_p1p1p2", "mass3_jitter"):
            W = I.space_p2_square(2)
        else:
            W = V
    T = oracle_mod.OracleTensor(m, V, W, form)
    D = dense(T)
    B = brute.dense_tensor(m, V, W, form)
    assert np.abs(D - B).max() <= 1e-14 * max(1.0, np.abs(B).max())
    # every structural triple kept (reading C7): nnz = number of distinct (I[a],J[b],W[c])
    trip = set()
    for K in range(m.n_cells):
        for a in V.cell_dofs[K]:
            for b in V.cell_dofs[K]:
                for c in W.cell_dofs[K]:
                    trip.add((a, b, c))
    assert T.nnz == len(trip)


@pytest.mark.parametrize("dim", [1, 2, 3])
def test_oracle_rules_monomial_exactness(oracle_mod, dim):
    """Every default rule the oracle's element loop takes integrates ∫_K λ^α = |K| d! α!/(|α|+d)!
    exactly for |α| ≤ the degree it is chosen for (2D: ≤ 4, reading C3) (T is an integral), and has
    positive weights summing to 1.  Pins the 3D degree ≥ 3 collapsed Gauss rule (MASS3, L327)."""
    import itertools
    from math import factorial
    import oracle
    for degree in range(0, 6):
        bary, w = oracle.rule(dim, degree)
        assert np.all(w > 0) and abs(w.sum() - 1) < 4e-15
        assert np.all(bary >= -1e-15) and np.allclose(bary.sum(axis=1), 1, atol=1e-15)
        # 1D: 3-point Gauss (degree 5) always; 2D degree ≥ 5 takes the 6-point degree-4 rule by
        # reading C3 (BJ cfg5 names "6-point quadrature")
        exact_to = 5 if dim == 1 else (min(degree, 4) if dim == 2 else degree)
        for al in itertools.product(range(exact_to + 1), repeat=dim + 1):
            if sum(al) > exact_to:
                continue
            exact = factorial(dim) * np.prod([factorial(a) for a in al]) / factorial(sum(al) + dim)
            got = float(np.sum(w * np.prod(bary ** np.array(al), axis=1)))
            assert abs(got - exact) <= 4e-15 * max(1.0, exact), (dim, degree, al, got, exact)


def test_tet_mass3_single_cell_closed_form(oracle_mod):
    """One Kuhn tet: M_abc = ∫ λ_a λ_b λ_c = |K|·3!·Π(mult)!/6!, i.e. |K|/20 (a=b=c), |K|/60 (two equal),
    |K|/120 (distinct) — the exact trilinear mass of PAPER.md L327 (the round-1 4-point rule gave 0.00905|K|)."""
    x = np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [1, 1, 1]], float)
    m = I.Mesh(3, x, np.array([[0, 1, 2, 3]], np.int32))
    V = I.space_p1(m)
    T = oracle_mod.OracleTensor(m, V, V, I.FORM_MASS3)
    D = dense(T)
    vol = 1.0 / 6
    for a in range(4):
        for b in range(4):
            for c in range(4):
                n = len({a, b, c})
                want = vol / (20 if n == 1 else 60 if n == 2 else 120)
                assert abs(D[a, b, c] - want) <= 4e-15 * want, (a, b, c, D[a, b, c], want)


def test_p2_six_point_rule_brute_force(oracle_mod):
    """cfg5 T is defined by the 6-point rule (reading C3): brute force with the same rule on jittered P2."""
    n = 2
    m = jitter(I.mesh_square(n), 0.2, 3)
    V = I.space_p2_square(n)
    T = oracle_mod.OracleTensor(m, V, V, I.FORM_CONV_J)
    B = brute.dense_tensor(m, V, V, I.FORM_CONV_J, quad=six_point_rule())
    assert np.abs(dense(T) - B).max() < 1e-15


def test_six_point_rule_monomial_exactness():
    """Dunavant degree 4: ∫ λ^α exact for |α| ≤ 4, not for 5."""
    bary, w = six_point_rule()
    from math import factorial
    worst = 0.0
    for a in range(5):
        for b in range(5 - a):
            for c in range(5 - a - b):
                exact = 2 * factorial(a) * factorial(b) * factorial(c) / factorial(a + b + c + 2)
                got = np.sum(w * bary[:, 0] ** a * bary[:, 1] ** b * bary[:, 2] ** c)
                worst = max(worst, abs(got - exact))
    assert worst < 1e-15
    assert abs(w.sum() - 1) < 1e-15


def test_p2_exact_moments_full_rule(oracle_mod):
    """Contractions of the 6-point cfg5 T whose integrand has degree ≤ 4 equal the EXACT integrals:
    k-slot with P2 interpolants of 1, x, y and j-slot with interpolants of x, y (reading C3)."""
    n = 3
    m = jitter(I.mesh_square(n), 0.15, 11)
    V = I.space_p2_square(n)
    x = V.dof_coords.copy()
    # dof coords of the jittered mesh: vertices move, midpoints are edge midpoints (affine P2)
    for K in range(m.n_cells):
        xs = m.coords[m.cells[K]]
        d = V.cell_dofs[K]
        x[d[:3]] = xs
        x[d[3]] = 0.5 * (xs[0] + xs[1]); x[d[4]] = 0.5 * (xs[1] + xs[2]); x[d[5]] = 0.5 * (xs[2] + xs[0])
    D = dense(oracle_mod.OracleTensor(m, V, V, I.FORM_CONV_J))
    Bx = brute.dense_tensor(m, V, V, I.FORM_CONV_J)  # exact integral
    for f in (np.ones(len(x)), x[:, 0], x[:, 1], 0.3 + x[:, 0] - 2 * x[:, 1]):
        assert np.abs(np.einsum("ijk,k->ij", D, f) - np.einsum("ijk,k->ij", Bx, f)).max() < 1e-14
    for g in (x[:, 0], x[:, 1]):
        assert np.abs(np.einsum("ijk,j->ik", D, g) - np.einsum("ijk,j->ik", Bx, g)).max() < 1e-14


# ----------------------------------------------------------------------------- invariants
@pytest.mark.parametrize("name,n", [("cfg1", 9), ("cfg2", 4), ("cfg3", 4), ("cfg4", 2), ("cfg5", 2)])
def test_partition_of_unity(oracle_mod, name, n):
    """SPEC.md L308/L316/L326: Σ_k T_ijk (w ≡ 1) reproduces the bilinear matrix (exact integration)."""
    pr = I.make_problem(name, n=n, batch=1)
    T = oracle_mod.OracleTensor(pr.mesh, pr.V, pr.W, pr.form)
    A = np.einsum("ijk->ij", dense(T))
    if name == "cfg1":
        B = np.zeros_like(A)  # ∫ φ_i φ_j ∂x(Σ φ_k) = 0
    elif name in ("cfg2", "cfg5"):
        B = brute.bilinear_matrix(pr.mesh, pr.V, "v", "dxdy")
    else:
        B = brute.bilinear_matrix(pr.mesh, pr.V, "grad", None)
    assert np.abs(A - B).max() < 1e-14


def test_plap_pou_stencils_full_size(oracle_mod):
    """PLAP PoU at BASELINE cfg3 size: 5-point stencil (4, −1, exactly 0 on diagonal neighbours)."""
    pr = I.make_problem("cfg3")
    T = oracle_mod.OracleTensor(pr.mesh, pr.V, pr.W, pr.form)
    ex = T.export()
    one = np.ones(T.n_f)
    A = T.jacobian(I.JAC_PICARD, I.INTERP_GRADPOW_P0, 4.0, np.zeros(T.n_u), one)
    n = 1024
    m = n + 1
    rows = np.repeat(np.arange(T.n_u), np.diff(ex["csr_row_ptr"]))
    cols = ex["csr_col"]
    ix, iy = rows % m, rows // m
    interior = (ix > 0) & (ix < n) & (iy > 0) & (iy < n)
    diff = cols - rows
    want = np.where(diff == 0, 4.0, np.where(np.isin(np.abs(diff), (1, m)), -1.0, 0.0))
    assert np.array_equal(A[interior], want[interior])


@pytest.mark.parametrize("dim", [2, 3])
def test_plap_symmetry(oracle_mod, dim):
    """PLAP slices symmetric in (i, j)."""
    m = jitter(I.mesh_square(4) if dim == 2 else I.mesh_cube(2), 0.2, 5)
    D = dense(oracle_mod.OracleTensor(m, I.space_p1(m), I.space_p0(m), I.FORM_PLAP))
    assert np.array_equal(D, D.transpose(1, 0, 2))


def test_integration_by_parts_identity(oracle_mod):
    """Reading C1: BASELINE's CONV_J vs the paper's N (CONV_I): with w = u,
    CONV_J(u,u)_i = −½ CONV_I(u,u)_i on every row whose node is off ∂Ω (P1, exact)."""
    n = 6
    pr = I.make_problem("cfg2", n=n)
    u = pr.u
    TJ = oracle_mod.OracleTensor(pr.mesh, pr.V, pr.V, I.FORM_CONV_J)
    TI = oracle_mod.OracleTensor(pr.mesh, pr.V, pr.V, I.FORM_CONV_I)
    rJ, rI = TJ.apply(u, u), TI.apply(u, u)
    x = pr.mesh.coords
    inner = np.all((x > 1e-12) & (x < 1 - 1e-12), axis=1)
    assert np.abs(rJ[inner] + 0.5 * rI[inner]).max() < 1e-15
    assert np.abs(rJ[~inner] + 0.5 * rI[~inner]).max() > 1e-6  # boundary rows differ (∮ term)


# ----------------------------------------------------------------------------- contractions
@pytest.mark.parametrize("name,n", [("cfg1", 8), ("cfg2", 4), ("cfg3", 4), ("cfg4", 2), ("cfg5", 2)])
def test_apply_and_picard_vs_dense(oracle_mod, name, n):
    """r = T:(u⊗w) and A = T·w (L182) vs einsum on the brute-force tensor."""
    pr = I.make_problem(name, n=n, batch=2)
    T = oracle_mod.OracleTensor(pr.mesh, pr.V, pr.W, pr.form)
    B = brute.dense_tensor(pr.mesh, pr.V, pr.W, pr.form, quad=six_point_rule() if name == "cfg5" else None)
    rng = np.random.default_rng(1)
    u, w = rng.standard_normal(T.n_u), rng.standard_normal(T.n_f)
    assert rel_l2(T.apply(u, w), np.einsum("ijk,j,k->i", B, u, w)) < 1e-14
    A = T.jacobian(I.JAC_PICARD, pr.interp, pr.p, u, w)
    ex = T.export()
    Ad = np.zeros((T.n_u, T.n_u))
    rows = np.repeat(np.arange(T.n_u), np.diff(ex["csr_row_ptr"]))
    Ad[rows, ex["csr_col"]] = A
    assert rel_l2(Ad, np.einsum("ijk,k->ij", B, w)) < 1e-14
    # consistency r = (T·w)·u = (T·₂u)·w
    assert rel_l2(Ad @ u, T.apply(u, w)) < 1e-14
    assert rel_l2(np.einsum("ijk,j->ik", B, u) @ w, T.apply(u, w)) < 1e-14
    # batched == per pair
    U, Wb = rng.standard_normal((3, T.n_u)), rng.standard_normal((3, T.n_f))
    R = T.apply_batched(U, Wb)
    for p in range(3):
        assert np.array_equal(R[p], T.apply(U[p], Wb[p]))


def test_apply_1d_closed_form(oracle_mod):
    """the 1D Galerkin Burgers stencil r_i = (u_{i+1}−u_{i−1})(u_{i−1}+u_i+u_{i+1})/6
    at w = u, and the general interior / end formulas."""
    pr = I.make_problem("cfg1")
    T = oracle_mod.OracleTensor(pr.mesh, pr.V, pr.W, pr.form)
    rng = np.random.default_rng(2)
    u, w = rng.standard_normal(T.n_u), rng.standard_normal(T.n_u)
    r = T.apply(u, w)
    i = np.arange(1, T.n_u - 1)
    want = (2 * u[i] * (w[i + 1] - w[i - 1]) + u[i + 1] * (w[i + 1] - w[i]) + u[i - 1] * (w[i] - w[i - 1])) / 6
    assert np.abs(r[i] - want).max() < 1e-14
    assert abs(r[0] - (w[1] - w[0]) * (2 * u[0] + u[1]) / 6) < 1e-14
    assert abs(r[-1] - (w[-1] - w[-2]) * (2 * u[-1] + u[-2]) / 6) < 1e-14
    u = pr.u
    r = T.apply(u, u)
    assert np.abs(r[i] - (u[i + 1] - u[i - 1]) * (u[i - 1] + u[i] + u[i + 1]) / 6).max() < 1e-14


def test_jacobian_1d_closed_forms(oracle_mod):
    """PICARD A_{i,i±1}, A_ii and NEWTON (w = u) J stencils of the 1D Burgers tensor."""
    pr = I.make_problem("cfg1")
    T = oracle_mod.OracleTensor(pr.mesh, pr.V, pr.W, pr.form)
    ex = T.export()
    rng = np.random.default_rng(3)
    u, w = rng.standard_normal(T.n_u), rng.standard_normal(T.n_u)
    A = T.jacobian(I.JAC_PICARD, I.INTERP_IDENTITY, 0, u, w)
    J = T.jacobian(I.JAC_NEWTON, I.INTERP_IDENTITY, 0, u, u)
    rp = ex["csr_row_ptr"]
    for i in range(1, T.n_u - 1):
        a = A[rp[i]:rp[i + 1]]
        assert np.allclose(a, [(w[i] - w[i - 1]) / 6, (w[i + 1] - w[i - 1]) / 3, (w[i + 1] - w[i]) / 6],
                           rtol=0, atol=1e-14)
        j = J[rp[i]:rp[i + 1]]
        assert np.allclose(j, [-(2 * u[i - 1] + u[i]) / 6, (u[i + 1] - u[i - 1]) / 6, (u[i] + 2 * u[i + 1]) / 6],
                           rtol=0, atol=1e-14)


def _residual(T, kind, p, u):
    return T.apply(u, T.interp(kind, p, u))


def _fd_jacobian(T, kind, p, u, eps):
    J = np.zeros((T.n_u, T.n_u))
    for m in range(T.n_u):
        e = np.zeros(T.n_u); e[m] = eps
        J[:, m] = (_residual(T, kind, p, u + e) - _residual(T, kind, p, u - e)) / (2 * eps)
    return J


def _csr_dense(T, vals):
    ex = T.export()
    D = np.zeros((T.n_u, T.n_u))
    rows = np.repeat(np.arange(T.n_u), np.diff(ex["csr_row_ptr"]))
    D[rows, ex["csr_col"]] = vals
    return D


@pytest.mark.parametrize("case", ["cfg1", "cfg2", "cfg2_square", "cfg3", "cfg4", "cfg4_p4", "cfg3_p25",
                                  "mass3_p2"])
def test_newton_jacobian_vs_finite_differences(oracle_mod, case):
    """J = T·w + (T·₂u)·D_u w (reading C10) equals D_u r(u) with w = w(u):
    central differences, exact for quadratic Burgers, ≤1e-6 relative for p-Laplace."""
    kind_override, p_override = None, None
    if case == "mass3_p2":
        m = jitter(I.mesh_square(2), 0.1, 1)
        V, W = I.space_p1(m), I.space_p2_square(2)
        T = oracle_mod.OracleTensor(m, V, W, I.FORM_MASS3)
        kind, p = I.INTERP_P1_TO_P2_SQUARE, 0.0
        u = np.random.default_rng(4).standard_normal(V.n_dofs)
        tol = 1e-9
    else:
        name = case.split("_")[0]
        pr = I.make_problem(name, n={"cfg1": 8, "cfg2": 3, "cfg3": 4, "cfg4": 2}[name])
        m = jitter(pr.mesh, 0.15, 2) if pr.mesh.dim > 1 else pr.mesh
        T = oracle_mod.OracleTensor(m, pr.V, pr.W, pr.form)
        kind, p, u = pr.interp, pr.p, pr.u
        if case == "cfg2_square":
            kind = I.INTERP_SQUARE
        if case == "cfg4_p4":
            p = 4.0
        if case == "cfg3_p25":
            p = 2.5
        tol = 1e-9 if pr.form != I.FORM_PLAP else 1e-6
    w = T.interp(kind, p, u)
    J = _csr_dense(T, T.jacobian(I.JAC_NEWTON, kind, p, u, w))
    Jfd = _fd_jacobian(T, kind, p, u, 1e-6 if tol < 1e-6 else 1e-5)
    assert rel_l2(J, Jfd) < tol


@pytest.mark.parametrize("name", ["cfg2", "cfg3", "cfg4"])
def test_euler_homogeneity(oracle_mod, name):
    """Burgers NEWTON: J·u = 2r; PLAP PICARD: A·u = r; PLAP NEWTON: J·u = (p−1) r (degree-p−1 homogeneous)."""
    pr = I.make_problem(name, n={"cfg2": 8, "cfg3": 8, "cfg4": 3}[name])
    T = oracle_mod.OracleTensor(pr.mesh, pr.V, pr.W, pr.form)
    u = pr.u
    w = T.interp(pr.interp, pr.p, u)
    r = T.apply(u, w)
    J = _csr_dense(T, T.jacobian(I.JAC_NEWTON, pr.interp, pr.p, u, w))
    A = _csr_dense(T, T.jacobian(I.JAC_PICARD, pr.interp, pr.p, u, w))
    assert rel_l2(A @ u, r) < 1e-13
    if pr.form == I.FORM_PLAP:
        assert rel_l2(J @ u, (pr.p - 1) * r) < 1e-12
        assert abs(r.sum()) < 1e-12 * np.abs(r).sum()  # Σ_i ∇φ_i = 0
        assert np.array_equal(J, J.T) or rel_l2(J, J.T) < 1e-14
    else:
        assert rel_l2(J @ u, 2 * r) < 1e-13


def test_bilinearity_and_zero(oracle_mod):
    pr = I.make_problem("cfg3", n=6)
    T = oracle_mod.OracleTensor(pr.mesh, pr.V, pr.W, pr.form)
    rng = np.random.default_rng(9)
    u, w = rng.standard_normal(T.n_u), rng.standard_normal(T.n_f)
    assert rel_l2(T.apply(2.5 * u, -0.5 * w), -1.25 * T.apply(u, w)) < 1e-15
    assert not np.any(T.apply(u, np.zeros(T.n_f)))


# ----------------------------------------------------------------------------- interpolation
@pytest.mark.parametrize("dim,p", [(2, 4.0), (3, 3.0), (2, 1.5)])
def test_gradpow_linear_field(oracle_mod, dim, p):
    """u = interpolant of α·x + β ⇒ ∇u_h ≡ α on every cell ⇒ w_K = |α|^{p−2}."""
    m = jitter(I.mesh_square(5) if dim == 2 else I.mesh_cube(3), 0.2, 8)
    T = oracle_mod.OracleTensor(m, I.space_p1(m), I.space_p0(m), I.FORM_PLAP)
    alpha = np.array([0.7, -1.3, 0.4][:dim])
    u = m.coords @ alpha + 0.25
    w = T.interp(I.INTERP_GRADPOW_P0, p, u)
    assert np.abs(w - np.linalg.norm(alpha) ** (p - 2)).max() < 1e-13


def test_p_laplace_egfem_p0_equals_sga(oracle_mod):
    """PAPER.md L594 / L626: with P1 trial space, EGFEM-P0 reproduces SGA exactly (a is constant per cell)."""
    for m, p in ((jitter(I.mesh_square(5), 0.2, 1), 4.0), (jitter(I.mesh_cube(2), 0.2, 2), 3.0)):
        T = oracle_mod.OracleTensor(m, I.space_p1(m), I.space_p0(m), I.FORM_PLAP)
        u = np.random.default_rng(5).standard_normal(m.n_vertices)
        r = T.apply(u, T.interp(I.INTERP_GRADPOW_P0, p, u))
        assert rel_l2(r, brute.sga_plap(m, u, p)) < 1e-13


def test_case1_exactness_mass3_p2(oracle_mod):
    """PAPER.md L338/L348 (Case 1): u² of P1 lies in P2, so M:(u⊗w) with w = P2-interp of u²
    equals the SGA term ∫ φ_i u_h³ (exact integration)."""
    n = 3
    m = jitter(I.mesh_square(n), 0.2, 4)
    V, W = I.space_p1(m), I.space_p2_square(n)
    T = oracle_mod.OracleTensor(m, V, W, I.FORM_MASS3)
    u = np.random.default_rng(6).standard_normal(V.n_dofs)
    r = T.apply(u, T.interp(I.INTERP_P1_TO_P2_SQUARE, 0, u))
    assert rel_l2(r, brute.sga_cubic_mass(m, u)) < 1e-13
    # GFEM (W = V, SQUARE) is only an approximation of the same term (Case 2)
    T1 = oracle_mod.OracleTensor(m, V, V, I.FORM_MASS3)
    r1 = T1.apply(u, T1.interp(I.INTERP_SQUARE, 0, u))
    assert rel_l2(r1, brute.sga_cubic_mass(m, u)) > 1e-3


def test_burgers_egfem_equals_sga(oracle_mod):
    """W = V with w = u is exact for P1 Burgers: T:(u⊗u) equals the tensor-free SGA integral."""
    pr = I.make_problem("cfg1", n=12)
    T = oracle_mod.OracleTensor(pr.mesh, pr.V, pr.W, pr.form)
    assert rel_l2(T.apply(pr.u, pr.u), brute.sga_burgers(pr.mesh, pr.V, pr.u, pr.u, "K")) < 1e-14
    m = jitter(I.mesh_square(4), 0.2, 3)
    V = I.space_p1(m)
    T = oracle_mod.OracleTensor(m, V, V, I.FORM_CONV_J)
    u = np.random.default_rng(7).standard_normal(V.n_dofs)
    assert rel_l2(T.apply(u, u), brute.sga_burgers(m, V, u, u, "J")) < 1e-14


def test_maps_consistency(oracle_mod):
    """Index maps: csr_col[slot_ij] = t_j, csr_col[slot_ik] = t_k, loc decodes i and j,
    (j,k) strictly increasing within a row."""
    for name, n in (("cfg2", 5), ("cfg4", 2), ("cfg5", 3)):
        pr = I.make_problem(name, n=n, batch=1)
        T = oracle_mod.OracleTensor(pr.mesh, pr.V, pr.W, pr.form)
        p0 = pr.W.family == I.P0
        ex = T.export(slot_ik=not p0, loc=p0)
        rows = np.repeat(np.arange(T.n_u), np.diff(ex["t_row_ptr"]))
        assert np.array_equal(ex["csr_col"][ex["slot_ij"]], ex["t_j"])
        crow = np.repeat(np.arange(T.n_u), np.diff(ex["csr_row_ptr"]))
        assert np.array_equal(crow[ex["slot_ij"]], rows)
        key = (rows.astype(np.int64) * T.n_u + ex["t_j"]) * T.n_f + ex["t_k"]
        assert np.all(np.diff(key) > 0)
        if p0:
            cv = pr.V.cell_dofs[ex["t_k"]]
            assert np.array_equal(cv[np.arange(T.nnz), ex["loc"] & 3], rows)
            assert np.array_equal(cv[np.arange(T.nnz), (ex["loc"] >> 2) & 3], ex["t_j"])
        else:
            assert np.array_equal(ex["csr_col"][ex["slot_ik"]], ex["t_k"])


def test_row_range_build_matches_full(oracle_mod):
    """The row-restricted build (used for sampled parity at full size) equals the full build on those rows."""
    pr = I.make_problem("cfg4", n=3)
    full = oracle_mod.OracleTensor(pr.mesh, pr.V, pr.W, pr.form).export()
    r0, r1 = 10, 41
    part = oracle_mod.OracleTensor(pr.mesh, pr.V, pr.W, pr.form, rows=(r0, r1)).export()
    a, b = full["t_row_ptr"][r0], full["t_row_ptr"][r1]
    assert np.array_equal(part["t_j"], full["t_j"][a:b])
    assert np.array_equal(part["t_k"], full["t_k"][a:b])
    assert np.array_equal(part["t_val"], full["t_val"][a:b])


# ----------------------------------------------------------------------------- F1 pointwise kinds
@pytest.mark.parametrize("dim", [2, 3])
def test_minsurf_linear_field(oracle_mod, dim):
    """u = interpolant of α·x + β ⇒ ∇u_h ≡ α ⇒ a_K = (1 + |α|²)^{-1/2} on every cell."""
    m = jitter(I.mesh_square(5) if dim == 2 else I.mesh_cube(3), 0.2, 8)
    T = oracle_mod.OracleTensor(m, I.space_p1(m), I.space_p0(m), I.FORM_PLAP)
    alpha = np.array([0.7, -1.3, 0.4][:dim])
    w = T.interp(I.INTERP_MINSURF_P0, 0.0, m.coords @ alpha + 0.25)
    assert np.abs(w - 1.0 / np.sqrt(1.0 + alpha @ alpha)).max() < 1e-15


@pytest.mark.parametrize("dim", [2, 3])
def test_minsurf_egfem_p0_equals_sga(oracle_mod, dim):
    """a(∇u_h) is constant per cell for P1 u_h, so EGFEM-P0 reproduces the SGA
    minimal-surface residual (tensor-free brute force)."""
    m = jitter(I.mesh_square(5) if dim == 2 else I.mesh_cube(2), 0.2, 11)
    T = oracle_mod.OracleTensor(m, I.space_p1(m), I.space_p0(m), I.FORM_PLAP)
    u = np.random.default_rng(12).standard_normal(m.n_vertices)
    r = T.apply(u, T.interp(I.INTERP_MINSURF_P0, 0.0, u))
    assert rel_l2(r, brute.sga_minsurf(m, u)) < 1e-13


@pytest.mark.parametrize("wfam", ["P1", "P0"])
def test_reciprocal_tensor_free(oracle_mod, wfam):
    """M_c̃:(u⊗c̃) with c̃ = 1/(k+u) interpolated onto W equals ∫ φ_i u_h c̃_h
    integrated exactly without the tensor (W = P1: nodal GFEM; W = P0: centroid value)."""
    m = jitter(I.mesh_square(4), 0.2, 13)
    V = I.space_p1(m)
    W = V if wfam == "P1" else I.space_p0(m)
    T = oracle_mod.OracleTensor(m, V, W, I.FORM_MASS3)
    u = 0.5 + np.random.default_rng(14).uniform(0.0, 1.0, V.n_dofs)
    k = 1.0
    r = T.apply(u, T.interp(I.INTERP_RECIPROCAL, k, u))
    assert rel_l2(r, brute.tensor_free_reciprocal(m, u, k, wfam)) < 1e-13


def test_reciprocal_closed_forms(oracle_mod):
    """Constant u = c ⇒ c̃ ≡ 1/(k+c) at the nodes; linear u ⇒ c̃_K = 1/(k + u(x̄_K)) at the centroid
    x̄_K = mean of the cell's vertices (u_h is exact for linear u)."""
    m = jitter(I.mesh_square(4), 0.2, 15)
    V = I.space_p1(m)
    T1 = oracle_mod.OracleTensor(m, V, V, I.FORM_MASS3)
    assert np.abs(T1.interp(I.INTERP_RECIPROCAL, 2.0, np.full(V.n_dofs, 0.5)) - 0.4).max() < 1e-16
    T0 = oracle_mod.OracleTensor(m, V, I.space_p0(m), I.FORM_MASS3)
    alpha = np.array([0.3, -0.2])
    u = m.coords @ alpha + 1.0
    xc = m.coords[m.cells].mean(axis=1)
    w = T0.interp(I.INTERP_RECIPROCAL, 1.0, u)
    assert np.abs(w - 1.0 / (1.0 + xc @ alpha + 1.0)).max() < 1e-15


@pytest.mark.parametrize("case", ["minsurf2d", "minsurf3d", "biochem_p1", "biochem_p0"])
def test_f1_newton_vs_finite_differences(oracle_mod, case):
    """J = T·w + (T·₂u)·D_u w for the F1 kinds equals central differences of r(u) = T:(u⊗w(u));
    the minimal-surface Newton matrix is symmetric (like p-Laplace)."""
    pr = I.make_problem(case, n={"minsurf2d": 4, "minsurf3d": 2, "biochem_p1": 3, "biochem_p0": 3}[case])
    m = jitter(pr.mesh, 0.15, 2)
    T = oracle_mod.OracleTensor(m, pr.V, pr.W, pr.form)
    u = pr.u
    w = T.interp(pr.interp, pr.p, u)
    J = _csr_dense(T, T.jacobian(I.JAC_NEWTON, pr.interp, pr.p, u, w))
    Jfd = _fd_jacobian(T, pr.interp, pr.p, u, 1e-5)
    assert rel_l2(J, Jfd) < 1e-8
    if pr.interp == I.INTERP_MINSURF_P0:
        assert rel_l2(J, J.T) < 1e-14


# ----------------------------------------------------------------------------- F2 quadrature-embedded W = I_k
# Reference rules typed here from the literature (Strang–Fix 3-point, Dunavant 6-point degree 4,
# the 4-point tetrahedral degree-2 rule), independent of the oracle's own tables.
RULE_3 = ([2 / 3, 1 / 6, 1 / 6, 1 / 6, 2 / 3, 1 / 6, 1 / 6, 1 / 6, 2 / 3], [1 / 3] * 3)
_A6, _B6 = 0.445948490915965, 0.091576213509771
RULE_6 = ([1 - 2 * _A6, _A6, _A6, _A6, 1 - 2 * _A6, _A6, _A6, _A6, 1 - 2 * _A6,
           1 - 2 * _B6, _B6, _B6, _B6, 1 - 2 * _B6, _B6, _B6, _B6, 1 - 2 * _B6],
          [0.223381589678011] * 3 + [0.109951743655322] * 3)


def test_table1_i4_space_size(oracle_mod):
    """PAPER.md Table 1: EGFEM (I4) has 4225 + 6·8192 = 53377 unknowns on the 64×64 mesh (N_f = N_q·N_el, L139)."""
    m = I.mesh_square(64)
    assert I.space_p1(m).n_dofs + I.space_quad(m, 6).n_dofs == 53377


@pytest.mark.parametrize("case", ["square_i4", "recip_i2"])
def test_case3_equivalence_with_sga_rule(oracle_mod, case):
    """Case 3: with W = I_k and w = f(u_h) at the rule's points, T:(u⊗w)
    reproduces the SGA term ∫ φ_i u f(u) evaluated with that same rule, to rounding."""
    m = jitter(I.mesh_square(4), 0.2, 21)
    V = I.space_p1(m)
    rule, nq, kind, k, f = {"square_i4": (RULE_6, 6, I.INTERP_SQUARE, 0.0, lambda x: x * x),
                            "recip_i2": (RULE_3, 3, I.INTERP_RECIPROCAL, 1.0, lambda x: 1.0 / (1.0 + x))}[case]
    T = oracle_mod.OracleTensor(m, V, I.space_quad(m, nq), I.FORM_MASS3)
    assert T.n_f == nq * m.n_cells
    u = 0.5 + np.random.default_rng(22).uniform(0.0, 1.0, V.n_dofs)
    r = T.apply(u, T.interp(kind, k, u))
    assert rel_l2(r, brute.sga_rule_mass(m, u, f, *rule)) < 1e-13


def test_i4_quadratic_is_exact(oracle_mod):
    """§5.1 (Table 1 'EGFEM (I4)'): the 6-point rule is exact to degree 4, so
    M:(u⊗w) with w = u_h² at its points equals the exact integral ∫ φ_i u_h³ of the SGA."""
    m = jitter(I.mesh_square(3), 0.2, 23)
    V = I.space_p1(m)
    T = oracle_mod.OracleTensor(m, V, I.space_quad(m, 6), I.FORM_MASS3)
    u = np.random.default_rng(24).standard_normal(V.n_dofs)
    r = T.apply(u, T.interp(I.INTERP_SQUARE, 0.0, u))
    assert rel_l2(r, brute.sga_cubic_mass(m, u)) < 1e-13


@pytest.mark.parametrize("dim,nq", [(2, 1), (2, 3), (3, 4)])
def test_plap_quad_equals_p0(oracle_mod, dim, nq):
    """PAPER.md L148/L616 (reading C20): I_1 and P0 give the same p-Laplace tensor values; for any
    rule (weights summing to 1) the P1 gradient is constant per cell, so r(I_k) = r(P0)."""
    m = jitter(I.mesh_square(4) if dim == 2 else I.mesh_cube(2), 0.2, 25)
    V = I.space_p1(m)
    Tq = oracle_mod.OracleTensor(m, V, I.space_quad(m, nq), I.FORM_PLAP)
    T0 = oracle_mod.OracleTensor(m, V, I.space_p0(m), I.FORM_PLAP)
    u = np.random.default_rng(26).standard_normal(V.n_dofs)
    p = 3.0
    rq = Tq.apply(u, Tq.interp(I.INTERP_GRADPOW_P0, p, u))
    r0 = T0.apply(u, T0.interp(I.INTERP_GRADPOW_P0, p, u))
    assert rel_l2(rq, r0) < 1e-14
    if nq == 1:
        assert np.abs(Tq.export()["t_val"] - T0.export()["t_val"]).max() < 1e-16


@pytest.mark.parametrize("case", ["quadratic_i4", "biochem_i2", "plap_i1", "plap3d_i2"])
def test_f2_newton_vs_finite_differences(oracle_mod, case):
    """J = T·w + (T·₂u)·D_u w with w at the quadrature points equals central differences of r(u)."""
    pr = I.make_problem(case, n={"quadratic_i4": 3, "biochem_i2": 3, "plap_i1": 4, "plap3d_i2": 2}[case])
    m = jitter(pr.mesh, 0.15, 2)
    T = oracle_mod.OracleTensor(m, pr.V, pr.W, pr.form)
    u = pr.u
    w = T.interp(pr.interp, pr.p, u)
    J = _csr_dense(T, T.jacobian(I.JAC_NEWTON, pr.interp, pr.p, u, w))
    Jfd = _fd_jacobian(T, pr.interp, pr.p, u, 1e-5)
    assert rel_l2(J, Jfd) < (1e-6 if pr.form == I.FORM_PLAP else 1e-8)


# ----------------------------------------------------------------------------- F3 bilinear GFEM forms
@pytest.mark.parametrize("form,ops", [(I.FORM_MASS3, ("v", "v")), (I.FORM_CONV_I, ("dxdy", "v"))])
def test_bilinear_matches_exact_and_pou(oracle_mod, form, ops):
    """F3: the oracle's bilinear M^c / N^f equals the exactly
    integrated matrix (brute force) and the u-slot contraction of the trilinear tensor with ones
    (partition of unity Σ_j φ_j = 1)."""
    m = jitter(I.mesh_square(4), 0.2, 31)
    V = I.space_p1(m)
    T = oracle_mod.OracleTensor(m, V, V, form)
    b = _csr_dense(T, T.bilinear())
    exact = brute.bilinear_matrix(m, V, *ops)
    assert np.abs(b - exact).max() < 1e-14 * max(1.0, np.abs(exact).max())
    ones = np.ones(T.n_u)
    Bpou = _csr_dense(T, T.jacobian(I.JAC_NEWTON, I.INTERP_IDENTITY, 0.0, ones, np.zeros(T.n_f)))
    assert np.abs(b - Bpou).max() < 1e-14 * max(1.0, np.abs(exact).max())


def test_gfem_burgers_residual_and_jacobian(oracle_mod):
    """GFEM Burgers term −½ N^f f with f = u² at the nodes: r = N^f f; its
    Jacobian N^f diag(2u) equals central differences of r(u) (r is quadratic: exact to rounding)."""
    m = jitter(I.mesh_square(3), 0.2, 32)
    V = I.space_p1(m)
    T = oracle_mod.OracleTensor(m, V, V, I.FORM_CONV_I)
    B = _csr_dense(T, T.bilinear())
    u = np.random.default_rng(33).standard_normal(V.n_dofs)
    r = lambda x: B @ (x * x)
    Jfd = np.column_stack([(r(u + e) - r(u - e)) / 2e-6 for e in np.eye(V.n_dofs) * 1e-6])
    assert rel_l2(B * (2 * u)[None, :], Jfd) < 1e-8


def test_gradient_u_slot_contracts_to_zero(oracle_mod):
    """Σ_j ∇φ_j = 0: forms whose u-slot is differentiated (CONV_J, PLAP) have T·₂1 = 0, so they
    have no bilinear GFEM counterpart of the B = T·₂1 kind (egfem_bilinear_build rejects them)."""
    m = jitter(I.mesh_square(3), 0.2, 34)
    V = I.space_p1(m)
    T = oracle_mod.OracleTensor(m, V, V, I.FORM_CONV_J)
    B = T.jacobian(I.JAC_NEWTON, I.INTERP_IDENTITY, 0.0, np.ones(T.n_u), np.zeros(T.n_f))
    assert np.abs(B).max() < 1e-15


@pytest.mark.parametrize("name", ["cfg2", "cfg4", "minsurf2d", "biochem_p0", "quadratic_i4"])
def test_oracle_threads_bitwise(oracle_mod, name):
    """the all-cores oracle timing splits the row / cell loops over OpenMP
    threads, each row still summed alone in its sequential order, so every output is bitwise the
    single-thread result; a cell-range interp equals the whole interp on its cells."""
    pr = I.make_problem(name, n=I.SMALL_N[name] + 2)
    o = oracle_mod.OracleTensor(pr.mesh, pr.V, pr.W, pr.form)
    outs = []
    for nt in (1, 4):
        oracle_mod.set_threads(nt)
        try:
            w = o.interp(pr.interp, pr.p, pr.u)
            outs.append((w, o.apply(pr.u, w), o.jacobian(0, pr.interp, pr.p, pr.u, w),
                         o.jacobian(1, pr.interp, pr.p, pr.u, w)))
        finally:
            oracle_mod.set_threads(1)
    for a, b in zip(*outs):
        assert np.array_equal(a, b)
    w = outs[0][0]
    cell_wise = pr.W.family in (I.P0, I.QUAD) or pr.interp == I.INTERP_P1_TO_P2_SQUARE
    n_items = pr.mesh.n_cells if cell_wise else pr.W.n_dofs
    c0, c1 = n_items // 3, 2 * n_items // 3
    wp = o.interp(pr.interp, pr.p, pr.u, items=(c0, c1))
    if cell_wise:
        dofs = np.asarray(pr.W.cell_dofs)[c0:c1].ravel()
    else:
        dofs = np.arange(c0, c1)
    assert np.array_equal(wp[dofs], w[dofs])
    rest = np.setdiff1d(np.arange(len(w)), dofs)
    assert np.all(wp[rest] == 0)
