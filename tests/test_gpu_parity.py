"""GPU ↔ oracle parity through the C ABI (-m gpu).

Bars (BASELINE.json north_star): integer arrays (pattern, slot and
index maps) bit-exact; fp64 relative L2 ≤ 1e-12; fp32 ≤ 2e-5 against the fp64
oracle on the fp64 inputs (reading C16).  Small cases run every element through
the oracle at sizes that span many tiles plus a ragged last tile; full BASELINE
sizes run whole (cfg1–3, cfg5) or on sampled row blocks the oracle builds row by
row (cfg4: first, middle and last blocks).
"""
import numpy as np
import pytest

import egfem_inputs as I
from gpu_helpers import SIX_PT, gpu_pass, oracle_pass
from helpers import rel_l2

pytestmark = pytest.mark.gpu

FP64_TOL = 1e-12
FP32_TOL = 2e-5
INT_KEYS = ("t_row_ptr", "t_j", "t_k", "csr_row_ptr", "csr_col", "slot_ij")


@pytest.fixture(scope="module")
def eg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    import paper_2005_06193_b200 as eg
    return eg


@pytest.fixture(scope="module")
def orc():
    import oracle
    oracle.build()
    return oracle


def _build_both(eg, orc, pr, dtype=0, rows=None):
    t = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, dtype=dtype, device=0)
    o = orc.OracleTensor(pr.mesh, pr.V, pr.W, pr.form, rows=rows)
    return t, o


def _maps_kw(pr):
    p0 = pr.W.family in (I.P0, I.QUAD)  # cell-wise W: loc map; W = V numbering: slot_ik
    return dict(slot_ik=not p0, loc=p0)


SMALL = [("cfg1", None), ("cfg2", None), ("cfg3", None), ("cfg4", None), ("cfg5", None),
         ("cfg2", 7), ("cfg3", 5), ("cfg4", 3), ("cfg4", 1), ("cfg3", 1), ("cfg1", 1), ("cfg5", 1),
         # SURVEY §8(f) F1 pointwise kinds: minimal surface (P0 W) and biochemical σ/(k+u) (W = P1, P0)
         ("minsurf2d", None), ("minsurf3d", None), ("minsurf3d", 2), ("biochem_p1", None), ("biochem_p0", None),
         # SURVEY §8(f) F2 quadrature-embedded W = I_k (Case 3)
         ("quadratic_i4", None), ("biochem_i2", None), ("plap_i1", None), ("plap3d_i2", None), ("plap3d_i2", 2)]


@pytest.mark.parametrize("name,n", SMALL)
def test_builder_bit_exact_small(eg, orc, name, n):
    """A0: canonical integer arrays memcmp-equal; values within 1e-12 (fp64)."""
    pr = I.make_problem(name, n=n if n else I.SMALL_N[name], batch=1)
    t, o = _build_both(eg, orc, pr)
    assert (t.nnz, t.nnz_csr) == (o.nnz, o.nnz_csr)
    kw = _maps_kw(pr)
    ex, oex = t.export(**kw), o.export(**kw)
    for key in INT_KEYS + tuple(k for k, v in kw.items() if v):
        assert np.array_equal(ex[key], oex[key]), key
    assert rel_l2(ex["t_val"], oex["t_val"]) <= FP64_TOL
    assert np.abs(ex["t_val"] - oex["t_val"]).max() <= 1e-15 * max(1.0, np.abs(oex["t_val"]).max()) * 8


@pytest.mark.parametrize("name,n", SMALL)
@pytest.mark.parametrize("fused", [False, True])
def test_hot_path_small(eg, orc, name, n, fused):
    """A1–A3 on every element: interp, apply, Picard and Newton Jacobians (fp64)."""
    pr = I.make_problem(name, n=n if n else I.SMALL_N[name], batch=1)
    u = pr.u[0] if pr.batch else pr.u
    t, o = _build_both(eg, orc, pr)
    g = gpu_pass(eg, t, pr, u, fused=fused)
    ref = oracle_pass(o, pr, u)
    if pr.interp == I.INTERP_IDENTITY:
        assert np.array_equal(g["w"], ref["w"])  # IDENTITY is a copy: bit-exact
    for key in ("w", "r", "A", "J"):
        assert rel_l2(g[key], ref[key]) <= FP64_TOL, (key, rel_l2(g[key], ref[key]))


def test_fused_equals_separate_bitwise(eg):
    """egfem_apply_jacobian is bitwise identical to egfem_apply + egfem_jacobian; runs are reproducible."""
    for name in ("cfg2", "cfg4"):
        pr = I.make_problem(name, n=I.SMALL_N[name])
        t = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, device=0)
        a = gpu_pass(eg, t, pr, pr.u, fused=False)
        b = gpu_pass(eg, t, pr, pr.u, fused=True)
        c = gpu_pass(eg, t, pr, pr.u, fused=False)
        for key in ("r", "A", "J", "w"):
            assert np.array_equal(a[key], b[key]), key
            assert np.array_equal(a[key], c[key]), key


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg5"])
def test_full_size_whole(eg, orc, name):
    """BASELINE sizes, every element: builder maps bit-exact, hot path within 1e-12."""
    pr = I.make_problem(name, batch=2)
    u = pr.u[0] if pr.batch else pr.u
    t, o = _build_both(eg, orc, pr)
    kw = _maps_kw(pr)
    ex, oex = t.export(**kw), o.export(**kw)
    for key in INT_KEYS + tuple(k for k, v in kw.items() if v):
        assert np.array_equal(ex[key], oex[key]), key
    assert rel_l2(ex["t_val"], oex["t_val"]) <= FP64_TOL
    newton = name != "cfg5"  # cfg5 is action-only (reading C24)
    g = gpu_pass(eg, t, pr, u, newton=newton)
    ref = oracle_pass(o, pr, u, newton=newton)
    for key in ("w", "r", "A") + (("J",) if newton else ()):
        assert rel_l2(g[key], ref[key]) <= FP64_TOL, key


def _row_blocks(n_u, size):
    return [(0, size), (n_u // 2 - size // 2, n_u // 2 + size // 2), (n_u - size, n_u)]


@pytest.mark.parametrize("dtype", [0, 1])
def test_cfg4_full_size_sampled_rows(eg, orc, dtype):
    """cfg4 at BASELINE size in the launch configuration bench.py times: whole w (interp over
    all 12.58M cells) and the first/middle/last row blocks of T, r, A, J vs a row-restricted
    oracle build.  fp32 compares against the fp64 oracle (reading C16)."""
    import torch
    pr = I.make_problem("cfg4")
    t = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, dtype=dtype, device=0)
    assert (t.nnz, t.nnz_csr) == (201326592, 31802497)
    g = gpu_pass(eg, t, pr, pr.u, fused=True)
    # the separate entry points too: egfem_apply (the apply-only kernel) and the separate
    # Newton egfem_jacobian, at full size in the same launch configuration
    gs = gpu_pass(eg, t, pr, pr.u, fused=False)
    ex = t.export(loc=True)
    tol = FP64_TOL if dtype == 0 else FP32_TOL
    o_full = orc.OracleTensor(pr.mesh, pr.V, pr.W, pr.form, rows=(0, 1))
    ow = o_full.interp(pr.interp, pr.p, pr.u)
    assert rel_l2(g["w"], ow) <= tol
    for r0, r1 in _row_blocks(t.n_u, 4000):
        o = orc.OracleTensor(pr.mesh, pr.V, pr.W, pr.form, rows=(r0, r1))
        oex = o.export(loc=True)
        a, b = ex["t_row_ptr"][r0], ex["t_row_ptr"][r1]
        for key in ("t_j", "t_k", "loc"):
            assert np.array_equal(ex[key][a:b], oex[key]), key
        assert np.array_equal(ex["t_row_ptr"][r0:r1 + 1] - a, oex["t_row_ptr"][r0:r1 + 1])
        assert rel_l2(ex["t_val"][a:b], oex["t_val"]) <= (FP64_TOL if dtype == 0 else 1e-7)
        ca, cb = ex["csr_row_ptr"][r0], ex["csr_row_ptr"][r1]
        assert np.array_equal(ex["csr_col"][ca:cb], oex["csr_col"])
        ref_r = o.apply(pr.u, ow)[r0:r1]
        ref_A = o.jacobian(0, pr.interp, pr.p, pr.u, ow)
        ref_J = o.jacobian(1, pr.interp, pr.p, pr.u, ow)
        for gg in (g, gs):
            assert rel_l2(gg["r"][r0:r1], ref_r) <= tol
            assert rel_l2(gg["A"][ca:cb], ref_A) <= tol
            assert rel_l2(gg["J"][ca:cb], ref_J) <= tol
    del t
    torch.cuda.empty_cache()


@pytest.mark.parametrize("name,n", [("cfg4", 6), ("cfg4", 10), ("cfg3", 9), ("cfg2", 17), ("cfg1", 300),
                                    ("biochem_p1", 20), ("minsurf2d", 12), ("minsurf3d", 8), ("plap3d_i2", 5),
                                    ("quadratic_i4", 16)])
def test_fp32_small(eg, orc, name, n):
    """fp32 handles (the fp64 build rounded once) on every single-vector kernel family: cell-major
    P0 (cfg3/cfg4), W = V dense blocks (cfg1/cfg2, RECIPROCAL Newton), MINSURF interp."""
    pr = I.make_problem(name, n=n)
    t, o = _build_both(eg, orc, pr, dtype=1)
    g = gpu_pass(eg, t, pr, pr.u)
    ref = oracle_pass(o, pr, pr.u)
    for key in ("w", "r", "A", "J"):
        assert rel_l2(g[key], ref[key]) <= FP32_TOL, key


@pytest.mark.parametrize("form,kind", [(I.FORM_CONV_J, I.INTERP_IDENTITY), (I.FORM_MASS3, I.INTERP_SQUARE),
                                       (I.FORM_MASS3, I.INTERP_RECIPROCAL), (I.FORM_CONV_I, I.INTERP_IDENTITY)])
def test_wv_3d_wide_stencils(eg, orc, form, kind):
    """W = V on a 3D P1 mesh: stencils up to 15 points take the 16-lane dense single-vector
    kernel; every W = V Newton factor (IDENTITY, SQUARE 2u, RECIPROCAL −1/(k+u)²), fused and
    separate, and a split row range, against the oracle."""
    import torch
    mesh = I.mesh_cube(5)
    V = I.space_p1(mesh)
    u = I.random_vector(V.n_dofs, 11, 0.5, 1.5)
    pr = I.Problem("wv3d", mesh, V, V, form, kind, 1.0, ("f64",), u)
    t, o = _build_both(eg, orc, pr)
    ref = oracle_pass(o, pr, u)
    for fused in (False, True):
        g = gpu_pass(eg, t, pr, u, fused=fused)
        for key in ("w", "r", "A", "J"):
            assert rel_l2(g[key], ref[key]) <= FP64_TOL, (fused, key)
    # two row ranges reproduce the whole-range call bitwise
    ud = torch.tensor(u, device="cuda")
    w = torch.empty(t.n_f, dtype=torch.float64, device="cuda")
    eg.egfem_interp(t, kind, 1.0, ud, w)
    r0, J0 = torch.empty(t.n_u, dtype=torch.float64, device="cuda"), torch.empty(t.nnz_csr, dtype=torch.float64,
                                                                                  device="cuda")
    eg.egfem_apply_jacobian(t, 1, kind, 1.0, ud, w, None, r0, J0)
    r1, J1 = torch.full_like(r0, float("nan")), torch.full_like(J0, float("nan"))
    cut = t.n_u // 3
    eg.egfem_apply_jacobian_rows(t, 1, kind, 1.0, ud, w, None, r1, J1, cut, t.n_u)
    eg.egfem_apply_jacobian_rows(t, 1, kind, 1.0, ud, w, None, r1, J1, 0, cut)
    torch.cuda.synchronize()
    assert torch.equal(r0, r1) and torch.equal(J0, J1)


@pytest.mark.parametrize("wfam", ["p1", "p0"])
@pytest.mark.parametrize("jit", [False, True])
def test_builder_3d_mass3_exact(eg, orc, wfam, jit):
    """A0 in 3D for a degree-3 integrand: the trilinear mass M from the builder's
    14-point rule vs the oracle's collapsed Gauss rule (two independent exact routes): integer
    arrays bit-exact, values within 1e-12, on a structured and a jittered cube."""
    mesh = I.mesh_cube(4)
    if jit:
        rng = np.random.default_rng(31)
        x = mesh.coords.copy()
        inner = np.all((x > 1e-12) & (x < 1 - 1e-12), axis=1)
        x[inner] += 0.2 / 4 * rng.uniform(-1, 1, (inner.sum(), 3))
        mesh = I.Mesh(3, x, mesh.cells)
    V = I.space_p1(mesh)
    W = V if wfam == "p1" else I.space_p0(mesh)
    t = eg.egfem_tensor_build(mesh, V, W, I.FORM_MASS3, dtype=0, device=0)
    o = orc.OracleTensor(mesh, V, W, I.FORM_MASS3)
    ex, oex = t.export(), o.export()
    for key in INT_KEYS:
        assert np.array_equal(ex[key], oex[key]), key
    assert rel_l2(ex["t_val"], oex["t_val"]) <= FP64_TOL


@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("B", [1, 8, 37, 64, 65, 130])
def test_batched_small(eg, orc, layout, B):
    """A2 batched: R_p = T:(U_p ⊗ W_p), NODE_MAJOR and PAIR_MAJOR, B not a multiple of 32."""
    import torch
    pr = I.make_problem("cfg5", n=I.SMALL_N["cfg5"], batch=B)
    t, o = _build_both(eg, orc, pr)
    U = pr.u
    rng = np.random.default_rng(5)
    Wv = U + 0.1 * rng.standard_normal(U.shape)  # w ≠ u to catch slot mix-ups
    R_ref = o.apply_batched(U, Wv)
    if layout == 0:
        Ud = torch.tensor(U.T.copy(), device="cuda").contiguous()
        Wd = torch.tensor(Wv.T.copy(), device="cuda").contiguous()
    else:
        Ud = torch.tensor(U, device="cuda")
        Wd = torch.tensor(Wv, device="cuda")
    R = torch.empty_like(Ud)
    eg.egfem_apply_batched(t, B, layout, Ud, Wd, R)
    Rh = R.cpu().numpy()
    Rh = Rh.T if layout == 0 else Rh
    assert rel_l2(Rh, R_ref) <= FP64_TOL


def test_cfg5_full_size_batched_sampled_pairs(eg, orc):
    """cfg5 at BASELINE size, B = 256 node-major (the bench launch): pairs 0, 77, 255 whole, and
    ALL 256 pairs (every pair chunk of the kernel) on the first / middle / last 3000-row blocks,
    each against a row-restricted oracle build (r is defined row by row)."""
    import torch
    pr = I.make_problem("cfg5")
    t = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, device=0)
    o = orc.OracleTensor(pr.mesh, pr.V, pr.W, pr.form)
    U = torch.tensor(pr.u.T.copy(), device="cuda")
    R = torch.empty_like(U)
    eg.egfem_apply_batched(t, 256, 0, U, U, R)
    Rh = R.cpu().numpy()
    for p in (0, 77, 255):
        assert rel_l2(Rh[:, p], o.apply(pr.u[p], pr.u[p])) <= FP64_TOL
    del o
    for r0, r1 in _row_blocks(t.n_u, 3000):
        ob = orc.OracleTensor(pr.mesh, pr.V, pr.W, pr.form, rows=(r0, r1))
        Rb = ob.apply_batched(pr.u, pr.u)[:, r0:r1]  # (256, rows)
        for p in range(256):
            assert rel_l2(Rh[r0:r1, p], Rb[p]) <= FP64_TOL, (r0, p)


def test_interp_kinds(eg, orc):
    """SQUARE (W = V) and P1_TO_P2_SQUARE (Case 1) interpolation plus their Jacobians."""
    import torch
    m = I.mesh_square(9)
    V, W2 = I.space_p1(m), I.space_p2_square(9)
    u = np.random.default_rng(3).standard_normal(V.n_dofs)
    # P1 -> P2 square with MASS3
    t = eg.egfem_tensor_build(m, V, W2, I.FORM_MASS3, device=0)
    o = orc.OracleTensor(m, V, W2, I.FORM_MASS3)
    ud = torch.tensor(u, device="cuda")
    w = torch.empty(t.n_f, dtype=torch.float64, device="cuda")
    eg.egfem_interp(t, I.INTERP_P1_TO_P2_SQUARE, 0, ud, w)
    ow = o.interp(I.INTERP_P1_TO_P2_SQUARE, 0, u)
    assert rel_l2(w.cpu().numpy(), ow) <= FP64_TOL
    r = torch.empty(t.n_u, dtype=torch.float64, device="cuda")
    eg.egfem_apply(t, ud, w, r)
    assert rel_l2(r.cpu().numpy(), o.apply(u, ow)) <= FP64_TOL
    # SQUARE with W = V
    t = eg.egfem_tensor_build(m, V, V, I.FORM_CONV_J, device=0)
    o = orc.OracleTensor(m, V, V, I.FORM_CONV_J)
    w = torch.empty(t.n_f, dtype=torch.float64, device="cuda")
    eg.egfem_interp(t, I.INTERP_SQUARE, 0, ud, w)
    ow = o.interp(I.INTERP_SQUARE, 0, u)
    assert rel_l2(w.cpu().numpy(), ow) <= FP64_TOL
    J = torch.empty(t.nnz_csr, dtype=torch.float64, device="cuda")
    eg.egfem_jacobian(t, I.JAC_NEWTON, I.INTERP_SQUARE, 0, ud, w, None, J)
    assert rel_l2(J.cpu().numpy(), o.jacobian(1, I.INTERP_SQUARE, 0, u, ow)) <= FP64_TOL


def test_user_quadrature_and_jittered_mesh(eg, orc):
    """Explicit quadrature (the 6-point rule passed in) on an unstructured (jittered) P2 mesh."""
    n = 8
    m = I.mesh_square(n)
    rng = np.random.default_rng(2)
    x = m.coords.copy()
    inner = np.all((x > 1e-12) & (x < 1 - 1e-12), axis=1)
    x[inner] += 0.2 / n * rng.uniform(-1, 1, (inner.sum(), 2))
    m = I.Mesh(2, x, m.cells)
    V = I.space_p2_square(n)
    bary, wq = [], []
    for a, ww in ((SIX_PT[0], SIX_PT[1]), (SIX_PT[2], SIX_PT[3])):
        for pnt in ((1 - 2 * a, a, a), (a, 1 - 2 * a, a), (a, a, 1 - 2 * a)):
            bary.append(pnt)
            wq.append(ww)
    t = eg.egfem_tensor_build(m, V, V, I.FORM_CONV_I, quad=(np.array(bary), np.array(wq)), device=0)
    o = orc.OracleTensor(m, V, V, I.FORM_CONV_I, quad=(np.array(bary), np.array(wq)))
    ex, oex = t.export(), o.export()
    for key in INT_KEYS:
        assert np.array_equal(ex[key], oex[key]), key
    assert rel_l2(ex["t_val"], oex["t_val"]) <= FP64_TOL


def test_from_coo_random_with_duplicates(eg):
    """egfem_tensor_from_coo: arbitrary order, duplicates summed; apply vs a dense einsum."""
    import torch
    rng = np.random.default_rng(11)
    n_u, n_f, nnz = 300, 300, 20000
    i = rng.integers(0, n_u, nnz)
    j = rng.integers(0, n_u, nnz)
    k = rng.integers(0, n_f, nnz)
    v = rng.standard_normal(nnz)
    t = eg.egfem_tensor_from_coo(n_u, n_f, i, j, k, v, device=0)
    D = np.zeros((n_u, n_u, n_f))
    np.add.at(D, (i, j, k), v)
    assert t.nnz == len(set(zip(i.tolist(), j.tolist(), k.tolist())))
    u, w = rng.standard_normal(n_u), rng.standard_normal(n_f)
    ud, wd = torch.tensor(u, device="cuda"), torch.tensor(w, device="cuda")
    r = torch.empty(n_u, dtype=torch.float64, device="cuda")
    eg.egfem_apply(t, ud, wd, r)
    assert rel_l2(r.cpu().numpy(), np.einsum("ijk,j,k->i", D, u, w)) <= FP64_TOL
    A = torch.empty(t.nnz_csr, dtype=torch.float64, device="cuda")
    eg.egfem_jacobian(t, 0, 0, 0, None, wd, None, A)
    ex = t.export()
    Ad = np.zeros((n_u, n_u))
    Ad[np.repeat(np.arange(n_u), np.diff(ex["csr_row_ptr"])), ex["csr_col"]] = A.cpu().numpy()
    assert rel_l2(Ad, np.einsum("ijk,k->ij", D, w)) <= FP64_TOL
    J = torch.empty_like(A)
    with pytest.raises(eg.EgfemError) as e:  # T·₂u leaves the (i,j) pattern of a random tensor
        eg.egfem_jacobian(t, 1, 0, 0, ud, wd, None, J)
    assert e.value.status == 3
    # a tensor whose (i,k) pairs are all fibers: k ∈ {i, j} plus the diagonal (i,i,i)
    k2 = np.where(rng.random(nnz) < 0.5, i, j)
    i2, j2 = np.concatenate([i, np.arange(n_u)]), np.concatenate([j, np.arange(n_u)])
    k2 = np.concatenate([k2, np.arange(n_u)])
    v2 = rng.standard_normal(len(i2))
    t2 = eg.egfem_tensor_from_coo(n_u, n_f, i2, j2, k2, v2, device=0)
    D2 = np.zeros((n_u, n_u, n_f))
    np.add.at(D2, (i2, j2, k2), v2)
    J = torch.empty(t2.nnz_csr, dtype=torch.float64, device="cuda")
    eg.egfem_jacobian(t2, 1, 0, 0, ud, wd, None, J)
    ex2 = t2.export()
    Jd = np.zeros((n_u, n_u))
    Jd[np.repeat(np.arange(n_u), np.diff(ex2["csr_row_ptr"])), ex2["csr_col"]] = J.cpu().numpy()
    assert rel_l2(Jd, np.einsum("ijk,k->ij", D2, w) + np.einsum("ijk,j->ik", D2, u)) <= FP64_TOL


def test_validation_errors(eg):
    """Validation happens before any launch and returns the documented status codes."""
    import torch
    pr = I.make_problem("cfg3", n=4)
    t = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, device=0)
    u = torch.zeros(t.n_u, dtype=torch.float64, device="cuda")
    w = torch.zeros(t.n_f, dtype=torch.float64, device="cuda")
    r = torch.zeros(t.n_u, dtype=torch.float64, device="cuda")
    with pytest.raises(eg.EgfemError) as e:
        eg.egfem_apply(t, u, None, r)
    assert e.value.status == 1
    with pytest.raises(eg.EgfemError) as e:
        eg.egfem_apply(t, u, w.cpu(), r)  # host pointer
    assert e.value.status == 1
    with pytest.raises(eg.EgfemError) as e:
        eg.egfem_interp(t, I.INTERP_IDENTITY, 0, u, w)  # W = P0 ≠ V
    assert e.value.status == 2
    with pytest.raises(eg.EgfemError) as e:
        eg.egfem_interp(t, I.INTERP_GRADPOW_P0, 1.0, u, w)  # p ≤ 1
    assert e.value.status == 1
    with pytest.raises(eg.EgfemError) as e:
        eg.egfem_apply(t, u[1:], w, r)  # misaligned
    assert e.value.status == 1
    # the C ABI itself (no binding checks): device pointers validated once are remembered per
    # handle, host pointers are still rejected after many accepted calls
    import ctypes
    L = eg.lib()
    pu, pw, pr_ = (ctypes.c_void_p(x.data_ptr()) for x in (u, w, r))
    for _ in range(40):
        assert L.egfem_apply(t.h, pu, pw, pr_, None) == 0
    hw = torch.zeros(t.n_f, dtype=torch.float64).pin_memory()
    for _ in range(3):
        assert L.egfem_apply(t.h, pu, ctypes.c_void_p(hw.data_ptr()), pr_, None) == 1
    r2 = torch.full_like(r, 7.0)
    assert L.egfem_apply(t.h, pu, pw, ctypes.c_void_p(r2.data_ptr()), None) == 0
    torch.cuda.synchronize()
    assert torch.equal(r2, r)
    bad = I.Mesh(2, pr.mesh.coords, pr.mesh.cells.copy())
    bad.cells[3, 1] = 10 ** 6
    with pytest.raises(eg.EgfemError) as e:
        eg.egfem_tensor_build(bad, pr.V, pr.W, pr.form, device=0)
    assert e.value.status == 1
    # F1/F2/F3 entry points
    with pytest.raises(eg.EgfemError) as e:
        eg.egfem_interp(t, I.INTERP_RECIPROCAL, float("nan"), u, w)  # k must be finite
    assert e.value.status == 1
    with pytest.raises(eg.EgfemError) as e:
        eg.egfem_interp(t, 6, 0.0, u, w)  # no such kind
    assert e.value.status == 1
    with pytest.raises(eg.EgfemError) as e:  # bilinear form needs W = V
        eg.egfem_bilinear_build(t, torch.zeros(t.nnz_csr, dtype=torch.float64, device="cuda"))
    assert e.value.status == 2
    with pytest.raises(eg.EgfemError) as e:  # x and y alias
        eg.egfem_csr_spmv(t, torch.zeros(t.nnz_csr, dtype=torch.float64, device="cuda"), u, u)
    assert e.value.status == 1
    with pytest.raises(eg.EgfemError) as e:  # QUAD with N_f not a multiple of the cell count
        eg.egfem_tensor_build(pr.mesh, pr.V, I.Space(I.QUAD, pr.mesh.n_cells * 3 + 1, None, None), pr.form, device=0)
    assert e.value.status == 2
    with pytest.raises(eg.EgfemError) as e:  # QUAD W cannot carry a differentiated k-slot
        m1 = I.mesh_interval(4)
        eg.egfem_tensor_build(m1, I.space_p1(m1), I.space_quad(m1, 3), I.FORM_CONV_K, device=0)
    assert e.value.status == 3


@pytest.mark.parametrize("name,nranks", [("cfg4", 2), ("cfg4", 3), ("cfg3", 4), ("cfg2", 3), ("cfg1", 5)])
def test_partition_emulation_bitwise(eg, name, nranks):
    """8(e): the G local problems run one after another on one GPU, each on its u window
    [col_begin, col_end), reproduce the single-GPU r and CSR values bitwise."""
    import torch
    pr = I.make_problem(name, n=I.SMALL_N[name])
    t = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, device=0)
    ref = gpu_pass(eg, t, pr, pr.u)
    r_all, J_all = [], []
    for rank in range(nranks):
        loc, win = eg.egfem_partition(t, nranks, rank)
        ul = torch.tensor(pr.u[win["col_begin"]:win["col_end"]], device="cuda")
        wl = torch.empty(loc.n_f, dtype=torch.float64, device="cuda")
        chain = None
        if pr.interp == I.INTERP_GRADPOW_P0:
            chain = torch.empty(loc.n_f * (pr.mesh.dim + 1), dtype=torch.float64, device="cuda")
        eg.egfem_interp(loc, pr.interp, pr.p, ul, wl, chain)
        r = torch.empty(loc.n_u, dtype=torch.float64, device="cuda")
        J = torch.empty(loc.nnz_csr, dtype=torch.float64, device="cuda")
        eg.egfem_apply_jacobian(loc, 1, pr.interp, pr.p, ul, wl, chain, r, J)
        torch.cuda.synchronize()
        assert loc.n_u == win["row_end"] - win["row_begin"]
        r_all.append(r.cpu().numpy())
        J_all.append(J.cpu().numpy())
    assert np.array_equal(np.concatenate(r_all), ref["r"])
    assert np.array_equal(np.concatenate(J_all), ref["J"])


@pytest.mark.parametrize("name,nranks", [("cfg4", 2), ("cfg4", 3), ("cfg3", 4), ("cfg2", 3), ("cfg1", 5),
                                          ("biochem_p0", 2)])
def test_overlap_split_reads_no_halo(eg, name, nranks):
    """8(e) overlap: with every halo entry of u poisoned (NaN), the interior phase — interp over
    egfem_interior's items, apply+Jacobian over its rows — already yields those rows' r and CSR
    values bitwise equal to the single-GPU pass (so it can run while the halo is in flight);
    after the halo arrives, the boundary phase completes r, J bitwise."""
    import torch
    pr = I.make_problem(name, n=I.SMALL_N[name])
    t = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, device=0)
    ref = gpu_pass(eg, t, pr, pr.u)
    grp = np.asarray(t.export(values=False)["csr_row_ptr"])
    cell_wise = pr.W.family in (I.P0, I.QUAD)
    n_inner = 0
    for rank in range(nranks):
        loc, win = eg.egfem_partition(t, nranks, rank)
        ra, rb, wa, wb = eg.egfem_interior(loc)
        n_items = loc.n_f  # P0: local cells = local W DOFs; W = V: W DOFs
        assert 0 <= ra <= rb <= loc.n_u and 0 <= wa <= wb
        n_inner += rb - ra
        cb, ce, r0, r1 = win["col_begin"], win["col_end"], win["row_begin"], win["row_end"]
        u_true = torch.tensor(pr.u[cb:ce], device="cuda")
        ul = torch.full_like(u_true, float("nan"))
        ul[r0 - cb:r1 - cb] = u_true[r0 - cb:r1 - cb]
        nan = float("nan")
        wl = torch.full((loc.n_f,), nan, dtype=torch.float64, device="cuda")
        chain = None
        if pr.W.family in (I.P0, I.QUAD) and pr.interp != I.INTERP_IDENTITY:
            chain = torch.full((loc.n_f * (pr.mesh.dim + 1),), nan, dtype=torch.float64, device="cuda")
        r = torch.full((loc.n_u,), nan, dtype=torch.float64, device="cuda")
        J = torch.full((loc.nnz_csr,), nan, dtype=torch.float64, device="cuda")
        lrp = np.asarray(loc.export(values=False)["csr_row_ptr"])
        f0 = grp[r0]
        # interior phase on the poisoned window
        eg.egfem_interp_range(loc, pr.interp, pr.p, ul, wl, chain, wa, wb)
        eg.egfem_apply_jacobian_rows(loc, 1, pr.interp, pr.p, ul, wl, chain, r, J, ra, rb)
        torch.cuda.synchronize()
        rr, JJ = r.cpu().numpy(), J.cpu().numpy()
        assert np.array_equal(rr[ra:rb], ref["r"][r0 + ra:r0 + rb])
        assert np.array_equal(JJ[lrp[ra]:lrp[rb]], ref["J"][f0 + lrp[ra]:f0 + lrp[rb]])
        assert np.all(np.isnan(rr[:ra])) and np.all(np.isnan(rr[rb:]))  # nothing else written
        # the halo arrives; boundary phase
        ul.copy_(u_true)
        eg.egfem_interp_range(loc, pr.interp, pr.p, ul, wl, chain, 0, wa)
        eg.egfem_interp_range(loc, pr.interp, pr.p, ul, wl, chain, wb, n_items)
        eg.egfem_apply_jacobian_rows(loc, 1, pr.interp, pr.p, ul, wl, chain, r, J, 0, ra)
        eg.egfem_apply_jacobian_rows(loc, 1, pr.interp, pr.p, ul, wl, chain, r, J, rb, loc.n_u)
        torch.cuda.synchronize()
        assert np.array_equal(r.cpu().numpy(), ref["r"][r0:r1])
        assert np.array_equal(J.cpu().numpy(), ref["J"][f0:grp[r1]])
        with pytest.raises(eg.EgfemError):
            eg.egfem_apply_jacobian_rows(loc, 1, pr.interp, pr.p, ul, wl, chain, r, J, 0, loc.n_u + 1)
        with pytest.raises(eg.EgfemError):
            eg.egfem_interp_range(loc, pr.interp, pr.p, ul, wl, chain, 1, 0)
    assert n_inner > 0
    # a global tensor has no halo: its interior is everything
    n_items = t.n_cells if cell_wise else t.n_f
    assert eg.egfem_interior(t) == (0, t.n_u, 0, n_items)


@pytest.mark.parametrize("name,nranks,w_null", [("cfg4", 3, False), ("cfg4", 3, True), ("cfg2", 2, False),
                                                ("biochem_p0", 2, False)])
def test_split_step_library_bitwise(eg, name, nranks, w_null):
    """dist.split_step — the N>1 bench step through the library — on each rank's local tensor
    with its window already filled (a plan without exchanges) reproduces the single-GPU r and J.
    w_null: the bench's N > 1 step for the packed gradient kinds (w_K only in the Newton record)."""
    import torch

    from paper_2005_06193_b200 import dist as edist
    pr = I.make_problem(name, n=I.SMALL_N[name])
    t = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, device=0)
    ref = gpu_pass(eg, t, pr, pr.u)
    grp = np.asarray(t.export(values=False)["csr_row_ptr"])
    for rank in range(nranks):
        loc, win = eg.egfem_partition(t, nranks, rank)
        wdw = edist.Window(win["row_begin"], win["row_end"], win["col_begin"], win["col_end"])
        plan = edist.HaloPlan(rank, wdw, [], [])
        ul = torch.tensor(pr.u[wdw.col_begin:wdw.col_end], device="cuda")
        wl = torch.empty(loc.n_f, dtype=torch.float64, device="cuda")
        chain = torch.empty(loc.n_f * (pr.mesh.dim + 1), dtype=torch.float64, device="cuda") \
            if pr.W.family in (I.P0, I.QUAD) and pr.interp != I.INTERP_IDENTITY else None
        r = torch.empty(loc.n_u, dtype=torch.float64, device="cuda")
        J = torch.empty(loc.nnz_csr, dtype=torch.float64, device="cuda")
        if w_null:
            assert "k_cell" in eg.egfem_kernel_name(loc, 2, eg.JAC_NEWTON, pr.interp, pr.p)
            wl = None
        edist.split_step(eg, loc, plan, eg.egfem_interior(loc), pr.interp, pr.p, ul, wl, chain, r, J)
        torch.cuda.synchronize()
        assert np.array_equal(r.cpu().numpy(), ref["r"][wdw.row_begin:wdw.row_end])
        assert np.array_equal(J.cpu().numpy(), ref["J"][grp[wdw.row_begin]:grp[wdw.row_end]])


@pytest.mark.parametrize("env", [{"EGFEM_PATH": "tile"}, {"EGFEM_PATH": "rows", "EGFEM_BATCHED": "csf"},
                                 {"EGFEM_CELLS_WORDS": "0"}])
def test_kernel_paths(eg, env):
    """The non-default kernels (TMA tile kernel, canonical-CSF row kernel for P0 W, CSF batched
    kernel) match the oracle: they are the fallbacks for long rows / wide stencils."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    res = subprocess.run([sys.executable, os.path.join(here, "path_check.py")], env=dict(os.environ, **env),
                         capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "path ok" in res.stdout


def test_packed_words_bitwise():
    """The cell-major kernels reading the packed 64-bit row words (default) and the staged
    (K, fiber|position) slices (EGFEM_CELLS_WORDS=0) compute the same sums in the same order:
    apply, Picard, Newton and fused outputs are bitwise equal at full cfg3 / cfg4 size, fp64 and
    fp32 (the staged kernels are oracle-checked)."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    out = []
    for env in ({}, {"EGFEM_CELLS_WORDS": "0"}):
        res = subprocess.run([sys.executable, os.path.join(here, "words_check.py")], env=dict(os.environ, **env),
                             capture_output=True, text=True, timeout=900)
        assert res.returncode == 0, res.stdout + res.stderr
        out.append([ln.split() for ln in res.stdout.splitlines() if ln.startswith("hash")])
    assert len(out[0]) == 4 and len(out[1]) == 4
    for a, b in zip(*out):
        assert a[1:3] == b[1:3] and a[-1] == b[-1], (a, b)
    # the default run took the packed words on the 3D fp64 tensor (the headline), the other the slices
    assert any("packed 64-bit row words" in " ".join(a) for a in out[0] if a[1] == "cfg4")
    assert all("packed" not in " ".join(b) for b in out[1])


@pytest.mark.parametrize("name", ["gfem2d", "biochem_p1"])
def test_bilinear_gfem(eg, orc, name):
    """F3: B = T·₂1 on the CSR pattern equals the oracle's element-by-element ∫ (slot φ_i) η_k
    (PAPER.md L196–203, L402–409); r = B f and J = B·diag(f'(u)) through the C ABI."""
    import torch
    pr = I.make_problem(name, n=I.SMALL_N[name])
    t, o = _build_both(eg, orc, pr)
    Bo = o.bilinear()
    B = torch.empty(t.nnz_csr, dtype=torch.float64, device="cuda")
    eg.egfem_bilinear_build(t, B)
    assert rel_l2(B.cpu().numpy(), Bo) <= FP64_TOL
    u = torch.tensor(pr.u, device="cuda")
    f = torch.empty(t.n_f, dtype=torch.float64, device="cuda")
    eg.egfem_interp(t, pr.interp, pr.p, u, f)
    r = torch.empty(t.n_u, dtype=torch.float64, device="cuda")
    eg.egfem_csr_spmv(t, B, f, r)
    J = torch.empty(t.nnz_csr, dtype=torch.float64, device="cuda")
    eg.egfem_bilinear_jacobian(t, B, pr.interp, pr.p, u, J)
    ex = o.export()
    rows = np.repeat(np.arange(t.n_u), np.diff(ex["csr_row_ptr"]))
    fo = o.interp(pr.interp, pr.p, pr.u)
    r_ref = np.zeros(t.n_u)
    np.add.at(r_ref, rows, Bo * fo[ex["csr_col"]])
    uc = pr.u[ex["csr_col"]]
    dfo = 2 * uc if pr.interp == I.INTERP_SQUARE else -1.0 / (pr.p + uc) ** 2
    assert rel_l2(r.cpu().numpy(), r_ref) <= FP64_TOL
    assert rel_l2(J.cpu().numpy(), Bo * dfo) <= FP64_TOL
    # the gradient u-slot form has no B = T·₂1 counterpart
    pr2 = I.make_problem("cfg2", n=4)
    t2 = eg.egfem_tensor_build(pr2.mesh, pr2.V, pr2.W, pr2.form, device=0)
    with pytest.raises(eg.EgfemError):
        eg.egfem_bilinear_build(t2, torch.empty(t2.nnz_csr, dtype=torch.float64, device="cuda"))


@pytest.mark.parametrize("name", ["cfg4", "cfg3", "cfg2"])
def test_cuda_graph_replay_bitwise(eg, name):
    """The bench step (interp + fused apply/Newton) captured into a CUDA graph and replayed gives
    bitwise the eager results (no host work in the launch path is stream-ordered)."""
    import torch
    pr = I.make_problem(name, n=I.SMALL_N[name])
    t = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, device=0)
    from gpu_helpers import needs_chain
    u = torch.tensor(pr.u, device="cuda")
    w = torch.empty(t.n_f, dtype=torch.float64, device="cuda")
    chain = torch.empty(t.n_f * (pr.mesh.dim + 1), dtype=torch.float64, device="cuda") if needs_chain(pr) else None
    r = torch.empty(t.n_u, dtype=torch.float64, device="cuda")
    J = torch.empty(t.nnz_csr, dtype=torch.float64, device="cuda")

    def step(s):
        eg.egfem_interp(t, pr.interp, pr.p, u, w, chain, s)
        eg.egfem_apply_jacobian(t, eg.JAC_NEWTON, pr.interp, pr.p, u, w, chain, r, J, s)
    step(torch.cuda.current_stream())
    torch.cuda.synchronize()
    r0, J0 = r.clone(), J.clone()
    r.zero_()
    J.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step(torch.cuda.current_stream())
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(r, r0) and torch.equal(J, J0)


@pytest.mark.parametrize("same", [True, False])
def test_batched_groups_graph_and_shards(eg, orc, same):
    """cfg5's batched action through the compiled row groups (fork/join over side streams):
    captured into a CUDA graph and replayed it is bitwise the eager result; batch shards (the
    multi-GPU split of the batch: pairs are independent) run as separate calls
    reproduce the full-batch columns bitwise; U ≠ W (the non-aliased kernel variant) and a batch
    that is not a multiple of the pair chunk (the guarded variant) match the oracle."""
    import torch
    pr = I.make_problem("cfg5", n=24, batch=96)
    t = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, device=0)
    name = eg.egfem_kernel_name(t, 3)
    # U == W launches take the symmetrized patterns (R = Σ_{j≤k} S_ijk u_j u_k, egfem_group.cu)
    assert "egfem_grp" in name and "symmetrized" in name
    o = orc.OracleTensor(pr.mesh, pr.V, pr.W, pr.form)
    U = torch.tensor(np.ascontiguousarray(pr.u.T), device="cuda")
    Wt = U if same else U * 0.5 + 0.25
    R = torch.empty_like(U)
    eg.egfem_apply_batched(t, 96, eg.LAYOUT_NODE_MAJOR, U, Wt, R)
    torch.cuda.synchronize()
    R0 = R.clone()
    Wn = Wt.cpu().numpy().T
    ref = o.apply_batched(pr.u, Wn)
    assert rel_l2(R0.cpu().numpy().T, ref) <= FP64_TOL
    R.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        eg.egfem_apply_batched(t, 96, eg.LAYOUT_NODE_MAJOR, U, Wt, R, torch.cuda.current_stream())
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(R, R0)
    # shards of the batch (as bench.py deals them to ranks) = the full batch's columns, bitwise
    for lo, hi in ((0, 64), (64, 96), (0, 37), (37, 96)):
        Us = U[:, lo:hi].contiguous()
        Ws = Us if same else Wt[:, lo:hi].contiguous()
        Rs = torch.empty_like(Us)
        eg.egfem_apply_batched(t, hi - lo, eg.LAYOUT_NODE_MAJOR, Us, Ws, Rs)
        torch.cuda.synchronize()
        assert torch.equal(Rs, R0[:, lo:hi]), (lo, hi)


@pytest.mark.parametrize("config", ["cfg1", "cfg5"])
def test_bench_line_contract(config):
    """bench.py on the GPU prints one JSON line with the contract's keys: value, roofline (named
    kernel, §8(d) bytes or flops, frac), e2e with its copy bytes, clocks, gpu_launches > 0 and a
    cpu_baseline whose parity against the GPU outputs is within tolerance."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    extra = ["--batch", "64"] if config == "cfg5" else []
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--config", config, "--steps", "3",
                          "--warmup", "3", *extra], capture_output=True, text=True, timeout=900, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "roofline", "e2e", "clocks",
              "gpu_launches", "cpu_baseline", "dtype", "config"):
        assert k in d, k
    assert d["value"] > 0 and d["gpu_launches"] > 0 and d["n_gpus"] == 1
    r = d["roofline"]
    assert r["kernel"] and r["frac"] > 0 and r["peak"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] == 1 and cb["all_cores"]["bitwise_equal_to_1_thread"]
    assert all(v <= 1e-12 for k, v in cb["parity_rel_l2"].items() if k not in ("rows", "pairs")), cb["parity_rel_l2"]


@pytest.mark.parametrize("B", [128, 96])
def test_batched_groups_fp32(eg, orc, B):
    """The compiled row-group kernels in fp32 (float records, float4 / float2 vectors): the batched
    action of the fp32 handle (fp64 build rounded once, reading C16) vs the fp64 oracle ≤ 2e-5,
    for a full (B = 128) and a guarded (B = 96) pair chunking."""
    import torch
    pr = I.make_problem("cfg5", n=20, batch=B)
    t = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, dtype=1, device=0)
    assert "egfem_grp" in eg.egfem_kernel_name(t, 3)
    o = orc.OracleTensor(pr.mesh, pr.V, pr.W, pr.form)
    U = torch.tensor(np.ascontiguousarray(pr.u.T), dtype=torch.float32, device="cuda")
    R = torch.empty_like(U)
    eg.egfem_apply_batched(t, B, eg.LAYOUT_NODE_MAJOR, U, U, R)
    torch.cuda.synchronize()
    ref = o.apply_batched(pr.u, pr.u)
    assert rel_l2(R.double().cpu().numpy().T, ref) <= FP32_TOL


@pytest.mark.parametrize("B,same", [(512, True), (300, False), (1000, True)])
def test_batched_groups_wide_batches(eg, orc, B, same):
    """Batches wider than one CTA's pairs: 512 (4 warps of 128 pairs, full variant), 300 and 1000
    (guarded variant; warps loop over the pair chunks), U aliased to W or not."""
    import torch
    pr = I.make_problem("cfg5", n=10, batch=B)
    t = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, device=0)
    o = orc.OracleTensor(pr.mesh, pr.V, pr.W, pr.form)
    U = torch.tensor(np.ascontiguousarray(pr.u.T), device="cuda")
    Wt = U if same else (0.5 * U - 0.125).contiguous()
    R = torch.empty_like(U)
    eg.egfem_apply_batched(t, B, eg.LAYOUT_NODE_MAJOR, U, Wt, R)
    torch.cuda.synchronize()
    ref = o.apply_batched(pr.u, Wt.cpu().numpy().T)
    assert rel_l2(R.cpu().numpy().T, ref) <= FP64_TOL


@pytest.mark.parametrize("name,n", [("plap3d_i2", 6), ("cfg4", 9), ("quadratic_i4", 20)])
def test_row_subranges_bitwise(eg, name, n):
    """egfem_apply_jacobian_rows over three row ranges (ragged, one of them empty) writes exactly the
    whole-tensor call's values in those rows (the cell-major kernel on a row view; 3D I_2 rows of
    384 nonzeros take the 32-lane configuration)."""
    import torch
    from gpu_helpers import needs_chain
    pr = I.make_problem(name, n=n)
    t = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, device=0)
    assert eg.egfem_kernel_name(t, 2, eg.JAC_NEWTON, pr.interp, pr.p).startswith("k_cell")
    u = torch.tensor(pr.u, device="cuda")
    w = torch.empty(t.n_f, dtype=torch.float64, device="cuda")
    chain = torch.empty(t.n_f * (pr.mesh.dim + 1), dtype=torch.float64, device="cuda") if needs_chain(pr) else None
    eg.egfem_interp(t, pr.interp, pr.p, u, w, chain)
    r = torch.empty(t.n_u, dtype=torch.float64, device="cuda")
    J = torch.empty(t.nnz_csr, dtype=torch.float64, device="cuda")
    eg.egfem_apply_jacobian(t, eg.JAC_NEWTON, pr.interp, pr.p, u, w, chain, r, J)
    r2 = torch.full_like(r, float("nan"))
    J2 = torch.full_like(J, float("nan"))
    cuts = [0, t.n_u // 3 + 1, t.n_u // 3 + 1, t.n_u - 7, t.n_u]
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        eg.egfem_apply_jacobian_rows(t, eg.JAC_NEWTON, pr.interp, pr.p, u, w, chain, r2, J2, lo, hi)
    torch.cuda.synchronize()
    assert torch.equal(r, r2) and torch.equal(J, J2)


@pytest.mark.parametrize("name,f32", [("cfg4", False), ("cfg4", True), ("cfg3", False), ("minsurf3d", False),
                                      ("plap3d_i2", False)])
def test_w_null_packed_record(eg, name, f32):
    """The gradient kinds keep w_K in the packed Newton record (include/egfem.h egfem_interp), so
    w may be NULL: egfem_interp then writes the record only (identical to the call with w, whose
    w equals the record's first entries), and the Newton calls on the cell-major path read w_K
    from the record — r and J bitwise equal to the calls with w.
    Calls that need the w array reject NULL before launching anything."""
    import torch
    pr = I.make_problem(name, n=I.SMALL_N[name])
    t = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, dtype=eg.F32 if f32 else eg.F64, device=0)
    td = t.torch_dtype
    d1 = pr.mesh.dim + 1
    u = torch.tensor(pr.u, dtype=td, device="cuda")
    w = torch.empty(t.n_f, dtype=td, device="cuda")
    ch0, ch1 = (torch.full((t.n_f * d1,), float("nan"), dtype=td, device="cuda") for _ in range(2))
    eg.egfem_interp(t, pr.interp, pr.p, u, w, ch0)
    eg.egfem_interp(t, pr.interp, pr.p, u, None, ch1)
    torch.cuda.synchronize()
    assert torch.equal(ch0, ch1)
    assert torch.equal(ch1.view(-1, d1)[:, 0], w)
    outs = []
    for wx, ch in ((w, ch0), (None, ch1)):
        r = torch.full((t.n_u,), float("nan"), dtype=td, device="cuda")
        J = torch.full((t.nnz_csr,), float("nan"), dtype=td, device="cuda")
        J2 = torch.full((t.nnz_csr,), float("nan"), dtype=td, device="cuda")
        r3 = torch.full((t.n_u,), float("nan"), dtype=td, device="cuda")
        J3 = torch.full((t.nnz_csr,), float("nan"), dtype=td, device="cuda")
        eg.egfem_apply_jacobian(t, eg.JAC_NEWTON, pr.interp, pr.p, u, wx, ch, r, J)
        eg.egfem_jacobian(t, eg.JAC_NEWTON, pr.interp, pr.p, u, wx, ch, J2)
        eg.egfem_step(t, pr.interp, pr.p, u, wx, ch, r3, J3)
        torch.cuda.synchronize()
        outs.append([x.cpu().numpy() for x in (r, J, J2, r3, J3)])
    for a, b in zip(*outs):
        assert np.array_equal(a, b)
    assert np.array_equal(outs[0][1], outs[0][2]) and np.array_equal(outs[0][0], outs[0][3])
    # row sub-ranges (the multi-GPU split step's calls) with w = NULL
    h = t.n_u // 2
    r = torch.full((t.n_u,), float("nan"), dtype=td, device="cuda")
    J = torch.full((t.nnz_csr,), float("nan"), dtype=td, device="cuda")
    eg.egfem_apply_jacobian_rows(t, eg.JAC_NEWTON, pr.interp, pr.p, u, None, ch1, r, J, 0, h)
    eg.egfem_apply_jacobian_rows(t, eg.JAC_NEWTON, pr.interp, pr.p, u, None, ch1, r, J, h, t.n_u)
    torch.cuda.synchronize()
    assert np.array_equal(r.cpu().numpy(), outs[0][0]) and np.array_equal(J.cpu().numpy(), outs[0][1])
    # w is required where it is read: apply alone, Picard, Newton without the record
    r = torch.empty(t.n_u, dtype=td, device="cuda")
    J = torch.empty(t.nnz_csr, dtype=td, device="cuda")
    for call in (lambda: eg.egfem_apply(t, u, None, r),
                 lambda: eg.egfem_jacobian(t, eg.JAC_PICARD, pr.interp, pr.p, None, None, None, J),
                 lambda: eg.egfem_interp(t, pr.interp, pr.p, u, None, None),
                 lambda: eg.egfem_apply_jacobian(t, eg.JAC_NEWTON, pr.interp, pr.p, u, None, None, r, J)):
        with pytest.raises(eg.EgfemError) as ex:
            call()
        assert ex.value.status in (1, 3)  # INVALID_ARGUMENT, UNSUPPORTED


def test_batched_row_partition(eg, orc):
    """The row-partitioned batched action (the SURVEY §8(e) alternative to batch sharding): each
    rank's local tensor (its rows, window columns) builds its own compiled row groups and, on its
    U window, reproduces its rows of the full action (rows are independent) within
    FP64_TOL, aliased (symmetrized patterns) and not."""
    import torch
    pr = I.make_problem("cfg5", n=24, batch=64)
    tg = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, device=0)
    o = orc.OracleTensor(pr.mesh, pr.V, pr.W, pr.form)
    U = torch.tensor(np.ascontiguousarray(pr.u.T), device="cuda")
    Wt = (0.5 * U - 0.125).contiguous()
    ref_same = o.apply_batched(pr.u, pr.u).T
    ref_diff = o.apply_batched(pr.u, Wt.cpu().numpy().T).T
    for N in (2, 3):
        for rank in range(N):
            loc, win = eg.egfem_partition(tg, N, rank)
            assert "egfem_grp" in eg.egfem_kernel_name(loc, 3)
            rb, re_, cb, ce = win["row_begin"], win["row_end"], win["col_begin"], win["col_end"]
            Ul = U[cb:ce].contiguous()
            Wl = Wt[cb:ce].contiguous()
            for Wx, ref in ((Ul, ref_same), (Wl, ref_diff)):
                Rl = torch.empty((re_ - rb, 64), dtype=U.dtype, device="cuda")
                eg.egfem_apply_batched(loc, 64, eg.LAYOUT_NODE_MAJOR, Ul, Wx, Rl)
                torch.cuda.synchronize()
                assert rel_l2(Rl.cpu().numpy(), ref[rb:re_]) <= FP64_TOL, (N, rank)


@pytest.mark.parametrize("name,f32", [("cfg1", False), ("cfg2", False), ("cfg2", True)])
def test_identity_newton_symmetric_blocks(eg, orc, name, f32):
    """The fused IDENTITY Newton with u and w the same array runs the symmetrized dense blocks:
    J_ij = Σ_b (M + Mᵀ)[a][b] u_b (= T·w + T·₂u at w = u) and r_i = ½ Σ_a u_a J_ia
    (= Σ_jk T_ijk u_j u_k, L183) — the same values as the call with a separate w, within the
    tolerance against the oracle."""
    import torch
    pr = I.make_problem(name, n=I.SMALL_N[name])
    t = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, dtype=eg.F32 if f32 else eg.F64, device=0)
    o = orc.OracleTensor(pr.mesh, pr.V, pr.W, pr.form)
    ref = oracle_pass(o, pr, pr.u)
    td = t.torch_dtype
    u = torch.tensor(pr.u, dtype=td, device="cuda")
    w = u.clone()
    tol = FP32_TOL if f32 else FP64_TOL
    outs = []
    for wx in (u, w):  # aliased: symmetrized blocks; separate: the plain blocks + reduce-scatter
        r = torch.empty(t.n_u, dtype=td, device="cuda")
        J = torch.empty(t.nnz_csr, dtype=td, device="cuda")
        eg.egfem_apply_jacobian(t, eg.JAC_NEWTON, eg.INTERP_IDENTITY, 0.0, u, wx, None, r, J)
        torch.cuda.synchronize()
        outs.append((r.double().cpu().numpy(), J.double().cpu().numpy()))
        assert rel_l2(outs[-1][0], ref["r"]) <= tol and rel_l2(outs[-1][1], ref["J"]) <= tol
    assert rel_l2(outs[0][0], outs[1][0]) <= tol and rel_l2(outs[0][1], outs[1][1]) <= tol
