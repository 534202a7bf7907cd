"""Geometry classes of the 3D interp (egfem_build.cu make_geo_classes, egfem_interp.cuh
interp_cells_geo): on a mesh made of translated copies of a few cells, step (1) of the gradient
kinds (PAPER.md L165–169, L582 / L605) reads each cell's (cofactors, 1/det) from its class
instead of gathering its vertex coordinates.  Both paths form the same numbers with the same
explicit roundings, so w and the packed Newton record are bitwise those of the gathering kernel
(EGFEM_GEOM_CLASSES=0), which test_gpu_parity.py checks against the oracle; here also against
the oracle directly.  Meshes without few classes (jittered vertices) keep the gathering kernel."""
import numpy as np
import pytest

import egfem_inputs as I
from helpers import rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2005_06193_b200 as m
    return m


def _interp(eg, t, pr, kind, p):
    import torch
    td = t.torch_dtype
    u = torch.tensor(pr.u, dtype=td, device="cuda")
    w = torch.empty(t.n_f, dtype=td, device="cuda")
    chain = torch.empty(t.n_f * 4, dtype=td, device="cuda")
    eg.egfem_interp(t, kind, p, u, w, chain)
    # row sub-ranges (the N > 1 interior / boundary phases) on the same buffers
    w2 = torch.full_like(w, float("nan"))
    c2 = torch.full_like(chain, float("nan"))
    n = t.n_cells
    for lo, hi in ((0, n // 3), (n // 3, n - 5), (n - 5, n)):
        eg.egfem_interp_range(t, kind, p, u, w2, c2, lo, hi)
    torch.cuda.synchronize()
    assert torch.equal(w, w2) and torch.equal(chain, c2)
    return w.cpu().numpy(), chain.cpu().numpy()


@pytest.mark.parametrize("n", [4, 32, 128])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("kind", ["gradpow", "minsurf"])
def test_geo_classes_bitwise(eg, monkeypatch, n, dtype, kind):
    """cfg4's mesh (n = 128 is the bench size): classes on, bitwise the gathering kernel."""
    pr = I.make_problem("cfg4", n=n)
    k, p = (I.INTERP_GRADPOW_P0, pr.p) if kind == "gradpow" else (I.INTERP_MINSURF_P0, 0.0)
    dt = eg.F64 if dtype == "f64" else eg.F32
    out = []
    for env in ("1", "0"):
        monkeypatch.setenv("EGFEM_GEOM_CLASSES", env)
        t = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, dtype=dt, device=0)
        name = eg.egfem_kernel_name(t, 5, eg.JAC_NEWTON, k, p)
        assert ("geo" in name) == (env == "1"), name
        if "geo" in name:
            assert "6 geometry classes" in name  # the six tetrahedra of a cube, translated
        out.append(_interp(eg, t, pr, k, p))
        del t
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1], out[1][1])


def test_geo_classes_vs_oracle(eg):
    """The class path (fp32 handle: fp64 geometry, fp32 outputs) against the oracle's interp at
    a small size, p = 3, 4, 2.5 and the minimal surface, at the fp32 tolerance of SURVEY §8.0."""
    import oracle
    pr = I.make_problem("cfg4", n=8)  # 1/8 exact: translated cells have bitwise equal edge vectors
    t = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, dtype=eg.F32, device=0)
    assert "geo" in eg.egfem_kernel_name(t, 5, eg.JAC_NEWTON, I.INTERP_GRADPOW_P0, 3.0)
    o = oracle.OracleTensor(pr.mesh, pr.V, pr.W, pr.form)
    for p in (3.0, 4.0, 2.5):
        w, c = _interp(eg, t, pr, I.INTERP_GRADPOW_P0, p)
        assert rel_l2(w, o.interp(I.INTERP_GRADPOW_P0, p, pr.u)) <= 2e-5
    w, _ = _interp(eg, t, pr, I.INTERP_MINSURF_P0, 0.0)
    assert rel_l2(w, o.interp(I.INTERP_MINSURF_P0, 0.0, pr.u)) <= 2e-5


def test_geo_classes_absent_on_jittered_mesh(eg):
    """Jittered interior vertices (and n = 6: 1/6 is not a double, so translated cells differ in
    the last bits): more than 32 distinct cells, so no table (gathering kernel)."""
    pr = I.make_problem("cfg4", n=6)
    rng = np.random.default_rng(3)
    x = pr.mesh.coords.copy()
    inner = np.all((x > 1e-12) & (x < 1 - 1e-12), axis=1)
    x[inner] += 0.2 / 6 * rng.uniform(-1, 1, (inner.sum(), 3))
    m = I.Mesh(3, x, pr.mesh.cells)
    for mesh in (m, pr.mesh):
        t = eg.egfem_tensor_build(mesh, pr.V, pr.W, pr.form, dtype=eg.F32, device=0)
        assert eg.egfem_kernel_name(t, 5, eg.JAC_NEWTON, I.INTERP_GRADPOW_P0, 3.0).startswith("k_interp_gradpow (")
