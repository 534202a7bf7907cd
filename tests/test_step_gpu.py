"""egfem_step — the single-pass Newton step: interp of the gradient kinds and
the fused apply / Newton Jacobian in one launch.

Parity: w, the packed chain, r and J bitwise equal to egfem_interp + egfem_apply_jacobian (the
two-launch path, itself checked against the oracle at every size in test_gpu_parity.py) and
within FP64_TOL of the oracle; the work-sequence synchronisation is stressed with tiny items and
no lag, across repeated launches (the epoch) and CUDA-graph replays."""
import numpy as np
import pytest

import egfem_inputs as I
from gpu_helpers import oracle_pass
from helpers import rel_l2

pytestmark = pytest.mark.gpu

FP64_TOL = 1e-12


@pytest.fixture(scope="module")
def eg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2005_06193_b200 as m
    return m


@pytest.fixture(autouse=True)
def single_pass(monkeypatch):
    """The single-pass plan is opt-in (EGFEM_STEP=1 when the tensor is built)."""
    monkeypatch.setenv("EGFEM_STEP", "1")


@pytest.fixture(scope="module")
def orc():
    import oracle
    return oracle


def _bufs(t, pr, torch, misalign=False):
    td = t.torch_dtype
    u = torch.tensor(pr.u, dtype=td, device="cuda")
    w = torch.empty(t.n_f, dtype=td, device="cuda")
    nch = t.n_f * (pr.mesh.dim + 1)
    if misalign:  # a chain 16 bytes past a 32-byte boundary (the API asks for 16-byte alignment)
        chain = torch.empty(nch + 4, dtype=td, device="cuda")[2:nch + 2]
    else:
        chain = torch.empty(nch, dtype=td, device="cuda")
    r = torch.empty(t.n_u, dtype=td, device="cuda")
    J = torch.empty(t.nnz_csr, dtype=td, device="cuda")
    return u, w, chain, r, J


def _two_launch(eg, t, pr, torch):
    u, w, chain, r, J = _bufs(t, pr, torch)
    eg.egfem_interp(t, pr.interp, pr.p, u, w, chain)
    eg.egfem_apply_jacobian(t, eg.JAC_NEWTON, pr.interp, pr.p, u, w, chain, r, J)
    torch.cuda.synchronize()
    return dict(w=w.cpu().numpy(), chain=chain.cpu().numpy(), r=r.cpu().numpy(), J=J.cpu().numpy())


def _step(eg, t, pr, torch, reps=1, misalign=False):
    u, w, chain, r, J = _bufs(t, pr, torch, misalign)
    outs = []
    for _ in range(reps):
        for x in (w, chain, r, J):
            x.fill_(float("nan"))
        eg.egfem_step(t, pr.interp, pr.p, u, w, chain, r, J)
        torch.cuda.synchronize()
        outs.append(dict(w=w.cpu().numpy(), chain=chain.cpu().numpy(), r=r.cpu().numpy(), J=J.cpu().numpy()))
    return outs


def _same(a, b):
    for key in ("w", "chain", "r", "J"):
        assert np.array_equal(a[key], b[key]), key


@pytest.mark.parametrize("name,n", [("cfg4", 6), ("cfg4", 10), ("cfg3", None), ("minsurf2d", None),
                                    ("minsurf3d", None)])
def test_step_single_pass_small(eg, orc, name, n):
    import torch
    pr = I.make_problem(name, n=n or I.SMALL_N[name])
    t = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, device=0)
    assert eg.egfem_kernel_name(t, 4, eg.JAC_NEWTON, pr.interp, pr.p).startswith("k_step")
    ref = _two_launch(eg, t, pr, torch)
    for out in _step(eg, t, pr, torch, reps=3):
        _same(out, ref)
    o = orc.OracleTensor(pr.mesh, pr.V, pr.W, pr.form)
    oref = oracle_pass(o, pr, pr.u)
    for key in ("w", "r", "J"):
        assert rel_l2(ref[key], oref[key]) <= FP64_TOL, key


@pytest.mark.parametrize("ci,ri,lag", [(1, 16, 0), (2, 16, 1), (16, 64, 0), (4, 32, 100000)])
def test_step_sync_stress(eg, monkeypatch, ci, ri, lag):
    """Tiny items and no lag: row items wait on in-flight interp items all the time."""
    import torch
    monkeypatch.setenv("EGFEM_STEP_CI", str(ci))
    monkeypatch.setenv("EGFEM_STEP_RI", str(ri))
    monkeypatch.setenv("EGFEM_STEP_LAG", str(lag))
    pr = I.make_problem("cfg4", n=24)
    t = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, device=0)
    ref = _two_launch(eg, t, pr, torch)
    for out in _step(eg, t, pr, torch, reps=4):
        _same(out, ref)


def test_step_graph_replay(eg):
    import torch
    pr = I.make_problem("cfg4", n=20)
    t = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, device=0)
    ref = _two_launch(eg, t, pr, torch)
    u, w, chain, r, J = _bufs(t, pr, torch)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        eg.egfem_step(t, pr.interp, pr.p, u, w, chain, r, J, s)  # eager warm-up on the capture stream
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        eg.egfem_step(t, pr.interp, pr.p, u, w, chain, r, J, torch.cuda.current_stream())
    for _ in range(3):
        for x in (w, chain, r, J):
            x.zero_()
        g.replay()
        torch.cuda.synchronize()
        _same(dict(w=w.cpu().numpy(), chain=chain.cpu().numpy(), r=r.cpu().numpy(), J=J.cpu().numpy()), ref)


@pytest.mark.parametrize("dtype", [0, 1])
def test_step_full_size_cfg4(eg, dtype):
    """BASELINE cfg4 (12.58M cells, 201M nonzeros) in the bench's launch configuration."""
    import torch
    pr = I.make_problem("cfg4")
    t = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, dtype=dtype, device=0)
    assert eg.egfem_kernel_name(t, 4, eg.JAC_NEWTON, pr.interp, pr.p).startswith("k_step")
    ref = _two_launch(eg, t, pr, torch)
    outs = _step(eg, t, pr, torch, reps=2)
    for out in outs:
        _same(out, ref)
    del t
    torch.cuda.empty_cache()


@pytest.mark.parametrize("name", ["plap3d_i2", "biochem_p0", "cfg4"])
def test_step_two_launch_fallback(eg, name):
    """Tensors / kinds / a misaligned chain outside the single-pass kernel: the two launches."""
    import torch
    pr = I.make_problem(name, n=I.SMALL_N[name])
    t = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, device=0)
    misalign = name == "cfg4"
    if not misalign:
        assert not eg.egfem_kernel_name(t, 4, eg.JAC_NEWTON, pr.interp, pr.p).startswith("k_step")
    ref = _two_launch(eg, t, pr, torch)
    c0 = eg.launch_count()
    out = _step(eg, t, pr, torch, misalign=misalign)[0]
    assert eg.launch_count() - c0 == 2
    _same(out, ref)


def test_step_default_is_two_launches(eg, monkeypatch):
    import torch
    monkeypatch.delenv("EGFEM_STEP")
    pr = I.make_problem("cfg4", n=8)
    t = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, device=0)
    assert eg.egfem_kernel_name(t, 4, eg.JAC_NEWTON, pr.interp, pr.p).startswith("k_interp_* + k_cell")
    ref = _two_launch(eg, t, pr, torch)
    c0 = eg.launch_count()
    _same(_step(eg, t, pr, torch)[0], ref)
    assert eg.launch_count() - c0 == 2


def test_step_validation(eg):
    import torch
    pr = I.make_problem("cfg4", n=4)
    t = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, device=0)
    u, w, chain, r, J = _bufs(t, pr, torch)
    with pytest.raises(eg.EgfemError):
        eg.egfem_step(t, pr.interp, pr.p, u, w, None, r, J)  # Newton needs the chain
    with pytest.raises(eg.EgfemError):
        eg.egfem_step(t, pr.interp, 1.0, u, w, chain, r, J)  # GRADPOW needs p > 1
