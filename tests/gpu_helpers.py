"""Shared helpers for the -m gpu parity tests (CUDA path through the C ABI vs the CPU oracle)."""
import numpy as np

import egfem_inputs as I

SIX_PT = (0.445948490915965, 0.2233815896780118, 0.091576213509770549, 0.10995174365532154)


def needs_chain(pr):
    """Cell-wise W (P0 or QUAD) kinds carry D_u w as per-DOF chain rows (include/egfem.h)."""
    return pr.W.family in (I.P0, I.QUAD) and pr.interp in (I.INTERP_GRADPOW_P0, I.INTERP_MINSURF_P0,
                                                          I.INTERP_RECIPROCAL, I.INTERP_SQUARE)


def gpu_pass(eg, t, pr, u_np, newton=True, fused=False, dtype=None):
    """interp → apply → jacobian on the GPU for problem `pr`; returns host arrays."""
    import torch
    dev = torch.device(f"cuda:{t.device}")
    td = t.torch_dtype
    u = torch.tensor(u_np, dtype=td, device=dev)
    w = torch.empty(t.n_f, dtype=td, device=dev)
    chain = None
    if needs_chain(pr):
        chain = torch.empty(t.n_f * (pr.mesh.dim + 1), dtype=td, device=dev)
    eg.egfem_interp(t, pr.interp, pr.p, u, w, chain)
    r = torch.empty(t.n_u, dtype=td, device=dev)
    A = torch.empty(t.nnz_csr, dtype=td, device=dev)
    J = torch.empty(t.nnz_csr, dtype=td, device=dev)
    if fused:
        eg.egfem_apply_jacobian(t, eg.JAC_NEWTON if newton else eg.JAC_PICARD, pr.interp, pr.p, u, w, chain, r,
                                J if newton else A)
        if newton:
            eg.egfem_jacobian(t, eg.JAC_PICARD, pr.interp, pr.p, None, w, None, A)
    else:
        eg.egfem_apply(t, u, w, r)
        eg.egfem_jacobian(t, eg.JAC_PICARD, pr.interp, pr.p, None, w, None, A)
        if newton:
            eg.egfem_jacobian(t, eg.JAC_NEWTON, pr.interp, pr.p, u, w, chain, J)
    torch.cuda.synchronize()
    out = dict(w=w.cpu().numpy(), r=r.cpu().numpy(), A=A.cpu().numpy())
    if newton:
        out["J"] = J.cpu().numpy()
    if chain is not None:
        out["chain"] = chain.cpu().numpy()
    return out


def oracle_pass(o, pr, u_np, newton=True):
    w = o.interp(pr.interp, pr.p, u_np)
    out = dict(w=w, r=o.apply(u_np, w), A=o.jacobian(0, pr.interp, pr.p, u_np, w))
    if newton:
        out["J"] = o.jacobian(1, pr.interp, pr.p, u_np, w)
    return out
