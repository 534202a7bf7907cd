"""Launch sequence for ncu: cfg4 apply, Picard, Newton, fused (once each, after one warm pass)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import egfem_inputs as I
import paper_2005_06193_b200 as eg

pr = I.make_problem("cfg4")
t = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, device=0)
u = torch.tensor(pr.u, device="cuda")
w = torch.empty(t.n_f, dtype=torch.float64, device="cuda")
chain = torch.empty(t.n_f * 4, dtype=torch.float64, device="cuda")
r = torch.empty(t.n_u, dtype=torch.float64, device="cuda")
J = torch.empty(t.nnz_csr, dtype=torch.float64, device="cuda")
eg.egfem_interp(t, pr.interp, pr.p, u, w, chain)
eg.egfem_apply(t, u, w, r)
eg.egfem_jacobian(t, eg.JAC_PICARD, pr.interp, pr.p, None, w, None, J)
eg.egfem_jacobian(t, eg.JAC_NEWTON, pr.interp, pr.p, u, w, chain, J)
eg.egfem_apply_jacobian(t, eg.JAC_NEWTON, pr.interp, pr.p, u, w, chain, r, J)
torch.cuda.synchronize()
print("done")
