"""Launch sequence for ncu: cfg4 apply, Picard, Newton, fused (once each, after one warm pass).
usage: python scripts/profile_cfg4_jac.py [f64|f32]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import egfem_inputs as I
import paper_2005_06193_b200 as eg

pr = I.make_problem("cfg4")
f32 = len(sys.argv) > 1 and sys.argv[1] == "f32"
td = torch.float32 if f32 else torch.float64
t = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, dtype=eg.F32 if f32 else eg.F64, device=0)
u = torch.tensor(pr.u, dtype=td, device="cuda")
w = torch.empty(t.n_f, dtype=td, device="cuda")
chain = torch.empty(t.n_f * 4, dtype=td, device="cuda")
r = torch.empty(t.n_u, dtype=td, device="cuda")
J = torch.empty(t.nnz_csr, dtype=td, device="cuda")
# the step's interp: w kept in the packed record only (w = NULL), as bench.py runs it; the separate
# apply / Picard launches read w, copied out of the record by a torch op (not a profiled kernel)
eg.egfem_interp(t, pr.interp, pr.p, u, None, chain)
w.copy_(chain.view(-1, 4)[:, 0])
eg.egfem_apply(t, u, w, r)
eg.egfem_jacobian(t, eg.JAC_PICARD, pr.interp, pr.p, None, w, None, J)
eg.egfem_jacobian(t, eg.JAC_NEWTON, pr.interp, pr.p, u, w, chain, J)
eg.egfem_apply_jacobian(t, eg.JAC_NEWTON, pr.interp, pr.p, u, None, chain, r, J)
torch.cuda.synchronize()
print("done")
