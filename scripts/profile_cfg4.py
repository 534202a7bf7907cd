"""Launch sequence for ncu: cfg4 interp, apply, Newton Jacobian, fused (each twice)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import egfem_inputs as I
import paper_2005_06193_b200 as eg

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
dt = eg.F64 if (len(sys.argv) < 3 or sys.argv[2] == "f64") else eg.F32
pr = I.make_problem(name, batch=1)
t = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, dtype=dt, device=0)
td = t.torch_dtype
u = torch.tensor(pr.u if not pr.batch else pr.u[0], dtype=td, device="cuda")
w = torch.empty(t.n_f, dtype=td, device="cuda")
gp = pr.interp == I.INTERP_GRADPOW_P0
chain = torch.empty(t.n_f * (pr.mesh.dim + 1), dtype=td, device="cuda") if gp else None
r = torch.empty(t.n_u, dtype=td, device="cuda")
J = torch.empty(t.nnz_csr, dtype=td, device="cuda")
for _ in range(2):
    eg.egfem_interp(t, pr.interp, pr.p, u, w, chain)
    eg.egfem_apply(t, u, w, r)
    eg.egfem_jacobian(t, eg.JAC_NEWTON, pr.interp, pr.p, u, w, chain, J)
    eg.egfem_apply_jacobian(t, eg.JAC_NEWTON, pr.interp, pr.p, u, w, chain, r, J)
torch.cuda.synchronize()
print("done", t.nnz)
