"""Small hot-path pass for compute-sanitizer runs: python scripts/debug_small.py cfg3 [n]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import egfem_inputs as I
import paper_2005_06193_b200 as eg

name = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else I.SMALL_N[name]
pr = I.make_problem(name, n=n, batch=1)
t = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, device=0)
torch.cuda.synchronize()
print("built", t.n_u, t.nnz, flush=True)
u = torch.tensor(pr.u if not pr.batch else pr.u[0], dtype=torch.float64, device="cuda")
w = torch.empty(t.n_f, dtype=torch.float64, device="cuda")
gp = pr.interp == I.INTERP_GRADPOW_P0
chain = torch.empty(t.n_f * (pr.mesh.dim + 1), dtype=torch.float64, device="cuda") if gp else None
r = torch.empty(t.n_u, dtype=torch.float64, device="cuda")
J = torch.empty(t.nnz_csr, dtype=torch.float64, device="cuda")
eg.egfem_interp(t, pr.interp, pr.p, u, w, chain)
torch.cuda.synchronize()
print("interp ok", flush=True)
eg.egfem_apply(t, u, w, r)
torch.cuda.synchronize()
print("apply ok", flush=True)
eg.egfem_jacobian(t, eg.JAC_PICARD, pr.interp, pr.p, None, w, None, J)
torch.cuda.synchronize()
print("picard ok", flush=True)
eg.egfem_jacobian(t, eg.JAC_NEWTON, pr.interp, pr.p, u, w, chain, J)
torch.cuda.synchronize()
print("newton ok", flush=True)
