"""Time the row kernels (apply / Picard / Newton / fused) on one config; env selects the variant.

usage: EGFEM_ROWS_CFG=G,NCH python scripts/rows_sweep.py cfg4 [f64|f32]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import egfem_inputs as I
import paper_2005_06193_b200 as eg

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
dt = eg.F32 if (len(sys.argv) > 2 and sys.argv[2] == "f32") else eg.F64
td = torch.float32 if dt == eg.F32 else torch.float64
pr = I.make_problem(name)
t = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, dtype=dt, device=0)
u = torch.tensor(pr.u, dtype=td, device="cuda")
w = torch.empty(t.n_f, dtype=td, device="cuda")
gp = pr.interp == I.INTERP_GRADPOW_P0
chain = torch.empty(t.n_f * (pr.mesh.dim + 1), dtype=td, device="cuda") if gp else None
r = torch.empty(t.n_u, dtype=td, device="cuda")
J = torch.empty(t.nnz_csr, dtype=td, device="cuda")
eg.egfem_interp(t, pr.interp, pr.p, u, w, chain)


def tm(fn, n=30):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


res = {"cfg": name, "dtype": "f32" if dt == eg.F32 else "f64", "impl": "seg",
       "rows_cfg": os.environ.get("EGFEM_ROWS_CFG", "auto")}
res["apply"] = tm(lambda: eg.egfem_apply(t, u, w, r))
res["picard"] = tm(lambda: eg.egfem_jacobian(t, eg.JAC_PICARD, pr.interp, pr.p, None, w, None, J))
res["newton"] = tm(lambda: eg.egfem_jacobian(t, eg.JAC_NEWTON, pr.interp, pr.p, u, w, chain, J))
res["fused"] = tm(lambda: eg.egfem_apply_jacobian(t, eg.JAC_NEWTON, pr.interp, pr.p, u, w, chain, r, J))
res["interp"] = tm(lambda: eg.egfem_interp(t, pr.interp, pr.p, u, w, chain))
if gp:  # w kept in the packed record only (w = NULL), as the bench step runs it
    res["interp_rec"] = tm(lambda: eg.egfem_interp(t, pr.interp, pr.p, u, None, chain))
print(json.dumps(res), flush=True)
