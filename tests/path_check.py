"""Run the hot path through a non-default kernel path and check it against the oracle.

EGFEM_PATH=tile  -> the TMA-pipelined tile kernel (general path for rows > 256 nonzeros)
EGFEM_PATH=rows  -> the canonical-CSF segmented row kernel for every tensor (P0 W too)
EGFEM_BATCHED=csf -> the CSF tile kernel for the batched action instead of the dense blocks
Invoked by test_gpu_parity.py::test_kernel_paths in a subprocess (the switches are read once)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np  # noqa: E402

import egfem_inputs as I  # noqa: E402
import oracle  # noqa: E402
import paper_2005_06193_b200 as eg  # noqa: E402
from gpu_helpers import gpu_pass, oracle_pass  # noqa: E402
from helpers import rel_l2  # noqa: E402

worst = 0.0
for name in ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5"):
    pr = I.make_problem(name, n=I.SMALL_N[name], batch=1)
    u = pr.u[0] if pr.batch else pr.u
    t = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, device=0)
    o = oracle.OracleTensor(pr.mesh, pr.V, pr.W, pr.form)
    ref = oracle_pass(o, pr, u)
    for fused in (False, True):
        g = gpu_pass(eg, t, pr, u, fused=fused)
        for key in ("w", "r", "A", "J"):
            e = rel_l2(g[key], ref[key])
            worst = max(worst, e)
            assert e <= 1e-12, (name, key, e)
# batched action (cfg5 form, W = V): B pairs against the single-pair oracle
import torch  # noqa: E402

pr = I.make_problem("cfg5", n=I.SMALL_N["cfg5"], batch=70)
t = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, device=0)
o = oracle.OracleTensor(pr.mesh, pr.V, pr.W, pr.form)
U = torch.tensor(np.ascontiguousarray(pr.u.T), dtype=torch.float64, device="cuda")  # node-major
R = torch.empty_like(U)
eg.egfem_apply_batched(t, pr.batch, eg.LAYOUT_NODE_MAJOR, U, U, R)
Rh = R.cpu().numpy()
for p in range(pr.batch):
    e = rel_l2(Rh[:, p], o.apply(pr.u[p], pr.u[p]))
    worst = max(worst, e)
    assert e <= 1e-12, ("batched", p, e)
print("path ok", os.environ.get("EGFEM_PATH"), os.environ.get("EGFEM_BATCHED"), worst)
