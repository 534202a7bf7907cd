"""Launch sequence for ncu: cfg5 batched action (B = 256, node-major), two launches.
usage: python scripts/profile_cfg5.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import egfem_inputs as I
import paper_2005_06193_b200 as eg

pr = I.make_problem("cfg5")
t = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, device=0)
print(eg.egfem_kernel_name(t, 3))
U = torch.tensor(np.ascontiguousarray(pr.u.T), device="cuda")
R = torch.empty_like(U)
for _ in range(2):
    eg.egfem_apply_batched(t, 256, eg.LAYOUT_NODE_MAJOR, U, U, R)
torch.cuda.synchronize()
print("done")
