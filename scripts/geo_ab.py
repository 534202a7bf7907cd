"""A/B of the 3D interp on cfg4: geometry classes (default) vs the gathering
kernel (EGFEM_GEOM_CLASSES=0); CUDA events, 50 launches each after warm-up, alternated 3 times.
profiles/r2_geo_ab_v1.json also has the fp64 class kernel (since dispatched for fp32 only) and the
table read through L1 instead of shared memory ("geo_smem" there = the kept variant)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import egfem_inputs as I
import paper_2005_06193_b200 as eg

pr = I.make_problem("cfg4")
res = {}
for dt, td in ((eg.F64, torch.float64), (eg.F32, torch.float32)):
    ts = {}
    for env in ("1", "0"):
        os.environ["EGFEM_GEOM_CLASSES"] = env
        ts[env] = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, dtype=dt, device=0)
    u = torch.tensor(pr.u, dtype=td, device="cuda")
    chain = torch.empty(ts["1"].n_f * 4, dtype=td, device="cuda")
    s = torch.cuda.current_stream()
    for rep in range(3):
        for env0 in ("1", "0"):
            env = env0
            t = ts[env]
            for _ in range(5):
                eg.egfem_interp(t, I.INTERP_GRADPOW_P0, 3.0, u, None, chain, s)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(50):
                eg.egfem_interp(t, I.INTERP_GRADPOW_P0, 3.0, u, None, chain, s)
            e1.record(s)
            torch.cuda.synchronize()
            res.setdefault(f"{'f64' if dt == eg.F64 else 'f32'}_{ {'1': 'geo', '0': 'gather', 's': 'geo_smem'}[env0]}", []).append(
                e0.elapsed_time(e1) / 50)
    res[f"{'f64' if dt == eg.F64 else 'f32'}_name"] = eg.egfem_kernel_name(ts["1"], 5, eg.JAC_NEWTON,
                                                                          I.INTERP_GRADPOW_P0, 3.0)
    del ts
print(json.dumps(res))
