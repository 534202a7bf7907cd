"""Experiment: the step (interp + fused apply/Newton) as S row slices, each preceded by the interp
of the cells it needs for the first time, so a slice's w / D_u w are read back from L2.
Each schedule is captured into one CUDA graph; prints the step time per S and checks r, J
bitwise against the two-launch step.

usage: python scripts/slice_sweep.py [cfg4] [f64|f32]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import egfem_inputs as I
import paper_2005_06193_b200 as eg

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
dt = eg.F32 if (len(sys.argv) > 2 and sys.argv[2] == "f32") else eg.F64
td = torch.float32 if dt == eg.F32 else torch.float64
pr = I.make_problem(name)
t = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, dtype=dt, device=0)
ex = t.export(values=False)
rp, tk = ex["t_row_ptr"], ex["t_k"]
kmax_pre = np.maximum.accumulate(np.maximum.reduceat(tk, rp[:-1]))  # rows are nonempty
del ex, tk
u = torch.tensor(pr.u, dtype=td, device="cuda")
w = torch.empty(t.n_f, dtype=td, device="cuda")
chain = torch.empty(t.n_f * (pr.mesh.dim + 1), dtype=td, device="cuda")
r = torch.empty(t.n_u, dtype=td, device="cuda")
J = torch.empty(t.nnz_csr, dtype=td, device="cuda")
N = eg.JAC_NEWTON


def whole(s):
    eg.egfem_interp(t, pr.interp, pr.p, u, w, chain, s)
    eg.egfem_apply_jacobian(t, N, pr.interp, pr.p, u, w, chain, r, J, s)


def sliced(S):
    bounds = np.linspace(0, t.n_u, S + 1).astype(np.int64)

    def run(s):
        done = 0
        for a, b in zip(bounds[:-1], bounds[1:]):
            need = int(kmax_pre[b - 1]) + 1
            if need > done:
                eg.egfem_interp_range(t, pr.interp, pr.p, u, w, chain, done, need, s)
                done = need
            eg.egfem_apply_jacobian_rows(t, N, pr.interp, pr.p, u, w, chain, r, J, int(a), int(b), s)
        if done < t.n_f:
            eg.egfem_interp_range(t, pr.interp, pr.p, u, w, chain, done, t.n_f, s)
    return run


def timed(fn, n=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn(torch.cuda.current_stream())
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


res = {"cfg": name, "dtype": "f32" if dt == eg.F32 else "f64", "whole": timed(whole)}
r0, J0 = r.clone(), J.clone()
for S in (2, 4, 8, 16, 32, 64):
    r.fill_(float("nan"))
    J.fill_(float("nan"))
    res[f"S{S}"] = timed(sliced(S))
    res[f"S{S}_bitwise"] = bool(torch.equal(r, r0) and torch.equal(J, J0))
print(json.dumps(res), flush=True)
