"""Single-pass step (egfem_step, k_step) vs the two launches (interp + fused apply/Newton), per
work-sequence setting (EGFEM_STEP_CI / _RI / _LAG, read when the tensor is built).  Each variant
is captured into a CUDA graph and replayed K times between CUDA events; one JSON line each.

usage: python scripts/step_sweep.py [cfg4] [f64|f32] [K] [ci,ri,lag[,mode] ...]
(mode 1: interp items only, 2: row items only — EGFEM_STEP_MODE diagnostics)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import egfem_inputs as I
import paper_2005_06193_b200 as eg


def timed(fn, K):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn(s)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn(torch.cuda.current_stream())
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(K):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / K


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
    dtype = 1 if (len(sys.argv) > 2 and sys.argv[2] == "f32") else 0
    K = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    variants = [v for v in sys.argv[4:] if v != "-"] if len(sys.argv) > 4 else ["32,64,2048"]
    pr = I.make_problem(name)
    for v in ["two", "interp", "fused"] + variants:
        base = v in ("two", "interp", "fused")
        if not base:
            f = v.split(",")
            os.environ.update(EGFEM_STEP="1", EGFEM_STEP_CI=f[0], EGFEM_STEP_RI=f[1], EGFEM_STEP_LAG=f[2],
                              EGFEM_STEP_MODE=f[3] if len(f) > 3 else "0")
        t = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, dtype=dtype, device=0)
        td = t.torch_dtype
        u = torch.tensor(pr.u, dtype=td, device="cuda")
        w = torch.empty(t.n_f, dtype=td, device="cuda")
        chain = torch.empty(t.n_f * (pr.mesh.dim + 1), dtype=td, device="cuda")
        r = torch.empty(t.n_u, dtype=td, device="cuda")
        J = torch.empty(t.nnz_csr, dtype=td, device="cuda")
        w = None  # the gradient kinds keep w_K in the packed record only, as bench.py runs the step
        if v == "two":
            def fn(s):
                eg.egfem_interp(t, pr.interp, pr.p, u, w, chain, s)
                eg.egfem_apply_jacobian(t, eg.JAC_NEWTON, pr.interp, pr.p, u, w, chain, r, J, s)
        elif v == "interp":
            def fn(s):
                eg.egfem_interp(t, pr.interp, pr.p, u, w, chain, s)
        elif v == "fused":
            eg.egfem_interp(t, pr.interp, pr.p, u, w, chain)

            def fn(s):
                eg.egfem_apply_jacobian(t, eg.JAC_NEWTON, pr.interp, pr.p, u, w, chain, r, J, s)
        else:
            def fn(s):
                eg.egfem_step(t, pr.interp, pr.p, u, w, chain, r, J, s)
        ms = timed(fn, K)
        print(json.dumps({"config": name, "dtype": "f32" if dtype else "f64", "variant": v, "ms": ms,
                          "kernel": "two launches" if base else
                          eg.egfem_kernel_name(t, 4, eg.JAC_NEWTON, pr.interp, pr.p)}), flush=True)
        del t, u, w, chain, r, J
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
