"""Per-rank COMPUTE of the row-partitioned step at N ranks, measured one rank at a time on one
GPU (no NCCL, no concurrent ranks — not a multi-GPU measurement): for each rank r of N, its
local tensor (egfem_partition) runs the bench step (interp + fused apply/Newton Jacobian) on its
u window with the halo already in place, timed with CUDA events over K steps.  The max over
ranks is the compute part of the N-GPU step; the halo exchange (≈ 134 KB per neighbour for
cfg4) is not included.  Writes one JSON line per N.

usage: python scripts/emulate_ranks.py [cfg4] [1,2,4,8] [steps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import egfem_inputs as I
import paper_2005_06193_b200 as eg


def step_ms(t, pr, u_np, K):
    dev = torch.device("cuda", 0)
    u = torch.tensor(u_np, device=dev)
    w = torch.empty(t.n_f, dtype=torch.float64, device=dev)
    chain = torch.empty(t.n_f * (pr.mesh.dim + 1), dtype=torch.float64, device=dev)
    r = torch.empty(t.n_u, dtype=torch.float64, device=dev)
    J = torch.empty(t.nnz_csr, dtype=torch.float64, device=dev)
    s = torch.cuda.current_stream()

    def step():
        eg.egfem_interp(t, pr.interp, pr.p, u, w, chain, s)
        eg.egfem_apply_jacobian(t, eg.JAC_NEWTON, pr.interp, pr.p, u, w, chain, r, J, s)
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(K):
        step()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / K


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
    Ns = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,2,4,8").split(",")]
    K = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    pr = I.make_problem(name)
    tg = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, device=0)
    t1 = None
    for N in Ns:
        per = []
        for rank in range(N):
            if N == 1:
                per.append(step_ms(tg, pr, pr.u, K))
                continue
            loc, win = eg.egfem_partition(tg, N, rank)
            per.append(step_ms(loc, pr, pr.u[win["col_begin"]:win["col_end"]], K))
            del loc
            torch.cuda.empty_cache()
        mx = max(per)
        t1 = mx if N == 1 else t1
        print(json.dumps({"config": name, "ranks": N, "per_rank_ms": per, "max_ms": mx,
                          "compute_speedup_vs_1": (t1 / mx) if t1 else None,
                          "note": "compute only, ranks timed one at a time on one GPU; halo exchange not included"}),
              flush=True)


if __name__ == "__main__":
    main()
