"""Helper of test_dist_nccl_gpu.py (run as its own process): a one-rank NCCL process group on
cuda:0 driving the distributed step — egfem_partition, gather_windows (all_gather over NCCL),
the halo plan and dist.split_step (interior / boundary phases with the exchange posted through
NCCL) — and the max-over-ranks timing all_reduce of bench.py.  Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

import egfem_inputs as I
import paper_2005_06193_b200 as eg
from paper_2005_06193_b200 import dist as edist


def main():
    name = sys.argv[1]
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{sys.argv[2]}", rank=0, world_size=1,
                            device_id=dev)
    pr = I.make_problem(name, n=I.SMALL_N[name])
    tg = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, device=0)
    u = torch.tensor(pr.u, device=dev)
    chain_len = tg.n_f * (pr.mesh.dim + 1)
    has_chain = pr.W.family in (I.P0, I.QUAD) and pr.interp != I.INTERP_IDENTITY
    # single-GPU reference step
    w = torch.empty(tg.n_f, dtype=torch.float64, device=dev)
    chain = torch.empty(chain_len, dtype=torch.float64, device=dev) if has_chain else None
    r = torch.empty(tg.n_u, dtype=torch.float64, device=dev)
    J = torch.empty(tg.nnz_csr, dtype=torch.float64, device=dev)
    eg.egfem_interp(tg, pr.interp, pr.p, u, w, chain)
    eg.egfem_apply_jacobian(tg, eg.JAC_NEWTON, pr.interp, pr.p, u, w, chain, r, J)
    # the N-rank code path with N = 1
    t, win = eg.egfem_partition(tg, 1, 0, 0)
    W = edist.Window(win["row_begin"], win["row_end"], win["col_begin"], win["col_end"])
    plan = edist.make_plan(edist.gather_windows(W), 0)
    ul = u[W.col_begin:W.col_end].clone()
    wl = torch.empty(t.n_f, dtype=torch.float64, device=dev)
    cl = torch.empty(t.n_f * (pr.mesh.dim + 1), dtype=torch.float64, device=dev) if has_chain else None
    rl = torch.empty(t.n_u, dtype=torch.float64, device=dev)
    Jl = torch.empty(t.nnz_csr, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record(stream)
    edist.split_step(eg, t, plan, eg.egfem_interior(t), pr.interp, pr.p, ul, wl, cl, rl, Jl, stream, ev)
    ev[3].record(stream)
    torch.cuda.synchronize()
    m = torch.tensor([ev[0].elapsed_time(ev[3])], dtype=torch.float64, device=dev)
    dist.all_reduce(m, op=dist.ReduceOp.MAX)
    dist.barrier()
    ok = bool(torch.equal(r, rl) and torch.equal(J, Jl))
    print(json.dumps({"config": name, "world": dist.get_world_size(), "backend": dist.get_backend(),
                      "rows": [W.row_begin, W.row_end], "halo": plan.halo_values, "bitwise": ok,
                      "ms_max": float(m.item())}), flush=True)
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
