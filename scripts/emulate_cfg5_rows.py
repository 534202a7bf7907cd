"""Row-partitioned cfg5 (the SURVEY §8(e) alternative to batch sharding): per-rank COMPUTE of the
batched action at N ranks, one rank at a time on one GPU (no NCCL; not a multi-GPU measurement).
Rank r's local tensor (egfem_partition: its rows, columns in its window, its own compiled row
groups) runs egfem_apply_batched on the node-major U window with the halo already in place; the
U halo a rank would receive per step (nodes outside its own rows × B pairs) is reported beside
it.  Each rank's R is checked against the full-tensor R (relative L2).  One JSON line per N.

usage: python scripts/emulate_cfg5_rows.py [1,2,4,8] [steps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import egfem_inputs as I
import paper_2005_06193_b200 as eg


def timed(fn, K):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(K):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / K


def main():
    Ns = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,2,4,8").split(",")]
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    pr = I.make_problem("cfg5")
    B = pr.batch
    tg = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, device=0)
    U = torch.tensor(np.ascontiguousarray(pr.u.T), device="cuda")  # node-major [n_u, B]
    R = torch.empty_like(U)
    t1 = timed(lambda: eg.egfem_apply_batched(tg, B, eg.LAYOUT_NODE_MAJOR, U, U, R), K)
    Rf = R.clone()
    for N in Ns:
        per, err, halo = [], 0.0, []
        for rank in range(N):
            if N == 1:
                per.append(t1)
                continue
            loc, win = eg.egfem_partition(tg, N, rank)
            Ul = U[win["col_begin"]:win["col_end"]].contiguous()
            Rl = torch.empty((win["row_end"] - win["row_begin"], B), dtype=U.dtype, device="cuda")
            per.append(timed(lambda: eg.egfem_apply_batched(loc, B, eg.LAYOUT_NODE_MAJOR, Ul, Ul, Rl), K))
            ref = Rf[win["row_begin"]:win["row_end"]]
            err = max(err, float(torch.linalg.norm(Rl - ref) / torch.linalg.norm(ref)))
            halo.append((win["col_end"] - win["col_begin"]) - (win["row_end"] - win["row_begin"]))
            name = eg.egfem_kernel_name(loc, 3)
            del loc
        out = {"config": "cfg5", "N": N, "batch": B, "max_rank_ms": max(per), "per_rank_ms": per,
               "compute_speedup": t1 / max(per), "rel_l2_vs_full": err,
               "halo_nodes_max": max(halo) if halo else 0,
               "halo_bytes_max": (max(halo) if halo else 0) * B * 8,
               "kernel": name[:160] if N > 1 else eg.egfem_kernel_name(tg, 3)[:160]}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
