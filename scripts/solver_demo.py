"""F4 evidence: the GPU Picard solve of the biochemical problem (§5.4) at increasing n;
prints one JSON line per n with Picard iterations, CG iterations, time split, nodal error."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2005_06193_b200.solver import biochemical_problem

for n in [int(a) for a in (sys.argv[1:] or ["64", "128", "256", "512"])]:
    s, d, ue = biochemical_problem(n)
    s.solve(d, ue, maxit=2, tol=0.0)  # warm-up
    torch.cuda.synchronize()
    t0 = time.time()
    res = s.solve(d, ue, tol=1e-12, maxit=100)
    torch.cuda.synchronize()
    dt = time.time() - t0
    print(json.dumps({"n": n, "unknowns": int(s.n), "picard_iterations": res.iterations, "converged": res.converged,
                      "cg_iterations": res.cg_iterations, "wall_s": dt,
                      "max_nodal_error": float(np.abs(res.u - ue).max()),
                      "last_increments": res.increments[-3:]}), flush=True)
