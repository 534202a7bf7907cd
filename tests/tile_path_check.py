"""Run the hot path through the TMA tile kernel (EGFEM_PATH=tile) and check it against the oracle.

Invoked by test_gpu_parity.py::test_tile_path in a subprocess (the path switch is read once)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
assert os.environ.get("EGFEM_PATH") == "tile"
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
    for fused in (False, True):
        g = gpu_pass(eg, t, pr, u, fused=fused)
        ref = oracle_pass(o, pr, u)
        for key in ("w", "r", "A", "J"):
            e = rel_l2(g[key], ref[key])
            worst = max(worst, e)
            assert e <= 1e-12, (name, key, e)
print("tile path ok", worst)
