"""bench.py host logic that needs no GPU (-m "not gpu"): the rank launcher, the partition plan
it deals to the ranks, and the byte model the roofline line divides by."""
import json
import os
import subprocess
import sys
import types

import numpy as np
import pytest

import egfem_inputs as I

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args, timeout=600):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


@pytest.mark.parametrize("n", [2, 3])
def test_launcher_spawns_ranks_row_partition(n):
    """`bench.py --gpus N` with no launcher starts N ranks itself (torch.distributed.run, gloo on
    CPU here): rank 0 prints one line with n_gpus = N; cfg4's rows are split into N contiguous,
    nnz-balanced ranges (egfem_partition_rows on the per-row nonzero counts)."""
    d = _bench("--plan-only", "--gpus", str(n), "--config", "cfg4")
    assert d["n_gpus"] == n and len(d["ranks"]) == n
    assert sorted(r["rank"] for r in d["ranks"]) == list(range(n))
    cuts = d["plan"]["row_cuts"]
    assert cuts[0] == 0 and cuts[-1] == 2146689 and all(a < b for a, b in zip(cuts, cuts[1:]))
    per = d["plan"]["nnz_per_rank"]
    assert sum(per) == 201326592
    assert max(per) - min(per) <= 96 * 2  # balanced to within a couple of rows


def test_launcher_cfg5_batch_shards():
    """cfg5 at N > 1 shards the batch (T replicated): contiguous pair ranges covering all 256."""
    d = _bench("--plan-only", "--gpus", "4", "--config", "cfg5")
    assert d["n_gpus"] == 4
    sh = d["plan"]["batch_shards"]
    assert sh[0][0] == 0 and sh[-1][1] == 256 and all(a[1] == b[0] for a, b in zip(sh, sh[1:]))
    assert "replicated" in d["plan"]["tensor"]


def test_single_rank_plan():
    d = _bench("--plan-only", "--config", "cfg4")
    assert d["n_gpus"] == 1 and d["plan"]["row_cuts"] == [0, 2146689]


SIZES = {  # N_u, N_f, N_el, nnz(T), nnz(CSR)
    "cfg2": (263169, 263169, 524288, 8133633, 1838081),
    "cfg3": (1050625, 2097152, 2097152, 18874368, 7346177),
    "cfg4": (2146689, 12582912, 12582912, 201326592, 31802497),
    "cfg5": (263169, 263169, 131072, 23081985, 3018753),
}


def _fake(name):
    n_u, n_f, n_el, nnz, csr = SIZES[name]
    pr = types.SimpleNamespace(name=name, mesh=types.SimpleNamespace(dim=3 if name == "cfg4" else 2, n_cells=n_el,
                                                                     n_vertices=n_u),
                               W=types.SimpleNamespace(family=I.P0 if name in ("cfg3", "cfg4") else I.P1),
                               interp=I.INTERP_GRADPOW_P0 if name in ("cfg3", "cfg4") else I.INTERP_IDENTITY)
    t = types.SimpleNamespace(n_u=n_u, n_f=n_f, nnz=nnz, nnz_csr=csr)
    return t, pr


@pytest.mark.parametrize("name,kind,mb", [("cfg4", "apply", 3373.41), ("cfg4", "jac", 4096.80),
                                          ("cfg4", "interp", 874.00), ("cfg3", "apply", 343.98),
                                          ("cfg3", "jac", 453.05), ("cfg3", "interp", 134.27),
                                          ("cfg2", "apply", 138.56), ("cfg2", "jac", 151.16)])
def test_model_bytes_match_survey_table(name, kind, mb):
    """The roofline's algorithmic bytes are SURVEY §8(d) D.3's per-call figures (its table of
    MB per call, computed from the §8(a) counts) — the numbers a by-hand recomputation uses."""
    import bench
    t, pr = _fake(name)
    assert abs(bench.model_bytes(t, pr, 8, kind) / 1e6 - mb) < 0.01


def test_model_bytes_fused_cfg4():
    """Fused apply + Newton on cfg4 fp64 = the T stream once plus both outputs: 4,131 MB
    (VERDICT r1's recomputation from §8(d))."""
    import bench
    t, pr = _fake("cfg4")
    assert abs(bench.model_bytes(t, pr, 8, "fused") / 1e6 - 4131.14) < 0.5


def test_oracle_sample_rows_and_items():
    """The cpu_baseline / reference sample: rows [0, R) and exactly the interp work items that
    feed them (cells touching a sampled row), bounded by the nonzero budget."""
    import bench
    pr = I.make_problem("cfg4", n=16)
    R, (c0, c1) = bench.oracle_sample(pr, 50_000)
    assert 0 < R < pr.n_u
    V = np.asarray(pr.V.cell_dofs)
    need = np.nonzero((V < R).any(axis=1))[0]
    assert c0 == need.min() and c1 == need.max() + 1


def test_reference_budget_bounds_total_work():
    """--impl reference: the per-step oracle sample is the cpu_baseline leg's up to
    REFERENCE_STEPS_FULL steps (the driver's K = 20 and the default K = 50 time the same rows),
    and shrinks as 1 / K beyond that so the total CPU work stays bounded."""
    import bench
    full = bench.ORACLE_SAMPLE_NNZ
    assert bench.reference_budget(full, 20) == full
    assert bench.reference_budget(full, bench.REFERENCE_STEPS_FULL) == full
    for K in (100, 400, 10_000):
        b = bench.reference_budget(full, K)
        assert 0 < b < full and b * K <= full * bench.REFERENCE_STEPS_FULL
    assert bench.reference_budget(1, 10_000) == 1
