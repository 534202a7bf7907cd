"""C-ABI library checks that need no GPU (-m "not gpu"): the .so loads, exports every
symbol include/egfem.h declares, and its host-only logic behaves."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def eg():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2005_06193_b200 as eg
    return eg


def header_functions():
    src = open(os.path.join(ROOT, "include", "egfem.h")).read()
    return sorted(set(re.findall(r"^\s*(?:egfem_status|uint64_t|const char\*)\s+(egfem_\w+)\s*\(", src, re.M)))


def test_header_declares_the_north_star_boundary():
    fns = header_functions()
    for name in ("egfem_tensor_build", "egfem_interp", "egfem_apply", "egfem_jacobian"):
        assert name in fns


def test_library_exports_every_declared_symbol(eg):
    import ctypes
    lib = ctypes.CDLL(eg.LIB_PATH)
    missing = [f for f in header_functions() if not hasattr(lib, f)]
    assert not missing, missing
    assert sorted(eg.EXPORTS) == header_functions()


def test_nm_shows_sm100a_cubin(eg):
    """The library carries sm_100a device code (cuobjdump lists the ELF arch)."""
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump missing")
    out = subprocess.run(["cuobjdump", "--list-elf", eg.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings(eg):
    L = eg.lib()
    for code, name in eg.STATUS.items():
        assert L.egfem_status_string(code).decode() == name


def test_null_handle_is_rejected_without_gpu(eg):
    """Validation runs before any CUDA call: a NULL tensor returns INVALID_ARGUMENT."""
    L = eg.lib()
    assert L.egfem_apply(None, None, None, None, None) == 1
    assert L.egfem_interp(None, 0, 0.0, None, None, None, None) == 1
    assert L.egfem_jacobian(None, 0, 0, 0.0, None, None, None, None, None) == 1
    assert "NULL" in L.egfem_last_error().decode()
    assert L.egfem_tensor_destroy(None) == 0
    assert L.egfem_interp_range(None, 0, 0.0, None, None, None, 0, 0, None) == 1
    assert L.egfem_apply_jacobian_rows(None, 0, 0, 0.0, None, None, None, None, None, 0, 0, None) == 1
    assert L.egfem_interior(None, None, None, None, None) == 1


def _py_partition(prefix, nranks):
    total = prefix[-1]
    b = [0]
    for r in range(1, nranks):
        target = -(-total * r // nranks)
        row = int(np.searchsorted(prefix, target, side="left"))
        b.append(min(max(row, b[-1]), len(prefix) - 1))
    b.append(len(prefix) - 1)
    return np.array(b)


@pytest.mark.parametrize("nranks", [1, 2, 3, 8, 17])
def test_partition_rows_matches_python(eg, nranks):
    rng = np.random.default_rng(nranks)
    counts = rng.integers(0, 100, 5000)
    prefix = np.concatenate([[0], np.cumsum(counts)])
    b = eg.egfem_partition_rows(prefix, nranks)
    assert np.array_equal(b, _py_partition(prefix, nranks))
    assert b[0] == 0 and b[-1] == 5000 and np.all(np.diff(b) >= 0)
    loads = prefix[b[1:]] - prefix[b[:-1]]
    assert loads.max() - loads.min() <= 2 * counts.max() + 1  # nnz-balanced


def test_partition_rows_edge_cases(eg):
    assert np.array_equal(eg.egfem_partition_rows(np.array([0]), 4), [0, 0, 0, 0, 0])
    assert np.array_equal(eg.egfem_partition_rows(np.array([0, 5]), 3), [0, 1, 1, 1])


def _brute_interior(rp, col, lo, hi):
    """Longest run of consecutive rows whose columns all lie in [lo, hi) (first on ties)."""
    n = len(rp) - 1
    ok = [bool(np.all((col[rp[i]:rp[i + 1]] >= lo) & (col[rp[i]:rp[i + 1]] < hi))) for i in range(n)]
    best = (0, 0)
    for a in range(n):
        for b in range(a + 1, n + 1):
            if all(ok[a:b]) and b - a > best[1] - best[0]:
                best = (a, b)
    return best


@pytest.mark.parametrize("seed", range(12))
def test_interior_rows_matches_brute_force(eg, seed):
    """egfem_interior_rows (the halo-free row run behind the overlapped exchange) against brute force."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(0, 40))
    counts = rng.integers(0, 5, n)
    rp = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    col = rng.integers(0, 30, int(rp[-1])).astype(np.int32)
    lo, hi = sorted(rng.integers(0, 31, 2))
    assert eg.egfem_interior_rows(rp, col, lo, hi) == _brute_interior(rp, col, lo, hi)


def test_interior_rows_band_structure(eg):
    """A banded pattern (the structured lexicographic numbering of a rank's window): the halo-free
    rows are the owned rows at least one bandwidth away from either end."""
    n_local, own_lo, own_hi, bw = 100, 10, 90, 10
    rows = range(own_lo, own_hi)
    rp, col = [0], []
    for i in rows:
        c = [j for j in range(i - bw, i + bw + 1) if 0 <= j < n_local]
        col += c
        rp.append(len(col))
    lo, hi = eg.egfem_interior_rows(np.array(rp), np.array(col), own_lo, own_hi)
    assert (lo, hi) == (bw, own_hi - own_lo - bw)
    assert eg.egfem_interior_rows(np.array([0]), np.array([], np.int32), 0, 1) == (0, 0)


def synthetic_group_key(n, g):
    """Pattern key (include/egfem.h egfem_group_compile) of g member rows on an n-point stencil,
    every member with fibers at every point and k positions (a + b + m) % 3 != 1."""
    key = [n, g]
    for m in range(g):
        key.append(n)
        for a in range(n):
            bs = [b for b in range(n) if (a + b + m) % 3 != 1]
            key += [a, len(bs)] + bs
    return key


@pytest.mark.parametrize("n,g,ppl,f64", [(19, 4, 2, 1), (9, 1, 1, 1), (12, 7, 4, 0), (1, 1, 2, 1)])
def test_group_kernel_generation_compiles(eg, n, g, ppl, f64):
    """The batched action's generated row-group kernels (egfem_group.cu) compile with NVRTC for
    sm_100a (no GPU needed): straight-line code for a synthetic pattern, fp64 and fp32, 1-4 pairs
    per lane; a malformed key is rejected before compiling."""
    eg.egfem_group_compile(synthetic_group_key(n, g), ppl, bool(f64))
    with pytest.raises(eg.EgfemError) as e:
        eg.egfem_group_compile(synthetic_group_key(n, g)[:-1] + [n + 5], ppl, bool(f64))
    assert e.value.status == 1
