"""CPU oracle for the EGFEM hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_2005_06193_b200``) never imports it and shares no code with it.

``liboracle.so`` is the plain C++17 oracle in ``egfem_oracle.cpp`` (fp64,
single-threaded, canonical order).  ``brute.py`` is an independent dense numpy
brute force + SGA quadrature used to pin the oracle on tiny meshes.

Parity status per function (DESIGN.md §4 restates it):
  build (T values, pattern, maps)  pinned: closed forms, dense brute force, PoU,
                                   symmetry, IBP identity, exact-integral moments
  interp                            pinned: linear-field closed form, brute force
  apply                             pinned: 1D closed form, brute force, Σr=0, SGA
  jacobian                          pinned: 1D closed forms, FD, Euler homogeneity
  bilinear (F3)                     pinned: exact-integration matrices (brute), PoU Σ_j T_ijk
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "egfem_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with the host C++ compiler (plain -O2, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-fopenmp", "-shared", "-fPIC", "-o", _LIB, _SRC])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i64, i32 = ctypes.c_int64, ctypes.c_int
        L.oracle_build.argtypes = [i32, i64, P, i64, P, i32, i64, i32, P, i32, i64, i32, P, i32, i32, P, P,
                                   i64, i64, ctypes.POINTER(ctypes.c_void_p)]
        L.oracle_build.restype = i32
        L.oracle_free.argtypes = [P]
        L.oracle_sizes.argtypes = [P, P, P, P, P]
        L.oracle_export.argtypes = [P] * 10
        L.oracle_export.restype = i32
        L.oracle_interp.argtypes = [P, i32, ctypes.c_double, P, P]
        L.oracle_interp.restype = i32
        L.oracle_apply.argtypes = [P, P, P, P]
        L.oracle_apply_batched.argtypes = [P, i32, P, P, P]
        L.oracle_jacobian.argtypes = [P, i32, i32, ctypes.c_double, P, P, P]
        L.oracle_jacobian.restype = i32
        L.oracle_bilinear.argtypes = [P, P]
        L.oracle_bilinear.restype = i32
        L.oracle_rule.argtypes = [i32, i32, i32, P, P]
        L.oracle_rule.restype = i32
        L.oracle_interp_range.argtypes = [P, i32, ctypes.c_double, P, P, i64, i64]
        L.oracle_interp_range.restype = i32
        L.oracle_set_threads.argtypes = [i32]
        L.oracle_set_threads(1)  # the plain sequential oracle unless a caller asks (bench all-cores timing)
        _lib = L
    return _lib


def rule(dim, degree):
    """The oracle's default quadrature rule for an integrand of `degree` in `dim` D:
    (bary[nq, dim+1], weights[nq]) with weights summing to 1."""
    L = lib()
    nq = L.oracle_rule(dim, degree, 0, None, None)
    if nq <= 0:
        raise ValueError(f"oracle_rule failed rc={nq}")
    bary = np.zeros((nq, dim + 1), np.float64)
    w = np.zeros(nq, np.float64)
    L.oracle_rule(dim, degree, nq, bary.ctypes.data_as(ctypes.c_void_p), w.ctypes.data_as(ctypes.c_void_p))
    return bary, w


def set_threads(n):
    """OpenMP threads of the row / cell loops (default 1; results are bitwise independent of n)."""
    lib().oracle_set_threads(int(n))


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


class OracleTensor:
    """Canonical T_ijk of (mesh, V, W, form) built element by element on the CPU."""

    def __init__(self, mesh, V, W, form, quad=None, rows=None):
        L = lib()
        self._keep = [np.ascontiguousarray(mesh.coords, np.float64), np.ascontiguousarray(mesh.cells, np.int32),
                      np.ascontiguousarray(V.cell_dofs, np.int32), np.ascontiguousarray(W.cell_dofs, np.int32)]
        nq, qb, qw = 0, None, None
        if quad is not None:
            qb = np.ascontiguousarray(quad[0], np.float64)
            qw = np.ascontiguousarray(quad[1], np.float64)
            nq = len(qw)
        r0, r1 = (-1, -1) if rows is None else rows
        h = ctypes.c_void_p()
        rc = L.oracle_build(mesh.dim, mesh.n_vertices, _p(self._keep[0]), mesh.n_cells, _p(self._keep[1]),
                            V.family, V.n_dofs, V.n_local, _p(self._keep[2]),
                            W.family, W.n_dofs, W.n_local, _p(self._keep[3]),
                            form, nq, _p(qb), _p(qw), r0, r1, ctypes.byref(h))
        if rc != 0:
            raise ValueError(f"oracle_build failed rc={rc}")
        self.h = h
        self.V, self.W = V, W
        self.n_u, self.n_f = V.n_dofs, W.n_dofs
        s = [np.zeros(1, np.int64) for _ in range(4)]
        L.oracle_sizes(self.h, *[_p(x) for x in s])
        self.nnz, self.nnz_csr = int(s[0][0]), int(s[1][0])

    def __del__(self):
        if getattr(self, "h", None) is not None and _lib is not None:
            _lib.oracle_free(self.h)
            self.h = None

    def export(self, slot_ik=False, loc=False, maps=True):
        L = lib()
        out = dict(t_row_ptr=np.zeros(self.n_u + 1, np.int64), t_j=np.zeros(self.nnz, np.int32),
                   t_k=np.zeros(self.nnz, np.int32), t_val=np.zeros(self.nnz, np.float64),
                   csr_row_ptr=np.zeros(self.n_u + 1, np.int64), csr_col=np.zeros(self.nnz_csr, np.int32),
                   slot_ij=np.zeros(self.nnz, np.int32) if maps else None)
        out["slot_ik"] = np.zeros(self.nnz, np.int32) if slot_ik else None
        out["loc"] = np.zeros(self.nnz, np.uint8) if loc else None
        keys = ["t_row_ptr", "t_j", "t_k", "t_val", "csr_row_ptr", "csr_col", "slot_ij", "slot_ik", "loc"]
        rc = L.oracle_export(self.h, *[_p(out[k]) for k in keys])
        if rc != 0:
            raise ValueError(f"oracle_export failed rc={rc}")
        return {k: v for k, v in out.items() if v is not None}

    def interp(self, kind, p, u, items=None):
        """w at the W-DOFs; items=(c0, c1) restricts to cells [c0, c1) (cell-wise kinds) or
        W-DOFs [c0, c1) (nodal kinds), the rest of w stays 0."""
        w = np.zeros(self.n_f, np.float64)
        u = np.ascontiguousarray(u, np.float64)
        c0, c1 = (0, -1) if items is None else items
        rc = lib().oracle_interp_range(self.h, kind, float(p), _p(u), _p(w), int(c0), int(c1))
        if rc != 0:
            raise ValueError(f"oracle_interp failed rc={rc}")
        return w

    def apply(self, u, w):
        r = np.zeros(self.n_u, np.float64)
        u = np.ascontiguousarray(u, np.float64)
        w = np.ascontiguousarray(w, np.float64)
        lib().oracle_apply(self.h, _p(u), _p(w), _p(r))
        return r

    def apply_batched(self, U, W):
        U = np.ascontiguousarray(U, np.float64)
        W = np.ascontiguousarray(W, np.float64)
        B = U.shape[0]
        R = np.zeros((B, self.n_u), np.float64)
        lib().oracle_apply_batched(self.h, B, _p(U), _p(W), _p(R))
        return R

    def bilinear(self):
        """F3: B_ik = ∫ (slot φ_i)(slot η_k) on the CSR pattern (W = V), element-by-element."""
        vals = np.zeros(self.nnz_csr, np.float64)
        rc = lib().oracle_bilinear(self.h, _p(vals))
        if rc != 0:
            raise ValueError(f"oracle_bilinear failed rc={rc}")
        return vals

    def jacobian(self, mode, kind, p, u, w):
        vals = np.zeros(self.nnz_csr, np.float64)
        u = np.ascontiguousarray(u, np.float64)
        w = np.ascontiguousarray(w, np.float64)
        rc = lib().oracle_jacobian(self.h, mode, kind, float(p), _p(u), _p(w), _p(vals))
        if rc != 0:
            raise ValueError(f"oracle_jacobian failed rc={rc}")
        return vals
