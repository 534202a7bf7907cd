"""paper_2005_06193_b200 — B200-native hot path of the extended group finite element method.

A thin ctypes binding over ``lib/libegfem.so`` (C ABI in ``include/egfem.h``).  It
only marshals arguments: every step of the path (tensor build, interpolation,
tensor action, Jacobian, batched action, partition, halo pack/unpack) runs in the
library's sm_100a CUDA kernels.  PyTorch supplies device memory and streams.

There is no CPU fallback: importing this package on a machine where
``libegfem.so`` is missing raises ImportError, and every call raises EgfemError
on a non-OK status.

Paper: Tolle & Marheineke, "Extended group finite element method", arXiv
2005.06193 — interp, T:(u⊗w) (L183, L251), T·w and
the Newton Jacobian (L182, L261, L290–292), offline tensors (L196–203, L304).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libegfem.so")

# enums (include/egfem.h)
F64, F32 = 0, 1
P0, P1, P2, QUAD = 0, 1, 2, 3
FORM_CONV_K, FORM_CONV_J, FORM_PLAP, FORM_MASS3, FORM_CONV_I = 0, 1, 2, 3, 4
INTERP_IDENTITY, INTERP_SQUARE, INTERP_GRADPOW_P0, INTERP_P1_TO_P2_SQUARE = 0, 1, 2, 3
INTERP_MINSURF_P0, INTERP_RECIPROCAL = 4, 5
JAC_PICARD, JAC_NEWTON = 0, 1
LAYOUT_NODE_MAJOR, LAYOUT_PAIR_MAJOR = 0, 1
STATUS = {0: "EGFEM_OK", 1: "EGFEM_ERR_INVALID_ARGUMENT", 2: "EGFEM_ERR_DIMENSION_MISMATCH",
          3: "EGFEM_ERR_UNSUPPORTED", 4: "EGFEM_ERR_INDEX_OVERFLOW", 5: "EGFEM_ERR_OUT_OF_MEMORY",
          6: "EGFEM_ERR_CUDA", 7: "EGFEM_ERR_NCCL"}

# every symbol include/egfem.h declares (tests check the .so exports all of them)
EXPORTS = ("egfem_tensor_build", "egfem_tensor_from_coo", "egfem_tensor_destroy", "egfem_tensor_info",
           "egfem_tensor_csr_pattern", "egfem_tensor_export", "egfem_interp", "egfem_apply",
           "egfem_apply_batched", "egfem_jacobian", "egfem_apply_jacobian", "egfem_partition",
           "egfem_partition_rows", "egfem_halo_pack", "egfem_halo_unpack", "egfem_launch_count",
           "egfem_status_string", "egfem_last_error", "egfem_bilinear_build", "egfem_csr_spmv",
           "egfem_bilinear_jacobian", "egfem_interior", "egfem_interp_range", "egfem_apply_jacobian_rows",
           "egfem_interior_rows", "egfem_kernel_name", "egfem_group_compile", "egfem_step")


class EgfemError(RuntimeError):
    def __init__(self, fn, status, detail):
        super().__init__(f"{fn}: {STATUS.get(status, status)}: {detail}")
        self.status = status


class _Mesh(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("n_vertices", ctypes.c_int64), ("coords", ctypes.c_void_p),
                ("n_cells", ctypes.c_int64), ("cells", ctypes.c_void_p)]


class _Space(ctypes.Structure):
    _fields_ = [("family", ctypes.c_int), ("n_dofs", ctypes.c_int64), ("cell_dofs", ctypes.c_void_p)]


class _Quad(ctypes.Structure):
    _fields_ = [("n_points", ctypes.c_int32), ("bary", ctypes.c_void_p), ("weights", ctypes.c_void_p)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libegfem.so not built ({LIB_PATH}); run __graft_entry__.build()")
    L = ctypes.CDLL(LIB_PATH)
    P, i64, i32, st = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int
    pp = ctypes.POINTER(ctypes.c_void_p)
    sig = {
        "egfem_tensor_build": [P, P, P, st, P, st, st, pp],
        "egfem_tensor_from_coo": [i64, i64, i64, P, P, P, P, st, st, pp],
        "egfem_tensor_destroy": [P],
        "egfem_tensor_info": [P, P, P, P, P, P],
        "egfem_tensor_csr_pattern": [P, pp, pp],
        "egfem_tensor_export": [P] * 10,
        "egfem_interp": [P, st, ctypes.c_double, P, P, P, P],
        "egfem_apply": [P, P, P, P, P],
        "egfem_apply_batched": [P, i32, st, P, P, P, P],
        "egfem_jacobian": [P, st, st, ctypes.c_double, P, P, P, P, P],
        "egfem_apply_jacobian": [P, st, st, ctypes.c_double, P, P, P, P, P, P],
        "egfem_partition": [P, i32, i32, st, pp, P, P, P, P, P, P],
        "egfem_partition_rows": [i64, P, i32, P],
        "egfem_halo_pack": [P, P, i64, P, P, P],
        "egfem_halo_unpack": [P, P, i64, P, P, P],
        "egfem_bilinear_build": [P, P, P],
        "egfem_csr_spmv": [P, P, P, P, P],
        "egfem_bilinear_jacobian": [P, P, st, ctypes.c_double, P, P, P],
        "egfem_interior": [P, P, P, P, P],
        "egfem_interp_range": [P, st, ctypes.c_double, P, P, P, i64, i64, P],
        "egfem_apply_jacobian_rows": [P, st, st, ctypes.c_double, P, P, P, P, P, i64, i64, P],
        "egfem_interior_rows": [i64, P, P, i64, i64, P, P],
        "egfem_kernel_name": [P, i32, st, st, ctypes.c_double, ctypes.c_char_p, ctypes.c_size_t],
        "egfem_group_compile": [P, i32, i32, i32],
        "egfem_step": [P, st, ctypes.c_double, P, P, P, P, P, P],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = st
    L.egfem_launch_count.restype = ctypes.c_uint64
    L.egfem_launch_count.argtypes = []
    L.egfem_status_string.restype = ctypes.c_char_p
    L.egfem_last_error.restype = ctypes.c_char_p
    return L


_lib = _load()


def lib():
    return _lib


def _check(fn, status):
    if status != 0:
        raise EgfemError(fn, status, _lib.egfem_last_error().decode())


def _np_ptr(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def _dptr(x):
    """Device pointer of a torch tensor (None -> NULL), unchecked (index buffers)."""
    if x is None:
        return None
    return ctypes.c_void_p(x.data_ptr())


def _buf(t, x, n, name, required=True):
    """Device pointer of a caller buffer after the checks the C ABI cannot make:
    a torch tensor on the handle's CUDA device, of the handle's dtype, contiguous, with at
    least `n` elements.  A failed check raises EgfemError(EGFEM_ERR_INVALID_ARGUMENT) before
    anything is launched, like the library's own validation.  None -> NULL (the library
    reports a missing required pointer itself)."""
    if x is None:
        return None
    bad = None
    if not x.is_cuda or x.device.index != t.device:
        bad = f"{name} must be on cuda:{t.device}, got {x.device}"
    elif x.dtype != t.torch_dtype:
        bad = f"{name} must be {t.torch_dtype}, got {x.dtype}"
    elif not x.is_contiguous():
        bad = f"{name} must be contiguous"
    elif x.numel() < n:
        bad = f"{name} has {x.numel()} elements, needs {n}"
    if bad:
        raise EgfemError("binding", 1, bad)
    return ctypes.c_void_p(x.data_ptr())


def _stream(stream, t=None):
    """The stream handle: a torch.cuda.Stream, a raw cudaStream_t int, or None = the current
    stream of the handle's device."""
    if stream is None:
        import torch
        dev = torch.device("cuda", t.device) if t is not None else None
        return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def _chain_len(t):
    return t.n_f * (t.dim + 1)


def launch_count() -> int:
    """Kernels this process launched through libegfem.so."""
    return int(_lib.egfem_launch_count())


class Tensor:
    """Owning handle of a device-resident EGFEM tensor T_ijk (egfem_tensor*)."""

    def __init__(self, handle, device, dim=0, n_cells=0, extra=None):
        self.h = handle
        self.device = device
        self.dim = dim
        self.n_cells = n_cells
        v = [np.zeros(1, np.int64) for _ in range(4)]
        dt = np.zeros(1, np.int32)
        _check("egfem_tensor_info", _lib.egfem_tensor_info(self.h, *[_np_ptr(x) for x in v], _np_ptr(dt)))
        self.n_u, self.n_f, self.nnz, self.nnz_csr = (int(x[0]) for x in v)
        self.dtype = int(dt[0])
        self.extra = extra or {}

    @property
    def torch_dtype(self):
        import torch
        return torch.float64 if self.dtype == F64 else torch.float32

    def close(self):
        if getattr(self, "h", None):
            _lib.egfem_tensor_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def csr_pattern(self):
        rp, col = ctypes.c_void_p(), ctypes.c_void_p()
        _check("egfem_tensor_csr_pattern", _lib.egfem_tensor_csr_pattern(self.h, ctypes.byref(rp), ctypes.byref(col)))
        return rp.value, col.value

    def export(self, slot_ik=False, loc=False, values=True):
        """Canonical host arrays (numpy) — SURVEY §8(a) A0 layout."""
        out = dict(t_row_ptr=np.zeros(self.n_u + 1, np.int64), t_j=np.zeros(self.nnz, np.int32),
                   t_k=np.zeros(self.nnz, np.int32),
                   t_val=np.zeros(self.nnz, np.float64 if self.dtype == F64 else np.float32) if values else None,
                   csr_row_ptr=np.zeros(self.n_u + 1, np.int64), csr_col=np.zeros(self.nnz_csr, np.int32),
                   slot_ij=np.zeros(self.nnz, np.int32),
                   slot_ik=np.zeros(self.nnz, np.int32) if slot_ik else None,
                   loc=np.zeros(self.nnz, np.uint8) if loc else None)
        keys = ["t_row_ptr", "t_j", "t_k", "t_val", "csr_row_ptr", "csr_col", "slot_ij", "slot_ik", "loc"]
        _check("egfem_tensor_export", _lib.egfem_tensor_export(self.h, *[_np_ptr(out[k]) for k in keys]))
        return {k: v for k, v in out.items() if v is not None}


def egfem_tensor_build(mesh, V, W, form, quad=None, dtype=F64, device=0) -> Tensor:
    """Assemble T on `device` (egfem_tensor_build)."""
    coords = np.ascontiguousarray(mesh.coords, np.float64)
    cells = np.ascontiguousarray(mesh.cells, np.int32)
    # cell_dofs None -> NULL: the canonical numbering (include/egfem.h egfem_space)
    vd = None if V.cell_dofs is None else np.ascontiguousarray(V.cell_dofs, np.int32)
    wd = None if W.cell_dofs is None else np.ascontiguousarray(W.cell_dofs, np.int32)
    m = _Mesh(mesh.dim, coords.shape[0], coords.ctypes.data, cells.shape[0], cells.ctypes.data)
    sv = _Space(V.family, V.n_dofs, None if vd is None else vd.ctypes.data)
    sw = _Space(W.family, W.n_dofs, None if wd is None else wd.ctypes.data)
    q = None
    if quad is not None:
        qb = np.ascontiguousarray(quad[0], np.float64)
        qw = np.ascontiguousarray(quad[1], np.float64)
        q = _Quad(len(qw), qb.ctypes.data, qw.ctypes.data)
    h = ctypes.c_void_p()
    _check("egfem_tensor_build", _lib.egfem_tensor_build(ctypes.byref(m), ctypes.byref(sv), ctypes.byref(sw), form,
                                                         ctypes.byref(q) if q is not None else None, dtype,
                                                         device, ctypes.byref(h)))
    return Tensor(h, device, mesh.dim, mesh.n_cells)


def egfem_tensor_from_coo(n_u, n_f, i, j, k, val, dtype=F64, device=0) -> Tensor:
    i, j, k = (np.ascontiguousarray(a, np.int32) for a in (i, j, k))
    val = np.ascontiguousarray(val, np.float64)
    h = ctypes.c_void_p()
    _check("egfem_tensor_from_coo", _lib.egfem_tensor_from_coo(n_u, n_f, len(val), _np_ptr(i), _np_ptr(j),
                                                               _np_ptr(k), _np_ptr(val), dtype, device,
                                                               ctypes.byref(h)))
    return Tensor(h, device)


def egfem_interp(t: Tensor, kind, p, u, w, chain=None, stream=None):
    """Step (1): w = f(Π_u u, Π_∇u ·₂ u)."""
    _check("egfem_interp", _lib.egfem_interp(t.h, kind, float(p), _buf(t, u, t.n_u, "u"), _buf(t, w, t.n_f, "w"),
                                             _buf(t, chain, _chain_len(t), "chain", False), _stream(stream, t)))


def egfem_apply(t: Tensor, u, w, r, stream=None):
    """Step (2): r = T:(u⊗w)."""
    _check("egfem_apply", _lib.egfem_apply(t.h, _buf(t, u, t.n_u, "u"), _buf(t, w, t.n_f, "w"), _buf(t, r, t.n_u, "r"),
                                           _stream(stream, t)))


def egfem_apply_batched(t: Tensor, batch, layout, U, W, R, stream=None):
    B = int(batch)
    _check("egfem_apply_batched", _lib.egfem_apply_batched(t.h, B, layout, _buf(t, U, B * t.n_u, "U"),
                                                           _buf(t, W, B * t.n_f, "W"), _buf(t, R, B * t.n_u, "R"),
                                                           _stream(stream, t)))


def egfem_jacobian(t: Tensor, mode, kind, p, u, w, chain, csr_vals, stream=None):
    """Step (3): A = T·w or J = T·w + (T·₂u)·D_u w into the CSR values."""
    _check("egfem_jacobian", _lib.egfem_jacobian(t.h, mode, kind, float(p), _buf(t, u, t.n_u, "u", False),
                                                 _buf(t, w, t.n_f, "w"), _buf(t, chain, _chain_len(t), "chain", False),
                                                 _buf(t, csr_vals, t.nnz_csr, "csr_vals"), _stream(stream, t)))


def egfem_bilinear_build(t: Tensor, b_vals, stream=None):
    """F3: the bilinear GFEM matrix B = T·₂1 on the CSR pattern (W = V)."""
    _check("egfem_bilinear_build", _lib.egfem_bilinear_build(t.h, _buf(t, b_vals, t.nnz_csr, "b_vals"),
                                                             _stream(stream, t)))


def egfem_csr_spmv(t: Tensor, vals, x, y, stream=None):
    """y = A x for values on the tensor's CSR pattern (the GFEM action r = B f)."""
    _check("egfem_csr_spmv", _lib.egfem_csr_spmv(t.h, _buf(t, vals, t.nnz_csr, "vals"), _buf(t, x, t.n_u, "x"),
                                                 _buf(t, y, t.n_u, "y"), _stream(stream, t)))


def egfem_bilinear_jacobian(t: Tensor, b_vals, kind, p, u, csr_vals, stream=None):
    """J = B·diag(f'(u)) for the GFEM term r = B f(u) (W = V)."""
    _check("egfem_bilinear_jacobian", _lib.egfem_bilinear_jacobian(t.h, _buf(t, b_vals, t.nnz_csr, "b_vals"), kind,
                                                                   float(p), _buf(t, u, t.n_u, "u"),
                                                                   _buf(t, csr_vals, t.nnz_csr, "csr_vals"),
                                                                   _stream(stream, t)))


def egfem_apply_jacobian(t: Tensor, mode, kind, p, u, w, chain, r, csr_vals, stream=None):
    _check("egfem_apply_jacobian", _lib.egfem_apply_jacobian(t.h, mode, kind, float(p), _buf(t, u, t.n_u, "u"),
                                                             _buf(t, w, t.n_f, "w"),
                                                             _buf(t, chain, _chain_len(t), "chain", False),
                                                             _buf(t, r, t.n_u, "r"),
                                                             _buf(t, csr_vals, t.nnz_csr, "csr_vals"),
                                                             _stream(stream, t)))


def egfem_step(t: Tensor, kind, p, u, w, chain, r, csr_vals, stream=None):
    """One Newton step's tensor work: egfem_interp then egfem_apply_jacobian(NEWTON) — in one
    launch (the single-pass kernel) where the tensor allows it."""
    _check("egfem_step", _lib.egfem_step(t.h, kind, float(p), _buf(t, u, t.n_u, "u"), _buf(t, w, t.n_f, "w"),
                                         _buf(t, chain, _chain_len(t), "chain", False), _buf(t, r, t.n_u, "r"),
                                         _buf(t, csr_vals, t.nnz_csr, "csr_vals"), _stream(stream, t)))


def egfem_interp_range(t: Tensor, kind, p, u, w, chain, lo, hi, stream=None):
    _check("egfem_interp_range", _lib.egfem_interp_range(t.h, kind, float(p), _buf(t, u, t.n_u, "u"),
                                                         _buf(t, w, t.n_f, "w"),
                                                         _buf(t, chain, _chain_len(t), "chain", False),
                                                         int(lo), int(hi), _stream(stream, t)))


def egfem_apply_jacobian_rows(t: Tensor, mode, kind, p, u, w, chain, r, csr_vals, row_lo, row_hi, stream=None):
    _check("egfem_apply_jacobian_rows",
           _lib.egfem_apply_jacobian_rows(t.h, mode, kind, float(p), _buf(t, u, t.n_u, "u"), _buf(t, w, t.n_f, "w"),
                                          _buf(t, chain, _chain_len(t), "chain", False), _buf(t, r, t.n_u, "r"),
                                          _buf(t, csr_vals, t.nnz_csr, "csr_vals"), int(row_lo), int(row_hi),
                                          _stream(stream, t)))


def egfem_interior(t: Tensor):
    """(row_lo, row_hi, w_lo, w_hi): the rows / interp items that read only owned u."""
    b = [np.zeros(1, np.int64) for _ in range(4)]
    _check("egfem_interior", _lib.egfem_interior(t.h, *[_np_ptr(x) for x in b]))
    return tuple(int(x[0]) for x in b)


def egfem_interior_rows(row_ptr, col, own_lo, own_hi):
    """Host helper: longest run of rows whose columns all lie in [own_lo, own_hi)."""
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    c = np.ascontiguousarray(col, dtype=np.int32)
    lo, hi = np.zeros(1, np.int64), np.zeros(1, np.int64)
    _check("egfem_interior_rows", _lib.egfem_interior_rows(len(rp) - 1, _np_ptr(rp), _np_ptr(c), int(own_lo),
                                                           int(own_hi), _np_ptr(lo), _np_ptr(hi)))
    return int(lo[0]), int(hi[0])


def egfem_partition_rows(prefix, nranks):
    """nnz-balanced contiguous row split (host only)."""
    prefix = np.ascontiguousarray(prefix, np.int64)
    out = np.zeros(nranks + 1, np.int64)
    _check("egfem_partition_rows", _lib.egfem_partition_rows(len(prefix) - 1, _np_ptr(prefix), nranks, _np_ptr(out)))
    return out


def egfem_partition(t: Tensor, nranks, rank, device=None):
    """Rank `rank`'s local tensor and its windows (row_begin, row_end, col_begin, col_end, w_begin, w_end)."""
    device = t.device if device is None else device
    h = ctypes.c_void_p()
    b = [np.zeros(1, np.int64) for _ in range(6)]
    _check("egfem_partition", _lib.egfem_partition(t.h, nranks, rank, device, ctypes.byref(h),
                                                   *[_np_ptr(x) for x in b]))
    names = ("row_begin", "row_end", "col_begin", "col_end", "w_begin", "w_end")
    win = {n: int(x[0]) for n, x in zip(names, b)}
    return Tensor(h, device, t.dim, 0, extra=win), win


def egfem_halo_pack(t: Tensor, idx, u_local, send_buf, stream=None):
    _check("egfem_halo_pack", _lib.egfem_halo_pack(t.h, _dptr(idx), idx.numel(), _buf(t, u_local, 0, "u_local"),
                                                   _buf(t, send_buf, idx.numel(), "send_buf"), _stream(stream, t)))


def egfem_halo_unpack(t: Tensor, idx, recv_buf, u_local, stream=None):
    _check("egfem_halo_unpack", _lib.egfem_halo_unpack(t.h, _dptr(idx), idx.numel(),
                                                       _buf(t, recv_buf, idx.numel(), "recv_buf"),
                                                       _buf(t, u_local, 0, "u_local"), _stream(stream, t)))


def egfem_kernel_name(t: Tensor, entry, mode=JAC_NEWTON, kind=INTERP_IDENTITY, p=0.0) -> str:
    """Kernel family an entry point runs for this handle (0 apply, 1 jacobian, 2 apply_jacobian,
    3 apply_batched node-major, 4 step, 5 interp); bench.py names its roofline kernel with it."""
    buf = ctypes.create_string_buffer(2048)
    _check("egfem_kernel_name", _lib.egfem_kernel_name(t.h, int(entry), mode, kind, float(p), buf, 2048))
    return buf.value.decode()


def egfem_group_compile(key, pairs_per_lane=2, f64=True):
    """NVRTC-compile the generated row-group kernel of one pattern (serialized key; no GPU needed)."""
    k = np.ascontiguousarray(key, np.int32)
    _check("egfem_group_compile", _lib.egfem_group_compile(_np_ptr(k), len(k), int(pairs_per_lane), int(bool(f64))))
