"""Host cost per call of the C ABI (validation + launch) and of the Python binding's checks,
on cfg1 (37 KB: the kernel itself is ~2 µs, so the loop is host-bound)."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import egfem_inputs as I
import paper_2005_06193_b200 as eg

pr = I.make_problem("cfg1")
t = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, device=0)
u = torch.tensor(pr.u, device="cuda")
w = u.clone()
r = torch.empty_like(u)
s = torch.cuda.current_stream()
N = 5000
for _ in range(100):
    eg.egfem_apply(t, u, w, r, s)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(N):
    eg.egfem_apply(t, u, w, r, s)
t1 = time.perf_counter()
torch.cuda.synchronize()
L = eg.lib()
pu, pw, pr_, ps = (ctypes.c_void_p(x.data_ptr()) for x in (u, w, r)), None, None, ctypes.c_void_p(s.cuda_stream)
pu, pw, pr_ = ctypes.c_void_p(u.data_ptr()), ctypes.c_void_p(w.data_ptr()), ctypes.c_void_p(r.data_ptr())
t2 = time.perf_counter()
for _ in range(N):
    L.egfem_apply(t.h, pu, pw, pr_, ps)
t3 = time.perf_counter()
torch.cuda.synchronize()
print({"binding_us_per_call": (t1 - t0) / N * 1e6, "c_abi_us_per_call": (t3 - t2) / N * 1e6,
       "python_checks_us": ((t1 - t0) - (t3 - t2)) / N * 1e6})
