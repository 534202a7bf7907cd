"""Hash the cell-major kernels' outputs (apply, Picard, Newton, fused) on full-size cfg3 / cfg4 in
fp64 and fp32, for test_gpu_parity.py::test_packed_words_bitwise: run once with the packed 64-bit
row words (default) and once with EGFEM_CELLS_WORDS=0 (the staged K / (fiber, position) slices);
the two kernels do the same arithmetic in the same order, so the hashes must agree."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import egfem_inputs as I  # noqa: E402
import paper_2005_06193_b200 as eg  # noqa: E402

for name in ("cfg3", "cfg4"):
    pr = I.make_problem(name)
    for dt in (eg.F64, eg.F32):
        td = torch.float64 if dt == eg.F64 else torch.float32
        t = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, dtype=dt, device=0)
        u = torch.tensor(pr.u, dtype=td, device="cuda")
        w = torch.empty(t.n_f, dtype=td, device="cuda")
        chain = torch.empty(t.n_f * (pr.mesh.dim + 1), dtype=td, device="cuda")
        eg.egfem_interp(t, pr.interp, pr.p, u, w, chain)
        h = hashlib.sha256()
        r = torch.empty(t.n_u, dtype=td, device="cuda")
        J = torch.empty(t.nnz_csr, dtype=td, device="cuda")
        for step in range(4):
            r.fill_(float("nan"))
            J.fill_(float("nan"))
            if step == 0:
                eg.egfem_apply(t, u, w, r)
            elif step == 1:
                eg.egfem_jacobian(t, eg.JAC_PICARD, pr.interp, pr.p, None, w, None, J)
            elif step == 2:
                eg.egfem_jacobian(t, eg.JAC_NEWTON, pr.interp, pr.p, u, w, chain, J)
            else:
                eg.egfem_apply_jacobian(t, eg.JAC_NEWTON, pr.interp, pr.p, u, w, chain, r, J)
            torch.cuda.synchronize()
            h.update(r.cpu().numpy().tobytes())
            h.update(J.cpu().numpy().tobytes())
        print("hash", name, "f64" if dt == eg.F64 else "f32", eg.egfem_kernel_name(t, 2, eg.JAC_NEWTON, pr.interp, pr.p),
              h.hexdigest(), flush=True)
        del t
