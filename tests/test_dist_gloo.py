"""Multi-process host logic of the row-partitioned driver on CPU with gloo.

world_size 2 and 3: every rank owns a contiguous row range and a column window; after
halo_exchange each rank's u_local must equal the global u on its whole window, and the
plans must be symmetric (what r sends to s is what s receives from r)."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _windows(n, nranks, reach):
    from paper_2005_06193_b200.dist import Window
    b = np.linspace(0, n, nranks + 1).astype(int)
    return [Window(int(b[r]), int(b[r + 1]), max(0, int(b[r]) - reach), min(n, int(b[r + 1]) + reach))
            for r in range(nranks)]


def test_plan_symmetry_and_coverage():
    from paper_2005_06193_b200.dist import make_plan
    for nranks, reach in ((2, 5), (4, 30), (5, 200), (8, 3)):
        n = 300
        ws = _windows(n, nranks, reach)
        plans = [make_plan(ws, r) for r in range(nranks)]
        for r, p in enumerate(plans):
            covered = np.zeros(p.n_local, bool)
            o = p.owned_offset
            covered[o:o + ws[r].row_end - ws[r].row_begin] = True
            for s, off, m in p.recvs:
                assert not covered[off:off + m].any()
                covered[off:off + m] = True
                # the sender's matching entry
                match = [x for x in plans[s].sends if x[0] == r]
                assert len(match) == 1 and match[0][2] == m
                assert ws[s].col_begin + match[0][1] == ws[r].col_begin + off
            assert covered.all()


def _worker(rank, world, port, n, reach, q):
    import torch
    import torch.distributed as dist

    from paper_2005_06193_b200.dist import Window, gather_windows, halo_exchange, make_plan
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        u = torch.arange(n, dtype=torch.float64) * 1.5 + 7
        b = np.linspace(0, n, world + 1).astype(int)
        me = Window(int(b[rank]), int(b[rank + 1]), max(0, int(b[rank]) - reach), min(n, int(b[rank + 1]) + reach))
        ws = gather_windows(me)
        plan = make_plan(ws, rank)
        ul = torch.full((plan.n_local,), float("nan"), dtype=torch.float64)
        o = plan.owned_offset
        ul[o:o + me.row_end - me.row_begin] = u[me.row_begin:me.row_end]
        halo_exchange(plan, ul)
        q.put((rank, bool(torch.equal(ul, u[me.col_begin:me.col_end]))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,reach", [(2, 17), (3, 40), (3, 400)])
def test_halo_exchange_gloo(world, reach):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 1000, reach, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(res.values()), res


def _overlap_worker(rank, world, port, n, reach, q):
    import torch
    import torch.distributed as dist

    import paper_2005_06193_b200 as eg
    from paper_2005_06193_b200.dist import Window, gather_windows, make_plan, overlapped_step
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        u = torch.sin(torch.arange(n, dtype=torch.float64)) + 2.0
        b = np.linspace(0, n, world + 1).astype(int)
        me = Window(int(b[rank]), int(b[rank + 1]), max(0, int(b[rank]) - reach), min(n, int(b[rank + 1]) + reach))
        plan = make_plan(gather_windows(me), rank)
        ul = torch.full((plan.n_local,), float("nan"), dtype=torch.float64)
        o, nr = plan.owned_offset, me.row_end - me.row_begin
        ul[o:o + nr] = u[me.row_begin:me.row_end]
        # a banded operator on the owned rows, columns in the local window
        rp, col, val = [0], [], []
        for i in range(me.row_begin, me.row_end):
            for j in range(max(0, i - reach), min(n, i + reach + 1)):
                col.append(j - me.col_begin)
                val.append(1.0 / (1 + abs(i - j)) + 1e-3 * i)
            rp.append(len(col))
        rp, col, val = np.array(rp), np.array(col, np.int32), torch.tensor(val, dtype=torch.float64)
        lo, hi = eg.egfem_interior_rows(rp, col, o, o + nr)
        r = torch.full((nr,), float("nan"), dtype=torch.float64)
        seen_nan = []

        def rows(a, z):
            for i in range(a, z):
                cs = torch.from_numpy(col[rp[i]:rp[i + 1]].astype(np.int64))
                r[i] = (val[rp[i]:rp[i + 1]] * ul[cs]).sum()

        def interior():
            rows(lo, hi)
            seen_nan.append(bool(torch.isnan(r[lo:hi]).any()))

        def boundary():
            rows(0, lo)
            rows(hi, nr)

        overlapped_step(plan, ul, interior, boundary)
        ug = u[me.col_begin:me.col_end]
        ref = torch.stack([(val[rp[i]:rp[i + 1]] * ug[torch.from_numpy(col[rp[i]:rp[i + 1]].astype(np.int64))]).sum()
                           for i in range(nr)])
        q.put((rank, (bool(torch.equal(r, ref)), not seen_nan[0], hi - lo)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,reach", [(2, 17), (3, 40), (3, 400)])
def test_overlapped_step_gloo(world, reach):
    """dist.overlapped_step with egfem_interior_rows' split: the interior rows, computed while the
    halo is in flight, read no halo entry (none is NaN-poisoned into them), and the step's result
    equals the serial one on every rank; with a reach wider than a rank (400) the interior is
    empty and the step degenerates to exchange-then-compute."""
    import multiprocessing as mp

    import __graft_entry__
    __graft_entry__.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_overlap_worker, args=(r, world, port, 600, reach, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for rank, (equal, clean, n_inner) in res.items():
        assert equal and clean, (rank, res)
        assert (n_inner > 0) == (reach < 100), (rank, n_inner)


class _MockEg:
    """Records the library calls of dist.split_step (no GPU): which interp items and rows each
    phase covers, and whether the halo had arrived when a call was made."""
    JAC_NEWTON = 1

    def __init__(self, ul, halo_mask):
        self.ul, self.halo = ul, halo_mask
        self.calls = []

    def _halo_ready(self):
        import torch
        return bool(not torch.isnan(self.ul[self.halo]).any())

    def egfem_interp_range(self, t, kind, p, u, w, chain, lo, hi, stream):
        self.calls.append(("interp", lo, hi, self._halo_ready()))

    def egfem_apply_jacobian_rows(self, t, mode, kind, p, u, w, chain, r, J, lo, hi, stream):
        self.calls.append(("rows", lo, hi, self._halo_ready()))


def _split_worker(rank, world, port, q):
    import types

    import torch
    import torch.distributed as dist

    from paper_2005_06193_b200.dist import Window, gather_windows, make_plan, split_step
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, reach = 400, 20
        b = np.linspace(0, n, world + 1).astype(int)
        me = Window(int(b[rank]), int(b[rank + 1]), max(0, int(b[rank]) - reach), min(n, int(b[rank + 1]) + reach))
        plan = make_plan(gather_windows(me), rank)
        ul = torch.full((plan.n_local,), float("nan"), dtype=torch.float64)
        o, nr = plan.owned_offset, me.row_end - me.row_begin
        ul[o:o + nr] = torch.arange(me.row_begin, me.row_end, dtype=torch.float64)
        halo = torch.ones(plan.n_local, dtype=torch.bool)
        halo[o:o + nr] = False
        eg = _MockEg(ul, halo)
        t = types.SimpleNamespace(n_u=nr, n_f=plan.n_local)
        split = (reach, nr - reach, o, o + nr)  # interior rows / items of a banded operator
        split_step(eg, t, plan, split, 0, 0.0, ul, None, None, None, None)
        q.put((rank, eg.calls, nr, plan.n_local, split))
    finally:
        dist.destroy_process_group()


def test_split_step_orchestration_gloo():
    """dist.split_step (the bench's N>1 step): the interior interp items and rows are issued
    before the halo is waited for, the boundary ones after it has arrived, and the ranges of
    each kind cover [0, n) exactly once."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_split_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    for rank, calls, nr, n_items, split in res:
        kinds = [c[0] for c in calls]
        assert kinds == ["interp", "rows", "interp", "interp", "rows", "rows"], calls
        assert all(c[3] for c in calls[2:]), calls  # boundary phase: halo in place
        for kind, n in (("interp", n_items), ("rows", nr)):
            cover = np.zeros(n, int)
            for c in calls:
                if c[0] == kind:
                    cover[c[1]:c[2]] += 1
            assert np.all(cover == 1), (kind, cover)
