"""Row-partitioned multi-GPU driver: one process per GPU, NCCL u-halo exchange.

T's rows are split into nnz-balanced contiguous ranges (egfem_partition).  Rank r
holds its rows and addresses a contiguous local vector u_local = u[col_begin:col_end)
(the structured lexicographic numbering makes the referenced columns one range), in
which its owned entries u[row_begin:row_end) sit at offset row_begin − col_begin.
Per iteration the only communication is the halo: every rank sends the part of its
owned range that each other rank's window covers — contiguous slices, so no pack
kernel is needed — with grouped point-to-point NCCL send/recv over NVLink.  w is not
exchanged: P0 W is recomputed locally from the window, W = V copies it.

This module holds only host logic (plans and torch.distributed calls); it runs on
CPU tensors under gloo for the multi-process tests.
"""
from __future__ import annotations

import dataclasses
from typing import List, Tuple


@dataclasses.dataclass(frozen=True)
class Window:
    row_begin: int
    row_end: int
    col_begin: int
    col_end: int


@dataclasses.dataclass
class HaloPlan:
    rank: int
    window: Window
    # (peer, local_offset, length): slices of u_local to send to / receive from peer
    sends: List[Tuple[int, int, int]]
    recvs: List[Tuple[int, int, int]]

    @property
    def n_local(self) -> int:
        return self.window.col_end - self.window.col_begin

    @property
    def owned_offset(self) -> int:
        return self.window.row_begin - self.window.col_begin

    @property
    def halo_values(self) -> int:
        return sum(n for _, _, n in self.recvs)


def make_plan(windows: List[Window], rank: int) -> HaloPlan:
    """Exchange plan of `rank` given every rank's window (deterministic, symmetric)."""
    me = windows[rank]
    sends, recvs = [], []
    for s, ws in enumerate(windows):
        if s == rank:
            continue
        # what `rank` needs from s: s's owned rows inside my window
        a, b = max(me.col_begin, ws.row_begin), min(me.col_end, ws.row_end)
        if a < b:
            recvs.append((s, a - me.col_begin, b - a))
        # what s needs from me: my owned rows inside s's window
        a, b = max(ws.col_begin, me.row_begin), min(ws.col_end, me.row_end)
        if a < b:
            sends.append((s, a - me.col_begin, b - a))
    return HaloPlan(rank, me, sends, recvs)


def gather_windows(win: Window, group=None) -> List[Window]:
    import torch
    import torch.distributed as dist
    ws = dist.get_world_size(group)
    be = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if be == "nccl" else torch.device("cpu")
    mine = torch.tensor([win.row_begin, win.row_end, win.col_begin, win.col_end], dtype=torch.int64, device=dev)
    allw = [torch.empty_like(mine) for _ in range(ws)]
    dist.all_gather(allw, mine, group=group)
    return [Window(*[int(x) for x in t.cpu().tolist()]) for t in allw]


def halo_start(plan: HaloPlan, u_local, group=None) -> list:
    """Post the halo exchange of u_local (grouped P2P send/recv of contiguous slices) and
    return its requests.  Under NCCL the transfers run on the communicator's stream, which
    first waits for the work already queued on the caller's stream (u is ready); kernels the
    caller queues next run concurrently with them."""
    import torch.distributed as dist
    ops = []
    for peer, off, n in plan.recvs:
        ops.append(dist.P2POp(dist.irecv, u_local[off:off + n], peer, group))
    for peer, off, n in plan.sends:
        ops.append(dist.P2POp(dist.isend, u_local[off:off + n], peer, group))
    return dist.batch_isend_irecv(ops) if ops else []


def halo_finish(reqs: list) -> None:
    """Wait for posted halo requests (NCCL: the caller's stream waits on the communicator's;
    gloo: the host blocks until the data is in place)."""
    for req in reqs:
        req.wait()


def halo_exchange(plan: HaloPlan, u_local, group=None) -> None:
    """Fill u_local's halo entries from their owners (grouped P2P send/recv)."""
    halo_finish(halo_start(plan, u_local, group))


def overlapped_step(plan: HaloPlan, u_local, interior, boundary, group=None) -> None:
    """One distributed step with the u-halo exchange hidden behind the interior work (§8(e)):
    post the exchange, run interior() — which must read owned entries of u_local only
    (egfem_interior's rows and interp items) — wait for the halo, run boundary()."""
    reqs = halo_start(plan, u_local, group)
    interior()
    halo_finish(reqs)
    boundary()


def split_step(eg, t, plan: HaloPlan, split, kind, p, u_local, w, chain, r, csr, stream=None, events=None,
               group=None) -> None:
    """One distributed step (interp + fused apply/Newton Jacobian) of a row-partitioned local
    tensor `t` with the u-halo exchange overlapped: `split` = egfem_interior(t) =
    (row_lo, row_hi, item_lo, item_hi).  The interior items / rows run while the halo is in
    flight; the boundary items [0, item_lo), [item_hi, n_items) and rows [0, row_lo),
    [row_hi, n_u) after it has arrived.  P0 local tensors: interp items are cells = W DOFs,
    W = V: W DOFs, so n_items = t.n_f.  `events` (optional, 4 CUDA events): [1] is recorded
    after the interior phase, [2] once the halo has arrived."""
    r0, r1, i0, i1 = split
    n_items = t.n_f

    def interior():
        eg.egfem_interp_range(t, kind, p, u_local, w, chain, i0, i1, stream)
        eg.egfem_apply_jacobian_rows(t, eg.JAC_NEWTON, kind, p, u_local, w, chain, r, csr, r0, r1, stream)
        if events:
            events[1].record(stream)

    def boundary():
        if events:
            events[2].record(stream)
        eg.egfem_interp_range(t, kind, p, u_local, w, chain, 0, i0, stream)
        eg.egfem_interp_range(t, kind, p, u_local, w, chain, i1, n_items, stream)
        eg.egfem_apply_jacobian_rows(t, eg.JAC_NEWTON, kind, p, u_local, w, chain, r, csr, 0, r0, stream)
        eg.egfem_apply_jacobian_rows(t, eg.JAC_NEWTON, kind, p, u_local, w, chain, r, csr, r1, t.n_u, stream)

    overlapped_step(plan, u_local, interior, boundary, group)
