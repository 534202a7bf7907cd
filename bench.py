#!/usr/bin/env python
"""EGFEM hot-path benchmark (BASELINE.json metric: tensor nonzeros/s and achieved HBM GB/s).

One step = one pass of the whole hot path (SURVEY §8(a) A1–A3) over the workload:
  (1) egfem_interp           w_K = |∇u_h|_K^{p−2} and D_u w       (GRADPOW_P0)
  (2)+(3) egfem_apply_jacobian  r = T:(u⊗w) and the Newton J = T·w + (T·₂u)·D_u w, fused
          into one pass over T (both outputs from a single stream of T's nonzeros).
Default workload: BASELINE configs[3] (3D p-Laplace p=3, 128³×6 tets, 201,326,592 nnz,
fp64) — the config the north star's headline target is quoted on ("≥70% of HBM at 1 GPU,
≥6× at 8 GPUs on the largest config"); it fits one B200.  Units: each step processes
2·nnz tensor nonzeros (apply + Jacobian, reading C25).

N>1 (torchrun): T's rows are partitioned (egfem_partition), each step adds the NCCL u-halo
exchange; value = all ranks' nonzeros / max-over-ranks device time ("scaling": "strong").

--impl reference: the CPU oracle (oracle/, test infrastructure) on a bounded row sample of
the same workload, timed on the host cores (rank 0 only).
"""
import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import egfem_inputs as I  # noqa: E402

ORACLE_SAMPLE_ROWS = 200_000


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _fp64_peak():
    """FP64 FMA peak: profiles/fp64_peak.json (tools/fp64_peak on this pool's B200) if present,
    else 148 SMs x 64 DFMA/clk x 2 x 1.965 GHz."""
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as f:
            return float(json.load(f)["fp64_fma_tflops"]), "measured (tools/fp64_peak)"
    except Exception:
        return 148 * 64 * 2 * 1.965e9 / 1e12, "derived (148 SM x 64 DFMA/clk x 1.965 GHz)"


def _traffic(workload, kernel):
    """Per-launch DRAM bytes from the committed ncu --set full summary, if any."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(workload, {}).get(kernel)
    except Exception:
        return None


class ClockSampler:
    """Samples SM clock + throttle reasons with NVML every ~2 ms during the timed region."""

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _sample(self):
        nv = self.nv
        self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        names = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                 "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}
        for k, bit in names.items():
            if r & bit:
                self.reasons.add(k)

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:
                return
            time.sleep(0.002)

    def __enter__(self):
        if self.nv:
            self._sample()
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self._stop.set()
            self.t.join()
            self._sample()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def algorithmic_bytes(t, pr, s, kind):
    """Minimal DRAM bytes of one launch in the CSF layout (DESIGN.md §5/§7).

    per nonzero: k (4) + value (s); per fiber: column (4) + offset (4); per row: offset (8);
    vectors read/written once.  kind: 'apply' | 'jac' (Newton) | 'fused' | 'interp'."""
    d1 = pr.mesh.dim + 1
    T = t.nnz * (4 + s) + t.nnz_csr * 8 + (t.n_u + 1) * 8
    if kind == "apply":
        return T + s * (2 * t.n_u + t.n_f)
    if kind == "jac":
        return T + s * (t.n_u + t.n_f + d1 * t.n_f) + s * t.nnz_csr
    if kind == "fused":
        return T + s * (2 * t.n_u + t.n_f + d1 * t.n_f) + s * t.nnz_csr
    if kind == "interp":  # cells (int32) + w + chain written + u and coords read
        return pr.mesh.n_cells * (4 * d1 + s * (1 + d1)) + t.n_u * (s + 8 * pr.mesh.dim)
    raise ValueError(kind)


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2005_06193_b200 as eg
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    pr = I.make_problem(args.config, batch=args.batch)
    dtype = eg.F64 if args.dtype == "f64" else eg.F32
    td = torch.float64 if dtype == eg.F64 else torch.float32
    s = 8 if dtype == eg.F64 else 4
    t0 = time.time()
    tg = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, dtype=dtype, device=local)
    torch.cuda.synchronize()
    build_s = time.time() - t0
    nnz_total = tg.nnz
    plan = None
    if world > 1:
        from paper_2005_06193_b200 import dist as edist
        t, win = eg.egfem_partition(tg, world, rank, local)
        del tg
        torch.cuda.empty_cache()
        W = edist.Window(win["row_begin"], win["row_end"], win["col_begin"], win["col_end"])
        plan = edist.make_plan(edist.gather_windows(W), rank)
        u_np = pr.u[win["col_begin"]:win["col_end"]]
        u_own = np.zeros_like(u_np)
        o = plan.owned_offset
        u_own[o:o + win["row_end"] - win["row_begin"]] = u_np[o:o + win["row_end"] - win["row_begin"]]
        u_np = u_own  # halos arrive through the exchange
    else:
        t = tg
        u_np = pr.u if not pr.batch else pr.u[0]
    batched = args.config == "cfg5"
    if batched:
        return run_batched(args, eg, t, pr, dev, td, s, build_s, world, rank)
    if args.config == "gfem2d" and world == 1:
        return run_gfem(args, eg, t, pr, dev, td, s, build_s)
    u = torch.tensor(u_np, dtype=td, device=dev)
    w = torch.empty(t.n_f, dtype=td, device=dev)
    gp = pr.W.family in (I.P0, I.QUAD) and pr.interp in (I.INTERP_GRADPOW_P0, I.INTERP_MINSURF_P0,
                                                         I.INTERP_RECIPROCAL, I.INTERP_SQUARE)
    chain = torch.empty(t.n_f * (pr.mesh.dim + 1), dtype=td, device=dev) if gp else None
    r = torch.empty(t.n_u, dtype=td, device=dev)
    J = torch.empty(t.nnz_csr, dtype=td, device=dev)
    stream = torch.cuda.current_stream(dev)

    if plan is not None:
        from paper_2005_06193_b200 import dist as edist
        # interior rows / interp items read owned u only: they run while the halo is in flight
        ir0, ir1, iw0, iw1 = eg.egfem_interior(t)

    def dist_step(ux, rx, e=None):
        """N>1: post the u-halo exchange, run the interior phase, wait for the halo (the
        compute stream waits on the communicator's), run the boundary phase."""
        edist.split_step(eg, t, plan, (ir0, ir1, iw0, iw1), pr.interp, pr.p, ux, w, chain, rx, J, stream, e)

    K, Wm = args.steps, args.warmup
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(K)]

    def step(e=None):
        if e:
            e[0].record(stream)
        if plan is not None:
            dist_step(u, r, e)
        else:
            eg.egfem_interp(t, pr.interp, pr.p, u, w, chain, stream)
            if e:
                e[2].record(stream)
            eg.egfem_apply_jacobian(t, eg.JAC_NEWTON, pr.interp, pr.p, u, w, chain, r, J, stream)
        if e:
            e[3].record(stream)

    # Timing rule: inputs larger than L2 or an L2 flush between timed steps.  The per-step working
    # set (T stream + vectors) of cfg4 is GBs; for the smaller configs a 512 MB write evicts L2
    # between steps and the step time is the sum of the per-step event intervals (flush excluded).
    ws_bytes = algorithmic_bytes(t, pr, s, "fused") + algorithmic_bytes(t, pr, s, "interp")
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = ws_bytes < 4 * l2_bytes
    scratch = torch.empty(512 << 20, dtype=torch.uint8, device=dev) if flush else None
    for _ in range(Wm):
        step()
    torch.cuda.synchronize()
    # Single GPU: each kernel of the step (interp, fused apply/Jacobian) is captured once into a
    # CUDA graph and replayed (no per-launch CPU overhead; matters for the small configs), with
    # CUDA events between the two replays so both kernels are timed inside the timed region.
    # N>1 keeps eager launches around the NCCL halo exchange.
    graph = None
    if world == 1 and not args.no_graph:
        side = torch.cuda.Stream(dev)
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            step()  # warm-up on the capture stream's family
        stream.wait_stream(side)
        torch.cuda.synchronize()
        graph = (torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph())
        with torch.cuda.graph(graph[0]):
            eg.egfem_interp(t, pr.interp, pr.p, u, w, chain, torch.cuda.current_stream(dev))
        with torch.cuda.graph(graph[1]):
            eg.egfem_apply_jacobian(t, eg.JAC_NEWTON, pr.interp, pr.p, u, w, chain, r, J,
                                    torch.cuda.current_stream(dev))
        torch.cuda.synchronize()
        for _ in range(Wm):
            graph[0].replay()
            graph[1].replay()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = eg.launch_count()
    with ClockSampler(local) as clk:
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record(stream)
        for k in range(K):
            if flush:
                scratch.zero_()
            if graph is not None:
                ev[k][0].record(stream)
                graph[0].replay()
                ev[k][2].record(stream)
                graph[1].replay()
                ev[k][3].record(stream)
            else:
                step(ev[k])
        stop.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches = eg.launch_count() - l0 if graph is None else 2 * K  # graph replays launch interp + fused
    ms = sum(e[0].elapsed_time(e[3]) for e in ev) if flush else start.elapsed_time(stop)
    phases = None
    if plan is not None:
        phases = {"interior_phase": float(np.mean([e[0].elapsed_time(e[1]) for e in ev])),
                  "exposed_halo_wait": float(np.mean([e[1].elapsed_time(e[2]) for e in ev])),
                  "boundary_phase": float(np.mean([e[2].elapsed_time(e[3]) for e in ev])),
                  "interior_rows": ir1 - ir0, "rows": t.n_u}
    if world > 1:
        m = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
        ms = float(m.item())
    units = 2 * nnz_total * K
    value = units / (ms * 1e-3)

    # separate apply / Jacobian launches (explanatory, outside the headline region)
    def avg_ms(fn, n=max(5, min(K, 50))):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fn()
        torch.cuda.synchronize()
        a.record(stream)
        for _ in range(n):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / n
    if plan is None:  # the step's two kernels, timed by the events inside the timed region
        t_interp = float(np.mean([e[0].elapsed_time(e[2]) for e in ev]))
        t_fused = float(np.mean([e[2].elapsed_time(e[3]) for e in ev]))
    else:  # N>1 splits them into phases: whole-range launches, outside the timed region
        t_interp = avg_ms(lambda: eg.egfem_interp(t, pr.interp, pr.p, u, w, chain, stream))
        t_fused = avg_ms(lambda: eg.egfem_apply_jacobian(t, eg.JAC_NEWTON, pr.interp, pr.p, u, w, chain, r, J,
                                                         stream))
    t_apply = avg_ms(lambda: eg.egfem_apply(t, u, w, r, stream))
    t_jac = avg_ms(lambda: eg.egfem_jacobian(t, eg.JAC_NEWTON, pr.interp, pr.p, u, w, chain, J, stream))
    t_pic = avg_ms(lambda: eg.egfem_jacobian(t, eg.JAC_PICARD, pr.interp, pr.p, None, w, None, J, stream))

    # end to end: every step copies its input u from pinned host memory and its result r back to
    # pinned host memory.  The copies run on their own streams with u and r double-buffered, so
    # step k's H2D and D2H overlap the compute of steps k±1 (PCIe is full duplex).
    u_host = torch.tensor(u_np, dtype=td).pin_memory()
    r_host = [torch.empty(t.n_u, dtype=td).pin_memory() for _ in range(2)]
    ub, rb = [u, torch.empty_like(u)], [r, torch.empty_like(r)]
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    ev_in, ev_c, ev_out = ([torch.cuda.Event() for _ in range(K)] for _ in range(3))

    def step_on(ux, rx):
        if plan is not None:
            dist_step(ux, rx)
            return
        eg.egfem_interp(t, pr.interp, pr.p, ux, w, chain, stream)
        eg.egfem_apply_jacobian(t, eg.JAC_NEWTON, pr.interp, pr.p, ux, w, chain, rx, J, stream)

    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    s_in.wait_event(a)
    s_out.wait_event(a)
    for k in range(K):
        x = k % 2
        if k >= 2:
            s_in.wait_event(ev_c[k - 2])  # step k-2's compute is done reading ub[x]
        with torch.cuda.stream(s_in):
            ub[x].copy_(u_host, non_blocking=True)
        ev_in[k].record(s_in)
        stream.wait_event(ev_in[k])
        if k >= 2:
            stream.wait_event(ev_out[k - 2])  # rb[x] has been read out
        step_on(ub[x], rb[x])
        ev_c[k].record(stream)
        s_out.wait_event(ev_c[k])
        with torch.cuda.stream(s_out):
            r_host[x].copy_(rb[x], non_blocking=True)
        ev_out[k].record(s_out)
    stream.wait_event(ev_out[K - 1])
    b.record(stream)
    torch.cuda.synchronize()
    e2e_ms = a.elapsed_time(b)
    if world > 1:
        m = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
        e2e_ms = float(m.item())

    peak, peak_kind = _peaks()
    fused_bytes = algorithmic_bytes(t, pr, s, "fused")
    achieved = fused_bytes / (t_fused * 1e-3) / 1e9
    workload = f"{args.config}-{args.dtype}"
    out = {
        "metric": "tensor nonzeros/s (apply + Newton Jacobian, 2 x nnz per step) and achieved HBM GB/s",
        "value": value, "unit": "nnz/s", "n_gpus": world, "steps": K, "warmup": Wm,
        "ms_per_step": ms / K, "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": args.dtype, "data": "synthetic (seeded, BASELINE.json recipe)",
        "config": {"workload": workload, "description": pr.description, "nnz": nnz_total,
                   "nnz_csr": t.nnz_csr if world == 1 else None, "n_u": pr.n_u, "n_f": pr.n_f,
                   "step": "interp(GRADPOW_P0 + D_u w) + fused apply/Newton-Jacobian" +
                           (" + NCCL u-halo overlapped with the interior rows" if world > 1 else ""),
                   "l2": (f"working set {ws_bytes / 1e9:.2f} GB < 4 x L2 ({l2_bytes >> 20} MB): 512 MB write "
                          "between timed steps, step time = sum of per-step intervals") if flush else
                         f"working set {ws_bytes / 1e9:.2f} GB >= 4 x L2 ({l2_bytes >> 20} MB); no flush",
                   "parallelism": f"row-partition x{world}" if world > 1 else "single GPU",
                   "launch": "CUDA graphs (interp; fused) replayed per step, events between" if graph is not None else "eager"},
        "roofline": {"bound": "hbm", "kernel": "k_cell<S,D1,G,CPL,FREG,DO_R=1,NewtonP0> (egfem_apply_jacobian, cell-major P0 path)",
                     "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": achieved / peak, "algorithmic_bytes": fused_bytes,
                     "traffic": _traffic(workload, "fused")},
        "kernels_ms": {"interp": t_interp, "apply_jacobian_fused": t_fused,
                       "apply": t_apply, "jacobian_newton": t_jac, "jacobian_picard": t_pic},
        "kernels_gbs": {"interp": algorithmic_bytes(t, pr, s, "interp") / (t_interp * 1e-3) / 1e9,
                        "apply": algorithmic_bytes(t, pr, s, "apply") / (t_apply * 1e-3) / 1e9,
                        "jacobian_newton": algorithmic_bytes(t, pr, s, "jac") / (t_jac * 1e-3) / 1e9,
                        "apply_nnz_per_s": t.nnz / (t_apply * 1e-3)},
        "e2e": {"value": units / (e2e_ms * 1e-3), "unit": "nnz/s", "h2d_bytes_per_step": u.numel() * s,
                "d2h_bytes_per_step": r.numel() * s, "ms_per_step": e2e_ms / K,
                "overlap": "H2D/D2H on copy streams, u and r double-buffered"},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "build_s": build_s,
    }
    if plan is not None:
        out["config"]["halo_values_per_rank"] = plan.halo_values
        out["phases_ms"] = phases
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(pr)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_batched(args, eg, t, pr, dev, td, s, build_s, world, rank):
    """cfg5: batched action, B pairs sharded across ranks (T replicated, no communication)."""
    import torch
    import torch.distributed as dist
    B = pr.batch
    lo, hi = rank * B // world, (rank + 1) * B // world
    Bl = hi - lo
    U = torch.tensor(np.ascontiguousarray(pr.u[lo:hi].T), dtype=td, device=dev)  # node-major
    R = torch.empty_like(U)
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        eg.egfem_apply_batched(t, Bl, eg.LAYOUT_NODE_MAJOR, U, U, R, stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    l0 = eg.launch_count()
    with ClockSampler(dev.index) as clk:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.steps):
            eg.egfem_apply_batched(t, Bl, eg.LAYOUT_NODE_MAJOR, U, U, R, stream)
        b.record(stream)
        torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    if world > 1:
        m = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
        ms = float(m.item())
    units = t.nnz * B * args.steps
    # end to end: this rank's pairs from pinned host memory, the action, R back to pinned host memory
    U_host = U.cpu().pin_memory()
    R_host = torch.empty(R.shape, dtype=td).pin_memory()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a2, b2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a2.record(stream)
    for _ in range(args.steps):
        U.copy_(U_host, non_blocking=True)
        eg.egfem_apply_batched(t, Bl, eg.LAYOUT_NODE_MAJOR, U, U, R, stream)
        R_host.copy_(R, non_blocking=True)
    b2.record(stream)
    torch.cuda.synchronize()
    e2e_ms = a2.elapsed_time(b2)
    if world > 1:
        m = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
        e2e_ms = float(m.item())
    byts = t.nnz * (4 + s) + t.nnz_csr * 8 + (t.n_u + 1) * 8 + s * (2 * t.n_u * Bl + t.n_f * Bl)
    flops = 2 * (t.nnz + t.nnz_csr) * Bl  # fiber-factored: per pair, an FMA per nonzero and per fiber
    per = ms / args.steps
    peak, kind = _peaks()
    fpeak, fkind = _fp64_peak()
    out = {"metric": "tensor nonzero-pairs/s (batched action) and achieved HBM GB/s", "value": units / (ms * 1e-3),
           "unit": "nnz*pair/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": per, "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
           "vs_baseline": None, "dtype": args.dtype, "data": "synthetic (seeded, BASELINE.json recipe)",
           "config": {"workload": f"cfg5-{args.dtype}", "batch": B, "nnz": t.nnz, "parallelism": f"batch-shard x{world}",
                      "l2": "inputs larger than L2 (T 0.3 GB + U, R 0.54 GB each); no flush"},
           "e2e": {"value": units / (e2e_ms * 1e-3), "unit": "nnz*pair/s", "h2d_bytes_per_step": U.numel() * s,
                   "d2h_bytes_per_step": R.numel() * s},
           "roofline": {"bound": "alu", "kernel": "k_dense<double,NODE_MAJOR> (egfem_apply_batched)",
                        "achieved": flops / (per * 1e-3) / 1e12, "peak": fpeak, "peak_kind": fkind,
                        "unit": "TFLOP/s", "frac": flops / (per * 1e-3) / 1e12 / fpeak,
                        "algorithmic_flops": flops, "traffic": None},
           "roofline_hbm": {"achieved": byts / (per * 1e-3) / 1e9, "peak": peak, "peak_kind": kind, "unit": "GB/s",
                            "frac": byts / (per * 1e-3) / 1e9 / peak, "algorithmic_bytes": byts},
           "gpu_launches": int(eg.launch_count() - l0), "clocks": clk.summary(), "build_s": build_s}
    if rank == 0:
        print(json.dumps(out), flush=True)


def run_gfem(args, eg, t, pr, dev, td, s, build_s):
    """F3: the GFEM (matrix) form of the Burgers term, r = N^f f with f = u² and J = N^f·diag(2u)
    (PAPER.md L402–409), timed beside the tensor form T:(u⊗u) + Newton Jacobian on the same mesh
    (the paper's tensor-vs-matrix comparison, L432).  Units: tensor nonzeros of the tensor form per
    step (2·nnz for apply + Jacobian), so both forms are on the same scale."""
    import torch
    stream = torch.cuda.current_stream(dev)
    u = torch.tensor(pr.u, dtype=td, device=dev)
    f = torch.empty(t.n_f, dtype=td, device=dev)
    r = torch.empty(t.n_u, dtype=td, device=dev)
    B = torch.empty(t.nnz_csr, dtype=td, device=dev)
    J = torch.empty(t.nnz_csr, dtype=td, device=dev)
    eg.egfem_bilinear_build(t, B, stream)

    def matrix_step():
        eg.egfem_interp(t, pr.interp, pr.p, u, f, None, stream)
        eg.egfem_csr_spmv(t, B, f, r, stream)
        eg.egfem_bilinear_jacobian(t, B, pr.interp, pr.p, u, J, stream)

    def tensor_step():
        eg.egfem_apply_jacobian(t, eg.JAC_NEWTON, eg.INTERP_IDENTITY, 0.0, u, u, None, r, J, stream)

    # the working set (~0.1 GB) fits L2: a 512 MB write between timed steps, per-step intervals summed
    scratch = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

    def timed(fn, K):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        for a, b in evs:
            scratch.zero_()
            a.record(stream)
            fn()
            b.record(stream)
        torch.cuda.synchronize()
        return sum(a.elapsed_time(b) for a, b in evs)
    l0 = eg.launch_count()
    with ClockSampler(dev.index) as clk:
        ms = timed(matrix_step, args.steps)
    launches = eg.launch_count() - l0
    ms_tensor = timed(tensor_step, args.steps)
    K = args.steps
    units = 2 * t.nnz * K
    # matrix step bytes: f from u (2 s N_u), B + cols (s+4) nnz_csr, row ptr, f gathered, r; J: B, cols, u, J
    byts = 2 * s * t.n_u + (s + 4) * t.nnz_csr + 8 * (t.n_u + 1) + 2 * s * t.n_u + (2 * s + 4) * t.nnz_csr + s * t.n_u
    peak, kind = _peaks()
    per = ms / K
    out = {"metric": "tensor nonzeros/s (GFEM matrix form of the same term, 2 x nnz(T) per step)",
           "value": units / (ms * 1e-3), "unit": "nnz/s", "n_gpus": 1, "steps": K, "warmup": args.warmup,
           "ms_per_step": per, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": args.dtype,
           "data": "synthetic (seeded)",
           "config": {"workload": f"{args.config}-{args.dtype}", "description": pr.description, "nnz": t.nnz,
                      "nnz_csr": t.nnz_csr, "step": "interp(SQUARE) + CSR SpMV r = N^f f + J = N^f diag(2u)",
                      "l2": "512 MB write between timed steps; step time = sum of per-step intervals"},
           "roofline": {"bound": "hbm", "kernel": "k_spmv + k_scale_cols (egfem_csr_spmv, egfem_bilinear_jacobian)",
                        "achieved": byts / (per * 1e-3) / 1e9, "peak": peak, "peak_kind": kind, "unit": "GB/s",
                        "frac": byts / (per * 1e-3) / 1e9 / peak, "algorithmic_bytes": byts, "traffic": None},
           "kernels_ms": {"matrix_step": per, "tensor_step_fused_apply_newton": ms_tensor / K},
           "gpu_launches": int(launches), "clocks": clk.summary(), "build_s": build_s}
    print(json.dumps(out), flush=True)


def cpu_baseline(pr, rows=ORACLE_SAMPLE_ROWS, steps=1):
    """The CPU oracle as it stands (single thread) on rows [0, rows) of the same workload."""
    import oracle
    o = oracle.OracleTensor(pr.mesh, pr.V, pr.W, pr.form, rows=(0, rows))
    t0 = time.time()
    for _ in range(steps):
        w = o.interp(pr.interp, pr.p, pr.u)
        o.apply(pr.u, w)
        o.jacobian(1, pr.interp, pr.p, pr.u, w)
    dt = (time.time() - t0) / steps
    return {"value": 2 * o.nnz / dt, "unit": "nnz/s", "cores": 1, "kind": "oracle",
            "sample": f"{pr.name} rows [0,{rows}) = {o.nnz} nnz; interp over all {pr.mesh.n_cells} cells "
                      f"+ apply + Newton Jacobian, {steps} step(s), {dt:.2f} s/step"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    pr = I.make_problem(args.config, batch=min(args.batch or 256, 256))
    if args.config == "cfg5":
        print(json.dumps({"impl": "reference", "unavailable": "reference arm implemented for cfg1-cfg4"}))
        return
    import oracle
    rows = min(ORACLE_SAMPLE_ROWS, pr.n_u)
    o = oracle.OracleTensor(pr.mesh, pr.V, pr.W, pr.form, rows=(0, rows))
    for _ in range(args.warmup if args.warmup <= 1 else 1):
        w = o.interp(pr.interp, pr.p, pr.u)
        o.apply(pr.u, w)
    t0 = time.time()
    for _ in range(args.steps):
        w = o.interp(pr.interp, pr.p, pr.u)
        o.apply(pr.u, w)
        o.jacobian(1, pr.interp, pr.p, pr.u, w)
    dt = time.time() - t0
    value = 2 * o.nnz * args.steps / dt
    sample = f"{pr.name} rows [0,{rows}) = {o.nnz} nnz per step (interp over all cells + apply + Newton Jacobian)"
    print(json.dumps({"impl": "reference", "metric": "tensor nonzeros/s (apply + Newton Jacobian, 2 x nnz per step) "
                      "and achieved HBM GB/s", "value": value, "unit": "nnz/s", "n_gpus": 1, "steps": args.steps,
                      "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps, "higher_is_better": True,
                      "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                      "config": {"workload": f"{args.config}-f64"},
                      "cpu_baseline": {"value": value, "unit": "nnz/s", "cores": 1, "kind": "oracle", "sample": sample},
                      "e2e": {"value": value, "unit": "nnz/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
          flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg4", choices=list(I.CONFIG_NAMES) + list(I.EXTRA_NAMES))
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="eager launches instead of a CUDA graph (N=1)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
