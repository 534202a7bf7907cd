#!/usr/bin/env python
"""EGFEM hot-path benchmark (BASELINE.json metric: tensor nonzeros/s and achieved HBM GB/s).

One step = one pass of the whole hot path (SURVEY §8(a) A1–A3) over the workload:
  (1) egfem_interp           w_K = |∇u_h|_K^{p−2} and D_u w       (GRADPOW_P0)
  (2)+(3) egfem_apply_jacobian  r = T:(u⊗w) and the Newton J = T·w + (T·₂u)·D_u w, fused
          into one pass over T (both outputs from a single stream of T's nonzeros).
Default workload: BASELINE configs[3] (3D p-Laplace p=3, 128³×6 tets, 201,326,592 nnz,
fp64) — the config the north star's headline target is quoted on ("≥70% of HBM at 1 GPU,
≥6× at 8 GPUs on the largest config"); it fits one B200.  Units: each step processes
2·nnz tensor nonzeros (apply + Jacobian, reading C25).  --config cfg5: the batched action
R = T:(U⊗W), B = 256 pairs (nnz·B units per step).

N>1: one process per GPU.  `python bench.py --gpus N` launches the N ranks itself
(torch.distributed.run) when WORLD_SIZE is not set; under torchrun it reads RANK /
LOCAL_RANK / WORLD_SIZE.  cfg1–4: T's rows are partitioned (egfem_partition), each step
adds the NCCL u-halo exchange overlapped with the interior rows; cfg5: T is replicated and
the batch is sharded (no communication).  value = all ranks' units / max-over-ranks device
time.  --plan-only prints the rank layout and partition plan without touching a GPU (the
CPU tests run it under gloo).

--impl reference: the CPU oracle (oracle/, test infrastructure) on a bounded row sample of
the same workload, timed on the host cores (rank 0 only).
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import egfem_inputs as I  # noqa: E402

# nonzeros of the oracle's bounded sample (about 8-10 s of single-core CPU work per step on the
# GPU box's host: 1.9e7 nnz/s for cfg4's interp + apply + Newton, 3.7e8 nnz·pairs/s batched)
ORACLE_SAMPLE_NNZ = 80_000_000
ORACLE_SAMPLE_NNZ_BATCHED = 3_000_000_000  # nnz·pairs for cfg5
REFERENCE_STEPS_FULL = 50  # --impl reference: the per-step sample shrinks beyond this many steps (≈3.5 min of CPU work in all)


def reference_budget(budget, steps):
    """Per-step oracle sample of the reference arm: the cpu_baseline leg's sample up to
    REFERENCE_STEPS_FULL steps, scaled down after that so --steps K stays within a few minutes."""
    return budget if steps <= REFERENCE_STEPS_FULL else max(1, budget * REFERENCE_STEPS_FULL // steps)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def _fp64_peak():
    """FP64 FMA peak: profiles/fp64_peak.json (tools/fp64_peak.sh on this pool's B200, with the
    SM clock sampled during the run) if present, else 148 SMs x 64 DFMA/clk x 2 x 1.965 GHz."""
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as f:
            d = json.load(f)
        return float(d["fp64_fma_tflops"]), "measured (tools/fp64_peak.sh)", d.get("clocks")
    except Exception:
        return 148 * 64 * 2 * 1.965e9 / 1e12, "derived (148 SM x 64 DFMA/clk x 1.965 GHz)", None


def _ncu(workload, kernel):
    """Per-launch ncu --set full numbers (DRAM bytes, L2 hit rate, time) from the committed
    summary profiles/traffic.json, if any: {"dram_bytes", "l2_hit_pct", "source"}."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        e = d.get(workload, {}).get(kernel)
        if e is None:
            return None
        if isinstance(e, (int, float)):
            return {"dram_bytes": e, "source": d.get("_source")}
        return e
    except Exception:
        return None


def host_cpu():
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"model": model, "cores": len(os.sched_getaffinity(0)), "logical_cpus": os.cpu_count()}


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


# ----------------------------------------------------------------------------- byte models
def model_bytes(t, pr, s, kind):
    """SURVEY §8(d) D.3 algorithmic bytes of one launch: the canonical format (val s + t_j 4 +
    t_k 4 per nonzero, an 8-byte row pointer per row), vectors read / written once; the slot
    maps are not counted.  kind: apply | jac | jac_picard | fused | interp."""
    d = pr.mesh.dim
    n_el = pr.mesh.n_cells
    T = t.nnz * (s + 8) + 8 * (t.n_u + 1)
    chain = pr.W.family in (I.P0, I.QUAD) and pr.interp in (I.INTERP_GRADPOW_P0, I.INTERP_MINSURF_P0,
                                                           I.INTERP_RECIPROCAL, I.INTERP_SQUARE)
    # Newton inputs besides T: P0-type W reads w and the chain data (c_aK, q_K: (d+2) per
    # cell, D.3); W = V reads u and w
    newton_in = s * t.n_f + s * (d + 2) * n_el if chain else s * (t.n_u + t.n_f)
    if kind == "apply":
        return T + s * (2 * t.n_u + t.n_f)
    if kind == "jac":
        return T + newton_in + s * t.nnz_csr
    if kind == "jac_picard":
        return T + s * t.n_f + s * t.nnz_csr
    if kind == "fused":  # one T stream; u read, r written, Newton inputs, J written
        return T + s * (2 * t.n_u) + (newton_in - (0 if chain else s * t.n_u)) + s * t.nnz_csr
    if kind == "interp":
        if chain:  # lean GRADPOW: connectivity + coordinates, u read, w and chain written
            return 4 * (d + 1) * n_el + s * d * pr.mesh.n_vertices + s * t.n_u + s * t.n_f + s * (d + 2) * n_el
        return s * (t.n_u + t.n_f)  # nodal: read u, write w
    raise ValueError(kind)


def layout_bytes(t, pr, s, kind):
    """Minimal bytes of the kernels' own CSF layout (k + value per nonzero, column + offset per
    fiber, a row offset): the layout-specific counterpart of model_bytes, for reference."""
    d1 = pr.mesh.dim + 1
    T = t.nnz * (4 + s) + t.nnz_csr * 8 + (t.n_u + 1) * 8
    if kind == "fused":
        return T + s * (2 * t.n_u + t.n_f + d1 * t.n_f) + s * t.nnz_csr
    return None


# ----------------------------------------------------------------------------- oracle sample
def oracle_sample(pr, budget_nnz):
    """A bounded, contiguous row sample [0, R) of the workload (about `budget_nnz` nonzeros) and
    the interp work items that feed exactly those rows (cells touching them, or the W-DOFs
    they reference) — what the CPU oracle is timed on."""
    mesh, V, W = pr.mesh, pr.V, pr.W
    per_row = {"cfg1": 7, "cfg2": 31, "cfg3": 18, "cfg4": 96, "cfg5": 88}.get(pr.name, 40)
    R = int(min(V.n_dofs, max(1, budget_nnz // per_row)))
    touch = np.asarray(V.cell_dofs) < R
    cells = np.nonzero(touch.any(axis=1))[0]
    cell_wise = W.family in (I.P0, I.QUAD) or pr.interp == I.INTERP_P1_TO_P2_SQUARE
    if cell_wise:
        items = (int(cells.min()), int(cells.max()) + 1)
    else:
        items = (0, int(np.asarray(W.cell_dofs)[cells].max()) + 1)
    return R, items


def cpu_baseline(pr, gpu_out=None, steps=1):
    """The CPU oracle as it stands on a bounded row sample of the same workload: one thread
    (the plain sequential oracle) and all host cores (OpenMP over rows / cells, each row in its
    sequential order: bitwise the same results).  Per step: interp over the sample's cells,
    apply and the Newton Jacobian of rows [0, R).  With `gpu_out` (the GPU's w, r, J) it also
    reports the relative L2 parity of the GPU outputs on the sample (reading C15)."""
    import oracle
    R, items = oracle_sample(pr, ORACLE_SAMPLE_NNZ)
    t0 = time.time()
    o = oracle.OracleTensor(pr.mesh, pr.V, pr.W, pr.form, rows=(0, R))
    build_s = time.time() - t0
    ncores = len(os.sched_getaffinity(0))
    res = {}
    for nt in (1, ncores):
        oracle.set_threads(nt)
        try:
            w = o.interp(pr.interp, pr.p, pr.u, items=items)  # warm-up
            t0 = time.time()
            for _ in range(steps):
                w = o.interp(pr.interp, pr.p, pr.u, items=items)
                r = o.apply(pr.u, w)
                J = o.jacobian(1, pr.interp, pr.p, pr.u, w)
            res[nt] = ((time.time() - t0) / steps, w, r, J)
        finally:
            oracle.set_threads(1)
    dt1, w, r, J = res[1]
    dtn = res[ncores][0]
    hc = host_cpu()
    out = {"value": 2 * o.nnz / dt1, "unit": "nnz/s", "cores": 1, "kind": "oracle",
           "sample": f"{pr.name} rows [0,{R}) = {o.nnz} nnz; interp over the {items[1] - items[0]} work items "
                     f"feeding them + apply + Newton Jacobian, {steps} step(s): {dt1:.2f} s/step on 1 thread",
           "all_cores": {"value": 2 * o.nnz / dtn, "cores": ncores, "s_per_step": dtn,
                         "bitwise_equal_to_1_thread": bool(all(np.array_equal(a, b) for a, b in
                                                                zip(res[1][1:], res[ncores][1:])))},
           "host_cpu": hc["model"], "host_cores": hc["cores"], "oracle_build_s": build_s}
    if gpu_out is not None:
        rr = slice(0, R)
        # the sample's rows are [0, R): their CSR slots are [0, csr_row_ptr[R]) on both sides (the
        # GPU pattern is memcmp-equal to the oracle's, tests/test_gpu_parity.py)
        ca, cb = 0, int(o.export(maps=False)["csr_row_ptr"][R])

        def rel(a, b):
            nb = float(np.linalg.norm(b))
            return float(np.linalg.norm(np.asarray(a, np.float64) - b) / nb) if nb > 0 else float(np.linalg.norm(a))
        c0, c1 = items
        if pr.W.family in (I.P0, I.QUAD) or pr.interp == I.INTERP_P1_TO_P2_SQUARE:
            wd = np.asarray(pr.W.cell_dofs)[c0:c1].ravel()
        else:
            wd = np.arange(c0, c1)
        out["parity_rel_l2"] = {"w": rel(gpu_out["w"][wd], w[wd]), "r": rel(gpu_out["r"][rr], r[rr]),
                                "J": rel(gpu_out["J"][ca:cb], J[ca:cb]), "rows": [0, R]}
    return out


def cpu_baseline_batched(pr, B, gpu_R=None):
    """cfg5: the oracle's batched action on rows [0, R) for all B pairs, 1 thread and all cores."""
    import oracle
    R, _ = oracle_sample(pr, ORACLE_SAMPLE_NNZ_BATCHED // B)
    o = oracle.OracleTensor(pr.mesh, pr.V, pr.W, pr.form, rows=(0, R))
    ncores = len(os.sched_getaffinity(0))
    U = np.ascontiguousarray(pr.u[:B])
    res = {}
    for nt in (1, ncores):
        oracle.set_threads(nt)
        try:
            t0 = time.time()
            Rr = o.apply_batched(U, U)
            res[nt] = (time.time() - t0, Rr)
        finally:
            oracle.set_threads(1)
    hc = host_cpu()
    out = {"value": o.nnz * B / res[1][0], "unit": "nnz*pair/s", "cores": 1, "kind": "oracle",
           "sample": f"cfg5 rows [0,{R}) = {o.nnz} nnz x {B} pairs (batched action): {res[1][0]:.2f} s on 1 thread",
           "all_cores": {"value": o.nnz * B / res[ncores][0], "cores": ncores, "s_per_step": res[ncores][0],
                         "bitwise_equal_to_1_thread": bool(np.array_equal(res[1][1], res[ncores][1]))},
           "host_cpu": hc["model"], "host_cores": hc["cores"]}
    if gpu_R is not None:  # node-major GPU R (N_u, B)
        ref = res[1][1][:, :R]
        got = gpu_R[:R, :B].T
        out["parity_rel_l2"] = {"R": float(np.linalg.norm(got - ref) / np.linalg.norm(ref)), "rows": [0, R],
                                "pairs": B}
    return out


# ----------------------------------------------------------------------------- ranks
def dist_env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def spawn_ranks(args):
    """`--gpus N` without a launcher: re-run this script under torch.distributed.run with N
    local ranks (rendezvous on 127.0.0.1) and return its exit code."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def row_nnz_host(pr):
    """Tensor nonzeros per row computed on the host from the DOF tables (P0-type W only: every
    (i, j, K) of a cell is its own nonzero, so row i has n_loc·(cells containing i))."""
    V = np.asarray(pr.V.cell_dofs)
    deg = np.bincount(V.ravel(), minlength=pr.V.n_dofs)
    return deg * V.shape[1] * pr.W.n_local


def plan_only(args):
    """The rank layout and partition plan (CPU, gloo): which rows / pairs each rank owns."""
    import torch.distributed as dist
    world, rank, local = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    pr = I.make_problem(args.config, batch=args.batch)
    plan = {}
    if args.config == "cfg5":
        B = pr.batch
        plan["batch_shards"] = [[r * B // world, (r + 1) * B // world] for r in range(world)]
        plan["tensor"] = "replicated (every rank holds all of T)"
    elif pr.W.family in (I.P0, I.QUAD):
        import paper_2005_06193_b200 as eg
        pref = np.concatenate([[0], np.cumsum(row_nnz_host(pr))]).astype(np.int64)
        cuts = eg.egfem_partition_rows(pref, world)
        plan["row_cuts"] = [int(x) for x in cuts]
        plan["nnz_per_rank"] = [int(pref[cuts[r + 1]] - pref[cuts[r]]) for r in range(world)]
    mine = {"rank": rank, "local_rank": local}
    if world > 1:
        allr = [None] * world
        dist.all_gather_object(allr, mine)
    else:
        allr = [mine]
    if rank == 0:
        print(json.dumps({"plan_only": True, "n_gpus": world, "gpus_flag": args.gpus, "config": args.config,
                          "ranks": allr, "plan": plan}), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2005_06193_b200 as eg
    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        # a bounded collective timeout: a hung exchange aborts the ranks instead of the whole run
        import datetime
        dist.init_process_group("nccl", device_id=dev, timeout=datetime.timedelta(seconds=300))
    pr = I.make_problem(args.config, batch=args.batch)
    dtype = eg.F64 if args.dtype == "f64" else eg.F32
    td = torch.float64 if dtype == eg.F64 else torch.float32
    s = 8 if dtype == eg.F64 else 4
    t0 = time.time()
    tg = eg.egfem_tensor_build(pr.mesh, pr.V, pr.W, pr.form, dtype=dtype, device=local)
    torch.cuda.synchronize()
    build_s = time.time() - t0
    if args.config == "cfg5":  # T replicated, the batch sharded: no row partition
        return run_batched(args, eg, tg, pr, dev, td, s, build_s, world, rank)
    if args.config == "gfem2d" and world == 1:
        return run_gfem(args, eg, tg, pr, dev, td, s, build_s)
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
        u_np = pr.u
    u = torch.tensor(u_np, dtype=td, device=dev)
    w = torch.empty(t.n_f, dtype=td, device=dev)
    gp = pr.W.family in (I.P0, I.QUAD) and pr.interp in (I.INTERP_GRADPOW_P0, I.INTERP_MINSURF_P0,
                                                         I.INTERP_RECIPROCAL, I.INTERP_SQUARE)
    chain = torch.empty(t.n_f * (pr.mesh.dim + 1), dtype=td, device=dev) if gp else None
    r = torch.empty(t.n_u, dtype=td, device=dev)
    J = torch.empty(t.nnz_csr, dtype=td, device=dev)
    stream = torch.cuda.current_stream(dev)
    # the gradient kinds keep w_K in the packed Newton record (include/egfem.h egfem_interp): on the
    # cell-major path the single-GPU step writes that one copy and the fused kernel reads w_K from
    # it, so the step passes w = NULL (a separate w array is a second copy nothing in the step reads)
    w_rec = (chain is not None and pr.interp in (I.INTERP_GRADPOW_P0, I.INTERP_MINSURF_P0)
             and "k_cell" in eg.egfem_kernel_name(t, 2, eg.JAC_NEWTON, pr.interp, pr.p))
    ws = None if w_rec else w
    # IDENTITY (W = V): w = u by definition, so the single-GPU step passes u as w — the interp is an
    # in-place copy and the fused Newton runs the symmetrized blocks (k_dense1 JAC 3)
    w_alias = plan is None and pr.interp == I.INTERP_IDENTITY and pr.W.family not in (I.P0, I.QUAD)
    if w_alias:
        ws = u

    if plan is not None:
        from paper_2005_06193_b200 import dist as edist
        # interior rows / interp items read owned u only: they run while the halo is in flight
        ir0, ir1, iw0, iw1 = eg.egfem_interior(t)

    def dist_step(ux, rx, e=None):
        """N>1: post the u-halo exchange, run the interior phase, wait for the halo (the
        compute stream waits on the communicator's), run the boundary phase."""
        edist.split_step(eg, t, plan, (ir0, ir1, iw0, iw1), pr.interp, pr.p, ux, ws, chain, rx, J, stream, e)

    K, Wm = args.steps, args.warmup
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(K)]

    def step(e=None):
        if e:
            e[0].record(stream)
        if plan is not None:
            dist_step(u, r, e)
        else:
            eg.egfem_interp(t, pr.interp, pr.p, u, ws, chain, stream)
            if e:
                e[2].record(stream)
            eg.egfem_apply_jacobian(t, eg.JAC_NEWTON, pr.interp, pr.p, u, ws, chain, r, J, stream)
        if e:
            e[3].record(stream)

    # Timing rule: inputs larger than L2 or an L2 flush between timed steps.  The per-step working
    # set (T stream + vectors) of cfg4 is GBs; for the smaller configs a 512 MB write evicts L2
    # between steps and the step time is the sum of the per-step event intervals (flush excluded).
    ws_bytes = model_bytes(t, pr, s, "fused") + model_bytes(t, pr, s, "interp")
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
        l_cap = eg.launch_count()
        with torch.cuda.graph(graph[0]):
            eg.egfem_interp(t, pr.interp, pr.p, u, ws, chain, torch.cuda.current_stream(dev))
        l_interp = eg.launch_count() - l_cap
        with torch.cuda.graph(graph[1]):
            eg.egfem_apply_jacobian(t, eg.JAC_NEWTON, pr.interp, pr.p, u, ws, chain, r, J,
                                    torch.cuda.current_stream(dev))
        l_graph = eg.launch_count() - l_cap
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
    launches = eg.launch_count() - l0 if graph is None else l_graph * K  # each replay launches the captured kernels
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
    gpu_out = None
    if world == 1:  # the last timed step's outputs, for the parity check of the cpu_baseline leg
        wv = chain.view(-1, pr.mesh.dim + 1)[:, 0] if w_rec else (u if w_alias else w)  # w_K from the packed record
        gpu_out = {"w": wv.double().cpu().numpy(), "r": r.double().cpu().numpy(), "J": J.double().cpu().numpy()}

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
    dist_ms = {}
    if plan is None:  # the step's two kernels, timed by the events inside the timed region
        ti = [e[0].elapsed_time(e[2]) for e in ev]
        tf = [e[2].elapsed_time(e[3]) for e in ev]
        t_interp = float(np.mean(ti))
        t_fused = float(np.mean(tf))
        dist_ms = {"interp": (float(np.median(ti)), float(np.min(ti))),
                   "apply_jacobian_fused": (float(np.median(tf)), float(np.min(tf)))}
    else:  # N>1 splits them into phases: whole-range launches, outside the timed region
        t_interp = avg_ms(lambda: eg.egfem_interp(t, pr.interp, pr.p, u, ws, chain, stream))
        t_fused = avg_ms(lambda: eg.egfem_apply_jacobian(t, eg.JAC_NEWTON, pr.interp, pr.p, u, ws, chain, r, J,
                                                         stream))
    if w_rec or w_alias:  # the separate apply / Picard launches below read the w array: fill it once
        eg.egfem_interp(t, pr.interp, pr.p, u, w, chain, stream)
    t_apply = avg_ms(lambda: eg.egfem_apply(t, u, w, r, stream))
    t_jac = avg_ms(lambda: eg.egfem_jacobian(t, eg.JAC_NEWTON, pr.interp, pr.p, u, w, chain, J, stream))
    t_pic = avg_ms(lambda: eg.egfem_jacobian(t, eg.JAC_PICARD, pr.interp, pr.p, None, w, None, J, stream))

    # end to end: every step copies its input u from pinned host memory and its result r back to
    # pinned host memory.  The copies run on their own streams with u and r double-buffered, so
    # step k's H2D and D2H overlap the compute of steps k±1 (PCIe is full duplex).  J stays on the
    # device (the Newton solve that consumes it runs on the GPU: solver.py); a second run also
    # reads J back every step.
    u_host = torch.tensor(u_np, dtype=td).pin_memory()
    r_host = [torch.empty(t.n_u, dtype=td).pin_memory() for _ in range(2)]
    J_host = [torch.empty(t.nnz_csr, dtype=td).pin_memory() for _ in range(2)]
    ub, rb, Jb = [u, torch.empty_like(u)], [r, torch.empty_like(r)], [J, torch.empty_like(J)]
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def step_on(ux, rx, Jx):
        if plan is not None:
            edist.split_step(eg, t, plan, (ir0, ir1, iw0, iw1), pr.interp, pr.p, ux, ws, chain, rx, Jx, stream)
            return
        wx = ux if w_alias else ws
        eg.egfem_interp(t, pr.interp, pr.p, ux, wx, chain, stream)
        eg.egfem_apply_jacobian(t, eg.JAC_NEWTON, pr.interp, pr.p, ux, wx, chain, rx, Jx, stream)

    def e2e_run(with_j):
        ev_in, ev_c, ev_out = ([torch.cuda.Event() for _ in range(K)] for _ in range(3))
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
                stream.wait_event(ev_out[k - 2])  # rb[x] (and Jb[x]) have been read out
            step_on(ub[x], rb[x], Jb[x] if with_j else J)
            ev_c[k].record(stream)
            s_out.wait_event(ev_c[k])
            with torch.cuda.stream(s_out):
                r_host[x].copy_(rb[x], non_blocking=True)
                if with_j:
                    J_host[x].copy_(Jb[x], non_blocking=True)
            ev_out[k].record(s_out)
        stream.wait_event(ev_out[K - 1])
        b.record(stream)
        torch.cuda.synchronize()
        e_ms = a.elapsed_time(b)
        if world > 1:
            m = torch.tensor([e_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(m, op=dist.ReduceOp.MAX)
            e_ms = float(m.item())
        return e_ms
    e2e_ms = e2e_run(False)
    e2e_j_ms = e2e_run(True)

    peak, peak_kind = _peaks()
    workload = f"{args.config}-{args.dtype}"
    fused_model = model_bytes(t, pr, s, "fused")
    achieved = fused_model / (t_fused * 1e-3) / 1e9
    fused_name = eg.egfem_kernel_name(t, 2, eg.JAC_NEWTON, pr.interp, pr.p)
    ncu = _ncu(workload, "fused") if world == 1 else None
    roof = {"bound": "hbm", "kernel": f"{fused_name}: egfem_apply_jacobian (apply + Newton Jacobian, one pass over T)",
            "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
            "algorithmic_bytes": fused_model,
            "bytes_model": "SURVEY §8(d) D.3: nnz(s+8) + 8(N_u+1) + 2s N_u + s N_f + s(d+2)N_el + s nnz_csr "
                           "(P0 W; W = V: nnz(s+8) + 8(N_u+1) + s(2N_u+N_f) + s nnz_csr)",
            "time_ms": t_fused, "time_from": "CUDA events around the kernel inside the timed region (mean)",
            "layout_bytes": layout_bytes(t, pr, s, "fused"),
            "traffic": ncu["dram_bytes"] if ncu else None}
    if ncu:
        roof["traffic_achieved"] = ncu["dram_bytes"] / (t_fused * 1e-3) / 1e9
        roof["traffic_frac"] = roof["traffic_achieved"] / peak
        roof["l2_hit_pct"] = ncu.get("l2_hit_pct")
        roof["traffic_source"] = ncu.get("source")
    kernels = {}
    for key, tm, kind, ent in (("interp", t_interp, "interp", None), ("apply", t_apply, "apply", 0),
                               ("jacobian_newton", t_jac, "jac", 1), ("jacobian_picard", t_pic, "jac_picard", 1),
                               ("apply_jacobian_fused", t_fused, "fused", 2)):
        mb = model_bytes(t, pr, s, kind)
        kn = None
        if ent is not None:
            kn = eg.egfem_kernel_name(t, ent, eg.JAC_PICARD if key == "jacobian_picard" else eg.JAC_NEWTON,
                                      pr.interp, pr.p)
        nc = (_ncu(workload, {"jac": "jac_newton"}.get(kind, kind)) or {}) if world == 1 else {}
        kernels[key] = {"ms": tm, "bytes_model": mb, "GBps": mb / (tm * 1e-3) / 1e9,
                        "frac_6543": mb / (tm * 1e-3) / 1e9 / peak, "frac_8000": mb / (tm * 1e-3) / 1e9 / 8000,
                        "nnz_per_s": t.nnz / (tm * 1e-3) if kind != "interp" else None, "kernel": kn,
                        "bytes_ncu": nc.get("dram_bytes"), "l2_hit_pct": nc.get("l2_hit_pct"),
                        "timing": "mean of in-region events" if key in dist_ms else f"mean of {max(5, min(K, 50))} "
                                  "back-to-back launches after the timed region"}
        if key in dist_ms:
            kernels[key]["ms_median"], kernels[key]["ms_min"] = dist_ms[key]
    out = {
        "metric": "tensor nonzeros/s (apply + Newton Jacobian, 2 x nnz per step) and achieved HBM GB/s",
        "value": value, "unit": "nnz/s", "n_gpus": world, "steps": K, "warmup": Wm,
        "ms_per_step": ms / K, "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": args.dtype, "data": "synthetic (seeded, BASELINE.json recipe)",
        "config": {"workload": workload, "description": pr.description, "nnz": nnz_total,
                   "nnz_csr": t.nnz_csr if world == 1 else None, "n_u": pr.n_u, "n_f": pr.n_f,
                   "step": ("interp(%s%s) + fused apply/Newton-Jacobian" % (
                       ["IDENTITY", "SQUARE", "GRADPOW_P0", "P1_TO_P2_SQUARE", "MINSURF_P0", "RECIPROCAL"][pr.interp],
                       " + D_u w" if chain is not None else "")) +
                           (" + NCCL u-halo overlapped with the interior rows" if world > 1 else "") +
                           ("; w_K kept in the packed Newton record only (w = NULL)" if w_rec else "") +
                           ("; w = u (IDENTITY): fused Newton on the symmetrized blocks" if w_alias else ""),
                   "l2": (f"working set {ws_bytes / 1e9:.2f} GB < 4 x L2 ({l2_bytes >> 20} MB): 512 MB write "
                          "between timed steps, step time = sum of per-step intervals") if flush else
                         f"working set {ws_bytes / 1e9:.2f} GB >= 4 x L2 ({l2_bytes >> 20} MB); no flush",
                   "parallelism": f"row-partition x{world}" if world > 1 else "single GPU",
                   "launch": "CUDA graphs (interp; fused) replayed per step, events between" if graph is not None
                             else "eager"},
        "roofline": roof,
        "kernels": kernels,
        "e2e": {"value": units / (e2e_ms * 1e-3), "unit": "nnz/s", "h2d_bytes_per_step": u.numel() * s,
                "d2h_bytes_per_step": r.numel() * s, "ms_per_step": e2e_ms / K,
                "jacobian": "device-resident: J (nnz_csr values) is consumed by the GPU Newton solve "
                            "(paper_2005_06193_b200/solver.py), not copied to the host",
                "overlap": "H2D/D2H on copy streams, u and r double-buffered"},
        "e2e_with_jacobian": {"value": units / (e2e_j_ms * 1e-3), "unit": "nnz/s",
                              "h2d_bytes_per_step": u.numel() * s,
                              "d2h_bytes_per_step": (r.numel() + J.numel()) * s, "ms_per_step": e2e_j_ms / K},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "build_s": build_s,
    }
    if plan is not None:
        out["config"]["halo_values_per_rank"] = plan.halo_values
        out["phases_ms"] = phases
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(pr, gpu_out)
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
    for _ in range(max(args.warmup, 1)):  # the first call compiles the row-group kernels (NVRTC)
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
    launches = eg.launch_count() - l0
    ms = a.elapsed_time(b)
    if world > 1:
        m = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
        ms = float(m.item())
    units = t.nnz * B * args.steps  # all ranks' pairs
    R_gpu = R.double().cpu().numpy() if world == 1 else None
    # end to end: this rank's pairs from pinned host memory, the action, R back to pinned host
    # memory; U / R double-buffered on copy streams so step k's copies overlap steps k±1
    K = args.steps
    U_host = U.cpu().pin_memory()
    R_host = [torch.empty(R.shape, dtype=td).pin_memory() for _ in range(2)]
    Ub, Rb = [U, torch.empty_like(U)], [R, torch.empty_like(R)]
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    ev_in, ev_c, ev_out = ([torch.cuda.Event() for _ in range(K)] for _ in range(3))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a2, b2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a2.record(stream)
    s_in.wait_event(a2)
    s_out.wait_event(a2)
    for k in range(K):
        x = k % 2
        if k >= 2:
            s_in.wait_event(ev_c[k - 2])
        with torch.cuda.stream(s_in):
            Ub[x].copy_(U_host, non_blocking=True)
        ev_in[k].record(s_in)
        stream.wait_event(ev_in[k])
        if k >= 2:
            stream.wait_event(ev_out[k - 2])
        eg.egfem_apply_batched(t, Bl, eg.LAYOUT_NODE_MAJOR, Ub[x], Ub[x], Rb[x], stream)
        ev_c[k].record(stream)
        s_out.wait_event(ev_c[k])
        with torch.cuda.stream(s_out):
            R_host[x].copy_(Rb[x], non_blocking=True)
        ev_out[k].record(s_out)
    stream.wait_event(ev_out[K - 1])
    b2.record(stream)
    torch.cuda.synchronize()
    e2e_ms = a2.elapsed_time(b2)
    if world > 1:
        m = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
        e2e_ms = float(m.item())
    # T once + the vectors x B (U, W read, R written) on this rank
    byts = t.nnz * (s + 8) + 8 * (t.n_u + 1) + s * (2 * t.n_u + t.n_f) * Bl
    flops = 2 * (t.nnz + t.nnz_csr) * Bl  # fiber-factored: per pair, an FMA per nonzero and per fiber
    per = ms / args.steps
    peak, kind = _peaks()
    fpeak, fkind, fclk = _fp64_peak()
    workload = f"cfg5-{args.dtype}"
    ncu = _ncu(workload, "batched") if world == 1 else None
    roof = {"bound": "alu", "kernel": eg.egfem_kernel_name(t, 3) + ": egfem_apply_batched (NODE_MAJOR)",
            "achieved": flops / (per * 1e-3) / 1e12, "peak": fpeak, "peak_kind": fkind, "peak_clocks": fclk,
            "unit": "TFLOP/s", "frac": flops / (per * 1e-3) / 1e12 / fpeak, "algorithmic_flops": flops,
            "flops_model": "SURVEY §8(d) D.3: 2(nnz + n_fib) per pair (an FMA per nonzero and per fiber)",
            "traffic": ncu["dram_bytes"] if ncu else None}
    # U == W runs the symmetrized patterns (egfem_group.cu): fewer FMAs than §8(d)'s count in the
    # compiled classes; the line states the executed share so the frac can be read either way
    import re
    msym = re.search(r"(\d+) instead of (\d+) FMAs per pair", roof["kernel"])
    if msym:
        roof["executed_fma_share_compiled_classes"] = int(msym.group(1)) / int(msym.group(2))
        roof["note"] = ("U == W: R = sum_{j<=k} S_ijk u_j u_k with S = T + T^T(j,k) (a quadratic form); frac is on "
                        "SURVEY §8(d)'s algorithmic flops, the kernels execute executed_fma_share of them")
    if ncu:
        roof["traffic_achieved_GBps"] = ncu["dram_bytes"] / (per * 1e-3) / 1e9
        roof["l2_hit_pct"] = ncu.get("l2_hit_pct")
        roof["fp64_pipe_pct"] = ncu.get("fp64_pipe_pct")
        roof["traffic_source"] = ncu.get("source")
    out = {"metric": "tensor nonzero-pairs/s (batched action) and achieved HBM GB/s", "value": units / (ms * 1e-3),
           "unit": "nnz*pair/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": per, "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
           "vs_baseline": None, "dtype": args.dtype, "data": "synthetic (seeded, BASELINE.json recipe)",
           "config": {"workload": workload, "batch": B, "batch_per_rank": Bl, "nnz": t.nnz,
                      "parallelism": f"batch-shard x{world} (T replicated)",
                      "l2": "inputs larger than L2 (T 0.37 GB + U, R 0.54 GB each); no flush"},
           "e2e": {"value": units / (e2e_ms * 1e-3), "unit": "nnz*pair/s", "h2d_bytes_per_step": U.numel() * s,
                   "d2h_bytes_per_step": R.numel() * s, "ms_per_step": e2e_ms / K,
                   "overlap": "H2D/D2H on copy streams, U and R double-buffered"},
           "roofline": roof,
           "roofline_hbm": {"achieved": byts / (per * 1e-3) / 1e9, "peak": peak, "peak_kind": kind, "unit": "GB/s",
                            "frac": byts / (per * 1e-3) / 1e9 / peak, "algorithmic_bytes": byts},
           "gpu_launches": int(launches), "clocks": clk.summary(), "build_s": build_s}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline_batched(pr, B, R_gpu)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


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


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    """The reference arm: the CPU oracle (the paper has no code) on the host cores,
    a bounded row sample of the same workload per step, rank 0 only."""
    _, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle
    pr = I.make_problem(args.config, batch=args.batch)
    hc = host_cpu()
    if args.config == "cfg5":
        B = pr.batch
        R, _ = oracle_sample(pr, reference_budget(ORACLE_SAMPLE_NNZ_BATCHED, args.steps) // B)
        o = oracle.OracleTensor(pr.mesh, pr.V, pr.W, pr.form, rows=(0, R))
        U = np.ascontiguousarray(pr.u[:B])
        o.apply_batched(U[:1], U[:1])
        t0 = time.time()
        for _ in range(args.steps):
            o.apply_batched(U, U)
        dt = time.time() - t0
        value = o.nnz * B * args.steps / dt
        unit = "nnz*pair/s"
        metric = "tensor nonzero-pairs/s (batched action) and achieved HBM GB/s"
        sample = f"cfg5 rows [0,{R}) = {o.nnz} nnz x {B} pairs per step (batched action)"
    else:
        R, items = oracle_sample(pr, reference_budget(ORACLE_SAMPLE_NNZ, args.steps))
        o = oracle.OracleTensor(pr.mesh, pr.V, pr.W, pr.form, rows=(0, R))
        w = o.interp(pr.interp, pr.p, pr.u, items=items)
        o.apply(pr.u, w)
        t0 = time.time()
        for _ in range(args.steps):
            w = o.interp(pr.interp, pr.p, pr.u, items=items)
            o.apply(pr.u, w)
            o.jacobian(1, pr.interp, pr.p, pr.u, w)
        dt = time.time() - t0
        value = 2 * o.nnz * args.steps / dt
        unit = "nnz/s"
        metric = "tensor nonzeros/s (apply + Newton Jacobian, 2 x nnz per step) and achieved HBM GB/s"
        sample = (f"{pr.name} rows [0,{R}) = {o.nnz} nnz per step (interp over the {items[1] - items[0]} work items "
                  "feeding them + apply + Newton Jacobian)")
    print(json.dumps({"impl": "reference", "metric": metric, "value": value, "unit": unit, "n_gpus": 1,
                      "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps,
                      "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                      "data": "synthetic", "config": {"workload": f"{args.config}-{args.dtype}"},
                      "cpu_baseline": {"value": value, "unit": unit, "cores": 1, "kind": "oracle", "sample": sample,
                                       "host_cpu": hc["model"], "host_cores": hc["cores"]},
                      "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
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
    ap.add_argument("--plan-only", action="store_true", help="print the rank layout / partition plan (no GPU)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if args.gpus > 1 and world == 0:  # no launcher: start the ranks ourselves
        sys.exit(spawn_ranks(args))
    if world and args.gpus != world and int(os.environ.get("RANK", "0")) == 0:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; using WORLD_SIZE", file=sys.stderr)
    if args.plan_only:
        plan_only(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
