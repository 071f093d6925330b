"""Benchmark of the B200 implicit-FEM solve path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg3|cfg1|cfg2|cfg5]
                    [--precond ldlt|jacobi] [--impl reference]

Default workload: config 3 of BASELINE.json (20x20x250 = 100k-node corotational
beam, nested-dissection LDL^T-PCG), the largest configuration that fits one GPU.
A step = one implicit time step of the scenario (assemble A, b on the device
+ device PCG + kinematic update) at scenario step 4 of a clamped corotational
beam under transverse gravity, LDL^T factors of step 1 replayed (fixed
staleness 3, SURVEY.md 8d / BASELINE.md section 2).  Every timed step repeats
the same step from the same state (nothing committed), L2 flushed between
steps.  The CPU oracle solves the same system with the same factors and the
run fails unless the iteration counts agree and x matches within 1e-10.
N > 1 (torchrun): the nested-dissection sharded solve of the same mesh
(strong scaling; --replicas: one independent simulation per GPU instead).
--impl reference: the CPU reference path (the NumPy oracle port, oracle/),
workload built from scratch by the oracle -- the product package is never
imported on that arm.
cfg5: 64 independent ~50k-node simulations (own gravity direction each)
split over the GPUs; a step advances all of them (strong scaling).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "PCG ms/time step + tri-solve GB/s vs HBM roofline per mesh size"
WORKLOADS = {
    "cfg1": dict(dims=(6, 6, 28), law="linear", desc="config 1: ~1k-node beam, linear elastic"),
    "cfg2": dict(dims=(10, 10, 100), law="corotational", desc="config 2: ~10k-node corotational beam"),
    "cfg3": dict(dims=(20, 20, 250), law="corotational", desc="config 3: ~100k-node corotational beam"),
    "cfg4": dict(dims=(20, 20, 2500), law="corotational",
                 desc="config 4: ~1M-node corotational beam (nested-dissection sharded across the GPUs)"),
    "cfg5": dict(dims=(20, 20, 125), law="corotational", batch=64,
                 desc="config 5: 64 independent ~50k-node corotational beams (batched, Jacobi-PCG)"),
}
STALE_FROM, AT_STEP = 1, 4
TOL, MAX_IT, LEAF, TILE = 1e-9, 8000, 64, 16


def workload_config(name, precond, world):
    """The `config` object of both arms' JSON lines (static: derived from the
    workload definition alone, so the reference arm reports the same dict)."""
    w = WORKLOADS[name]
    nx, ny, nz = w["dims"]
    return {
        "workload": w["desc"], "mesh": "x".join(map(str, w["dims"])), "law": w["law"],
        "nodes": nx * ny * nz, "tets": 6 * (nx - 1) * (ny - 1) * (nz - 1), "dofs": 3 * nx * ny * nz,
        "precond": precond, "staleness": AT_STEP - STALE_FROM, "scenario_step": AT_STEP, "tol": TOL,
        "leaf": LEAF, "tile": TILE, "l2": "flushed (256 MB write) before every timed step",
        "parallelism": f"replicas x{world}",
    }


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text()), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback"


# ---------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------

def build_workload(name, device=True, with_factors=True):
    import paper_2306_05893_b200 as P
    from paper_2306_05893_b200 import krylov, ndprecond as ND
    from paper_2306_05893_b200.integrator import BackwardEulerIntegrator, IntegratorConfig, SimState

    w = WORKLOADS[name]
    mesh = P.generate_beam(*w["dims"], 0.1)
    mesh = mesh.with_fixed_nodes(np.flatnonzero(mesh.nodes[:, 2] == 0.0))
    params = P.MaterialParams(1e5, 0.3, 1000.0)
    integ = BackwardEulerIntegrator(mesh, P.make_model(w["law"], mesh, params),
                                    IntegratorConfig(dt=0.01, gravity=(0.0, -9.81, 0.0)))
    cfg = krylov.SolverConfig(TOL, MAX_IT)

    def jacobi(a, b):
        return krylov.pcg(a, b, krylov.jacobi_precond(a), cfg)

    jacobi.accepts_device = True
    t0 = time.perf_counter()
    plan = ND.expand_plan(ND.nested_dissection(P.vertex_adjacency(mesh), LEAF)) if with_factors else None
    t_nd = time.perf_counter() - t0
    st = SimState.rest(mesh, device=True)
    factors = None
    t_factor = 0.0
    for k in range(1, AT_STEP):
        res = integ.step(st, jacobi)
        if with_factors and k == STALE_FROM:
            t0 = time.perf_counter()
            factors = ND.ldlt_factor(res.matrix, plan, tile=TILE, source_step=k)
            t_factor = time.perf_counter() - t0
    if factors is not None:
        factors.device()

    def ldlt(a, b):
        return krylov.pcg(a, b, factors, cfg)

    ldlt.accepts_device = True
    return dict(name=name, mesh=mesh, integ=integ, state=st, factors=factors, plan=plan,
                solvers={"jacobi": jacobi, "ldlt": ldlt}, t_nd=t_nd, t_factor=t_factor, cfg=cfg)


class L2Flush:
    def __init__(self):
        import torch

        self.buf = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MB > L2

    def __call__(self):
        self.buf.zero_()


def time_steps(W, mode, steps, warmup, flush, graph=False):
    """Device step time.  graph=True replays the step captured as one CUDA
    graph (integrator.CapturedStep: the same kernels, no host work between
    them); otherwise compute_step runs eagerly."""
    import gc

    import torch
    from paper_2306_05893_b200 import _lib

    integ, st, solve = W["integ"], W["state"], W["solvers"][mode]
    step = integ.compute_step
    per_replay = None
    if graph:
        cap = integ.capture(st, solve)
        step = lambda s_, _solve: cap.replay(s_)  # noqa: E731
        per_replay = cap.kernels
    gc.disable()  # collector runs between steps (outside the events), never inside one
    for _ in range(warmup):
        flush()
        step(st, solve)
        gc.collect(0)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    iters, asm, slv = [], [], []
    launches = 0
    res = None
    for k in range(steps):
        res = None
        gc.collect(0)  # frees the previous step's device buffers held in reference cycles
        flush()
        l0 = _lib.launch_count()
        ev[k][0].record()
        res = step(st, solve)
        ev[k][1].record()
        # every libtsb kernel launch (the PCG solve is one); a graph replay runs the captured ones
        launches += per_replay if per_replay is not None else _lib.launch_count() - l0
        iters.append(res.report.iterations)
        asm.append(res.assembly_time * 1e3)
        slv.append(res.solve_time * 1e3)
    torch.cuda.synchronize()
    gc.enable()
    per = [a.elapsed_time(b) for a, b in ev]
    return dict(total_ms=sum(per), ms=statistics.median(per), iterations=statistics.median(iters),
                assembly_ms=statistics.median(asm), solve_ms=statistics.median(slv), launches=launches,
                per_step=per)


def time_apply(W, reps, flush):
    """Isolated LDL^T apply (both sweeps + perm/D), CUDA events on the launching stream."""
    import torch

    f = W["factors"]
    dev = f.device()
    r = torch.randn(f.plan.n, dtype=torch.float64, device="cuda")
    z = torch.empty_like(r)
    for _ in range(3):
        dev.run("apply", r, z)
    ts = []
    for _ in range(reps):
        flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dev.run("apply", r, z)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    nnzL = f.fill_in
    n = f.plan.n
    bytes_apply = 16 * nnzL + 48 * n  # two sweeps + perm gather + D + iperm
    ms = statistics.median(ts)
    return dict(ms=ms, bytes=bytes_apply, gbs=bytes_apply / (ms * 1e-3) / 1e9, nnzL=nnzL,
                stored_bytes=sum(dev.bytes.values()))


def time_spmv(W, reps, flush):
    """Isolated SpMV kernel (tsb_spmv through the C ABI, buffers preallocated):
    the flush is enqueued first, so the host launch of the SpMV overlaps the
    flush and the events bracket the kernel alone."""
    import torch
    from paper_2306_05893_b200 import _lib, krylov

    integ, st = W["integ"], W["state"]
    a, b, _ = integ.assemble_system(st)
    x = torch.randn(a.ncols, dtype=torch.float64, device="cuda")
    y = torch.empty(a.nrows, dtype=torch.float64, device="cuda")
    d_rp, d_ci = a.device_pattern()
    dv = a.device_values()
    lib = _lib.load()
    args = (a.nrows, _lib.ptr(d_rp), _lib.ptr(d_ci), _lib.ptr(dv), _lib.ptr(x), _lib.ptr(y), _lib.stream_ptr())
    for _ in range(3):
        krylov.spmv(a, x)
        lib.tsb_spmv(*args)
    ts = []
    for _ in range(reps):
        flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lib.tsb_spmv(*args)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    byts = 12 * a.nnz + 20 * a.nrows
    return dict(ms=ms, bytes=byts, gbs=byts / (ms * 1e-3) / 1e9, nnz=a.nnz)


def time_assembly(W, reps, flush):
    """Fused device assembly of the step (elem + gather launches), CUDA events, L2 flushed."""
    import torch

    integ, st = W["integ"], W["state"]
    x, v, fe = (integ._flat_dev(a) for a in (st.positions, st.velocities, st.f_ext))
    for _ in range(3):
        integ._assemble_device(x, v, fe)
    ts = []
    for _ in range(reps):
        flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        integ._assemble_device(x, v, fe)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    mesh = W["mesh"]
    nnz = len(integ.assembler.pattern["col_ind"])
    byts = 8 * nnz + mesh.element_count * (16 + 104 + 64) + mesh.node_count * 144
    return dict(ms=ms, bytes=byts, gbs=byts / (ms * 1e-3) / 1e9)


FP64_PEAK_TFLOPS = 37.0  # DMMA (the refactorisation's tile path), measured on this B200 (tools/ubench_fp64.cu); not in MEASURED_PEAKS.json


def time_refactor(W, reps=3):
    """Device LDL^T refactorisation (csrc/refactor.cu) of the current step's matrix."""
    import torch
    from paper_2306_05893_b200 import refactor as R

    a, _, _ = W["integ"].assemble_system(W["state"])
    t0 = time.perf_counter()
    rf = R.DeviceRefactor(a, W["plan"], TILE)
    t_plan = time.perf_counter() - t0
    img = rf.images[0]
    ts = []
    for i in range(1 + reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rf.enqueue(a, img)
        e1.record()
        e1.synchronize()
        if i:
            ts.append(e0.elapsed_time(e1))
    if rf.failed_block() >= 0:
        raise RuntimeError("device refactorisation hit a non-positive pivot")
    ms = statistics.median(ts)
    tf = rf.rplan.flops / (ms * 1e-3) / 1e12
    out = dict(ms=ms, gflop=rf.rplan.flops / 1e9, tflops=tf, peak_tflops=FP64_PEAK_TFLOPS,
               frac=tf / FP64_PEAK_TFLOPS, bound="fp64", plan_s=t_plan, workspace_gb=rf.workspace_bytes / 1e9)
    W["refactor"] = rf
    return out


def time_async_device(W, steps, flush):
    """Steady state of AsyncPreconditioner(device=True) on a running simulation
    (a copy of the scenario state, committed every step): each step polls,
    solves with the newest published factor (Jacobi until the first lands) and
    submits the step's matrix for refactorisation on a side stream."""
    import torch
    from paper_2306_05893_b200 import krylov, ndprecond as ND

    pre = ND.AsyncPreconditioner(W["plan"], tile=TILE, device=True)
    cfg = W["cfg"]
    integ = W["integ"]
    st = W["state"].copy()  # the run advances its own copy of the scenario state
    t0 = time.perf_counter()
    pre.prepare(integ.assemble_system(st)[0])  # setup: refactorisation planning off the stepping path
    t_prep = time.perf_counter() - t0
    stale, iters, per = [], [], []
    k0 = 1000
    for k in range(steps + 5):
        pre.poll()
        ready = pre.status is ND.PrecondStatus.READY
        solve = (lambda a, b: krylov.pcg(a, b, pre, cfg)) if ready else W["solvers"]["jacobi"]
        flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res = integ.step(st, solve)
        pre.update(res.matrix, k0 + k)
        e1.record()
        e1.synchronize()
        if k >= 5:
            per.append(e0.elapsed_time(e1))
            iters.append(res.report.iterations)
            stale.append(pre.staleness(k0 + k) if ready else -1)
    pre.close()
    return dict(ms_per_step=statistics.median(per), iterations=statistics.median(iters),
                staleness_median=statistics.median(stale), steps=len(per), prepare_s=t_prep,
                first_ready_step=next((k for k, sv in enumerate(stale) if sv >= 0), -1))


def time_e2e(W, mode, steps):
    """Same step through the reference-facing API with HOST (NumPy) state in
    pinned memory: H2D of x, v, f_ext and D2H of the step's results inside the
    timed region."""
    import torch
    from paper_2306_05893_b200.integrator import SimState

    st = W["state"]

    def pinned(a):  # the step's inputs live in pinned host memory (straight DMA, as a time loop's results do)
        t = a.detach().cpu() if torch.is_tensor(a) else torch.from_numpy(np.ascontiguousarray(a))
        return t.pin_memory().numpy()

    host = SimState(pinned(st.positions), pinned(st.velocities), pinned(st.accelerations), pinned(st.f_int),
                    pinned(st.f_ext), st.time)
    solve = W["solvers"][mode]
    for _ in range(2):
        W["integ"].compute_step(host, solve)
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        res = W["integ"].compute_step(host, solve)
        _ = res.positions.sum()  # results are host arrays
        ts.append((time.perf_counter() - t0) * 1e3)
    n = 3 * W["mesh"].node_count
    return dict(ms=statistics.median(ts), h2d=3 * 8 * n, d2h=6 * 8 * n)


# ---------------------------------------------------------------------------
# CPU baseline: the oracle port of the reference on the host cores
# ---------------------------------------------------------------------------

def oracle_step(W, mode, rest, pattern, host_state):
    """One reference step on the host: the oracle's fused assembly through the
    cached mapping (the reference's fast path) + PCG with the same
    preconditioner as the GPU arm (the very same host LdlFactors object)."""
    from oracle import tetsim_oracle as O

    mesh = W["mesh"]
    x, v, fe = host_state
    out = O.assemble_system(mesh.nodes, mesh.elements, mesh.fixed_nodes, rest, x, v, fe, 0.01,
                            (0.0, -9.81, 0.0), linear=WORKLOADS[W["name"]]["law"] == "linear", pattern=pattern)
    if mode == "ldlt":
        f = W["factors"]
        pre = lambda r: O.apply(f, r)  # noqa: E731
    else:
        inv = O.jacobi_inv_diag(out["row_ptr"], out["col_ind"], out["values"], len(out["b"]))
        pre = lambda r: r * inv  # noqa: E731
    return O.pcg(out["row_ptr"], out["col_ind"], out["values"], out["b"], pre, TOL, MAX_IT)


def cpu_baseline(W, mode, budget_s=20.0, max_steps=10, threads=1):
    """The oracle port of the reference step on one host core (median of full
    steps within the budget) -- and the parity check of the GPU step: same
    state, same preconditioner, the oracle's iterations and x."""
    from oracle import tetsim_oracle as O
    from threadpoolctl import threadpool_limits

    st = W["state"].to_host()
    host_state = (st.positions, st.velocities, st.f_ext)
    mesh = W["mesh"]
    with threadpool_limits(limits=threads):
        rest = O.rest_data(mesh.nodes, mesh.elements, 1e5, 0.3, 1000.0)
        pattern = O.assembly_pattern(mesh.nodes, mesh.elements, mesh.fixed_nodes, rest)
        ts = []
        t_start = time.perf_counter()
        while len(ts) < max_steps and (time.perf_counter() - t_start) < budget_s:
            t0 = time.perf_counter()
            x, it, res, conv = oracle_step(W, mode, rest, pattern, host_state)
            ts.append((time.perf_counter() - t0) * 1e3)
    return dict(ms=statistics.median(ts), steps=len(ts), iterations=it, x=x, residual=res, converged=conv)


def check_parity(W, mode, cpu):
    """The GPU step must reproduce the oracle: same PCG iteration count, x
    within 1e-10 relative (north_star tolerance); raises otherwise."""
    res = W["integ"].compute_step(W["state"], W["solvers"][mode])
    x = res.accelerations.reshape(-1).cpu().numpy()
    it = int(res.report.iterations)
    ref = cpu["x"]
    err = float(np.abs(x - ref).max() / max(np.abs(ref).max(), 1e-300))
    out = {"iterations_gpu": it, "iterations_oracle": int(cpu["iterations"]), "x_rel_err": err,
           "tolerance": 1e-10, "ok": it == int(cpu["iterations"]) and err <= 1e-10}
    if not out["ok"]:
        raise SystemExit(f"parity check failed: {out}")
    return out


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------

class ClockSampler:
    """nvidia-smi samples clocks into a file while the timed region runs (no
    Python reader thread competing for the GIL with the launch path)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, gpu):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def __enter__(self):
        import tempfile

        self.path = tempfile.NamedTemporaryFile(prefix="clocks_", suffix=".csv", delete=False).name
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "50", "-i", str(self.gpu)], stdout=self.fh,
                                         stderr=subprocess.DEVNULL, text=True)
            # nvidia-smi's start-up (NVML init, first query) stalls the device for
            # tens of ms: let it settle before the timed region starts
            t0 = time.time()
            while time.time() - t0 < 5.0 and os.path.getsize(self.path) < 2:
                time.sleep(0.05)
            time.sleep(0.2)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()
            try:
                self.lines = [ln.strip() for ln in open(self.path) if ln.strip()]
                os.unlink(self.path)
            except Exception:
                self.lines = []
        return False

    def summary(self):
        rows = []
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) >= 7:
                try:
                    rows.append((float(p[0]), float(p[1]), p[2:6], float(p[6])))
                except ValueError:
                    pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i, v in enumerate(r[2]) if v.lower() == "active"})
        loaded = [r for r in rows if r[3] > 0] or rows
        return {"sm_mhz": statistics.median(r[0] for r in loaded), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows), "samples_under_load": len(loaded)}


def traffic_from_profiles(workload):
    p = ROOT / "profiles" / "ncu_traffic.json"
    try:
        return json.loads(p.read_text()).get(workload)
    except Exception:
        return None


# ---------------------------------------------------------------------------
# config 5: a batch of independent simulations per GPU
# ---------------------------------------------------------------------------

def batch_config(world):
    w = WORKLOADS["cfg5"]
    nx, ny, nz = w["dims"]
    return {"workload": w["desc"], "mesh": "x".join(map(str, w["dims"])), "simulations": w["batch"],
            "nodes": nx * ny * nz, "dofs": 3 * nx * ny * nz, "precond": "jacobi", "scenario_step": 4, "tol": TOL,
            "parallelism": f"batch split over {world} GPU(s), no collective",
            "l2": "flushed (256 MB write) before every batch step",
            "step": "one implicit step of every simulation (CUDA-graph replays, one after another)"}


def batch_gravity(i):
    """Gravity of simulation i: a random unit direction (default_rng(i)) x 9.81."""
    g = np.random.default_rng(i).standard_normal(3)
    return tuple(float(v) for v in 9.81 * g / np.linalg.norm(g))


def build_batch(world, rank):
    import paper_2306_05893_b200 as P
    from paper_2306_05893_b200 import krylov
    from paper_2306_05893_b200.integrator import BackwardEulerIntegrator, IntegratorConfig, SimState

    w = WORKLOADS["cfg5"]
    mesh = P.generate_beam(*w["dims"], 0.1)
    mesh = mesh.with_fixed_nodes(np.flatnonzero(mesh.nodes[:, 2] == 0.0))
    params = P.MaterialParams(1e5, 0.3, 1000.0)
    cfg = krylov.SolverConfig(TOL, MAX_IT)

    def jacobi(a, b):
        return krylov.pcg(a, b, krylov.jacobi_precond(a), cfg)

    jacobi.accepts_device = True
    sims = []
    for i in range(w["batch"]):
        if i % world != rank:
            continue
        integ = BackwardEulerIntegrator(mesh, P.make_model(w["law"], mesh, params),
                                        IntegratorConfig(dt=0.01, gravity=batch_gravity(i)))
        st = SimState.rest(mesh, device=True)
        for _ in range(3):  # a few scenario steps: non-trivial velocities and rotations
            integ.step(st, jacobi)
        sims.append({"id": i, "integ": integ, "state": st})
    return mesh, sims, jacobi


def run_batched(args, world, rank, local, dist):
    """Config 5: every rank steps its share of the 64 simulations (sequentially,
    each as a captured CUDA graph); value = ms per batch step (all 64
    simulations), max over ranks; strong scaling (the batch is fixed)."""
    import gc

    import torch
    from paper_2306_05893_b200 import _lib, krylov
    from paper_2306_05893_b200.integrator import SimState

    mesh, sims, solve = build_batch(world, rank)
    for sm in sims:
        sm["cap"] = sm["integ"].capture(sm["state"], solve)
    flush = L2Flush()
    pk, pk_kind = peaks()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    gc.disable()

    def batch_step():
        its = []
        for sm in sims:
            its.append(sm["cap"].replay(sm["state"]).report.iterations)
        return its

    for _ in range(args.warmup):
        flush()
        batch_step()
    torch.cuda.synchronize()
    per, iters = [], []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            iters += batch_step()
            e1.record()
            e1.synchronize()
            per.append(e0.elapsed_time(e1))
    gc.enable()
    t_local = torch.tensor([sum(per)], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
        dist.barrier()
    ms = float(t_local.item()) / args.steps
    # isolated SpMV of simulation 0's matrix (the Jacobi-PCG iteration is SpMV-bound)
    W0 = {"integ": sims[0]["integ"], "state": sims[0]["state"]}
    spmv_r = time_spmv(W0, 20, flush)
    # e2e: one batch step through the public API with host (NumPy) state
    hosts = [SimState(*(a.detach().cpu().numpy() for a in (sm["state"].positions, sm["state"].velocities,
                                                          sm["state"].accelerations, sm["state"].f_int,
                                                          sm["state"].f_ext)), sm["state"].time) for sm in sims]

    def host_solve(a, b):
        return krylov.pcg(a, b, krylov.jacobi_precond(a), krylov.SolverConfig(TOL, MAX_IT))

    host_solve.accepts_device = True
    e2e = []
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for sm, hs in zip(sims, hosts):
            res = sm["integ"].compute_step(hs, host_solve)
            _ = res.positions.sum()
        e2e.append((time.perf_counter() - t0) * 1e3)
    t_e2e = torch.tensor([min(e2e)], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(t_e2e, op=dist.ReduceOp.MAX)
    n = mesh.ndof
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return 0
    hbm = pk.get("hbm_gbs", 6650.0)
    batch = WORKLOADS["cfg5"]["batch"]
    line = {
        "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": batch_config(world), "per_rank": len(sims),
        "sim_steps_per_s": batch / (ms * 1e-3),
        "iterations_median": statistics.median(iters),
        "spmv": {"ms": spmv_r["ms"], "gbs": spmv_r["gbs"], "frac": spmv_r["gbs"] / hbm},
        "roofline": {"bound": "hbm", "kernel": "CSR SpMV (bit-exact), the Jacobi-PCG iteration's dominant part",
                     "achieved": spmv_r["gbs"], "peak": hbm, "peak_kind": pk_kind, "unit": "GB/s",
                     "frac": spmv_r["gbs"] / hbm, "traffic": None},
        "e2e": {"value": float(t_e2e.item()), "unit": "ms", "h2d_bytes_per_step": 3 * 8 * n * len(sims),
                "d2h_bytes_per_step": 6 * 8 * n * len(sims)},
        "gpu_launches": sum(sm["cap"].kernels for sm in sims) * args.steps,
        "clocks": clk.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        cb = batch_cpu_baseline(sims[0])
        line["cpu_baseline"] = {"value": cb * batch, "unit": "ms", "cores": 1, "kind": "port",
                                "sample": f"one oracle step (assembly + Jacobi-PCG) of simulation 0 ({cb:.0f} ms), "
                                          f"x {batch} simulations, 1 BLAS thread"}
    print(json.dumps(line))
    if dist:
        dist.destroy_process_group()
    return 0


def batch_cpu_baseline(sim, threads=1):
    from oracle import tetsim_oracle as O
    from threadpoolctl import threadpool_limits

    integ, st = sim["integ"], sim["state"].to_host()
    mesh = integ.mesh
    with threadpool_limits(limits=threads):
        rest = O.rest_data(mesh.nodes, mesh.elements, 1e5, 0.3, 1000.0)
        t0 = time.perf_counter()
        out = O.assemble_system(mesh.nodes, mesh.elements, mesh.fixed_nodes, rest, st.positions, st.velocities,
                                st.f_ext, 0.01, integ.config.gravity)
        inv = O.jacobi_inv_diag(out["row_ptr"], out["col_ind"], out["values"], len(out["b"]))
        O.pcg(out["row_ptr"], out["col_ind"], out["values"], out["b"], lambda r: r * inv, TOL, MAX_IT)
        return (time.perf_counter() - t0) * 1e3


# ---------------------------------------------------------------------------
# nested-dissection sharded step: one process per GPU
# ---------------------------------------------------------------------------

def run_sharded(args, world, rank, local, dist):
    """Every rank assembles only its subtrees' elements (shard.rank_mesh), the
    rank's local system is gathered on the device (shard.LocalSystem) and the
    LDL^T-PCG runs sharded (shard.DistributedPcg: owned subtrees + replicated
    top separators, top-row exchanges by NCCL or by our peer-memory kernels,
    device stop flag, iterations replayed as CUDA graphs).  A step = sharded
    assembly + local extraction + sharded solve of the scenario step's system;
    ms per step = max over ranks; strong scaling (the mesh is fixed).  Rank 0
    checks the result against the single-GPU PCG on the same factors."""
    import gc

    import torch
    import paper_2306_05893_b200 as P
    from paper_2306_05893_b200 import _lib, krylov, shard as S
    from paper_2306_05893_b200.integrator import BackwardEulerIntegrator, IntegratorConfig, SimState

    W = build_workload(args.workload)
    mesh, f = W["mesh"], W["factors"]
    sp = S.shard_blocks(f, world)
    perm = np.asarray(f.plan.perm)
    sub, nr = S.rank_mesh(mesh, sp, perm, rank)
    integ = BackwardEulerIntegrator(sub, P.make_model(WORKLOADS[args.workload]["law"], sub,
                                                      P.MaterialParams(1e5, 0.3, 1000.0)),
                                    IntegratorConfig(dt=0.01, gravity=(0.0, -9.81, 0.0)))
    full = W["state"]
    n = mesh.ndof
    fe = torch.from_numpy(S.rank_f_ext(full.f_ext.cpu().numpy(), nr, rank)).cuda()
    st = SimState(full.positions.clone(), full.velocities.clone(), torch.zeros_like(full.positions),
                  torch.zeros(n, dtype=torch.float64, device="cuda"), fe)
    a, b, _ = integ.assemble_system(st)
    fixed = mesh.fixed_dofs()
    t0 = time.perf_counter()
    ls = S.LocalSystem(np.asarray(a.row_ptr), np.asarray(a.col_ind), sp, perm, rank, fixed)
    t_plan = time.perf_counter() - t0
    grid = 32 if args.share_gpu else 0
    dp = S.DistributedPcg(None, f, rank=rank, world=world, grid=grid, exchange=args.exchange,
                          local=ls.system(a.device_values(), b))

    def step():
        a_, b_, _ = integ.assemble_system(st)
        dp.set_values(ls.values(a_.device_values()), ls.rhs(b_))
        return dp.solve(None, TOL, MAX_IT)

    flush = L2Flush()
    x, it, res, conv = step()
    # parity: the sharded solve vs the single-GPU device PCG of the same system and factors
    parity = None
    if rank == 0:
        af, bf_, _ = W["integ"].assemble_system(full)
        xr, rep = krylov.pcg(af, bf_, f, W["cfg"])
        xr = xr.cpu().numpy()
        err = float(np.abs(x.cpu().numpy() - xr).max() / max(np.abs(xr).max(), 1e-300))
        parity = {"iterations_sharded": it, "iterations_single_gpu": int(rep.iterations), "x_rel_err": err,
                  "tolerance": 1e-10, "ok": it == int(rep.iterations) and err <= 1e-10 and conv}
        if not parity["ok"]:
            raise SystemExit(f"sharded parity check failed: {parity}")
    for _ in range(args.warmup):
        flush()
        step()
    dist.barrier() if dist else None
    torch.cuda.synchronize()
    gc.disable()
    per = []
    launches = 0
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            l0 = _lib.launch_count()
            e0.record()
            step()
            e1.record()
            e1.synchronize()
            launches += _lib.launch_count() - l0 + dp.last_replayed  # eager + graph-replayed kernels
            per.append(e0.elapsed_time(e1))
    gc.enable()
    t_local = torch.tensor([sum(per)], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
        dist.barrier()
    ms = float(t_local.item()) / args.steps
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return 0
    cfgd = workload_config(args.workload, "ldlt", world)
    cfgd["parallelism"] = (f"nested-dissection shards x{world} ({args.exchange} exchange)"
                           + (", all ranks on one GPU" if args.share_gpu else ""))
    cfgd["step"] = "sharded assembly + device local-system gather + sharded LDL^T-PCG (graph-replayed, device stop flag)"
    line = {
        "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": cfgd, "iterations": it, "parity": parity,
        "shards": {"top_rows": int(len(sp.top_rows)), "load": [float(v) for v in sp.load],
                   "local_plan_s": t_plan},
        "gpu_launches": launches, "clocks": clk.summary(),
    }
    print(json.dumps(line))
    if dist:
        dist.destroy_process_group()
    return 0


def reference_workload(name, gravity=(0.0, -9.81, 0.0), at_step=AT_STEP, with_factors=True):
    """The whole workload built by the oracle alone (no product import):
    beam, rest data, cached assembly mapping, dissection, the scenario run
    from rest to step AT_STEP with Jacobi-PCG steps, the factors of step
    STALE_FROM's matrix."""
    from oracle import tetsim_nd as OND, tetsim_oracle as O

    w = WORKLOADS[name]
    linear = w["law"] == "linear"
    nodes, el = OND.generate_beam(*w["dims"], 0.1)
    fixed = OND.clamped_nodes(nodes)
    t0 = time.perf_counter()
    rest = O.rest_data(nodes, el, 1e5, 0.3, 1000.0)
    pattern = O.assembly_pattern(nodes, el, fixed, rest)
    plan = (OND.expand_plan(OND.nested_dissection(*OND.vertex_adjacency(len(nodes), el), LEAF))
            if with_factors else None)
    x, v, fe = nodes.copy(), np.zeros_like(nodes), np.zeros(3 * len(nodes))
    factors = None
    for k in range(1, at_step):
        out = O.assemble_system(nodes, el, fixed, rest, x, v, fe, 0.01, gravity, linear=linear, pattern=pattern)
        inv = O.jacobi_inv_diag(out["row_ptr"], out["col_ind"], out["values"], len(out["b"]))
        acc, _, _, _ = O.pcg(out["row_ptr"], out["col_ind"], out["values"], out["b"], lambda r: r * inv, TOL, MAX_IT)
        if with_factors and k == STALE_FROM:
            factors = OND.ldlt_factor(out["row_ptr"], out["col_ind"], out["values"], plan, TILE)
        x, v, _ = O.advance(acc, x, v, 0.01, fixed)
    return dict(nodes=nodes, el=el, fixed=fixed, rest=rest, pattern=pattern, plan=plan, factors=factors,
                state=(x, v, fe), linear=linear, gravity=gravity, setup_s=time.perf_counter() - t0)


def reference_sample(R, precond, part, nparts):
    """One bounded sample of the reference step (ms of the full step it stands
    for): the oracle's element pass + merge over element chunk `part` of
    `nparts` (x nparts) and the rest of the fused pass (mass share, rhs), then
    ONE PCG iteration (SpMV, preconditioner, dots, updates) x the iteration
    count of the full solve at this state."""
    from oracle import tetsim_oracle as O

    nodes, el, rest, pat = R["nodes"], R["el"], R["rest"], R["pattern"]
    x, v, fe = R["state"]
    m = len(el)
    c0, c1 = part * m // nparts, (part + 1) * m // nparts
    sub = {k: (val[c0:c1] if isinstance(val, np.ndarray) and len(val) == m else val) for k, val in rest.items()}
    t0 = time.perf_counter()
    _, _, krot = O.corotational(nodes, el[c0:c1], sub, x, v, R["linear"])
    lo, hi = 12 * m + 144 * c0, 12 * m + 144 * c1
    sel = (pat["kept"] >= lo) & (pat["kept"] < hi)
    np.bincount(pat["kept_slots"][sel], weights=(0.01 * 0.01) * krot.reshape(-1)[pat["kept"][sel] - lo],
                minlength=len(pat["col_ind"]))
    t_chunk = time.perf_counter() - t0
    t0 = time.perf_counter()
    np.bincount(rest["gdof"].reshape(-1), weights=np.repeat(rest["share"], 12), minlength=3 * len(nodes))
    t_rest = time.perf_counter() - t0
    sysm = R["system"]
    rp, ci, vals, b = sysm["row_ptr"], sysm["col_ind"], sysm["values"], sysm["b"]
    pre = R["pre"]
    p = pre(b)
    t0 = time.perf_counter()
    ap = O.spmv(rp, ci, vals, p)
    alpha = float(b @ p) / float(p @ ap)
    xx = alpha * p
    r = b - alpha * ap
    float(np.linalg.norm(r))
    z = pre(r)
    beta = float(r @ z) / float(b @ p)
    p = z + beta * p
    t_iter = time.perf_counter() - t0
    del xx
    return (nparts * t_chunk + t_rest + R["iterations"] * t_iter) * 1e3


def reference_system(R, precond):
    """Assemble the timed step's system with the oracle and solve it once in
    full (iteration count of the step; the samples time one iteration)."""
    from oracle import tetsim_oracle as O

    x, v, fe = R["state"]
    out = O.assemble_system(R["nodes"], R["el"], R["fixed"], R["rest"], x, v, fe, 0.01, R["gravity"],
                            linear=R["linear"], pattern=R["pattern"])
    if precond == "ldlt":
        f = R["factors"]
        pre = lambda r: O.apply(f, r)  # noqa: E731
    else:
        inv = O.jacobi_inv_diag(out["row_ptr"], out["col_ind"], out["values"], len(out["b"]))
        pre = lambda r: r * inv  # noqa: E731
    t0 = time.perf_counter()
    _, it, _, conv = O.pcg(out["row_ptr"], out["col_ind"], out["values"], out["b"], pre, TOL, MAX_IT)
    R.update(system=out, pre=pre, iterations=it)
    return it, conv, time.perf_counter() - t0


def run_reference(args):
    """Reference arm: the reference's CPU path (the NumPy oracle port of tetsim,
    oracle/) on the host cores, all BLAS threads; the product package is never
    imported.  Rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    if args.workload == "cfg5":
        return run_reference_batched(args)
    from oracle import tetsim_oracle as O

    R = reference_workload(args.workload)
    it, conv, t_full_solve = reference_system(R, args.precond)
    nparts = 8 if args.workload in ("cfg3",) else 1
    for k in range(args.warmup):
        reference_sample(R, args.precond, k % nparts, nparts)
    ts = [reference_sample(R, args.precond, k % nparts, nparts) for k in range(args.steps)]
    ms = statistics.median(ts)
    ncores = os.cpu_count()
    sample = (f"per step: the oracle's element pass + merge over 1/{nparts} of the elements (x{nparts}), the rest "
              f"of the fused pass, and one PCG iteration x {it} iterations (the full {args.precond}-PCG solve of "
              f"this system took {it} iterations, {t_full_solve * 1e3:.0f} ms); median of {args.steps} steps; "
              "workload built by the oracle (beam, dissection, scenario steps, stale factors)")
    assert not any(k.startswith("paper_2306_05893_b200") for k in sys.modules), "reference arm imported the product"
    line = {
        "impl": "reference", "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.workload, args.precond, args.gpus),
        "iterations": it, "converged": bool(conv), "setup_s": R["setup_s"],
        "cpu_baseline": {"value": ms, "unit": "ms", "cores": ncores, "kind": "port", "sample": sample},
        "e2e": {"value": ms, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def run_reference_batched(args):
    """Reference arm of config 5: simulation 0 (own gravity direction) built by
    the oracle from rest (3 Jacobi steps, as the GPU arm), then bounded samples
    of its step (1/4 of the elements + one Jacobi-PCG iteration x the
    iteration count); the batch step is 64 x that.  No product import."""
    R = reference_workload("cfg5", gravity=batch_gravity(0), at_step=4, with_factors=False)
    it, conv, t_full = reference_system(R, "jacobi")
    nparts = 4
    for k in range(args.warmup):
        reference_sample(R, "jacobi", k % nparts, nparts)
    ts = [reference_sample(R, "jacobi", k % nparts, nparts) for k in range(args.steps)]
    batch = WORKLOADS["cfg5"]["batch"]
    ms = statistics.median(ts) * batch
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": batch_config(args.gpus), "iterations": it, "converged": bool(conv),
        "cpu_baseline": {"value": ms, "unit": "ms", "cores": os.cpu_count(), "kind": "port",
                         "sample": f"simulation 0: element pass + merge over 1/{nparts} of the elements (x{nparts}) "
                                   f"+ one Jacobi-PCG iteration x {it} iterations, median of {args.steps}, "
                                   f"x {batch} simulations; all host BLAS threads"},
        "e2e": {"value": ms, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default 100; the reference arm's CPU samples default to 10)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="cfg3", choices=sorted(WORKLOADS))
    ap.add_argument("--precond", default="ldlt", choices=["ldlt", "jacobi"])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--eager", action="store_true", help="time compute_step eagerly instead of the captured graph")
    ap.add_argument("--shard", action="store_true",
                    help="nested-dissection sharded solve (the default for N > 1; N = 1 runs it on one rank)")
    ap.add_argument("--replicas", action="store_true", help="N > 1: independent replicas instead of shards")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "peer"])
    ap.add_argument("--share-gpu", action="store_true",
                    help="all ranks on cuda:0 (gloo group + peer exchange): exercises the N > 1 path on one GPU")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.steps is None:  # defaults that finish within minutes on either arm
        args.steps = 10 if args.impl == "reference" else 100
    if args.impl == "reference":
        return run_reference(args)

    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.share_gpu:
        local = 0
        args.exchange = "peer"
        os.environ["TSB_SHARED_DEVICE"] = "1"
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if args.share_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2306_05893_b200 import _lib

    if args.workload == "cfg5":
        return run_batched(args, world, rank, local, dist)
    if args.shard or (world > 1 and not args.replicas):
        return run_sharded(args, world, rank, local, dist)
    ldlt_extras = args.precond == "ldlt" or args.workload != "cfg4"  # cfg4 Jacobi: no 25 GB host factor
    W = build_workload(args.workload, with_factors=ldlt_extras)
    flush = L2Flush()
    pk, pk_kind = peaks()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        main_r = time_steps(W, args.precond, args.steps, args.warmup, flush, graph=not args.eager)
    eager_r = time_steps(W, args.precond, max(10, args.steps // 4), 3, flush)
    other = "jacobi" if args.precond == "ldlt" else "ldlt"
    other_r = (time_steps(W, other, max(10, args.steps // 4), 3, flush, graph=not args.eager) if ldlt_extras
               else None)
    torch.cuda.synchronize()
    t_local = torch.tensor([main_r["total_ms"]], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
        dist.barrier()
    total_ms = float(t_local.item())
    apply_r = time_apply(W, 20, flush) if ldlt_extras else None
    spmv_r = time_spmv(W, 20, flush)
    asm_r = time_assembly(W, 20, flush)
    e2e_r = time_e2e(W, args.precond, max(5, min(args.steps, 30)))
    # the device refactorisation's workspace (fronts of every block at once) is 17 GB at
    # cfg3 and ~10x that at 1M nodes: not run at cfg4
    refac_ok = ldlt_extras and args.workload != "cfg4"
    refac_r = time_refactor(W) if refac_ok else None
    async_r = time_async_device(W, max(10, min(args.steps, 30)), flush) if refac_ok else None
    ms = total_ms / args.steps
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return 0
    cpu = parity = None
    if world == 1 and not args.no_cpu_baseline and args.workload != "cfg4":  # the oracle needs ~10 min at 1M nodes
        cpu = cpu_baseline(W, args.precond)
        parity = check_parity(W, args.precond, cpu)
    hbm = pk.get("hbm_gbs", 6650.0)
    traffic = traffic_from_profiles(args.workload)
    mesh, f = W["mesh"], W["factors"]
    line = {
        "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.workload, args.precond, world),
        "sizes": {"nnz": spmv_r["nnz"], "nnz_L": apply_r["nnzL"] if apply_r else None},
        "iterations": main_r["iterations"], "assembly_ms": eager_r["assembly_ms"], "pcg_ms": eager_r["solve_ms"],
        "step_mode": "eager compute_step" if args.eager else "CUDA graph replay of compute_step (CapturedStep)",
        "eager_ms_per_step": eager_r["ms"],
        "step_ms": {"min": min(main_r["per_step"]), "median": statistics.median(main_r["per_step"]),
                    "max": max(main_r["per_step"]),
                    "argmax": int(max(range(len(main_r["per_step"])), key=lambda k: main_r["per_step"][k]))},
        other: {"ms_per_step": other_r["ms"], "iterations": other_r["iterations"]} if other_r else None,
        "trisolve": {"apply_ms": apply_r["ms"], "gbs": apply_r["gbs"], "frac": apply_r["gbs"] / hbm,
                     "algorithmic_bytes": apply_r["bytes"], "stored_bytes": apply_r["stored_bytes"]} if apply_r else None,
        "spmv": {"ms": spmv_r["ms"], "gbs": spmv_r["gbs"], "frac": spmv_r["gbs"] / hbm},
        "assembly": {"ms": asm_r["ms"], "gbs": asm_r["gbs"], "frac": asm_r["gbs"] / hbm,
                     "algorithmic_bytes": asm_r["bytes"]},
        "roofline": ({"bound": "hbm", "kernel": "ldlt apply (level-scheduled L and L^T sweeps)",
                      "achieved": apply_r["gbs"], "peak": hbm, "peak_kind": pk_kind, "unit": "GB/s",
                      "frac": apply_r["gbs"] / hbm, "traffic": traffic} if args.precond == "ldlt" else
                     {"bound": "hbm", "kernel": "CSR SpMV (bit-exact), the Jacobi-PCG iteration's dominant part",
                      "achieved": spmv_r["gbs"], "peak": hbm, "peak_kind": pk_kind, "unit": "GB/s",
                      "frac": spmv_r["gbs"] / hbm, "traffic": None}),
        "e2e": {"value": e2e_r["ms"], "unit": "ms", "h2d_bytes_per_step": e2e_r["h2d"],
                "d2h_bytes_per_step": e2e_r["d2h"]},
        "gpu_launches": main_r["launches"],
        "clocks": clk.summary(),
        "setup_s": {"nested_dissection": W["t_nd"], "host_factor": W["t_factor"]},
        "refactor": dict(refac_r, host_factor_s=W["t_factor"],
                         kernel="device LDL^T refactorisation (multifrontal 64x64 tiles, csrc/refactor.cu)")
        if refac_r else None,
        "ldlt_async_device": async_r,
    }
    if cpu is not None:
        line["cpu_baseline"] = {"value": cpu["ms"], "unit": "ms", "cores": 1, "kind": "port",
                                "sample": f"median of {cpu['steps']} oracle steps (fused assembly through the cached "
                                          f"mapping + {args.precond}-PCG, {cpu['iterations']} it, same host factors) "
                                          f"of the same {args.workload} state, 1 BLAS thread"}
        line["parity"] = parity
    print(json.dumps(line))
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
