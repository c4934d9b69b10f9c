#!/usr/bin/env python
"""Benchmark: MGRIT time-to-solution / fine time-step*DOF/s (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

One "step" = one complete MGRIT solve (residual-norm stop at 1e-7) of the
headline workload, BASELINE config 4 (BASELINE.json configs[3], the config
the 1/2/4/8-GPU metric is defined on): 2D P1 eddy-current model on a
512 x 512 grid (261,121 DOFs), three-phase PWM, 2^16 implicit-Euler steps on
[0, 0.02] s, 4-level V-cycle, FCF, m = 16, C-intervals partitioned across
the N GPUs.  Spatial coarsening on the coarsest level ("delayed", 2 grids):
the literal direct coarsening stalls in the reference's own algorithm on
this model (tests/golden/mgrit_cfg2_direct_n128.npz).  Factors
are shared between 1/dt values within 1e-12 relative (configs.config4;
tests/test_gpu_full.py pins that option against the reference engine's
4-level fixture).

value  : whole-job fine time-step*DOF/s = n_steps * n_dofs * K / t, inputs
         (problem data) resident in HBM, CUDA events on the launch stream,
         barrier + synchronize on both sides, max over ranks; profiling off.
e2e    : the same metric through the public API from host data: problem
         construction (host assembly, H2D of the level data and excitation
         tables), factorisation, solve, D2H of this rank's C-point iterate into
         pinned host memory.
roofline: per-kernel table from a separate, untimed profiling solve (CUDA
         events around every launch on the launching stream): the band-chain
         kernels (fp64 DMMA; algorithmic 2 n w flops per direction and column,
         the reference's dpbtrs) against the measured DMMA peak, and their
         HBM bytes against MEASURED_PEAKS.json.
config2: the config-2 leg (127^2, 2^14 steps, 3 levels): time-to-solution and
         its residual history checked against the reference engine's own
         full-size run (tests/golden/mgrit_cfg2_full.npz).
config3: the nonlinear config-3 leg at its stated size: one solve.
phi_microbench: BASELINE config 5 (256^2 Jacobi-PCG Phi, B = 64 .. 4096).
sequential_gpu: GPU sequential stepping on a window of the headline,
         extrapolated to the whole horizon (labelled).
cpu_baseline: the CPU oracle (reference algorithm: banded Cholesky Phi via
         scipy/LAPACK) stepping the headline model, one core.
--impl reference: the oracle on all host cores, same metric; rank 0 only.
"""

import os as _os

# one BLAS/OpenMP thread per process before numpy loads: the CPU arms run
# one oracle process per core (no oversubscription in the reference arm)
for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    _os.environ.setdefault(_v, "1")

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_NOMINAL_TFLOPS = 40.0      # B200 fp64 / fp64-tensor nominal (fallback only)
SEQ_WINDOW_STEPS = 256          # GPU sequential leg: timed window, extrapolated
CPU_SAMPLE_STEPS = 8            # oracle Phi steps per CPU sample (after one factorisation)
METRIC = "MGRIT time-to-solution as fine time-step*DOF/s"


def headline_spec():
    from paper_1912_03106_b200 import configs
    return configs.config4(grids=2, strategy="delayed")


def config2_spec():
    from paper_1912_03106_b200 import configs
    return configs.config2(grids=2, strategy="delayed")


def workload_config(spec, world):
    mg = spec["mgrit"]
    return {
        "workload": "BASELINE config 4 (configs[3]): linear 2D P1 eddy-current, 3-phase PWM, "
                    "512x512 grid, 2^16 steps, MGRIT V(FCF) 4 levels m=16, spatial coarsening "
                    "on the coarsest level",
        "mesh": f"{spec['N']}x{spec['N']} cells, {(spec['N'] - 1) ** 2} DOFs",
        "n_steps": spec["n_steps"],
        "levels": len(mg["factors"]) + 1,
        "m": mg["factors"][0],
        "spatial_strategy": mg["spatial_strategy"],
        "n_spatial_grids": spec["n_spatial_grids"],
        "tolerance": mg["tolerance"],
        "inner_solver": "banded Cholesky (direct), fp64 DMMA solves; on the 511^2 grid by the "
                        "strip solve (8 / 16 strips + separator Schur complement: the same "
                        "direct solve, ~2.7x fewer flops), on the coarse grid in the "
                        "reference's natural order; factors shared within dt_merge_rtol "
                        f"{spec['inner'].get('dt_merge_rtol', 0.0)}",
        "parallelism": f"time-parallel C-intervals over {world} GPU(s)",
        "l2": "working set > L2 (level-0 batch vectors 8.6 GB each); no flush needed",
    }


# --- clocks ------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.dev = device_index
        self.samples = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", str(self.dev), "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=2)
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4)
                          if s[2 + k].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def fp64_peak():
    """Measured fp64 tensor-core (DMMA m8n8k4) peak of this GPU, TFLOP/s:
    tools/fp64_peak.cu (8 independent accumulator chains per warp, 4-32 warps
    per SM, all SMs), compiled on first use.  Falls back to the nominal
    40 TFLOP/s."""
    src = os.path.join(ROOT, "tools", "fp64_peak.cu")
    exe = os.path.join(ROOT, "tools", "fp64_peak")
    try:
        if not os.path.exists(exe) or os.path.getmtime(exe) < os.path.getmtime(src):
            subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", exe,
                            src], check=True, capture_output=True, timeout=300)
        out = subprocess.run([exe], check=True, capture_output=True, text=True, timeout=120).stdout
        runs = json.loads(out)["runs"]
        best = max(r["tflops"] for r in runs if r.get("kind") == "dmma_m8n8k4")
        return best, "measured: DMMA m8n8k4 issue rate, all SMs (tools/fp64_peak.cu, this run)"
    except Exception as e:  # noqa: BLE001 -- the bench must still print its line
        return FP64_NOMINAL_TFLOPS, f"nominal B200 fp64 tensor (measurement failed: {e!r:.80})"


def ncu_traffic():
    """Per-launch DRAM bytes of the dominant kernel from this round's ncu
    capture (profiles/kernel_traffic.json), or None."""
    path = os.path.join(ROOT, "profiles", "kernel_traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return None


# --- CPU oracle arms ----------------------------------------------------------------
# The oracle Phi on the headline model: scipy/LAPACK banded Cholesky (the
# reference's own cholesky_banded / cho_solve_banded path, problems.py:130-146)
# on the 261,121-DOF operator.  A full CPU solve is infeasible (the
# sequential solve alone is 65,536 x 0.39 s = 7 h on one core), so both CPU
# legs time a bounded sample of Phi steps at the workload's dt after one
# factorisation and report the fine time-step*DOF rate of SEQUENTIAL stepping
# -- an upper bound for the CPU: MGRIT needs >= 3 Phi per fine step.

_CPU = {}


def _cpu_setup():
    from oracle import fem2d, time_hierarchy as oth
    spec = headline_spec()
    prob = fem2d.make_problem(spec)
    grid = oth.build_uniform_grid(0.0, spec["tf"], spec["n_steps"]).points
    u = prob.initial_state(0)
    u, _ = prob.step(u, grid[0], grid[1], 0)          # factorisation of the first dt
    _CPU.update(prob=prob, t0=float(grid[0]), t1=float(grid[1]), u=u)
    return prob.spatial.size(0)


def _cpu_steps(k):
    """k oracle Phi steps at the cached dt; returns seconds."""
    prob, u = _CPU["prob"], _CPU["u"]
    t0 = time.perf_counter()
    for _ in range(k):
        u, _ = prob.step(u, _CPU["t0"], _CPU["t1"], 0)
    _CPU["u"] = u
    return time.perf_counter() - t0


def cpu_baseline_single():
    n = _cpu_setup()
    _cpu_steps(1)
    secs = _cpu_steps(CPU_SAMPLE_STEPS)
    return {"value": CPU_SAMPLE_STEPS * n / secs, "unit": "fine time-step*DOF/s",
            "cores": 1, "kind": "port",
            "sample": f"oracle Phi (banded Cholesky, scipy/LAPACK: the reference's path) on the "
                      f"headline model, {CPU_SAMPLE_STEPS} sequential steps at the workload dt "
                      f"after one factorisation ({secs / CPU_SAMPLE_STEPS:.3f} s per step); "
                      "rate of sequential stepping, an upper bound for CPU MGRIT"}


def _pool_steps(k):
    return _cpu_steps(k)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import multiprocessing as mp
    cores = len(os.sched_getaffinity(0))
    n = _cpu_setup()                    # assembly + factor once, shared copy-on-write
    ctx = mp.get_context("fork")
    times = []
    with ctx.Pool(cores) as pool:
        for k in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            pool.map(_pool_steps, [CPU_SAMPLE_STEPS] * cores)
            dt = time.perf_counter() - t0
            if k >= args.warmup:
                times.append(dt)
    total = sum(times)
    value = args.steps * cores * CPU_SAMPLE_STEPS * n / total
    spec = headline_spec()
    line = {
        "metric": METRIC, "impl": "reference",
        "value": value, "unit": "fine time-step*DOF/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(spec, 1),
        "cpu_baseline": {"value": value, "unit": "fine time-step*DOF/s", "cores": cores,
                         "kind": "port",
                         "sample": f"each step: {cores} processes x {CPU_SAMPLE_STEPS} oracle "
                                   "Phi steps (banded Cholesky, scipy/LAPACK, one shared "
                                   "factor) of the headline model; extrapolated: the rate of "
                                   f"{cores} perfectly time-parallel sequential steppers, no "
                                   "MGRIT overhead (MGRIT needs >= 3 Phi per fine step)"},
        "e2e": {"value": value, "unit": "fine time-step*DOF/s",
                "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --- B200 arm ------------------------------------------------------------------------

def summarize_kernels(prof, elapsed, hbm_peak, fp64_peak_tf):
    """Per-kernel table of a profiling solve: launches, mean duration,
    algorithmic bytes / flops per launch, achieved GB/s and TFLOP/s and their
    fractions of the measured peaks, share of the solve."""
    out = []
    for k in prof:
        if not k["launches"] or k["name"] == "k_band_solve":
            continue
        avg_ms = k["total_ms"] / k["launches"]
        d = dict(name=k["name"], launches=k["launches"], avg_ms=avg_ms,
                 total_ms=k["total_ms"], share_of_step=(k["total_ms"] / 1e3) / elapsed)
        if k["alg_bytes"]:
            gbs = k["alg_bytes"] / (k["total_ms"] * 1e-3) / 1e9
            d.update(alg_bytes_per_launch=k["alg_bytes"] / k["launches"], achieved_gbs=gbs,
                     hbm_frac=gbs / hbm_peak)
        if k["alg_flops"]:
            tf = k["alg_flops"] / (k["total_ms"] * 1e-3) / 1e12
            d.update(alg_flops_per_launch=k["alg_flops"] / k["launches"], achieved_tflops=tf,
                     dmma_frac=tf / fp64_peak_tf)
        out.append(d)
    out.sort(key=lambda k: -k["total_ms"])
    return out


def phi_microbench(problem_cls, local, peak, batches=(64, 256, 1024, 4096)):
    """BASELINE config 5: one batched Jacobi-PCG Phi (rtol 1e-10) over B
    N(0,1) states on the 256^2 mesh per batch size; CUDA-event timing of the
    call, per-kernel events for B = 1024, and the true relative residual of
    every column checked on the device (torch CSR product of the same
    operator) against the stopping rule."""
    import torch
    from paper_1912_03106_b200 import configs
    spec = configs.config5()
    prob = problem_cls(spec, device=local, inner="pcg")
    n = prob.spatial.size(0)
    dev = prob.device
    g = prob.grids[0]
    A = torch.sparse_csr_tensor(torch.as_tensor(g.row_ptr, dtype=torch.int64),
                                torch.as_tensor(g.col_idx, dtype=torch.int64),
                                torch.as_tensor(g.k_val + g.m_val / spec["dt"]),
                                size=(n, n)).to(dev)
    M = torch.sparse_csr_tensor(torch.as_tensor(g.row_ptr, dtype=torch.int64),
                                torch.as_tensor(g.col_idx, dtype=torch.int64),
                                torch.as_tensor(g.m_val / spec["dt"]), size=(n, n)).to(dev)
    stream = torch.cuda.current_stream(dev)
    rows = []
    kernels = None
    for B in batches:
        U = torch.as_tensor(np.random.default_rng(0).standard_normal((B, n)), device=dev)
        inv = torch.full((B,), 1.0 / spec["dt"], dtype=torch.float64, device=dev)
        src = torch.zeros(B, 0, dtype=torch.float64, device=dev)
        out = torch.empty_like(U)
        prob.phi_batch(0, U, inv, src, out)              # warm-up
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        prob.phi_batch(0, U, inv, src, out)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        st = prob.last_stats()
        t = e0.elapsed_time(e1) / 1e3
        rhs = (M @ U.T).T
        res = torch.linalg.vector_norm((A @ out.T).T - rhs, dim=1) / \
            torch.linalg.vector_norm(rhs, dim=1)
        alg = st["column_iters"] * 80.0 * n + B * 40.0 * n
        rows.append({"B": B, "value": B * n / t, "seconds": t,
                     "batch_iters": st["batch_iters"], "column_iters": st["column_iters"],
                     "alg_bytes": alg, "achieved_gbs": alg / t / 1e9,
                     "frac_of_peak": alg / t / 1e9 / peak,
                     "max_true_residual": float(res.max())})
        if B == 1024:
            prob.profile(True)
            prob.phi_batch(0, U, inv, src, out)
            torch.cuda.synchronize(dev)
            kernels = summarize_kernels(prob.profile_read(reset=True), t, peak, 1.0)
            prob.profile(False)
        del U, out, rhs
    prob.close()
    ok = all(r["max_true_residual"] <= 1.05 * spec["inner"]["rtol"] for r in rows)
    main = next(r for r in rows if r["B"] == 1024)
    return {"workload": "BASELINE config 5: 256x256 (65,025 DOFs), N(0,1) states (seed 0), "
                        "dt=0.02/2^14, f=0, x0=u_prev, Jacobi-PCG rtol 1e-10",
            "unit": "time-step*DOF/s", "value": main["value"], "frac_of_peak": main["frac_of_peak"],
            "bytes_model": "80 n per column-iteration (k_sdir 32 n + k_supd 48 n) + 40 n setup",
            "batches": rows, "kernels_B1024": kernels,
            "residual_check": "true relative residual of every column <= 1.05 rtol: "
                              + ("pass" if ok else "FAIL")}


def _history(run):
    return [run.initial_residual] + list(run.residual_norms)


def config2_leg(local, transport, reps=3):
    """Config 2 at its stated size: time-to-solution and the residual history
    against the reference engine's full-size run (same iterations, <= 1e-8)."""
    import torch
    from paper_1912_03106_b200 import (CycleSpec, GpuFemProblem, MgritSolver, StoppingCriterion,
                                       TimeHierarchy, build_uniform_grid)
    spec = config2_spec()
    mg = spec["mgrit"]
    prob = GpuFemProblem(spec, device=local)
    grid = build_uniform_grid(0.0, spec["tf"], spec["n_steps"])
    solver = MgritSolver(prob, TimeHierarchy.build(grid, mg["factors"]),
                         CycleSpec(kind=mg["kind"], gamma=mg["gamma"], max_iters=mg["max_iters"],
                                   spatial_strategy=mg["spatial_strategy"]),
                         StoppingCriterion(tolerance=mg["tolerance"]), transport)
    dev = prob.device
    run, _ = solver.solve(gather_solution=False)
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    e0.record(stream)
    for _ in range(reps):
        run, _ = solver.solve(gather_solution=False)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    t = e0.elapsed_time(e1) / 1e3 / reps
    res = {"workload": "BASELINE config 2: 128x128 grid (16,129 DOFs), 2^14 steps, 3 levels, "
                       "delayed spatial coarsening",
           "time_to_solution_s": t, "value": spec["n_steps"] * prob.spatial.size(0) / t,
           "unit": "fine time-step*DOF/s", "iterations": run.iterations,
           "residual_history": _history(run)}
    fx = os.path.join(ROOT, "tests", "golden", "mgrit_cfg2_full.npz")
    if os.path.exists(fx):
        z = np.load(fx)
        ref = z["history"]
        h = np.array(res["residual_history"])
        same = run.iterations == int(z["iterations"]) and len(h) == len(ref)
        rel = float(np.max(np.abs(h - ref) / ref)) if same else None
        res["parity_vs_reference_engine"] = {
            "fixture": "tests/golden/mgrit_cfg2_full.npz (pintmg.mgrit_solve, full size)",
            "same_iterations": bool(same), "max_rel_history_diff": rel,
            "pass": bool(same and rel is not None and rel <= 1e-8)}
    prob.close()
    return res


def config3_leg(local, transport):
    """Config 3 at its stated size (nonlinear Brauer iron, 127^2, 2^14 steps,
    3 levels): one solve -- damped Newton per column, CG on the Newton systems
    preconditioned by frozen-Jacobian banded factors."""
    import torch
    from paper_1912_03106_b200 import (CycleSpec, GpuFemProblem, MgritSolver, StoppingCriterion,
                                       TimeHierarchy, build_uniform_grid, configs)
    spec = configs.config3(grids=2, strategy="delayed")
    mg = spec["mgrit"]
    prob = GpuFemProblem(spec, device=local)
    grid = build_uniform_grid(0.0, spec["tf"], spec["n_steps"])
    solver = MgritSolver(prob, TimeHierarchy.build(grid, mg["factors"]),
                         CycleSpec(kind=mg["kind"], gamma=mg["gamma"], max_iters=mg["max_iters"],
                                   spatial_strategy=mg["spatial_strategy"]),
                         StoppingCriterion(tolerance=mg["tolerance"]), transport)
    dev = prob.device
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    e0.record(stream)
    run, _ = solver.solve(gather_solution=False)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    t = e0.elapsed_time(e1) / 1e3
    st = prob.total_stats()
    res = {"workload": "BASELINE config 3: nonlinear (Brauer iron annulus), 128x128 grid, 2^14 "
                       "steps, 3 levels, delayed spatial coarsening, Newton tol 1e-8",
           "time_to_solution_s": t, "value": spec["n_steps"] * prob.spatial.size(0) / t,
           "unit": "fine time-step*DOF/s", "iterations": run.iterations,
           "converged": run.converged, "failure": run.failure,
           "residual_history": _history(run),
           "newton_iterations": st["newton_iters"], "batched_cg_iterations": st["column_iters"],
           "note": "first solve of a fresh problem (includes building the frozen-Jacobian "
                   "factors); parity pinned at 63^2 by tests/golden/mgrit_cfg3_n64.npz"}
    prob.close()
    return res


def run_b200(args):
    import torch
    import torch.distributed as dist
    from paper_1912_03106_b200 import (CycleSpec, DistTransport, GpuFemProblem, MgritSolver,
                                       NullTransport, StoppingCriterion, TimeHierarchy,
                                       build, build_uniform_grid)
    build.build()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    # dev check of the multi-rank plumbing on a 1-GPU box: every rank on
    # cuda:0, gloo (host-staged) instead of NCCL -- never a measurement
    share = os.environ.get("PINTGPU_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
        transport = DistTransport(device=dev)
    else:
        transport = NullTransport()
    spec = headline_spec()
    mg = spec["mgrit"]
    n_steps = spec["n_steps"]

    def make_solver(problem):
        grid = build_uniform_grid(0.0, spec["tf"], n_steps)
        hier = TimeHierarchy.build(grid, mg["factors"])
        return MgritSolver(problem, hier,
                           CycleSpec(kind=mg["kind"], gamma=mg["gamma"],
                                     max_iters=mg["max_iters"],
                                     spatial_strategy=mg["spatial_strategy"]),
                           StoppingCriterion(tolerance=mg["tolerance"]), transport)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(x):
        if world > 1:
            t = torch.tensor([x], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())
        return x

    problem = GpuFemProblem(spec, device=local)
    solver = make_solver(problem)
    n0 = problem.spatial.size(0)
    for _ in range(args.warmup):
        run, _ = solver.solve(gather_solution=False)
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = problem.launch_count()
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(stream)
    runs = []
    for _ in range(args.steps):
        run, _ = solver.solve(gather_solution=False)
        runs.append(run)
    e1.record(stream)
    barrier()
    clk = clocks.stop()
    elapsed = max_over_ranks(e0.elapsed_time(e1) / 1e3)
    launches = problem.launch_count() - launches0
    value = args.steps * n_steps * n0 / elapsed
    hists = [_history(r) for r in runs]
    deterministic = all(h == hists[0] for h in hists)

    # --- per-kernel profile: one more solve with CUDA events around every
    # launch (synchronising; untimed) -- explains `value`, never measures it
    barrier()
    problem.profile(True)
    tp0 = time.perf_counter()
    solver.solve(gather_solution=False)
    torch.cuda.synchronize(dev)
    prof_elapsed = time.perf_counter() - tp0
    prof = problem.profile_read(reset=True)
    problem.profile(False)

    # --- GPU sequential time stepping on a window of the horizon
    # (extrapolated: 2^16 dependent single-column Phi calls take minutes)
    seq = None
    if world == 1 and not args.no_seq:
        from paper_1912_03106_b200 import sequential_solve
        grid = build_uniform_grid(0.0, spec["tf"], n_steps)
        pts = grid.points[:SEQ_WINDOW_STEPS + 1]
        try:
            sequential_solve(problem, pts[:17])                       # warm
            barrier()
            e0.record(stream)
            traj = sequential_solve(problem, pts)
            e1.record(stream)
            barrier()
            w = e0.elapsed_time(e1) / 1e3
            del traj
            est = w * n_steps / SEQ_WINDOW_STEPS
            seq = {"window_steps": SEQ_WINDOW_STEPS, "window_s": w,
                   "extrapolated_s": est, "label": "extrapolated from the timed window",
                   "mgrit_speedup_vs_sequential": est / (elapsed / args.steps)}
        except Exception as e:      # noqa: BLE001 -- the headline line must still print
            seq = {"skipped": f"{type(e).__name__}: {e!s:.200}"}

    # --- (last on this problem: its SPIKE chunk responses take ~20 GB more)
    # --- the same solve with the natural-order band solve (the reference's
    # dpbtrs ordering) instead of the strip solve: one solve, its time and how
    # far the two direct solvers' residual histories are apart
    natural = None
    if getattr(problem, "opts", None) is not None and problem.opts.strips and not args.no_natural:
        try:
            problem.use_strips(False)
            barrier()
            e0.record(stream)
            run_n, _ = solver.solve(gather_solution=False)
            e1.record(stream)
            barrier()
            hn, hs = np.array(_history(run_n)), np.array(_history(runs[-1]))
            same = len(hn) == len(hs)
            rel = np.abs(hn - hs) / hn if same else None
            above = hn >= mg["tolerance"] if same else None
            natural = {"time_to_solution_s": max_over_ranks(e0.elapsed_time(e1) / 1e3),
                       "iterations": run_n.iterations,
                       "residual_history": list(map(float, hn)),
                       "same_iterations_as_strip_solve": bool(run_n.iterations == runs[-1].iterations),
                       "max_rel_history_diff_vs_strip_solve_down_to_tolerance":
                           float(rel[above].max()) if same else None,
                       "rel_diff_of_the_converged_residual": float(rel[-1]) if same else None,
                       "note": "two exact direct solvers: entries down to the stopping tolerance "
                               "agree to < 1e-8; the converged residual (below it) sits on the "
                               "rounding floor of Phi"}
        except Exception as e:      # noqa: BLE001 -- e.g. no room for the SPIKE responses
            natural = {"skipped": f"{type(e).__name__}: {e!s:.200}"}
        finally:
            problem.use_strips(True)

    # the timed problem holds ~170 GB (factors, SPIKE responses, level
    # buffers): free it before the end-to-end run builds a fresh one
    lvl0_K, lvl0_n = solver.levels[0].K, solver.levels[0].n
    del solver
    problem.close()
    torch.cuda.empty_cache()

    # --- end to end through the public API: host spec in (assembly + H2D of
    # the level data and excitation tables, factorisation), solve, D2H of this
    # rank's C-point iterate (the MGRIT solution at the C-points) into pinned
    # host memory (allocated before the timed region)
    host = torch.empty((lvl0_K, lvl0_n), dtype=torch.float64, pin_memory=True)
    e2e_runs = []
    for _ in range(max(1, args.e2e_reps)):
        barrier()
        t0 = time.perf_counter()
        p2 = GpuFemProblem(spec, device=local)
        h2d = sum(g.row_ptr.nbytes + g.col_idx.nbytes + g.m_val.nbytes + g.k_val.nbytes
                  + g.shapes.nbytes + g.weights.nbytes for g in p2.grids)
        torch.cuda.synchronize(dev)
        t1 = time.perf_counter()
        s2 = make_solver(p2)                    # includes the banded factorisations
        h2d += sum(lv.inv_dt_all.numel() * 8 + sum(t.numel() * 8 for t in lv.src_all)
                   for lv in s2.levels)
        torch.cuda.synchronize(dev)
        t2 = time.perf_counter()
        run2, _ = s2.solve(gather_solution=False)
        torch.cuda.synchronize(dev)
        t3 = time.perf_counter()
        host.copy_(s2.levels[0].c_store, non_blocking=True)
        barrier()
        e2e_s = max_over_ranks(time.perf_counter() - t0)
        parts = {"problem_s": t1 - t0, "solver_setup_s": t2 - t1, "solve_s": t3 - t2,
                 "d2h_s": time.perf_counter() - t3}
        e2e_runs.append((e2e_s, parts))
        del s2
        p2.close()
        torch.cuda.empty_cache()
    e2e_sorted = sorted(e2e_runs, key=lambda x: x[0])
    e2e_s, e2e_parts = e2e_sorted[len(e2e_sorted) // 2]
    d2h = int(host.numel() * 8)
    del host

    cfg2 = config2_leg(local, transport) if not args.no_cfg2 else None
    cfg3 = config3_leg(local, transport) if not args.no_cfg3 else None
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0
    peak, peak_src = measured_peak()
    fpk, fpk_src = fp64_peak()
    kernels = summarize_kernels(prof, prof_elapsed, peak, fpk)
    # dominant kernel: the 32-column-group chains (k_band_rb<32, ...>) of the
    # GPU-filling level-0 batches; narrower batches (fewer ranks' worth of
    # columns) fall back to all chain launches
    chains = [k for k in kernels if k["name"].startswith("chain32")]
    wide = bool(chains)
    if not chains:
        chains = [k for k in kernels if k["name"].startswith("band_chain")]
    roofline = None
    if chains:
        ms = sum(k["total_ms"] for k in chains)
        fl = sum(k["alg_flops_per_launch"] * k["launches"] for k in chains)
        by = sum(k["alg_bytes_per_launch"] * k["launches"] for k in chains)
        nl = sum(k["launches"] for k in chains)
        tr = ncu_traffic()
        traffic = None
        if wide and tr and tr.get("workload") == "cfg4-headline":
            traffic = tr.get("dram_bytes_per_launch")
        roofline = {"bound": "tensor",
                    "kernel": ("k_band_wcol<64, 1, ...> (strip-system band chains of the "
                               "4,096-column level-0 batches, 2 solves x fwd + bwd)" if wide else
                               "band chains (k_band_rb / k_band_chain_ks, fwd + bwd)"),
                    "achieved": fl / (ms * 1e-3) / 1e12, "peak": fpk, "unit": "TFLOP/s",
                    "frac": fl / (ms * 1e-3) / 1e12 / fpk, "traffic": traffic,
                    "traffic_source": (tr.get("source") if traffic else None),
                    "alg_bytes_per_launch": by / nl,
                    "peak_source": fpk_src,
                    "share_of_step": (ms / 1e3) / prof_elapsed,
                    "avg_launch_ms": ms / nl, "launches": nl,
                    "hbm_achieved_gbs": by / (ms * 1e-3) / 1e9, "hbm_peak_gbs": peak,
                    "hbm_frac": by / (ms * 1e-3) / 1e9 / peak,
                    "hbm_peak_source": peak_src,
                    "alg_model": "flops 2 n w per direction, column and solve (n, w = size and "
                                 "lower bandwidth of the banded systems the kernel solves: "
                                 "dpbtrs; strip systems n = 257,792, w = 64); bytes = Y "
                                 "in/out + each distinct factor once",
                    "timing": "CUDA events around every launch in a separate profiling solve "
                              f"({prof_elapsed:.2f} s with its per-call syncs)",
                    "kernels": kernels}
    phi_bench = phi_microbench(problem_cls=GpuFemProblem, local=local, peak=peak) \
        if not args.no_phi else None
    cpu = cpu_baseline_single() if world == 1 and not args.no_cpu else None
    r = runs[-1]
    line = {
        "metric": METRIC,
        "value": value, "unit": "fine time-step*DOF/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE config 4 model, no external data)",
        "config": workload_config(spec, world),
        "time_to_solution_s": elapsed / args.steps,
        "mgrit": {"iterations": r.iterations, "converged": r.converged,
                  "residual_history": _history(r), "identical_across_steps": deterministic,
                  "phi_columns_per_solve": r.phi_columns, "phi_calls_per_solve": r.phi_calls,
                  "parity": "no CPU reference run at this size (days of CPU); pinned by "
                            "tests/golden/mgrit_cfg4shape_n128.npz (4-level cycle, reference "
                            "engine; natural-order and strip solve, tests/test_gpu_full.py, "
                            "test_gpu_strips.py), the 511^2 Phi tests and the "
                            "natural_band_solve leg of this line"},
        "e2e": {"value": n_steps * n0 / e2e_s, "unit": "fine time-step*DOF/s",
                "seconds": e2e_s, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": d2h,
                "parts": {k: round(v, 4) for k, v in e2e_parts.items()},
                "reps_s": [round(x[0], 4) for x in e2e_runs],
                "stat": "median of the repetitions in reps_s"},
        "roofline": roofline,
        "natural_band_solve": natural,
        "sequential_gpu": seq,
        "config2": cfg2,
        "config3": cfg3,
        "phi_microbench": phi_bench,
        "cpu_baseline": cpu,
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def self_launch(args):
    """--gpus N without a launcher: start N ranks on this node (one per GPU,
    NCCL), the way the driver does, and pass rank 0's line through."""
    import socket
    import torch
    share = os.environ.get("PINTGPU_BENCH_SHARE_GPU") == "1"
    if not share and torch.cuda.device_count() < args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but only "
                         f"{torch.cuda.device_count()} CUDA device(s) visible")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")          # communicator lines on stderr
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--no-phi", action="store_true", help="skip the config-5 batched-Phi leg")
    ap.add_argument("--no-cfg2", action="store_true", help="skip the config-2 leg")
    ap.add_argument("--no-cfg3", action="store_true", help="skip the config-3 (nonlinear) leg")
    ap.add_argument("--e2e-reps", type=int, default=1,
                    help="end-to-end repetitions (median reported)")
    ap.add_argument("--no-seq", action="store_true", help="skip the GPU sequential-stepping leg")
    ap.add_argument("--no-natural", action="store_true",
                    help="skip the natural-order band-solve leg")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)          # rank 0 only, host cores
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
