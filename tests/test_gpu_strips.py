"""The strip solve (csrc/strips.cuh: strips + separator Schur complement, the
path config 4's 4,096-column level-0 batches take) against the REFERENCE
engine's fixtures.  The library only switches to strips on grids of 255^2
and more and batches that fill the GPU, so these tests force it through the
127^2 fixtures (PG_STRIPS_MIN_SIDE / PG_STRIPS_MIN_B are read once per
process: the solve runs in a child process) and apply the gates of test_gpu_full.py: same iteration count,
residual history within 1e-8 relative for every entry down to the stopping
tolerance, C-point iterate within 1e-9.  The converged residual itself (below
the tolerance, ~2e-8 absolute) is only required within 1e-7: it sits on the
rounding floor of Phi, where the strip solve -- measured closer to a
long-double solution than LAPACK's natural-order dpbtrs, 1.5e-15 against
8.9e-15 at 63^2 -- cannot share the reference's rounding errors the way the
natural-order solve does."""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys
sys.path.insert(0, {tests!r})
import numpy as np, torch
import test_gpu_full as full
from conftest import load_golden
fx = load_golden({name!r})
prob, grid, run, sol = full._solve(fx)
hist = np.array([run.initial_residual] + run.residual_norms)
ref = fx["history"]
assert run.iterations == int(fx["iterations"]) and run.converged == bool(fx["converged"])
rel = np.abs(hist - ref) / ref
# 1e-8 down to the stopping tolerance; the entry below it (the converged
# residual, ~1e-8 absolute) sits on the rounding floor of Phi itself, where
# two exact direct solvers agree to ~1e-16 of the initial residual
above = ref >= float(fx["tol"])
assert rel[above].max() < 1e-8, rel
assert rel.max() < 1e-7 and np.abs(hist - ref).max() < 1e-14 * ref[0], rel
full._check_c_points(sol, fx, 1e-9)
print("STRIPS_OK", run.iterations, float(rel.max()))
"""


@pytest.mark.parametrize("name", ["mgrit_cfg2_full", "mgrit_cfg4shape_n128"])
def test_strip_solve_matches_reference_engine(cuda, name):
    env = dict(os.environ, PG_STRIPS="1", PG_STRIPS_MIN_SIDE="63", PG_STRIPS_MIN_B="8",
               PYTHONPATH=ROOT)
    code = CHILD.format(tests=os.path.join(ROOT, "tests"), name=name)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "STRIPS_OK" in r.stdout, r.stdout[-2000:]


def test_strip_solve_matches_natural_band_solve(cuda):
    """Phi of one batch through both direct solves, 255^2 (the smallest grid
    the library uses strips on), mixed dt, with the rhs add: agreement to
    rounding, far inside the 1e-12 bar of the banded-Cholesky Phi tests."""
    code = r"""
import os, sys
sys.path.insert(0, {root!r})
import numpy as np, torch
from paper_1912_03106_b200 import GpuFemProblem, configs
spec = configs.config2(N=256, n_steps=2 ** 14, levels=1)
prob = GpuFemProblem(spec, inner="cholesky")
dev, n, B = prob.device, prob.spatial.size(0), 600
rng = np.random.default_rng(1)
U = torch.as_tensor(rng.standard_normal((B, n)) * 1e-3, device=dev)
dt = 0.02 / 2 ** 14
inv_h = np.where(np.arange(B) % 3 == 0, 1.0 / (2 * dt), 1.0 / dt)
src = torch.as_tensor(prob.source_values(np.linspace(0.001, 0.019, B)), device=dev)
G = torch.as_tensor(rng.standard_normal((2, n)), device=dev)
gi = torch.as_tensor((np.arange(B) % 3 - 1).astype(np.int32), device=dev)
out = torch.empty_like(U)
prob.phi_batch(0, U, torch.as_tensor(inv_h, device=dev), src, out, g=G, g_idx=gi, inv_dt_host=inv_h)
np.save(sys.argv[1], out.cpu().numpy())
"""
    import tempfile
    outs = []
    with tempfile.TemporaryDirectory() as tmp:
        for mode in ("0", "1"):
            path = os.path.join(tmp, f"o{mode}.npy")
            env = dict(os.environ, PG_STRIPS=mode, PG_STRIPS_MIN_B="8", PYTHONPATH=ROOT)
            r = subprocess.run([sys.executable, "-c", code.format(root=ROOT), path], env=env,
                               capture_output=True, text=True, timeout=600, cwd=ROOT)
            assert r.returncode == 0, r.stderr[-4000:]
            outs.append(np.load(path))
    rel = np.linalg.norm(outs[0] - outs[1], axis=1) / np.linalg.norm(outs[0], axis=1)
    assert rel.max() < 1e-12, rel.max()


def test_use_strips_switches_at_run_time(cuda):
    """`GpuFemProblem.use_strips` (pg_solver_opts.strips) on a live problem: a
    GPU-filling batch on the 255^2 grid through the strip solve, then through
    the natural-order band solve, same inputs -- agreement to rounding."""
    import torch
    from paper_1912_03106_b200 import GpuFemProblem, configs
    spec = configs.config2(N=256, n_steps=2 ** 14, levels=1)
    prob = GpuFemProblem(spec, inner="cholesky")
    n, B = prob.spatial.size(0), 3904
    gen = torch.Generator(device=cuda).manual_seed(5)
    U = torch.randn(B, n, dtype=torch.float64, device=cuda, generator=gen) * 1e-3
    dt = 0.02 / 2 ** 14
    inv_h = np.full(B, 1.0 / dt)
    inv = torch.as_tensor(inv_h, device=cuda)
    src = torch.as_tensor(prob.source_values(np.linspace(0.001, 0.019, B)), device=cuda)
    outs = []
    for on in (True, False):
        prob.use_strips(on)
        out = torch.empty_like(U)
        prob.phi_batch(0, U, inv, src, out, inv_dt_host=inv_h)
        outs.append(out)
    rel = (torch.linalg.vector_norm(outs[0] - outs[1], dim=1)
           / torch.linalg.vector_norm(outs[1], dim=1)).max().item()
    assert 0.0 < rel < 1e-12, rel          # two different direct solvers, same answer
    prob.close()


def test_engine_on_the_511_grid_strips_vs_natural(cuda):
    """A short MGRIT solve on the 511^2 grid (64 steps, 2 levels): the engine's
    setup factors the natural-order system and both strip systems concurrently
    (pg_prefactor), every Phi call takes a strip path; the same solve with
    strips off (natural-order chains + SPIKE) gives the same iteration count
    and residual history down to the stopping tolerance."""
    from paper_1912_03106_b200 import (CycleSpec, GpuFemProblem, MgritSolver, StoppingCriterion,
                                       TimeHierarchy, build_uniform_grid, configs)
    spec = configs.config2(N=512, n_steps=64, levels=2, grids=1, strategy="none")
    spec["inner"]["dt_merge_rtol"] = 1e-12
    tf = spec["tf"] * 64 / 2 ** 14
    hists = []
    for on in (True, False):
        spec["inner"]["strips"] = on
        prob = GpuFemProblem(spec, inner="cholesky")
        grid = build_uniform_grid(0.0, tf, 64)
        solver = MgritSolver(prob, TimeHierarchy.build(grid, [8]),
                             CycleSpec(kind="V", gamma=1, max_iters=10, spatial_strategy="none"),
                             StoppingCriterion(tolerance=1e-7))
        run, _ = solver.solve(gather_solution=False)
        hists.append((run.iterations, np.array([run.initial_residual] + run.residual_norms)))
        del solver
        prob.close()
    assert hists[0][0] == hists[1][0]
    hs, hn = hists[0][1], hists[1][1]
    above = hn >= 1e-7
    assert np.max(np.abs(hs - hn)[above] / hn[above]) < 1e-8
    assert np.max(np.abs(hs - hn)) < 1e-13 * hn[0]
