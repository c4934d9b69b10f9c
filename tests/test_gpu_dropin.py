"""The drop-in boundary from the reference's side (INTEGRATION.md route A):

* the reference's OWN 1D operator (problems.py:111-146) through pg_phi_batch,
  against fixtures produced by the reference's LinearDiffusionProblem and
  engine (tests/golden/make_golden_1d.py) and a dense solve -- the settings
  of the reference's test_problems.py:56-66 and test_acceptance.py:47-62,
  :248-267;
* an engine written against the reference contract (the oracle's restatement
  of MgritSolver, one problem.step per interval) driving the GPU problem
  through ReferenceProblemAdapter.
"""

import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN, load_golden

pytestmark = pytest.mark.gpu


def _npz(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    return {k: z[k] for k in z.files}


def _sawtooth_pwm():
    """The reference's default PwmSource (excitation.py:61-92): phase 1,
    T = 0.02, 400 pulses, modulation 0.8, sawtooth carrier, no ramp."""
    from paper_1912_03106_b200.excitation import Excitation
    ex = Excitation(kind="pwm", carrier="sawtooth")
    return lambda times, smooth: ex.table([1], times, smooth)


def _dense_step(n, nu, sigma, dt, u_prev, f):
    dx = 1.0 / (n + 1)
    K = nu / dx ** 2 * (2.0 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1))
    return np.linalg.solve(K + sigma / dt * np.eye(n), f + sigma / dt * u_prev)


@pytest.mark.parametrize("inner", ["cholesky", "pcg"])
def test_reference_1d_operator_through_phi_batch(cuda, inner):
    from paper_1912_03106_b200.dropin import GpuOperatorProblem, reference_1d_levels
    fx = _npz("ref1d_step")
    n, nu, sigma = int(fx["n"]), float(fx["diffusivity"]), float(fx["mass_coeff"])
    prob = GpuOperatorProblem(reference_1d_levels(n, 1, nu, sigma), source=_sawtooth_pwm(),
                              inner=inner)
    assert np.array_equal(prob.grids[0].shapes[0], fx["shape"])
    assert np.allclose(prob.loss_weights(0).cpu().numpy(), fx["weights"], rtol=0, atol=0)
    B = fx["U"].shape[0]
    # the banded direct solve is the reference's algorithm (1e-12, its own
    # test's bar); Jacobi-PCG at rtol 1e-13 is an iterative stand-in
    rtol = 1e-12 if inner == "cholesky" else 1e-9
    U = torch.as_tensor(fx["U"], device=cuda)
    inv = 1.0 / (fx["t_next"] - fx["t_prev"])
    for smooth, key, skey in ((False, "out", "src"), (True, "out_smooth", "src_smooth")):
        src = prob.source_values(fx["t_next"], smooth)
        assert np.array_equal(src[:, 0], fx[skey])              # same excitation bits
        out = torch.empty_like(U)
        prob.phi_batch(0, U, torch.as_tensor(inv, device=cuda), torch.as_tensor(src, device=cuda),
                       out, inv_dt_host=np.ascontiguousarray(inv))
        got = out.cpu().numpy()
        assert np.allclose(got, fx[key], rtol=rtol, atol=1e-14)
        for b in range(B):
            dense = _dense_step(n, nu, sigma, 1.0 / inv[b], fx["U"][b], src[b, 0] * fx["shape"])
            assert np.allclose(got[b], dense, rtol=rtol, atol=1e-14)
    # the B = 1 contract view: fresh state, inputs untouched, deterministic
    from paper_1912_03106_b200 import BlockState
    u0 = BlockState(U[0].clone())
    a, diag = prob.step(u0, float(fx["t_prev"][0]), float(fx["t_next"][0]))
    b, _ = prob.step(u0, float(fx["t_prev"][0]), float(fx["t_next"][0]))
    assert torch.equal(a.field, b.field) and torch.equal(u0.field, U[0]) and diag.converged
    assert np.allclose(a.field.cpu().numpy(), fx["out"][0], rtol=rtol, atol=1e-14)
    prob.close()


def test_reference_1d_mgrit_matches_reference_engine(cuda):
    """Two-level exactness (reference acceptance test 1) and a 5-level V-cycle
    on the reference's own 1D problem: same iteration counts, histories and
    iterates as pintmg.mgrit_solve; MGRIT = sequential stepping to 1e-10."""
    from paper_1912_03106_b200 import (CycleSpec, StoppingCriterion, TimeHierarchy,
                                       build_uniform_grid, mgrit_solve, sequential_solve)
    from paper_1912_03106_b200.dropin import GpuOperatorProblem, reference_1d_levels
    fx = _npz("ref1d_mgrit")
    prob = GpuOperatorProblem(reference_1d_levels(31), source=_sawtooth_pwm())
    grid = build_uniform_grid(0.0, 0.02, 64)
    assert np.array_equal(grid.points, fx["times"])
    seq = sequential_solve(prob, grid.points).cpu().numpy()
    scale = np.abs(fx["seq"]).max()
    assert np.abs(seq - fx["seq"]).max() <= 1e-12 * scale
    hier = TimeHierarchy.build(grid, [4])
    for gamma, cap in ((0, 16), (1, 8)):
        run, sol = mgrit_solve(prob, hier, CycleSpec(kind="two-level", gamma=gamma, max_iters=cap),
                               StoppingCriterion(tolerance=1e-12))
        assert run.iterations == int(fx[f"iters_g{gamma}"])
        hist = np.array([run.initial_residual] + run.residual_norms)
        ref = fx[f"hist_g{gamma}"]
        # entries above the rounding floor agree to 1e-8 relative
        big = ref > 1e-9 * ref[0]
        assert np.all(np.abs(hist - ref)[big] <= 1e-8 * ref[big])
        assert np.all(hist[~big] <= 1e-9 * ref[0])
        got = sol.cpu().numpy()
        assert np.abs(got - fx[f"sol_g{gamma}"]).max() <= 1e-11 * scale
        assert np.abs(got - seq).max() <= 1e-10 * max(scale, 1.0)
    grid5 = build_uniform_grid(0.0, 0.02, 256)
    run, sol = mgrit_solve(prob, TimeHierarchy.build(grid5, [2, 2, 2, 2]),
                           CycleSpec(kind="V", gamma=1, max_iters=30),
                           StoppingCriterion(tolerance=1e-10))
    assert run.iterations == int(fx["iters5"])
    ref = fx["hist5"]
    hist = np.array([run.initial_residual] + run.residual_norms)
    big = ref > 1e-9 * ref[0]
    assert np.all(np.abs(hist - ref)[big] <= 1e-8 * ref[big])
    assert np.abs(sol.cpu().numpy() - fx["sol5"]).max() <= 1e-10 * np.abs(fx["sol5"]).max()
    prob.close()


class _OneIntervalAtATime:
    """Feeds the oracle engine's step_batch from problem.step calls with
    B = 1, in interval order: the loop of the reference's MgritSolver
    (mgrit.py:361-393)."""

    def __init__(self, adapter, oracle_problem):
        self.a = adapter
        self.spatial = oracle_problem.spatial          # host transfers (oracle)
        self.n_scalars = 0
        self.levels = oracle_problem.levels

    def loss_weights(self, level=0):
        return self.a.loss_weights(level)

    def step_batch(self, U, t_prev, t_next, spatial_level=0, smooth=False):
        from oracle.state import BlockState
        out = np.empty_like(U)
        for b in range(U.shape[0]):
            s, diag = self.a.step(BlockState(U[b], None, spatial_level), float(t_prev[b]),
                                  float(t_next[b]), spatial_level, smooth=smooth)
            assert diag.converged and s.field is not U[b]
            out[b] = s.field
        return out


def test_route_a_reference_engine_order_drives_gpu_step(cuda):
    """Config 1 (32^2, 2^10 steps, 2 levels): the restated reference engine
    calls the GPU Phi one interval at a time through the adapter and
    reproduces the reference engine's own run (tests/golden/mgrit_cfg1)."""
    from oracle import fem2d, mgrit as om, time_hierarchy as oth
    from oracle.state import BlockState
    from paper_1912_03106_b200 import GpuFemProblem
    from paper_1912_03106_b200.dropin import ReferenceProblemAdapter
    fx = load_golden("mgrit_cfg1")
    spec = fx["spec"]
    gpu = GpuFemProblem(spec, inner="cholesky")
    adapter = ReferenceProblemAdapter(gpu, BlockState)
    shim = _OneIntervalAtATime(adapter, fem2d.make_problem(spec))
    grid = oth.build_uniform_grid(0.0, spec["tf"], spec["n_steps"])
    mg = spec["mgrit"]
    run, sol = om.mgrit_solve(shim, oth.TimeHierarchy.build(grid, mg["factors"]),
                              om.CycleSpec(kind=mg["kind"], gamma=mg["gamma"],
                                           max_iters=int(fx["max_iters"])),
                              om.StoppingCriterion(tolerance=float(fx["tol"])))
    assert run.iterations == int(fx["iterations"])
    hist = np.array([run.initial_residual] + list(run.residual_norms))
    assert np.max(np.abs(hist - fx["history"]) / fx["history"]) < 1e-8
    m = int(fx["factors"][0])
    err = np.linalg.norm(sol[::m] - fx["sol_c"]) / np.linalg.norm(fx["sol_c"])
    assert err < 1e-9, err
    assert adapter.calls >= run.iterations * spec["n_steps"]      # really one call per step
    gpu.close()


def test_csr_streamed_pcg_on_an_irregular_pattern(cuda):
    """An operator that is neither a few diagonals (DIA path) nor small enough
    for the CTA-resident solver: a 5-point Laplacian + mass on an 80 x 80 grid
    in a random node ordering (6,400 unknowns, ~6,000 distinct offsets) goes
    through the CSR streamed Jacobi-PCG (pcg.cuh k_pcg_setup / k_pcg_dir /
    k_pcg_upd).  Checked against a sparse direct solve, mixed dt, with rhs add."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla
    from paper_1912_03106_b200.dropin import GpuOperatorProblem, OperatorLevel
    m = 80
    n = m * m
    rng = np.random.default_rng(3)
    T = sp.diags([-1.0, 2.0, -1.0], [-1, 0, 1], shape=(m, m))
    K = (sp.kron(sp.identity(m), T) + sp.kron(T, sp.identity(m))).tocsr() * float(m * m)
    M = sp.diags(rng.uniform(0.5, 2.0, n)).tocsr()
    perm = rng.permutation(n)
    P = sp.identity(n, format="csr")[perm]
    K, M = (P @ K @ P.T).tocsr(), (P @ M @ P.T).tocsr()
    pattern = (abs(K) + abs(M)).tocsr()
    pattern.sort_indices()
    rows, cols = pattern.nonzero()
    kv = np.asarray(K[rows, cols]).ravel()
    mv = np.asarray(M[rows, cols]).ravel()
    shape = rng.standard_normal(n)
    prob = GpuOperatorProblem([OperatorLevel(pattern.indptr, pattern.indices, mv, kv,
                                             shapes=shape[None, :])],
                              source=lambda t, smooth: np.cos(40.0 * np.asarray(t))[:, None],
                              inner="pcg", rtol=1e-12)
    B = 24
    U = rng.standard_normal((B, n))
    dts = np.where(np.arange(B) % 3 == 0, 2e-4, 1e-4)
    t_next = 0.01 + 1e-3 * np.arange(B)
    src = prob.source_values(t_next)
    G = rng.standard_normal((2, n))
    g_idx = torch.as_tensor(np.where(np.arange(B) % 4 == 1, 1, -1).astype(np.int32), device=cuda)
    out = torch.empty(B, n, dtype=torch.float64, device=cuda)
    prob.phi_batch(0, torch.as_tensor(U, device=cuda), torch.as_tensor(1.0 / dts, device=cuda),
                   torch.as_tensor(src, device=cuda), out, g=torch.as_tensor(G, device=cuda),
                   g_idx=g_idx)
    st = prob.last_stats()
    assert st["failed"] == 0 and st["batch_iters"] > 10
    got = out.cpu().numpy()
    for b in range(B):
        A = (K + M / dts[b]).tocsc()
        x = spla.spsolve(A, (M @ U[b]) / dts[b] + src[b, 0] * shape)
        if b % 4 == 1:
            x = x + G[1]
        assert np.linalg.norm(got[b] - x) <= 1e-9 * np.linalg.norm(x), b
    prob.close()
