"""The CPU oracle against the reference's own outputs and closed forms.

Fixtures in tests/golden/ were produced by the reference engine
(/root/reference/pkg/src/pintmg/mgrit.py) driving the oracle's 2D problem
(tests/golden/make_golden.py).  The oracle's own batched engine must
reproduce them (same order of operations -> same bits)."""

import math

import numpy as np
import pytest

from conftest import load_golden
from oracle import excitation as oexc
from oracle import fem2d, mgrit as om, spatial2d, time_hierarchy as oth


def _oracle_run(fx):
    spec = fx["spec"]
    prob = fem2d.make_problem(spec)
    grid = oth.build_uniform_grid(0.0, spec["tf"], spec["n_steps"])
    mg = spec["mgrit"]
    hier = oth.TimeHierarchy.build(grid, mg["factors"])
    return om.mgrit_solve(prob, hier,
                          om.CycleSpec(kind=mg["kind"], gamma=mg["gamma"],
                                       max_iters=int(fx["max_iters"]),
                                       spatial_strategy=mg["spatial_strategy"],
                                       nested_iterations=mg.get("nested_iterations", False)),
                          om.StoppingCriterion(tolerance=float(fx["tol"])))


@pytest.mark.parametrize("name", ["mgrit_cfg1", "mgrit_cfg2_delayed_n32",
                                  "mgrit_cfg2_direct_n32", "mgrit_cfg2_fcycle_n32",
                                  "mgrit_cfg2_nested_n32"])
def test_oracle_engine_reproduces_reference_engine(name):
    fx = load_golden(name)
    run, sol = _oracle_run(fx)
    hist = np.array([run.initial_residual] + run.residual_norms)
    assert run.iterations == int(fx["iterations"])
    np.testing.assert_allclose(hist, fx["history"], rtol=1e-12, atol=0)
    if "sol_c" in fx:
        m = int(fx["factors"][0])
        np.testing.assert_allclose(sol[::m], fx["sol_c"], rtol=1e-12, atol=1e-18)


def test_oracle_engine_surrogate_scalars_match_reference_engine():
    """f3: (theta, omega) ride along every state through the reference engine
    (reference SurrogateMachineProblem semantics, problems.py:247-287): the
    oracle engine's augmented rows [field | theta, omega] reproduce it."""
    fx = load_golden("mgrit_cfg1_surrogate")
    run, sol = _oracle_run(fx)
    hist = np.array([run.initial_residual] + run.residual_norms)
    assert run.iterations == int(fx["iterations"])
    np.testing.assert_allclose(hist, fx["history"], rtol=1e-12, atol=0)
    m = int(fx["factors"][0])
    n = fx["sol_c"].shape[1]
    np.testing.assert_allclose(sol[::m, :n], fx["sol_c"], rtol=1e-12, atol=1e-18)
    np.testing.assert_allclose(sol[::m, n:], fx["sol_c_scalars"], rtol=1e-10, atol=1e-22)


def test_surrogate_step_restates_reference_update():
    """One surrogate step by hand: field step of the base problem, torque with
    the new field, backward-Euler speed then angle (problems.py:269-287)."""
    from paper_1912_03106_b200 import configs
    spec = configs.with_surrogate(configs.config1(), inertia=2.0, friction=0.5)
    prob = fem2d.make_problem(spec)
    base = fem2d.make_problem(configs.config1())
    n = prob.spatial.size(0)
    rng = np.random.default_rng(1)
    u = fem2d.BlockState(rng.standard_normal(n) * 1e-3, [0.3, -0.7])
    out, _ = prob.step(u, 0.001, 0.0015)
    f, _ = base.step(fem2d.BlockState(u.field), 0.001, 0.0015)
    assert np.array_equal(out.field, f.field)
    dt = 0.0015 - 0.001
    T = float(fem2d.surrogate_coupling(32) @ f.field)
    om_ = (-0.7 + dt * T / 2.0) / (1.0 + dt * 0.5 / 2.0)
    assert out.scalars[1] == om_ and out.scalars[0] == 0.3 + dt * om_
    with pytest.raises(ValueError):
        configs.with_surrogate(configs.config1(), inertia=0.0)


def test_direct_spatial_coarsening_stalls_in_reference():
    """Documented behaviour: config 2's literal direct coarsening stalls."""
    fx = load_golden("mgrit_cfg2_direct_n32")
    h = fx["history"]
    assert not bool(fx["converged"])
    assert h[-1] / h[-2] > 0.7          # ~15-20 % per iteration at best


def test_linear_step_matches_dense_solve():
    """test_problems.py:56-66 analogue: banded Cholesky vs dense solve."""
    from paper_1912_03106_b200 import configs
    spec = configs.config2(N=8, n_steps=64, levels=1)
    prob = fem2d.make_problem(spec)
    lv = prob.levels[0]
    rng = np.random.default_rng(0)
    u = rng.normal(size=lv.mesh.n)
    dt, t = 1e-4, 0.0123
    out, _ = prob.step(fem2d.BlockState(u), t - dt, t)
    A = (lv.K + lv.M / dt).toarray()
    f = prob.forcing(t)
    expect = np.linalg.solve(A, f + (lv.M @ u) / dt)
    np.testing.assert_allclose(out.field, expect, rtol=1e-11, atol=1e-14 * np.abs(expect).max())


def test_nonlinear_jacobian_fd_check():
    """test_problems.py:286-304 analogue on the 2D Brauer operator."""
    from paper_1912_03106_b200 import configs
    spec = configs.config3(N=8, n_steps=64, levels=1)
    prob = fem2d.make_problem(spec)
    lv = prob.levels[0]
    assert lv.iron.any()
    rng = np.random.default_rng(1)
    u = rng.normal(size=lv.mesh.n) * 0.05
    v = rng.normal(size=lv.mesh.n)
    inv_dt = 1e4
    J = lv.jacobian(u, inv_dt)

    def F(w):
        return inv_dt * (lv.M @ w) + lv.operator(w)
    eps = 1e-7
    fd = (F(u + eps * v) - F(u - eps * v)) / (2 * eps)
    assert np.linalg.norm(J @ v - fd) / np.linalg.norm(fd) < 1e-6


def test_nonlinear_reduces_to_linear_when_saturation_off():
    """k1 = 0: the Newton step equals the linear step after one iteration
    (test_problems.py:127-142 analogue)."""
    from paper_1912_03106_b200 import configs
    spec = configs.config3(N=8, n_steps=64, levels=1)
    spec["nonlinear"].update(k1=0.0, k3=1.0)
    nl = fem2d.NonlinearFemProblem(spec)
    lin_spec = dict(spec)
    lin_spec["nonlinear"] = None
    lin = fem2d.LinearFemProblem(lin_spec)
    u = fem2d.BlockState(1e-3 * np.random.default_rng(2).normal(size=nl.spatial.size(0)))
    a, da = nl.step(u, 0.001, 0.0011)
    b, _ = lin.step(u, 0.001, 0.0011)
    assert da.iterations <= 2
    np.testing.assert_allclose(a.field, b.field, rtol=1e-9, atol=1e-12)


def test_transfers_are_tensor_products_of_reference_1d():
    """Injection = field[1::2] per dimension (spatial.py:71); bilinear =
    the reference's linear interpolation per dimension (spatial.py:73-84);
    injection(prolong(e)) == e exactly (test_spatial.py:43-49)."""
    h = spatial2d.SpatialHierarchy2D(8, 2, "injection", "bilinear")
    m = h.side(0)
    f = np.arange(m * m, dtype=float)
    c = h.restrict_field(f, 0).reshape(h.side(1), h.side(1))
    assert np.array_equal(c, f.reshape(m, m)[1::2, 1::2])
    e = np.array([[1.0, 2.0, 1.0], [0.0, 3.0, 0.5], [2.0, 1.0, 4.0]])
    up = h.prolong_field(e.reshape(-1), 1).reshape(m, m)

    def lin1d(v):       # reference spatial.py:79-83
        fine = np.empty(2 * len(v) + 1)
        fine[1::2] = v
        pad = np.concatenate(([0.0], v, [0.0]))
        fine[0::2] = 0.5 * (pad[:-1] + pad[1:])
        return fine
    expect = np.array([lin1d(col) for col in np.array([lin1d(row) for row in e]).T]).T
    np.testing.assert_allclose(up, expect, rtol=0, atol=1e-15)
    assert np.array_equal(h.restrict_field(up.reshape(-1), 0), e.reshape(-1))


def test_full_weighting_is_scaled_transpose_of_bilinear():
    h = spatial2d.SpatialHierarchy2D(16, 2, "full-weighting", "bilinear")
    nf, nc = h.size(0), h.size(1)
    P = np.stack([h.prolong_field(np.eye(nc)[k], 1) for k in range(nc)], axis=1)
    R = np.stack([h.restrict_field(np.eye(nf)[k], 0) for k in range(nf)], axis=1)
    np.testing.assert_allclose(R, 0.25 * P.T, atol=1e-15)


def test_excitation_reference_values():
    """Closed forms from reference test_excitation.py / test_acceptance.py [8]."""
    T = 0.02
    assert oexc.reference(1, T / 4.0, T) == pytest.approx(1.0, abs=1e-15)
    assert oexc.reference(2, 0.0, T) == pytest.approx(-math.sqrt(3.0) / 2.0, abs=1e-15)
    assert oexc.carrier(2, 0.0, T) == pytest.approx(-1.0)
    assert oexc.carrier(2, T / 4.0, T) == pytest.approx(0.0, abs=1e-15)
    assert oexc.carrier(1, 0.75 * T, T) == pytest.approx(0.5, abs=1e-14)
    assert oexc.pwm(1, 0.01, T, 1, 0.0) == 1.0
    for pulses in (1, 40, 400):
        assert oexc.pwm(1, 0.0, T, pulses, 0.8) == 1.0
    assert oexc.ramp(T, T) == pytest.approx(0.5)
    # triangle carrier: -1 at period starts, +1 mid-period
    assert oexc.carrier(400, 0.0, T, "triangle") == -1.0
    assert oexc.carrier(400, T / 800.0, T, "triangle") == pytest.approx(1.0, abs=1e-12)


def test_time_hierarchy_matches_reference_semantics():
    g = oth.build_uniform_grid(0.0, 0.02, 2 ** 10)
    h = oth.TimeHierarchy.build(g, [16])
    assert h.grids[1].n_points == 65
    assert np.array_equal(h.grids[1].points, g.points[::16])       # bitwise
    assert h.splittings[1].factor == 16 and h.splittings[1].n_intervals == 4


def test_oracle_jacobi_pcg_matches_direct_solve():
    """oracle/pcg.py (config 5's Jacobi-PCG, checker for the GPU's) on a
    small config-5 operator: residual meets the stopping rule, the iterate is
    within kappa * rtol of the direct solve, and a tighter rtol converges to it."""
    import scipy.sparse.linalg as spla
    from oracle import fem2d
    from oracle.pcg import jacobi_pcg
    from paper_1912_03106_b200 import configs
    spec = configs.config5(N=32)
    lv = fem2d.make_problem(spec).levels[0]
    A = (lv.K + lv.M * (1.0 / spec["dt"])).tocsr()
    U = np.random.default_rng(0).standard_normal((4, A.shape[0]))
    rhs = (1.0 / spec["dt"]) * (lv.M @ U.T).T
    exp = spla.splu(A.tocsc()).solve(rhs.T).T
    for rtol, tol in ((1e-10, 1e-5), (1e-14, 1e-9)):
        x, its = jacobi_pcg(A, rhs, U, rtol)
        res = np.linalg.norm((A @ x.T).T - rhs, axis=1) / np.linalg.norm(rhs, axis=1)
        assert res.max() < 1.05 * rtol + 1e-15
        err = np.linalg.norm(x - exp, axis=1) / np.linalg.norm(exp, axis=1)
        assert err.max() < tol, (rtol, err.max())
        assert (its > 0).all()
