"""The five BASELINE.json workloads as plain model/solver specs.

A spec is a JSON-able dict read by both the product (`mesh.py`) and the CPU
oracle (`oracle/fem2d.py`), so both sides discretise exactly the same model.
Every choice the configs leave open is fixed here
once and documented in DESIGN.md 2:

* "N x N grid" = N x N cells, (N-1)^2 interior unknowns (G1).
* sigma per element by centroid; the "1e-6 regularisation added to the mass
  matrix" is a conductivity floor sigma_reg = 1e-6 S/m on every element
  (G10).
* config 1's "two opposite 0.1 x 0.1 boxes": centred at (0.15, 0.5) and
  (0.85, 0.5), opposite signs (go/return conductor) (G10).
* config 2's six slots: 0.1 x 0.1 boxes centred on r = 0.4 at 60 degree
  steps carrying A+, C-, B+, A-, C+, B- (G5); PWM modulation 0.8, no ramp
  (reference defaults, excitation.py:21-23, :68) (G6); triangle carrier as
  the config says (the reference's sawtooth stays available) (G4).
* config 3: the iron annulus 0.3 <= r <= 0.45 minus the slot boxes is
  nonlinear; config 1's disc conductivity, config 2's PWM slots (G7, G10).
* MGRIT: fixed m = 16 on every level via TimeHierarchy.build (G9), V-cycle
  (G12), FCF (gamma = 1), residual-norm stop at 1e-7, max 50 iterations.
"""

import copy
import math

MU0 = 4e-7 * math.pi
NU0 = 1.0 / MU0

_BASE = {
    "N": 32,
    "t0": 0.0,
    "tf": 0.02,
    "n_steps": 1024,
    "nu0": NU0,
    "sigma_disc": 3.7e7,
    "disc_radius": 0.25,
    "disc_center": [0.5, 0.5],
    "sigma_reg": 1e-6,
    "amplitude": 1e6,
    "sources": [],
    "excitation": None,
    "nonlinear": None,
    "n_spatial_grids": 1,
    "restriction": "injection",
    "prolongation": "bilinear",
    "mgrit": {"factors": [16], "kind": "V", "gamma": 1, "max_iters": 50,
              "spatial_strategy": "none", "tolerance": 1e-7,
              "nested_iterations": False},
    # inner solve of Phi: "cholesky" = banded Cholesky per distinct dt (the
    # reference's own cholesky_banded path); "pcg" = batched Jacobi-PCG
    "inner": {"kind": "cholesky", "rtol": 1e-13, "max_iters": 20000},
}


def _box(cx, cy, w=0.1):
    return [cx - w / 2, cy - w / 2, cx + w / 2, cy + w / 2]


def slot_sources(radius=0.4, width=0.1):
    """A+, C-, B+, A-, C+, B- at 60 degree steps (phase 1 = A, 2 = B, 3 = C)."""
    pattern = [(1, 1.0), (3, -1.0), (2, 1.0), (1, -1.0), (3, 1.0), (2, -1.0)]
    out = []
    for k, (ph, sg) in enumerate(pattern):
        th = k * math.pi / 3.0
        out.append({"box": _box(0.5 + radius * math.cos(th),
                                0.5 + radius * math.sin(th), width),
                    "phase": ph, "sign": sg})
    return out


def config1(N=32, n_steps=1024):
    s = copy.deepcopy(_BASE)
    s.update(N=N, n_steps=n_steps,
             sources=[{"box": _box(0.15, 0.5), "phase": 1, "sign": 1.0},
                      {"box": _box(0.85, 0.5), "phase": 1, "sign": -1.0}],
             excitation={"kind": "sine", "period": 0.02})
    s["name"] = "cfg1"
    return s


def config2(N=128, n_steps=2 ** 14, levels=3, carrier="triangle", grids=None,
            strategy="direct"):
    """grids/strategy default to the config's literal "coarsening by 2 per
    level" (direct, one grid per level); DESIGN.md 2 explains the
    'delayed' variant (grids=2) used where the literal one stalls."""
    s = copy.deepcopy(_BASE)
    s.update(N=N, n_steps=n_steps, sources=slot_sources(),
             excitation={"kind": "pwm", "period": 0.02, "pulses": 400,
                         "modulation": 0.8, "carrier": carrier,
                         "ramp_enabled": False},
             n_spatial_grids=levels if grids is None else grids,
             restriction="full-weighting", prolongation="bilinear")
    s["mgrit"].update(factors=[16] * (levels - 1), spatial_strategy=strategy)
    s["name"] = "cfg2"
    return s


def config3(N=128, n_steps=2 ** 14, levels=3, carrier="triangle", grids=None,
            strategy="direct"):
    s = config2(N, n_steps, levels, carrier, grids, strategy)
    s["nonlinear"] = {"r_in": 0.3, "r_out": 0.45, "k1": 3.8e-4, "k2": 2.17,
                      "k3": 3.96e-4,
                      "newton": {"tol": 1e-8, "max_iters": 10, "damping": 0.5,
                                 "max_halvings": 8}}
    # config 3's "PCG inner solve": CG on the Newton system, preconditioned by
    # the banded-Cholesky factor of the linearised operator ("cholesky"); the
    # Jacobi-preconditioned variant is inner kind "pcg"
    s["inner"].update(kind="cholesky", rtol=1e-12)
    s["name"] = "cfg3"
    return s


def config4(N=512, n_steps=2 ** 16, levels=4, carrier="triangle", grids=None,
            strategy="direct"):
    s = config2(N, n_steps, levels, carrier, grids, strategy)
    # rounding of t_{i+1} - t_i gives ~10 bitwise-distinct dt per level; at
    # 511^2 every banded factor is 2.4 GB, so factors are shared between 1/dt
    # values within 1e-12 relative (1e-16-level effect on Phi; the exact
    # reference cache key is dt_merge_rtol = 0)
    s["inner"]["dt_merge_rtol"] = 1e-12
    s["name"] = "cfg4"
    return s


def config5(N=256):
    """Isolated batched-Phi microbenchmark: config-1 coefficients on the
    256^2 mesh, dt = 0.02 / 2^14, f = 0, x0 = u_prev, Jacobi-PCG rtol 1e-10."""
    s = copy.deepcopy(_BASE)
    s.update(N=N, n_steps=2 ** 14)
    s["inner"] = {"kind": "pcg", "rtol": 1e-10, "max_iters": 20000}
    s["dt"] = 0.02 / 2 ** 14
    s["batches"] = [64, 256, 1024, 4096]
    s["name"] = "cfg5"
    return s


def with_surrogate(spec, inertia=1.0, friction=0.1):
    """Rotor angle / speed (theta, omega) one-way coupled to the field: the 2D
    form of the reference's SurrogateMachineProblem (problems.py:247-287).
    Torque = sum_i c_i u_i with c_i = sin(2 pi x_i) h^2 over the interior
    nodes (the 2D analogue of the reference's sin(2 pi x) dx); after the field
    step omega' = (omega + dt T / I) / (1 + dt friction / I), theta' = theta +
    dt omega'.  The two scalars ride along every state (norms include them,
    transfers pass them through bitwise)."""
    if inertia <= 0.0 or friction < 0.0:
        raise ValueError("need inertia > 0 and friction >= 0")
    s = copy.deepcopy(spec)
    s["surrogate"] = {"inertia": float(inertia), "friction": float(friction)}
    s["name"] = spec.get("name", "spec") + "+surrogate"
    return s


CONFIGS = {"cfg1": config1, "cfg2": config2, "cfg3": config3,
           "cfg4": config4, "cfg5": config5}
