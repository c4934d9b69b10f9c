"""Source waveforms evaluated on the host, once per level and time point.

Same formulas as reference excitation.py: reference sine with three-phase
shifts (:19, :26-30), sawtooth carrier 2 frac(p t / T) - 1 (:33-38) or the
triangle carrier BASELINE config 2 names, pwm = sign(a r - c) with ties to
+1 (:41-49), startup ramp (:52-57), PwmSource.value / smooth_value (:84-92).
Values are tabulated per time point at setup and uploaded, so the device
forcing is bit-identical to the host formula.
"""

import math

import numpy as np

PHASE_SHIFTS = {1: 0.0, 2: -2.0 * math.pi / 3.0, 3: -4.0 * math.pi / 3.0}


def reference(phase, t, period=0.02):
    if phase not in PHASE_SHIFTS:
        raise ValueError(f"phase must be 1, 2 or 3, got {phase!r}")
    return np.sin(2.0 * math.pi * np.asarray(t) / period + PHASE_SHIFTS[phase])


def carrier(pulses, t, period=0.02, kind="sawtooth"):
    if pulses < 1:
        raise ValueError(f"pulses must be a positive integer, got {pulses!r}")
    x = np.asarray(t) * (pulses / period)
    frac = x - np.floor(x)
    if kind == "sawtooth":
        return 2.0 * frac - 1.0
    if kind == "triangle":
        return 1.0 - 4.0 * np.abs(frac - 0.5)
    raise ValueError(f"unknown carrier {kind!r}")


def pwm(phase, t, period=0.02, pulses=400, modulation=0.8, kind="sawtooth"):
    gap = modulation * reference(phase, t, period) - carrier(pulses, t, period, kind)
    out = np.where(gap >= 0.0, 1.0, -1.0)
    return out if out.ndim else float(out)


def ramp(t, period=0.02):
    x = np.asarray(t)
    out = np.where(x < 2.0 * period,
                   0.5 * (1.0 - np.cos(math.pi * x / (2.0 * period))), 1.0)
    return out if out.ndim else float(out)


class Excitation:
    """Per-phase source values; kind "sine" (config 1) or "pwm"."""

    def __init__(self, kind="pwm", period=0.02, pulses=400, modulation=0.8,
                 carrier="sawtooth", ramp_enabled=False):
        if kind not in ("sine", "pwm"):
            raise ValueError(f"excitation kind must be sine or pwm, got {kind!r}")
        if period <= 0.0:
            raise ValueError(f"period must be positive, got {period!r}")
        if pulses < 1:
            raise ValueError(f"pulses must be >= 1, got {pulses!r}")
        if not 0.0 <= modulation <= 1.0:
            raise ValueError(f"modulation must lie in [0, 1], got {modulation!r}")
        self.kind, self.period, self.pulses = kind, float(period), int(pulses)
        self.modulation, self.carrier = float(modulation), carrier
        self.ramp_enabled = bool(ramp_enabled)

    def _ramp(self, t):
        return ramp(t, self.period) if self.ramp_enabled else 1.0

    def value(self, phase, t):
        if self.kind == "sine":
            return self._ramp(t) * reference(phase, t, self.period)
        return self._ramp(t) * pwm(phase, t, self.period, self.pulses,
                                   self.modulation, self.carrier)

    def smooth_value(self, phase, t):
        if self.kind == "sine":
            return self._ramp(t) * reference(phase, t, self.period)
        return self._ramp(t) * self.modulation * reference(phase, t, self.period)

    def table(self, phases, times, smooth=False):
        """[len(times), len(phases)] values, the same formulas evaluated on the
        whole time array at once (tests/test_host.py checks them against the
        scalar oracle bit for bit)."""
        f = self.smooth_value if smooth else self.value
        times = np.asarray(times, dtype=float)
        out = np.zeros((len(times), len(phases)))
        for k, ph in enumerate(phases):
            out[:, k] = np.broadcast_to(f(ph, times), times.shape)
        return out
