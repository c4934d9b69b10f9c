"""Excitation restatement (oracle).  Follows reference excitation.py.

reference()  -- excitation.py:26-30     sin(2 pi t / T + shift)
carrier()    -- excitation.py:33-38     sawtooth 2 frac(p t / T) - 1
               plus the "triangle" carrier BASELINE config 2 names (G4)
pwm()        -- excitation.py:41-49     sign(a r - c), ties -> +1
ramp()       -- excitation.py:52-57
PwmSource    -- excitation.py:61-92
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
    gap = (modulation * reference(phase, t, period)
           - carrier(pulses, t, period, kind))
    out = np.where(gap >= 0.0, 1.0, -1.0)
    return out if out.ndim else float(out)


def ramp(t, period=0.02):
    x = np.asarray(t)
    out = np.where(x < 2.0 * period,
                   0.5 * (1.0 - np.cos(math.pi * x / (2.0 * period))), 1.0)
    return out if out.ndim else float(out)


class Excitation:
    """Per-phase scalar source values v_phase(t).

    kind "sine": v = reference(phase, t) (BASELINE config 1's 50 Hz source);
    kind "pwm": v = ramp * pwm(phase, t) (excitation.py:84-87), smooth
    surrogate modulation * reference (excitation.py:89-92).
    """

    def __init__(self, kind="pwm", period=0.02, pulses=400, modulation=0.8,
                 carrier="sawtooth", ramp_enabled=False):
        if kind not in ("sine", "pwm"):
            raise ValueError(kind)
        self.kind = kind
        self.period = float(period)
        self.pulses = int(pulses)
        self.modulation = float(modulation)
        self.carrier = carrier
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
        return self._ramp(t) * self.modulation * reference(phase, t,
                                                           self.period)
