"""Scheme knobs of the FV core (reference hydro.py:20-33)."""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class NumericsParams:
    """Limiter sharpness theta and the CFL target of the step controller."""

    theta: float = 1.5
    cfl_target: float = 0.125

    def __post_init__(self):
        if not 1.0 <= self.theta <= 2.0:
            raise ValueError(f"theta must be in [1, 2], got {self.theta}")
        if not 0.0 < self.cfl_target < 0.25:
            raise ValueError(f"cfl_target must be in (0, 0.25), got {self.cfl_target}")
