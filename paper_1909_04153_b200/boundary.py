"""Side policies and their per-step host scalars.

Same policy types and validation as the reference
(/root/reference/pkg/src/boussim/boundary.py:22-354).  On the B200 path the
ghost strips and sponge damping are applied by device kernels; the host
only evaluates, once per step, the scalars those kernels need:

* a wavemaker's surface displacement and normal flux at t
  (:func:`maker_surface_flux`, reference boundary.py:190-199), and
* a sponge band's damping factors for the step's dt
  (:func:`sponge_band`, reference boundary.py:264-300),

with the reference's own float / numpy expressions, so the device sees the
bit-identical values the reference would have applied.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .grid import GHOST

SIDES = ("north", "south", "east", "west")  # ghost-fill order (boundary.py:25)


class ConfigurationError(ValueError):
    """A boundary configuration that cannot be run."""


@dataclass(frozen=True)
class WaveComponent:
    amplitude: float
    omega: float
    k: float
    phase: float = 0.0

    def __post_init__(self):
        if self.amplitude < 0:
            raise ValueError("wave amplitude must be non-negative")
        if self.omega <= 0 or self.k <= 0:
            raise ValueError("wave frequency and wavenumber must be positive")


@dataclass(frozen=True)
class SpectrumSpec:
    hs: float
    tp: float
    n_components: int
    df: float
    seed: int
    gamma: float = 3.3

    def __post_init__(self):
        if self.hs <= 0 or self.tp <= 0 or self.df <= 0:
            raise ValueError("Hs, Tp and df must be positive")
        if self.n_components < 1:
            raise ValueError("need at least one wave component")
        if self.gamma < 1:
            raise ValueError("peak enhancement must be >= 1")


@dataclass(frozen=True)
class Wall:
    kind: str = field(default="wall", init=False)


@dataclass(frozen=True)
class SineMaker:
    components: tuple
    kind: str = field(default="sine", init=False)

    def __post_init__(self):
        object.__setattr__(self, "components", tuple(self.components))
        if len(self.components) != 1:
            raise ValueError("sine maker carries exactly one component")


@dataclass(frozen=True)
class IrregularMaker:
    components: tuple
    kind: str = field(default="irregular", init=False)

    def __post_init__(self):
        object.__setattr__(self, "components", tuple(self.components))
        if not self.components:
            raise ValueError("irregular maker needs at least one component")


@dataclass(frozen=True)
class Sponge:
    width: float
    lambda_max: float
    kind: str = field(default="sponge", init=False)

    def __post_init__(self):
        if self.width <= 0:
            raise ValueError("sponge width must be positive")
        if self.lambda_max < 0:
            raise ValueError("sponge strength must be non-negative")


@dataclass
class Boundaries:
    west: object
    east: object
    south: object
    north: object

    def side(self, name: str):
        return getattr(self, name)

    def validate(self, bathy) -> None:
        """Makers need wet edges; sponges need two cells (boundary.py:332-354)."""
        validate_boundaries(self, bathy)


def policy_kind(policy) -> str:
    """'wall' | 'maker' | 'sponge' for any policy object carrying the
    reference's ``kind`` tag (ours or boussim's own dataclasses)."""
    kind = getattr(policy, "kind", None)
    if kind == "wall":
        return "wall"
    if kind in ("sine", "irregular"):
        return "maker"
    if kind == "sponge":
        return "sponge"
    raise ConfigurationError(f"unknown boundary policy {policy!r}")


def validate_boundaries(boundaries, bathy) -> None:
    grid = bathy.grid
    g = GHOST
    edge_depth = {
        "west": bathy.depth[g:-g, g], "east": bathy.depth[g:-g, -g - 1],
        "south": bathy.depth[g, g:-g], "north": bathy.depth[-g - 1, g:-g],
    }
    for name in SIDES:
        pol = boundaries.side(name) if hasattr(boundaries, "side") else getattr(boundaries, name)
        kind = policy_kind(pol)
        if kind == "maker" and edge_depth[name].min() <= 0.0:
            raise ConfigurationError(
                f"wavemaker on {name} side requires positive still-water depth "
                f"along the whole boundary")
        if kind == "sponge":
            cell = grid.dx if name in ("west", "east") else grid.dy
            if pol.width < 2.0 * cell:
                raise ConfigurationError(
                    f"sponge on {name} side must span at least two cells "
                    f"(width {pol.width} < {2 * cell})")


def solve_dispersion(omega: float, d: float, g: float = 9.81) -> float:
    """k from omega^2 = g k tanh(k d): bracketed Newton from the deep-water
    seed (reference boundary.py:107-131)."""
    if omega <= 0 or d <= 0 or g <= 0:
        raise ValueError("omega, depth and g must all be positive")
    target = omega * omega
    lo = target / g
    hi = 2.0 * max(lo, omega / math.sqrt(g * d))
    for _ in range(200):
        if target - g * hi * math.tanh(hi * d) < 0:
            break
        lo = hi
        hi *= 2.0
    k = target / g
    for _ in range(100):
        th = math.tanh(k * d)
        resid = target - g * k * th
        if abs(resid) <= 1e-13 * target:
            return k
        if resid > 0:
            lo = k
        else:
            hi = k
        slope = -g * (th + k * d * (1.0 - th * th))
        k_new = k - resid / slope
        if not (lo < k_new < hi):
            k_new = 0.5 * (lo + hi)
        k = k_new
    raise RuntimeError(f"dispersion solve did not converge for omega={omega}, d={d}")


def sine_component(amplitude: float, period: float, d_boundary: float,
                   g: float = 9.81, phase: float = 0.0) -> WaveComponent:
    omega = 2.0 * math.pi / period
    return WaveComponent(amplitude=amplitude, omega=omega,
                         k=solve_dispersion(omega, d_boundary, g), phase=phase)


def jonswap_density(f: float, fp: float, gamma: float, g: float = 9.81) -> float:
    sigma = 0.07 if f <= fp else 0.09
    r = math.exp(-((f - fp) ** 2) / (2.0 * sigma ** 2 * fp ** 2))
    return (g * g * (2.0 * math.pi) ** -4 * f ** -5
            * math.exp(-1.25 * (fp / f) ** 4) * gamma ** r)


def jonswap_components(spec: SpectrumSpec, d_boundary: float,
                       g: float = 9.81) -> list:
    """Peak-centred JONSWAP discretization rescaled to Hs, seeded phases
    (reference boundary.py:160-187)."""
    if d_boundary <= 0:
        raise ConfigurationError("spectral wavemaker needs positive still-water depth")
    fp = 1.0 / spec.tp
    n = spec.n_components
    freqs = fp + (np.arange(n) - n // 2) * spec.df
    freqs = freqs[freqs > 0.0]
    dens = np.array([jonswap_density(f, fp, spec.gamma, g) for f in freqs])
    amps = np.sqrt(2.0 * dens * spec.df)
    amps *= spec.hs / (4.0 * math.sqrt(np.sum(amps ** 2) / 2.0))
    phases = np.random.default_rng(spec.seed).uniform(0.0, 2.0 * math.pi, size=freqs.size)
    out = []
    for a, f, phi in zip(amps, freqs, phases):
        omega = 2.0 * math.pi * f
        out.append(WaveComponent(amplitude=float(a), omega=float(omega),
                                 k=solve_dispersion(omega, d_boundary, g), phase=float(phi)))
    return out


def maker_surface_flux(components, t: float) -> tuple[float, float]:
    """(eta, normal flux) of a maker at time t, summed in component order."""
    eta = 0.0
    flux = 0.0
    for c in components:
        s = c.amplitude * math.sin(c.omega * t + c.phase)
        eta += s
        flux += s * (c.omega / c.k)
    return eta, flux


def sponge_band(grid, side: str, width: float, lambda_max: float):
    """Static band geometry of one sponge: (first index, distances s of the
    band cells from the edge in ascending index order) or None when there
    is nothing to damp.  Index is a column for east/west, a row otherwise."""
    if lambda_max == 0.0:
        return None
    if side in ("west", "east"):
        s = (np.arange(grid.nx) + 0.5) * grid.dx
        if side == "east":
            s = s[::-1]
    else:
        s = (np.arange(grid.ny) + 0.5) * grid.dy
        if side == "north":
            s = s[::-1]
    in_band = s < width
    if not in_band.any():
        return None
    idx = np.flatnonzero(in_band)
    return int(idx[0]), s[in_band].copy()


def sponge_factors(s_band: np.ndarray, width: float, lambda_max: float,
                   dt: float) -> np.ndarray:
    """exp(-lambda dt) per band cell, the reference's numpy expression."""
    lam = lambda_max * ((width - s_band) / width) ** 2
    return np.exp(-lam * dt)
