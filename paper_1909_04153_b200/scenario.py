"""Synthetic inputs for the benchmark configurations.

Generators restate the reference's (/root/reference/pkg/src/boussim/
scenario.py:28-134) with identical numpy expressions so the static fields
and initial states are bitwise those the reference builds.  ``make_case``
assembles the named configs used by tests and bench.py.
"""

from __future__ import annotations

import dataclasses
import math
import warnings
from dataclasses import dataclass

import numpy as np

from . import boundary as bc
from .grid import GHOST, Grid, PhysParams, build_bathymetry, build_bathymetry_rows, still_state


@dataclass(frozen=True)
class SolitaryWaveSpec:
    height: float
    depth: float
    crest_x: float
    direction: str = "+x"
    breaking_ratio: float = 0.78

    def __post_init__(self):
        if self.depth <= 0.0:
            raise ValueError("ambient depth must be positive")
        if not 0.0 < self.height < self.breaking_ratio * self.depth:
            raise ValueError(f"waveheight {self.height} outside (0, "
                             f"{self.breaking_ratio}*depth) breaking guard")
        if self.direction not in ("+x", "-x"):
            raise ValueError("direction must be '+x' or '-x'")

    @property
    def decay_rate(self) -> float:
        return math.sqrt(3.0 * self.height / (4.0 * self.depth ** 3))


def solitary_wave_ic(spec: SolitaryWaveSpec, bathy, g: float = 9.81):
    """sech^2 surface with P = eta sqrt(g d0)(1 + eta/d0) on wet cells
    (reference scenario.py:105-134)."""
    state = still_state(bathy)
    grid = bathy.grid
    x = grid.x_centers_padded()
    eta = spec.height / np.cosh(spec.decay_rate * (x - spec.crest_x)) ** 2
    edge = max(eta[GHOST], eta[GHOST + grid.nx - 1])
    if edge > 1e-6 * spec.height:
        warnings.warn(f"solitary wave tail not contained: boundary elevation "
                      f"{edge:.3g} m exceeds {1e-6 * spec.height:.3g} m", stacklevel=2)
    eta2d = np.broadcast_to(eta, state.w.shape)
    flux = eta2d * np.sqrt(g * spec.depth) * (1.0 + eta2d / spec.depth)
    if spec.direction == "-x":
        flux = -flux
    state.w[:] = np.maximum(bathy.bed_eff, bathy.ws + eta2d)
    wet = state.w - bathy.bed_eff > 0.0
    state.p[:] = np.where(wet, flux, 0.0)
    state.q[:] = 0.0
    return state


def rip_channel_bed(grid: Grid, j0: int = 0, j1: int | None = None) -> np.ndarray:
    """Interior bed rows [j0, j1) of the rip-channel beach (reference
    scenario.py:57-72, paper Eq. 48): the same elementwise expression on the
    same cell centres, so any row range is bitwise the whole grid's rows."""
    xc, yc = np.meshgrid(grid.x_centers(), grid.y_centers()[j0:j1])
    reach = (18.0 - xc) / 30.0
    bump = 3.0 * np.exp(-(18.0 - xc) / 3.0) * np.cos(np.pi * yc / 30.0) ** 10
    return 0.1 - reach * (1.0 + bump)


def rip_channel_bathymetry(grid: Grid, h_eps=None):
    """Plane beach with a rip channel (reference scenario.py:57-72, paper Eq. 48)."""
    return build_bathymetry(grid, rip_channel_bed(grid), ws=0.0, h_eps=h_eps)


def berkhoff_bed(grid: Grid, ws: float = 0.0) -> np.ndarray:
    """Elliptic shoal on a 1:50 slope rotated 20 degrees."""
    xc, yc = np.meshgrid(grid.x_centers(), grid.y_centers())
    xs = grid.x0 + 0.5 * grid.nx * grid.dx
    ys = grid.y0 + 0.5 * grid.ny * grid.dy
    th = math.radians(20.0)
    xr = (yc - ys) * math.cos(th) - (xc - xs) * math.sin(th)
    yr = (yc - ys) * math.sin(th) + (xc - xs) * math.cos(th)
    d = np.where(yr < -5.82, 0.45, np.maximum(0.10, 0.45 - 0.02 * (5.82 + yr)))
    inside = (xr / 4.0) ** 2 + (yr / 3.0) ** 2 < 1.0
    lift = -0.3 + 0.5 * np.sqrt(np.maximum(0.0, 1.0 - (xr / 5.0) ** 2 - (yr / 3.75) ** 2))
    d = np.where(inside, d - lift, d)
    return ws - d


@dataclass
class Case:
    """Everything needed to construct a Simulator for one configuration."""

    name: str
    bathy: object
    state: object
    boundaries: object
    phys: PhysParams
    dt_init: float
    h_dry: float | None = None


def _walls():
    return bc.Boundaries(west=bc.Wall(), east=bc.Wall(), south=bc.Wall(), north=bc.Wall())


def make_case(name: str, gpus: int = 1, scale: int = 1) -> Case:
    """C1..C5 of SURVEY.md 8(d).  ``scale`` divides the C3/C4/C5 grid
    (keeping the physical domain) for quick tests; ``gpus`` sets the C5
    global extent 4096 x (4096 * gpus)."""
    if name == "C1":
        grid = Grid(1024, 5, 0.05, 0.05)
        bathy = build_bathymetry(grid, np.full((5, 1024), -0.32), ws=0.0)
        state = solitary_wave_ic(SolitaryWaveSpec(0.0576, 0.32, crest_x=15.0), bathy)
        return Case(name, bathy, state, _walls(), PhysParams(), 0.002)
    if name == "C2":
        grid = Grid(2048, 64, 0.05, 0.05)
        xc, _ = np.meshgrid(grid.x_centers(), grid.y_centers())
        bed = np.where(xc < 40.0, -0.32, -0.32 + (xc - 40.0) / 20.0)
        bathy = build_bathymetry(grid, bed, ws=0.0)
        state = solitary_wave_ic(SolitaryWaveSpec(0.0576, 0.32, crest_x=33.0), bathy)
        return Case(name, bathy, state, _walls(), PhysParams(), 0.002, h_dry=1e-3)
    if name in ("C3", "C3J"):
        # C3J: the irregular (JONSWAP) variant of the shoal
        n = 1024 // scale
        grid = Grid(n, n, 0.025 * scale, 0.025 * scale)
        bathy = build_bathymetry(grid, berkhoff_bed(grid), ws=0.0)
        d_west = float(bathy.depth[GHOST:-GHOST, GHOST].min())
        if name == "C3J":
            west = bc.IrregularMaker(tuple(bc.jonswap_components(
                bc.SpectrumSpec(0.05, 1.0, 64, 2.0 / 64, 0), d_west)))
        else:
            west = bc.SineMaker((bc.sine_component(0.0232, 1.0, d_west),))
        bounds = bc.Boundaries(west=west, east=bc.Sponge(2.0, 10.0), south=bc.Sponge(1.0, 10.0),
                               north=bc.Sponge(1.0, 10.0))
        return Case(name, bathy, still_state(bathy), bounds, PhysParams(), 0.002)
    if name in ("C4", "C5"):
        grid = rip_grid(name, gpus, scale)
        bathy = rip_channel_bathymetry(grid)
        d_west = float(bathy.depth[GHOST:-GHOST, GHOST].min())
        return Case(name, bathy, still_state(bathy), _rip_bounds(d_west),
                    PhysParams(c_f=0.0025), 0.001)
    raise ValueError(f"unknown case {name!r}")


def rip_grid(name: str, gpus: int = 1, scale: int = 1) -> Grid:
    """The C4 (4096^2) / C5 (4096 x 4096*gpus) rip-channel grid."""
    n = 4096 // scale
    ny = n * (gpus if name == "C5" else 1)
    return Grid(n, ny, 20.48 / n, 30.0 / n, x0=0.0, y0=-15.0)


def _rip_bounds(d_west: float):
    comps = bc.jonswap_components(bc.SpectrumSpec(0.13, 1.6, 68, 0.01, 7), d_west)
    return bc.Boundaries(west=bc.IrregularMaker(tuple(comps)), east=bc.Wall(),
                         south=bc.Wall(), north=bc.Wall())


@dataclass
class StripCase(Case):
    """One rank's y-strip of a case: ``bathy``/``state`` hold padded rows
    [row0, row0 + ny + 4) of the global arrays; ``grid`` is the global grid."""

    grid: Grid | None = None
    row0: int = 0


def make_strip_case(name: str, rank: int, world: int, reduce=None, scale: int = 1) -> StripCase:
    """Rank ``rank``'s strip of C4 / C5 split over ``world`` y-strips
    (parallel.split_rows), built from its own rows only -- no rank holds the
    global grid.  The two global scalars the whole-grid build derives (h_eps
    from the maximum depth, the maker's west depth from a column minimum) come
    through ``reduce(value, "max" | "min")`` (an all-reduce across ranks; None:
    single process, the values of this strip).  Bitwise the rows of
    ``make_case(name, world, scale)`` (tests/test_parallel_host.py)."""
    from .parallel import split_rows
    if name not in ("C4", "C5"):
        raise ValueError(f"strip-local build supports C4 / C5, not {name!r}")
    reduce = reduce or (lambda v, op: v)
    grid = rip_grid(name, world, scale)
    row0, ny = split_rows(grid.ny, world)[rank]
    bathy = build_bathymetry_rows(grid, lambda a, b: rip_channel_bed(grid, a, b), row0, ny,
                                  ws=0.0, h_eps=1.0)
    # build_bathymetry: h_eps = 1e-6 * max(1, depth.max()) over every padded row
    h_eps = 1e-6 * max(1.0, float(reduce(float(bathy.depth.max()), "max")))
    bathy = dataclasses.replace(bathy, h_eps=h_eps)
    d_west = float(reduce(float(bathy.depth[GHOST:-GHOST, GHOST].min()), "min"))
    return StripCase(name, bathy, still_state(bathy), _rip_bounds(d_west),
                     PhysParams(c_f=0.0025), 0.001, grid=grid, row0=row0)
