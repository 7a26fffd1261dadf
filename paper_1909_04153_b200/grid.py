"""Grid, physical constants, bathymetry preprocessing and the prognostic
state -- the host-side data model the B200 step consumes.

Same public names and semantics as the reference data model
(/root/reference/pkg/src/boussim/grid.py:19-194) so a caller's setup code
ports unchanged; the derived static fields are computed with the same
numpy expressions, so they are bitwise identical to the reference's
(pinned by tests/test_abi_host.py::test_build_bathymetry_bitwise against
tests/golden/).

Layout: every field is float64, row-major ``[j, i]`` (j north, i east),
padded with a ``GHOST``-wide frame: shape ``(ny + 4, nx + 4)``.
``bed_face_x[j, i]`` is the bed on the face between padded cells i and i+1
(shape ``(ny + 4, nx + 3)``); ``bed_face_y[j, i]`` between rows j and j+1
(shape ``(ny + 3, nx + 4)``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

GHOST = 2


@dataclass(frozen=True)
class Grid:
    """Uniform cell-centred grid (reference grid.py:23-61)."""

    nx: int
    ny: int
    dx: float
    dy: float
    x0: float = 0.0
    y0: float = 0.0

    def __post_init__(self):
        if self.nx < 5 or self.ny < 5:
            raise ValueError(
                f"grid needs at least 5x5 interior cells, got {self.nx}x{self.ny}")
        if not (self.dx > 0.0 and self.dy > 0.0):
            raise ValueError("cell sizes must be positive")

    @property
    def shape_padded(self) -> tuple[int, int]:
        return (self.ny + 2 * GHOST, self.nx + 2 * GHOST)

    @property
    def interior(self) -> tuple[slice, slice]:
        return (slice(GHOST, GHOST + self.ny), slice(GHOST, GHOST + self.nx))

    def x_centers(self) -> np.ndarray:
        return self.x0 + (np.arange(self.nx) + 0.5) * self.dx

    def y_centers(self) -> np.ndarray:
        return self.y0 + (np.arange(self.ny) + 0.5) * self.dy

    def x_centers_padded(self) -> np.ndarray:
        return self.x0 + (np.arange(-GHOST, self.nx + GHOST) + 0.5) * self.dx

    def y_centers_padded(self) -> np.ndarray:
        return self.y0 + (np.arange(-GHOST, self.ny + GHOST) + 0.5) * self.dy

    def zeros_padded(self) -> np.ndarray:
        return np.zeros(self.shape_padded)


@dataclass(frozen=True)
class PhysParams:
    """Gravity, dispersion coefficient B and quadratic friction c_f
    (reference grid.py:64-78)."""

    g: float = 9.81
    b_disp: float = 1.0 / 15.0
    c_f: float = 0.0

    def __post_init__(self):
        if not (self.g > 0.0 and math.isfinite(self.g)):
            raise ValueError("g must be positive")
        if self.c_f < 0.0:
            raise ValueError("friction coefficient must be non-negative")
        if not math.isfinite(self.b_disp):
            raise ValueError("dispersion coefficient must be finite")


@dataclass(frozen=True)
class Bathymetry:
    """Bed and every static field the step reads (reference grid.py:86-117)."""

    grid: Grid
    ws: float
    bed: np.ndarray
    bed_eff: np.ndarray
    depth: np.ndarray
    depth_dx: np.ndarray
    depth_dy: np.ndarray
    bed_face_x: np.ndarray
    bed_face_y: np.ndarray
    h_eps: float


def build_bathymetry(grid: Grid, bed_interior, ws: float,
                     h_eps: float | None = None) -> Bathymetry:
    """Corner-averaged bed, face beds, clamped still-water depth and its
    centred slopes (reference grid.py:120-154).

    The bed is reflected three cells deep so every padded cell has four
    interior-derived corners; corner and cell means use the reference's
    pairing so ``2*bed_eff == face_w + face_e`` holds bitwise in x.
    """
    b = np.asarray(bed_interior, dtype=np.float64)
    if b.shape != (grid.ny, grid.nx):
        raise ValueError(
            f"bed shape {b.shape} does not match grid ({grid.ny}, {grid.nx})")
    if not np.all(np.isfinite(b)):
        raise ValueError("bed contains non-finite values")
    ext = np.pad(b, GHOST + 1, mode="symmetric")
    sw, nw_, se, ne = ext[:-1, :-1], ext[1:, :-1], ext[:-1, 1:], ext[1:, 1:]
    corner = 0.25 * ((sw + nw_) + (se + ne))
    fx = 0.5 * (corner[:-1, 1:-1] + corner[1:, 1:-1])
    fy = 0.5 * (corner[1:-1, :-1] + corner[1:-1, 1:])
    eff = 0.25 * ((corner[:-1, :-1] + corner[1:, :-1])
                  + (corner[:-1, 1:] + corner[1:, 1:]))
    depth = np.maximum(ws - eff, 0.0)
    ddy, ddx = np.gradient(depth, grid.dy, grid.dx)
    if h_eps is None:
        h_eps = 1e-6 * max(1.0, float(depth.max()))
    if h_eps <= 0.0:
        raise ValueError("h_eps must be positive")
    return Bathymetry(grid=grid, ws=float(ws), bed=ext[1:-1, 1:-1].copy(),
                      bed_eff=eff, depth=depth, depth_dx=ddx, depth_dy=ddy,
                      bed_face_x=fx, bed_face_y=fy, h_eps=float(h_eps))


def build_bathymetry_rows(grid: Grid, bed_rows, row0: int, ny: int, ws: float,
                          h_eps: float) -> Bathymetry:
    """The static fields of padded rows [row0, row0 + ny + 4) of the grid --
    one y-strip of ``build_bathymetry(grid, bed, ws, h_eps)`` -- computed from
    bed rows only: ``bed_rows(j0, j1)`` returns interior bed rows [j0, j1)
    (clipped to the grid).  Every value is the one the whole-grid call makes:
    the 3-cell symmetric pad is applied at the global edges only, the corner /
    face / cell means are the same elementwise expressions, and the y slope
    uses central differences inside the grid and np.gradient's one-sided ones
    at its edges (one extra depth row each side makes the strip's rows
    central).  ``h_eps`` must be the whole grid's (it depends on the global
    maximum depth).  The returned Bathymetry's grid is the strip's own
    (``ny`` rows starting at ``y0 + row0 * dy``); bed_face_y has ny + 3 rows."""
    G3 = GHOST + 1
    # ext rows [e0, e1) of the 3-padded bed (global ext row e is bed row e - 3,
    # reflected symmetrically at the grid edges like np.pad 'symmetric'):
    # enough for cell rows row0 - 1 .. row0 + ny + 4 and face rows of the strip
    e0, e1 = row0 - 1, row0 + ny + 2 * GHOST + 3
    e0c, e1c = max(e0, 0), min(e1, grid.ny + 2 * G3)
    src = np.arange(e0c, e1c) - G3
    src = np.where(src < 0, -src - 1, src)
    src = np.where(src >= grid.ny, 2 * grid.ny - 1 - src, src)
    lo, hi = int(src.min()), int(src.max()) + 1
    b = np.asarray(bed_rows(lo, hi), dtype=np.float64)
    if b.shape != (hi - lo, grid.nx):
        raise ValueError(f"bed rows shape {b.shape}, expected {(hi - lo, grid.nx)}")
    if not np.all(np.isfinite(b)):
        raise ValueError("bed contains non-finite values")
    ext = np.pad(b[src - lo], ((0, 0), (G3, G3)), mode="symmetric")
    sw, nw_, se, ne = ext[:-1, :-1], ext[1:, :-1], ext[:-1, 1:], ext[1:, 1:]
    corner = 0.25 * ((sw + nw_) + (se + ne))            # rows e0c .. e1c - 2
    fx = 0.5 * (corner[:-1, 1:-1] + corner[1:, 1:-1])
    fy = 0.5 * (corner[1:-1, :-1] + corner[1:-1, 1:])   # rows e0c .. e1c - 3
    eff = 0.25 * ((corner[:-1, :-1] + corner[1:, :-1])
                  + (corner[:-1, 1:] + corner[1:, 1:]))  # padded rows e0c .. e1c - 3
    depth = np.maximum(ws - eff, 0.0)
    ddy, ddx = np.gradient(depth, grid.dy, grid.dx)
    k = row0 - e0c  # padded row row0 within the computed blocks
    n = ny + 2 * GHOST
    sg = Grid(grid.nx, ny, grid.dx, grid.dy, grid.x0, grid.y0 + row0 * grid.dy)
    return Bathymetry(grid=sg, ws=float(ws), bed=ext[k + 1:k + 1 + n, 1:-1].copy(),
                      bed_eff=eff[k:k + n].copy(), depth=depth[k:k + n].copy(),
                      depth_dx=ddx[k:k + n].copy(), depth_dy=ddy[k:k + n].copy(),
                      bed_face_x=fx[k:k + n].copy(), bed_face_y=fy[k:k + n - 1].copy(), h_eps=float(h_eps))


@dataclass
class FieldState:
    """Surface elevation w and volume fluxes P (x) and Q (y), padded
    (reference grid.py:157-187)."""

    w: np.ndarray
    p: np.ndarray
    q: np.ndarray

    def copy(self) -> "FieldState":
        return FieldState(self.w.copy(), self.p.copy(), self.q.copy())

    def validate(self, bathy: Bathymetry) -> None:
        ii = bathy.grid.interior
        for name, arr in (("w", self.w), ("p", self.p), ("q", self.q)):
            if arr.shape != bathy.grid.shape_padded:
                raise ValueError(f"{name} has shape {arr.shape}, expected "
                                 f"{bathy.grid.shape_padded}")
            if not np.all(np.isfinite(arr[ii])):
                raise ValueError(f"{name} contains non-finite values")
        col = self.w[ii] - bathy.bed_eff[ii]
        if col.min() < -1e-10:
            j, i = np.unravel_index(np.argmin(col), col.shape)
            raise ValueError(f"negative water column at interior cell ({j}, {i}): "
                             f"w - bed = {col[j, i]:.3e}")

    def mass(self, bathy: Bathymetry) -> float:
        ii = bathy.grid.interior
        return float(np.sum(self.w[ii] - bathy.bed_eff[ii])) * bathy.grid.dx * bathy.grid.dy


def still_state(bathy: Bathymetry) -> FieldState:
    """Lake at rest (reference grid.py:190-194)."""
    w = np.maximum(bathy.ws, bathy.bed_eff)
    return FieldState(w=w, p=np.zeros_like(w), q=np.zeros_like(w))
