"""Per-step observers of the run loop, on device.

The reference run loop (cli.py:635-649) calls, after every step,
``recorder.record(sim.state, t)`` and ``tracker.update(sim.state)``: both read
the host state, which for a GPU simulator would mean a full device-to-host
copy per step.  These classes keep the reference API (scenario.py:142-299)
and accept either a host ``FieldState`` (the reference behaviour, unchanged)
or the ``Simulator`` itself, in which case:

- ``GaugeRecorder.record(sim, t)`` reads only the gauge cells: every step's
  finalize kernel samples them in its last CTA and they come back with the
  step's 104-byte result (no extra launch or synchronization);
- ``MaxSurfaceTracker.update(sim)`` folds interior w into a device-resident
  running ``np.maximum``; the fold rides on the next step's stage kernel,
  which reads w anyway.

The host arithmetic on the sampled values is the reference's, so gauge series
are bitwise equal to recording from the downloaded state.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .grid import GHOST, FieldState, Grid

GAUGE_CSV_HEADER = "t,eta,P,Q,u,v"


@dataclass(frozen=True)
class GaugeSpec:
    """A surface/flux sampling point; interval 0 records every call
    (scenario.py:142-152)."""

    gauge_id: str
    x: float
    y: float
    record_interval: float = 0.0

    def __post_init__(self):
        if self.record_interval < 0.0:
            raise ValueError("record interval must be >= 0")


def gauge_cell(grid: Grid, x: float, y: float) -> tuple[int, int]:
    """Padded (row, col) of the cell whose centre is nearest (x, y)
    (scenario.py:155-161: round half to even, as np.rint)."""
    i = int(np.rint((x - grid.x0) / grid.dx - 0.5))
    j = int(np.rint((y - grid.y0) / grid.dy - 0.5))
    if not (0 <= i < grid.nx and 0 <= j < grid.ny):
        raise ValueError(f"gauge position ({x}, {y}) outside the domain")
    return j + GHOST, i + GHOST


def _is_sim(source) -> bool:
    return hasattr(source, "watch_cells") and hasattr(source, "cell_values")


class GaugeRecorder:
    """Per-gauge time series of (t, eta, P, Q, u, v) (scenario.py:164-214).

    Velocities are fluxes over the local water column floored at ``h_eps``.
    ``record`` takes a host FieldState or the Simulator (device sampling).
    """

    def __init__(self, bathy, gauges, h_eps: float | None = None):
        self.bathy = bathy
        self.gauges = list(gauges)
        self.h_eps = bathy.h_eps if h_eps is None else h_eps
        self._cells = [gauge_cell(bathy.grid, g.x, g.y) for g in self.gauges]
        self._due = [-math.inf] * len(self.gauges)
        self.samples: dict[str, list[tuple]] = {g.gauge_id: [] for g in self.gauges}
        self._sim = None
        self._slots = None

    def _values(self, source):
        """(w, p, q) per gauge from a host state or the simulator's device."""
        if _is_sim(source):
            if source is not self._sim:
                self._sim = source
                self._slots = source.watch_cells(self._cells)
            vals = source.cell_values()
            return [tuple(vals[s]) for s in self._slots]
        return [(source.w[j, i], source.p[j, i], source.q[j, i]) for j, i in self._cells]

    def record(self, source, t: float) -> int:
        """Sample every gauge whose interval has elapsed; returns how many
        were sampled (scenario.py:184-202)."""
        due = [k for k in range(len(self.gauges)) if not (t + 1e-12 < self._due[k])]
        if not due:
            return 0
        vals = self._values(source)
        be, ws = self.bathy.bed_eff, self.bathy.ws
        for k in due:
            gauge = self.gauges[k]
            j, i = self._cells[k]
            w, p, q = (float(v) for v in vals[k])
            h = max(w - be[j, i], self.h_eps)
            self.samples[gauge.gauge_id].append((t, w - ws, p, q, p / h, q / h))
            self._due[k] = t + gauge.record_interval
        return len(due)

    def series(self, gauge_id: str) -> np.ndarray:
        """(n, 6) float array of one gauge's samples."""
        return np.array(self.samples[gauge_id], dtype=float).reshape(-1, 6)

    def write_csv(self, directory, prefix: str = "gauge_") -> list[str]:
        """One CSV per gauge (``%.12g`` columns); returns the paths."""
        from .artifacts import atomic_write_text
        written = []
        for gauge in self.gauges:
            rows = [GAUGE_CSV_HEADER]
            rows += [",".join(f"{v:.12g}" for v in rec) for rec in self.samples[gauge.gauge_id]]
            path = os.path.join(str(directory), f"{prefix}{gauge.gauge_id}.csv")
            atomic_write_text(path, "\n".join(rows) + "\n")
            written.append(path)
        return written


def record_gauges(state, recorder: GaugeRecorder, t: float) -> int:
    """Functional alias for GaugeRecorder.record (scenario.py:217-220)."""
    return recorder.record(state, t)


class MaxSurfaceTracker:
    """Per-cell running maximum of the interior water surface
    (scenario.py:289-299).

    ``update(state)`` with a host FieldState is the reference's
    ``np.maximum``; ``update(sim)`` keeps the maximum on the device (fold
    deferred into the next stage kernel) and ``max_w`` downloads it.
    """

    def __init__(self, bathy):
        self.grid = bathy.grid
        self._host = np.full((bathy.grid.ny, bathy.grid.nx), -np.inf)
        self._sim = None

    def update(self, source) -> "MaxSurfaceTracker":
        if _is_sim(source):
            if self._sim is None:
                if np.isfinite(self._host).any() or np.isnan(self._host).any():
                    raise ValueError("this tracker already holds host maxima")
                self._sim = source
                source.max_tracker(nat.MAX_RESET)
            elif source is not self._sim:
                raise ValueError("a tracker follows one simulator")
            source.max_tracker(nat.MAX_FOLD)
            return self
        if self._sim is not None:
            raise ValueError("this tracker is bound to a device simulator")
        g = GHOST
        np.maximum(self._host, source.w[g:g + self.grid.ny, g:g + self.grid.nx], out=self._host)
        return self

    @property
    def max_w(self) -> np.ndarray:
        if self._sim is not None:
            return self._sim.download_max()
        return self._host

    @max_w.setter
    def max_w(self, value):
        if self._sim is not None:
            raise ValueError("max_w of a device tracker is read-only")
        self._host = value


__all__ = ["GAUGE_CSV_HEADER", "GaugeSpec", "gauge_cell", "GaugeRecorder", "record_gauges",
           "MaxSurfaceTracker", "FieldState"]
