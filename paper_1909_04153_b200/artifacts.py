"""On-disk formats either side of the run loop.

Byte-identical to the reference writers: ESRI-ASCII rasters (grid.py:198-268),
``dt_history.csv`` (cli.py:596-603), ``summary.json`` (cli.py:606-610) and the
snapshot naming (cli.py:572-593).  Gauge CSVs are ``observers.GaugeRecorder.
write_csv``.  Raster data blocks are formatted by ``bsq_append_rows`` in the
native library (host code, all cores) instead of one Python format per cell.
"""

from __future__ import annotations

import json
import os
import tempfile
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .grid import GHOST

DT_HISTORY_HEADER = "step,time,dt,max_cfl,max_speed,max_depth"
SNAPSHOT_FIELDS = ("w", "P", "Q", "max_w")


def atomic_write_text(path, text: str) -> None:
    """Write via a sibling temporary file and rename (grid.py:271-284)."""
    path = os.fspath(path)
    fd, tmp = tempfile.mkstemp(dir=os.path.dirname(path) or ".", prefix=".tmp-", suffix="~")
    try:
        with os.fdopen(fd, "w") as fh:
            fh.write(text)
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


@dataclass(frozen=True)
class AsciiGrid:
    values: np.ndarray  # [j, i], j increasing northward
    xll: float
    yll: float
    cellsize: float


_REQUIRED_KEYS = ("ncols", "nrows", "xllcorner", "yllcorner", "cellsize")


def load_ascii_grid(path) -> AsciiGrid:
    """Read an ESRI-ASCII raster (grid.py:212-247); NODATA cells are an error."""
    with open(path, "r") as fh:
        lines = fh.read().split("\n")
    header: dict[str, float] = {}
    row = 0
    keys = (*_REQUIRED_KEYS, "nodata_value")
    while row < len(lines):
        parts = lines[row].split()
        if len(parts) != 2 or parts[0].lower() not in keys:
            break
        header[parts[0].lower()] = float(parts[1])
        row += 1
    for key in _REQUIRED_KEYS:
        if key not in header:
            raise ValueError(f"{path}: missing required header key {key!r}")
    ncols, nrows = int(header["ncols"]), int(header["nrows"])
    data = [[float(v) for v in ln.split()] for ln in lines[row:] if ln.strip()]
    if len(data) != nrows or any(len(r) != ncols for r in data):
        raise ValueError(f"{path}: data block does not match declared {nrows} rows x {ncols} cols")
    values = np.array(data, dtype=np.float64).reshape(nrows, ncols)
    nodata = header.get("nodata_value")
    if nodata is not None and np.any(values == nodata):
        raise ValueError(f"{path}: NODATA cells present; gaps are not supported")
    return AsciiGrid(values=values[::-1].copy(), xll=header["xllcorner"],
                     yll=header["yllcorner"], cellsize=header["cellsize"])


def write_ascii_grid(path, values: np.ndarray, cellsize: float, xll: float = 0.0,
                     yll: float = 0.0, nodata: float = -9999.0) -> None:
    """ESRI-ASCII raster at full float64 precision, north row first, written
    atomically (grid.py:250-268)."""
    values = np.asarray(values, dtype=np.float64)
    if values.ndim != 2:
        raise ValueError("raster values must be 2-D")
    if values.strides[1] != values.itemsize or values.strides[0] % values.itemsize:
        values = np.ascontiguousarray(values)
    ny, nx = values.shape
    head = "\n".join([f"ncols {nx}", f"nrows {ny}", f"xllcorner {xll:.17g}",
                      f"yllcorner {yll:.17g}", f"cellsize {cellsize:.17g}",
                      f"NODATA_value {nodata:.17g}"]) + "\n"
    path = os.fspath(path)
    fd, tmp = tempfile.mkstemp(dir=os.path.dirname(path) or ".", prefix=".tmp-", suffix="~")
    try:
        with os.fdopen(fd, "w") as fh:
            fh.write(head)
        stride = values.strides[0] // values.itemsize
        n = nat.lib().bsq_append_rows(tmp.encode(), nat.ptr(values), ny, nx, stride, 1)
        if n < 0:
            raise OSError(f"formatting the raster data block into {tmp} failed")
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


def snapshot_paths(out_dir: str, fields, t: float) -> dict[str, str]:
    """``<field>_<t:012.6f>.asc`` (cli.py:572-574)."""
    stamp = f"{t:012.6f}"
    return {f: os.path.join(out_dir, f"{f}_{stamp}.asc") for f in fields}


def write_snapshots(out_dir: str, fields, sim, tracker, t: float) -> list[str]:
    """One raster per requested field of the committed state (cli.py:577-593).
    The state is downloaded once per snapshot, not per step."""
    grid = sim.bathy.grid
    ii = (slice(GHOST, GHOST + grid.ny), slice(GHOST, GHOST + grid.nx))
    need_state = any(f in ("w", "P", "Q") for f in fields)
    st = sim.download_state() if need_state else None
    sources = {"w": lambda: st.w[ii], "P": lambda: st.p[ii], "Q": lambda: st.q[ii],
               "max_w": lambda: tracker.max_w}
    written = []
    for name, path in snapshot_paths(out_dir, fields, t).items():
        write_ascii_grid(path, sources[name](), cellsize=grid.dx, xll=grid.x0, yll=grid.y0)
        written.append(path)
    return written


def write_dt_history(out_dir: str, records) -> str:
    """``dt_history.csv``, ``%.12g`` columns (cli.py:596-603)."""
    rows = [DT_HISTORY_HEADER]
    rows += [f"{r.step_index},{r.sim_time:.12g},{r.dt:.12g},{r.max_cfl:.12g},"
             f"{r.max_speed:.12g},{r.max_depth:.12g}" for r in records]
    path = os.path.join(out_dir, "dt_history.csv")
    atomic_write_text(path, "\n".join(rows) + "\n")
    return path


def write_summary(out_dir: str, payload: dict) -> str:
    """``summary.json``: indent 2, sorted keys (cli.py:606-610)."""
    path = os.path.join(out_dir, "summary.json")
    atomic_write_text(path, json.dumps(payload, indent=2, sort_keys=True) + "\n")
    return path
