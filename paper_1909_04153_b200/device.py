"""Device side of one Boussinesq simulation: a libbsq context whose device
memory is a single torch-owned CUDA tensor, driven through the C ABI.

This is the only place the Python host touches device memory; everything
per cell happens in the library's sm_100a kernels.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native as nat
from .grid import GHOST


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


class DeviceStep:
    """Owns the library context for one grid.

    ``desc`` is a filled :class:`_native.Desc`; ``bathy`` supplies the
    static fields in the reference layout.
    """

    def __init__(self, desc: "nat.Desc", bathy, device=None, stream=None, cw_south=None):
        L = nat.lib()
        if not torch.cuda.is_available():
            raise RuntimeError("the B200 step needs a CUDA device (no CPU fallback)")
        self.device = torch.device(device if device is not None else "cuda")
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.desc = desc
        nbytes = L.bsq_workspace_bytes(ctypes.byref(desc))
        if nbytes == 0:
            raise ValueError(L.bsq_last_error().decode())
        self.nbytes = int(nbytes)
        with torch.cuda.device(self.device):
            self.workspace = torch.empty(self.nbytes, dtype=torch.uint8, device=self.device)
            self.stream = stream if stream is not None else torch.cuda.Stream(self.device)
        self._static = [_f64(a) for a in (bathy.bed_eff, bathy.depth, bathy.depth_dx,
                                          bathy.depth_dy, bathy.bed_face_x, bathy.bed_face_y)]
        cws = None if cw_south is None else _f64(cw_south)
        st = nat.Static(*[nat.ptr(a) for a in self._static],
                        nat.ptr(cws) if cws is not None else None)
        h = ctypes.c_void_p()
        rc = L.bsq_create(ctypes.byref(desc), ctypes.byref(st),
                          ctypes.c_void_p(self.workspace.data_ptr()), self.nbytes,
                          ctypes.c_void_p(self.stream.cuda_stream), ctypes.byref(h))
        nat.check(rc, "bsq_create")
        self._h = h
        self._static = None
        self.ny, self.nx = desc.ny, desc.nx
        self.shape = (desc.ny + 2 * GHOST, desc.nx + 2 * GHOST)
        self._res = nat.StepResult()

    def close(self):
        h = getattr(self, "_h", None)
        if h:
            nat.lib().bsq_destroy(h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- state ----------------------------------------------------------
    def upload(self, w, p, q):
        w, p, q = _f64(w), _f64(p), _f64(q)
        for a in (w, p, q):
            if a.shape != self.shape:
                raise ValueError(f"state array has shape {a.shape}, expected {self.shape}")
        nat.check(nat.lib().bsq_upload_state(self._h, nat.ptr(w), nat.ptr(p), nat.ptr(q)),
                  "upload_state")

    def download(self, pending: bool = False, out=None):
        if out is None:
            out = tuple(np.empty(self.shape) for _ in range(3))
        w, p, q = out
        nat.check(nat.lib().bsq_download_state(self._h, 1 if pending else 0, nat.ptr(w),
                                               nat.ptr(p), nat.ptr(q)), "download_state")
        return w, p, q

    # -- BSQ_Y_SPIKE strips ---------------------------------------------------------
    def spike_coeffs(self) -> np.ndarray:
        """(4, nx): v_first, v_last, w_first, w_last of this strip's spikes."""
        out = np.empty((4, self.nx))
        nat.check(nat.lib().bsq_spike_coeffs(self._h, nat.ptr(out)), "spike_coeffs")
        return out

    def set_spike_table(self, table: np.ndarray, rank: int):
        t = _f64(table)
        nat.check(nat.lib().bsq_set_spike_table(self._h, nat.ptr(t), t.shape[0], rank),
                  "set_spike_table")

    def spike_fix(self, solve: int, ybound: torch.Tensor):
        """Couple this strip's solve ``solve`` (1 or 2) to the others; ybound
        is the (G, 2, nx) device tensor of every strip's first / last row."""
        self._keep_yb = ybound  # alive until the stream has consumed it
        nat.check(nat.lib().bsq_spike_fix(self._h, solve, ctypes.c_void_p(ybound.data_ptr())),
                  "spike_fix")

    # -- observers -------------------------------------------------
    def set_gauges(self, cells):
        """Padded (row, col) cells sampled by every step's k_final."""
        rows = np.ascontiguousarray([c[0] for c in cells], dtype=np.int32)
        cols = np.ascontiguousarray([c[1] for c in cells], dtype=np.int32)
        nat.check(nat.lib().bsq_set_gauges(self._h, nat.iptr(rows), nat.iptr(cols), len(rows)),
                  "set_gauges")
        self._ngauge = len(rows)

    def gauge_values(self) -> np.ndarray:
        """(n, 3) w, P, Q at the gauges, committed state."""
        out = np.empty((getattr(self, "_ngauge", 0), 3))
        if out.shape[0]:
            nat.check(nat.lib().bsq_gauge_values(self._h, nat.ptr(out)), "gauge_values")
        return out

    def max_tracker(self, op: int):
        nat.check(nat.lib().bsq_max_tracker(self._h, op), "max_tracker")

    def download_max(self) -> np.ndarray:
        out = np.empty((self.ny, self.nx))
        nat.check(nat.lib().bsq_download_max(self._h, nat.ptr(out)), "download_max")
        return out

    def history(self, level: int, field: int) -> np.ndarray:
        out = np.empty((self.ny, self.nx))
        nat.check(nat.lib().bsq_download_history(self._h, level, field, nat.ptr(out)), "history")
        return out

    # -- stepping ---------------------------------------------------------
    def step(self, params: "nat.StepParams") -> tuple[int, "nat.StepResult"]:
        rc = nat.lib().bsq_step(self._h, ctypes.byref(params), ctypes.byref(self._res))
        if rc not in (nat.BSQ_OK, nat.BSQ_ERR_SINGULAR):
            nat.check(rc, "bsq_step")
        return rc, self._res

    def commit(self):
        nat.check(nat.lib().bsq_commit(self._h), "commit")

    # -- y-strip sharding: phased step and workspace views -----------------------
    def phase(self, ph: int, params=None):
        p = ctypes.byref(params) if params is not None else None
        rc = nat.lib().bsq_phase(self._h, ph, p, ctypes.byref(self._res))
        if rc not in (nat.BSQ_OK, nat.BSQ_ERR_SINGULAR):
            nat.check(rc, f"bsq_phase({ph})")
        return rc, self._res

    def factor_tail(self) -> np.ndarray:
        out = np.empty(self.nx)
        nat.check(nat.lib().bsq_factor_tail(self._h, nat.ptr(out)), "factor_tail")
        return out

    def pivot_flags(self):
        pos, sing = ctypes.c_int(), ctypes.c_int()
        nat.check(nat.lib().bsq_pivot_flags(self._h, ctypes.byref(pos), ctypes.byref(sing)),
                  "pivot_flags")
        return bool(pos.value), bool(sing.value)

    def _layout(self, which: int):
        off, pitch, xo, eb = ctypes.c_size_t(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        nat.check(nat.lib().bsq_array_layout(self._h, which, ctypes.byref(off), ctypes.byref(pitch),
                                             ctypes.byref(xo), ctypes.byref(eb)), "array_layout")
        return off.value, pitch.value, xo.value, eb.value

    def rows(self, which: int) -> torch.Tensor:
        """Torch view (ny+4, nx+4) of a padded device field inside the workspace."""
        off, pitch, xo, eb = self._layout(which)
        dt = torch.float64 if eb == 8 else torch.float32
        n = (self.ny + 4) * pitch * eb
        return self.workspace[off:off + n].view(dt).view(self.ny + 4, pitch)[:, xo:xo + self.nx + 4]

    def result_rate(self) -> torch.Tensor:
        """Torch view of the device step result's max CFL rate (one double)."""
        off, _, _, _ = self._layout(nat.ARR_RESULT)
        return self.workspace[off:off + 8].view(torch.float64)

    def vector(self, which: int) -> torch.Tensor:
        """Torch view of an nx-long device vector (strip boundary values)."""
        off, _, _, eb = self._layout(which)
        dt = torch.float64 if eb == 8 else torch.float32
        return self.workspace[off:off + self.nx * eb].view(dt)

    # -- kernel-level seams -------------------------------------------------
    def stage_rates(self):
        outs = [np.empty((self.ny, self.nx)) for _ in range(5)]
        nat.check(nat.lib().bsq_stage_rates(self._h, *[nat.ptr(a) for a in outs]), "stage_rates")
        return outs

    def solve_momentum(self, us, vs, pg_w, pg_e, qg_s, qg_n):
        arrs = [_f64(a) for a in (us, vs, pg_w, pg_e, qg_s, qg_n)]
        p, q = np.empty((self.ny, self.nx)), np.empty((self.ny, self.nx))
        nat.check(nat.lib().bsq_solve_momentum(self._h, *[nat.ptr(a) for a in arrs],
                                               nat.ptr(p), nat.ptr(q)), "solve_momentum")
        return p, q

    def speed_extrema(self):
        out = np.zeros(3)
        nat.check(nat.lib().bsq_speed_extrema(self._h, nat.ptr(out)), "speed_extrema")
        return float(out[0]), float(out[1]), float(out[2])

    def fill_ghosts(self, eta, flux):
        e, f = _f64(eta), _f64(flux)
        nat.check(nat.lib().bsq_fill_ghosts(self._h, nat.ptr(e), nat.ptr(f)), "fill_ghosts")

    # -- timing ---------------------------------------------------------------
    def set_timing(self, on: bool):
        nat.check(nat.lib().bsq_set_timing(self._h, 1 if on else 0), "set_timing")

    def kernel_times(self):
        n = ctypes.c_int()
        ms = (ctypes.c_float * 16)()
        names = (ctypes.c_char_p * 16)()
        nat.check(nat.lib().bsq_kernel_times(self._h, 16, ms, names, ctypes.byref(n)), "times")
        return [(names[k].decode(), float(ms[k])) for k in range(n.value)]

    def kernels_per_step(self) -> int:
        return int(nat.lib().bsq_kernels_per_step(self._h))
