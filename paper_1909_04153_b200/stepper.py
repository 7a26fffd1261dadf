"""Drop-in for ``boussim.stepper`` whose step runs on a B200.

``Simulator`` keeps the reference constructor, methods, attributes and
error behaviour (/root/reference/pkg/src/boussim/stepper.py:145-340) so the
one production construction site (cli.py:544-547) and the reference's
tests can switch to it.  Per step the host evaluates only the reference's
fp64 scalars -- AB3/VFD weights, maker values, sponge factors, the lazy-EMA
controller -- and one ``bsq_step`` call runs the whole per-cell pipeline on
the device (see include/bsq.h); the host reads back five reductions and a
few flags.  The state stays resident in HBM: ``Simulator.state`` is a
host copy downloaded on access (and uploaded again if the caller edits it).

Inputs may be this package's data model or the reference's own objects
(anything with the same attributes): policies are dispatched on their
``kind`` tag.
"""

from __future__ import annotations

import math
import warnings
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from . import boundary as bc
from . import multistep
from .device import DeviceStep
from .grid import GHOST, FieldState, PhysParams
from .hydro import NumericsParams

DT_MIN_DEFAULT = 1e-7
MODES = ("adaptive", "fixed")
SOLVERS = ("thomas", "cr")
_KIND_CODE = {"wall": nat.WALL, "maker": nat.MAKER, "sponge": nat.SPONGE}
_STAGE_NAMES = ("e", "f", "g", "fstar", "gstar")


try:  # the reference package, when it is installed beside this one
    from boussim.stepper import InstabilityError as _InstabilityBase
except Exception:  # noqa: BLE001 -- absent (or unimportable): a plain RuntimeError
    _InstabilityBase = RuntimeError


class InstabilityError(_InstabilityBase):
    """The run blew up; carries a snapshot of the offending state.

    A subclass of ``boussim.stepper.InstabilityError`` whenever boussim is
    importable, so the reference's own ``except stepper.InstabilityError``
    (cli.py:654) catches it after the one-line swap of INTEGRATION.md."""

    def __init__(self, message: str, step_index: int, sim_time: float, state=None):
        RuntimeError.__init__(self, message)  # the same fields either base sets
        self.step_index = step_index
        self.sim_time = sim_time
        self.state = state


@dataclass
class TimeController:
    """Step-size state and controller parameters (reference stepper.py:34-67)."""

    dt_init: float
    cfl_target: float = 0.125
    alpha: float = 0.2
    mode: str = "adaptive"
    dt_min: float = DT_MIN_DEFAULT
    dt_max: float | None = None
    dt: float = field(init=False)
    dt_prev: float = field(init=False, default=math.nan)
    dt_prev2: float = field(init=False, default=math.nan)
    step_index: int = field(init=False, default=1)
    sim_time: float = field(init=False, default=0.0)

    def __post_init__(self):
        if not (math.isfinite(self.dt_init) and self.dt_init > 0):
            raise ValueError(f"dt_init must be positive, got {self.dt_init}")
        if self.dt_max is None:
            self.dt_max = 10.0 * self.dt_init
        if not (0.0 < self.dt_min <= self.dt_init <= self.dt_max):
            raise ValueError(f"need 0 < dt_min <= dt_init <= dt_max, got "
                             f"({self.dt_min}, {self.dt_init}, {self.dt_max})")
        if not 0.0 < self.alpha <= 1.0:
            raise ValueError(f"alpha must be in (0, 1], got {self.alpha}")
        if not 0.0 < self.cfl_target < 0.25:
            raise ValueError(f"cfl_target must be in (0, 0.25), got {self.cfl_target}")
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}, got {self.mode!r}")
        self.dt = self.dt_init


@dataclass(frozen=True)
class StepRecord:
    step_index: int
    sim_time: float
    dt: float
    max_cfl: float
    max_speed: float
    max_depth: float


def lazy_ema(dt_candidate: float, dt_prev: float, alpha: float) -> float:
    """Decreases pass through, increases are blended (paper Eq. 47,
    reference stepper.py:101-106)."""
    if dt_candidate <= dt_prev:
        return dt_candidate
    return alpha * dt_candidate + (1.0 - alpha) * dt_prev


def cfl_candidate(max_rate: float, cfl_target: float, dt_min: float, dt_max: float) -> float:
    """cfl / max((|u|+c)/dx, (|v|+c)/dy) clamped to [dt_min, dt_max]; a still
    or dry domain gives dt_max (reference stepper.py:95-98)."""
    if max_rate <= 0.0:
        return dt_max
    return min(max(cfl_target / max_rate, dt_min), dt_max)


class _Stage:
    """One history level, downloaded on first access."""

    def __init__(self, dev: DeviceStep, level: int):
        self._dev, self._level, self._cache = dev, level, {}

    def __getattr__(self, name):
        if name in _STAGE_NAMES:
            if name not in self._cache:
                self._cache[name] = self._dev.history(self._level, _STAGE_NAMES.index(name))
            return self._cache[name]
        raise AttributeError(name)


class DeviceHistory:
    """Newest-first view of the device-resident stage ring
    (reference dispersion.py:38-64)."""

    def __init__(self, dev: DeviceStep):
        self._dev = dev
        self.n = 0

    def __len__(self):
        return self.n

    @property
    def newest(self):
        return _Stage(self._dev, 0)

    @property
    def middle(self):
        return _Stage(self._dev, 1)

    @property
    def oldest(self):
        return _Stage(self._dev, 2)


def _validate_state(state, bathy) -> None:
    ii = bathy.grid.interior
    for name, arr in (("w", state.w), ("p", state.p), ("q", state.q)):
        if arr.shape != bathy.grid.shape_padded:
            raise ValueError(f"{name} has shape {arr.shape}, expected {bathy.grid.shape_padded}")
        if not np.all(np.isfinite(arr[ii])):
            raise ValueError(f"{name} contains non-finite values")
    col = state.w[ii] - bathy.bed_eff[ii]
    if col.min() < -1e-10:
        j, i = np.unravel_index(np.argmin(col), col.shape)
        raise ValueError(f"negative water column at interior cell ({j}, {i}): "
                         f"w - bed = {col[j, i]:.3e}")


def _coefficients(d, slope, delta, bp13):
    curv = bp13 * d * d / delta ** 2
    drift = d * slope / (6.0 * delta)
    return drift - curv, 1.0 + 2.0 * curv, -drift - curv


class Simulator:
    """Adaptive-AB3 Boussinesq simulation whose per-step work runs on a B200.

    Constructor, ``advance``/``run`` and attributes as the reference
    (stepper.py:170-340).  Extra keywords: ``device`` (torch device spec),
    ``precision``: "fp64" (default; bitwise equal to the reference) or "fp32"
    (device storage and arithmetic in float; host API stays float64), and
    ``exact_subnormal``: the line solves and the CFL extrema also divide
    numerators under 2^-960 (values below ~1e-289, e.g. a far field decayed
    into the subnormal range) with IEEE rounding.  Off, those quotients are
    Markstein's and can miss IEEE's by an ulp; the stage is exact either way
    (bsq_device.cuh "Tiny numerators"; tests/test_gpu_tiny.py).
    """

    def __init__(self, bathy, state, boundaries, controller,
                 numerics: NumericsParams | None = None, phys: PhysParams | None = None,
                 solver: str = "thomas", blowup_bound: float | None = None,
                 cross_correction: bool = True, h_dry: float | None = None,
                 device=None, precision: str = "fp64", exact_subnormal: bool = False):
        self.bathy = bathy
        self.boundaries = boundaries
        self.controller = controller
        self.numerics = numerics if numerics is not None else \
            NumericsParams(cfl_target=controller.cfl_target)
        self.phys = phys if phys is not None else PhysParams()
        if solver not in SOLVERS:
            raise ValueError(f"unknown solver {solver!r}; expected one of {SOLVERS}")
        self.solver = solver
        self.h_dry = h_dry if h_dry is not None else 100.0 * bathy.h_eps
        if self.h_dry < 0.0:
            raise ValueError("h_dry must be non-negative")
        self._validate_inputs(state, bathy, boundaries)
        grid = self._desc_grid(bathy.grid)
        self._policies = [getattr(boundaries, s) for s in bc.SIDES]
        self._kinds = [bc.policy_kind(p) for p in self._policies]
        self._warn_dominance()

        if precision not in ("fp64", "fp32"):
            raise ValueError(f"precision must be 'fp64' or 'fp32', got {precision!r}")
        self.precision = precision
        d = nat.Desc()
        d.nx, d.ny = grid.nx, grid.ny
        d.precision = nat.FP64 if precision == "fp64" else nat.FP32
        d.solver = nat.THOMAS if solver == "thomas" else nat.CR
        d.cross_correction = 1 if cross_correction else 0
        d.exact_tiny = 1 if exact_subnormal else 0
        self._bands = [None] * 4
        for k, (side, pol, kind) in enumerate(zip(bc.SIDES, self._policies, self._kinds)):
            d.side_kind[k] = _KIND_CODE[kind]
            if kind == "sponge":
                band = bc.sponge_band(grid, side, pol.width, pol.lambda_max)
                if band is not None:
                    self._bands[k] = (band[1], pol.width, pol.lambda_max)
                    d.sponge_lo[k], d.sponge_len[k] = band[0], band[1].size
        d.dx, d.dy = grid.dx, grid.dy
        d.dx2, d.dy2 = grid.dx ** 2, grid.dy ** 2
        ph = self.phys
        d.g, d.b_disp, d.bp13, d.c_f = ph.g, ph.b_disp, ph.b_disp + 1.0 / 3.0, ph.c_f
        d.theta, d.h_eps, d.h_dry, d.ws = self.numerics.theta, bathy.h_eps, self.h_dry, bathy.ws
        self._fac_keep: list = [None] * 4
        self._dev = self._make_device(d, bathy, device)
        self._dev.upload(state.w, state.p, state.q)
        self._host_state = None      # FieldState handed out by .state
        self._host_pristine = None   # what the device held when it was handed out
        self.workspace = self._dev.workspace
        self.history = DeviceHistory(self._dev)
        self.records: list[StepRecord] = []
        self._rest = np.maximum(bathy.ws, bathy.bed_eff)
        ii = bathy.grid.interior
        amp0 = self._global_max(float(np.max(np.abs(state.w[ii] - self._rest[ii]))))
        self.initial_amplitude = amp0
        self.blowup_bound = blowup_bound if blowup_bound is not None else 10.0 * amp0 + 1.0
        self.clamped_volume = 0.0
        self.last_scheme: str | None = None
        self.cross_correction = cross_correction
        self._chain = controller.dt_init
        self._extrema = self._dev.speed_extrema()
        self._params = nat.StepParams()
        self.speculate = True  # queue the next stage behind each step (bsq_step_params.spec)
        # maker components as (amplitude, omega, k, phase) rows for the
        # native per-step sums (bsq_maker_sums == boundary.maker_surface_flux)
        self._maker_rows = [
            np.ascontiguousarray([(c.amplitude, c.omega, c.k, c.phase) for c in pol.components],
                                 dtype=np.float64).reshape(-1, 4)
            if kind == "maker" else None
            for pol, kind in zip(self._policies, self._kinds)]
        self._maker_out = np.zeros(2)
        self._maker_call = [
            (nat.lib().bsq_maker_sums, nat.ptr(r), r.shape[0], nat.ptr(self._maker_out))
            if r is not None else None for r in self._maker_rows]

    def _maker(self, k: int, t: float):
        fn, rows, n, out = self._maker_call[k]
        fn(rows, n, t, out)
        o = self._maker_out
        return float(o[0]), float(o[1])

    def _make_device(self, desc, bathy, device):
        """The device engine for the whole grid (ShardedSimulator overrides)."""
        return DeviceStep(desc, bathy, device=device)

    # hooks a strip-local ShardedSimulator overrides (its inputs are one y-strip)
    def _validate_inputs(self, state, bathy, boundaries):
        _validate_state(state, bathy)
        bc.validate_boundaries(boundaries, bathy)

    def _desc_grid(self, grid):
        """The grid the device descriptor and the sponge bands describe."""
        return grid

    def _global_max(self, x: float) -> float:
        return x

    # -- implicit operator (host copy, for inspection and the warning) ----------
    def _warn_dominance(self):
        g = self.bathy.grid
        ii = g.interior
        d = self.bathy.depth[ii]
        bp13 = self.phys.b_disp + 1.0 / 3.0
        for slope, delta, tag in ((self.bathy.depth_dx[ii], g.dx, "x"),
                                  (self.bathy.depth_dy[ii], g.dy, "y")):
            a, b, c = _coefficients(d, slope, delta, bp13)
            bad = np.abs(b) - np.abs(a) - np.abs(c) <= 0.0
            if bad.any():
                warnings.warn(f"{int(bad.sum())} {tag}-direction rows lose diagonal dominance "
                              "(steep bed relative to depth); solves may be inaccurate there",
                              UserWarning, stacklevel=3)

    @property
    def coef(self):
        """Tridiagonal coefficients (implicit.py:93-119 layout: y transposed)."""
        g = self.bathy.grid
        ii = g.interior
        d = self.bathy.depth[ii]
        bp13 = self.phys.b_disp + 1.0 / 3.0
        ax, bx, cx = _coefficients(d, self.bathy.depth_dx[ii], g.dx, bp13)
        ay, by, cy = _coefficients(d, self.bathy.depth_dy[ii], g.dy, bp13)
        from types import SimpleNamespace
        return SimpleNamespace(ax=ax, bx=bx, cx=cx, ay_t=np.ascontiguousarray(ay.T),
                               by_t=np.ascontiguousarray(by.T), cy_t=np.ascontiguousarray(cy.T))

    # -- state access -------------------------------------------------------
    def _sync_host_edits(self):
        hs = self._host_state
        if hs is None:
            return
        if self._host_pristine is None:  # large grid: no pristine copy to diff against,
            self._dev.upload(hs.w, hs.p, hs.q)  # so whatever the caller holds goes back
            self._host_state = None
            return
        pw, pp, pq = self._host_pristine
        changed = any(a.shape != b.shape or (a.view(np.uint64) != b.view(np.uint64)).any()
                      for a, b in ((hs.w, pw), (hs.p, pp), (hs.q, pq)))
        if changed:
            self._dev.upload(hs.w, hs.p, hs.q)
        self._host_state = None
        self._host_pristine = None

    @property
    def state(self) -> FieldState:
        """Host copy of the committed state, downloaded on first access after a
        step.  In-place edits of ``sim.state`` take effect at the next step,
        as in the reference: small grids (<= EDIT_TRACK_BYTES) keep a pristine
        copy and upload only if something changed; larger grids upload the
        handed-out arrays before the next step (one host-to-device copy of
        the state per access, instead of a second host copy and a diff).
        ``download_state()`` reads without that write-back."""
        if self._host_state is None:
            w, p, q = self._dev.download()
            if 3 * w.nbytes <= self.EDIT_TRACK_BYTES:
                self._host_pristine = (w.copy(), p.copy(), q.copy())
            else:
                self._host_pristine = None
            self._host_state = FieldState(w, p, q)
        return self._host_state

    @state.setter
    def state(self, new_state):
        shape = self.bathy.grid.shape_padded
        for a in (new_state.w, new_state.p, new_state.q):
            if a.shape != shape:
                raise ValueError(f"state array has shape {a.shape}, expected {shape}")
        self._host_state = None
        self._host_pristine = None
        self._dev.upload(new_state.w, new_state.p, new_state.q)

    EDIT_TRACK_BYTES = 64 << 20

    def download_state(self, out=None) -> FieldState:
        """Copy the committed state into ``out`` (a FieldState or (w, p, q),
        e.g. pinned arrays) or fresh arrays, without edit tracking."""
        arrs = None if out is None else (
            (out.w, out.p, out.q) if hasattr(out, "w") else tuple(out))
        return FieldState(*self._dev.download(out=arrs))

    def _pending_state(self) -> FieldState:
        return FieldState(*self._dev.download(pending=True))

    # -- device observers (used by observers.py) -------------------
    def watch_cells(self, cells) -> list[int]:
        """Register padded (row, col) cells that every step samples on the
        device; returns their slots in :meth:`cell_values`."""
        if not hasattr(self, "_watch"):
            self._watch, self._watch_slot = [], {}
        slots, grew = [], False
        for c in cells:
            c = (int(c[0]), int(c[1]))
            if c not in self._watch_slot:
                self._watch_slot[c] = len(self._watch)
                self._watch.append(c)
                grew = True
            slots.append(self._watch_slot[c])
        if grew:
            self._dev.set_gauges(self._watch)
        return slots

    def cell_values(self) -> np.ndarray:
        """(n, 3) w, P, Q of the committed state at the watched cells."""
        self._sync_host_edits()
        return self._dev.gauge_values()

    def max_tracker(self, op: int):
        """Running max of interior w on the device (include/bsq.h BSQ_MAX_*)."""
        self._sync_host_edits()
        self._dev.max_tracker(op)

    def download_max(self) -> np.ndarray:
        self._sync_host_edits()
        return self._dev.download_max()

    # -- single step ----------------------------------------------------------
    def advance(self, dt: float | None = None) -> StepRecord:
        c = self.controller
        dt_used = c.dt if dt is None else dt
        try:
            return self._advance(dt_used)
        except FloatingPointError as err:
            raise InstabilityError(f"aborted at step {c.step_index}, t={c.sim_time:.6g}: {err}",
                                   step_index=c.step_index, sim_time=c.sim_time,
                                   state=self.state) from err

    def _fill_params(self, t: float, dt_used: float, euler: bool) -> "nat.StepParams":
        c = self.controller
        pr = self._params
        pr.t, pr.dt, pr.euler = t, dt_used, 1 if euler else 0
        # controller state: lets the library queue the next step's stage
        # behind this one (verified against the host's own values next step)
        pr.spec = 1 if self.speculate else 0
        pr.adaptive = 1 if c.mode == "adaptive" else 0
        pr.step_index = c.step_index
        pr.cfl_target, pr.alpha, pr.dt_min, pr.dt_max = c.cfl_target, c.alpha, c.dt_min, c.dt_max
        pr.dt_init, pr.chain, pr.dt_fixed = c.dt_init, self._chain, c.dt
        pr.dt_prev = c.dt_prev if math.isfinite(c.dt_prev) else 0.0
        if not euler:
            steps = multistep.StepTriple(dt_used, c.dt_prev, c.dt_prev2)
            w = multistep.ab3_weights(steps, ratio_policy="clamp")
            s = multistep.increment_weights(steps, ratio_policy="clamp")
            pr.wc, pr.wp, pr.wp2 = w.w_cur, w.w_prev, w.w_prev2
            pr.sc, pr.sp, pr.sp2 = s
        for k, (pol, kind) in enumerate(zip(self._policies, self._kinds)):
            if kind == "maker":
                pr.maker_eta_t[k], pr.maker_flux_t[k] = self._maker(k, t)
                pr.maker_eta_n[k], pr.maker_flux_n[k] = self._maker(k, t + dt_used)
            band = self._bands[k]
            if band is not None:
                fac = np.ascontiguousarray(bc.sponge_factors(band[0], band[1], band[2], dt_used))
                self._fac_keep[k] = fac
                pr.sponge_fac[k] = nat.ptr(fac)
        return pr

    def _advance(self, dt_used: float) -> StepRecord:
        c = self.controller
        t = c.sim_time
        nx = self.bathy.grid.nx
        self._sync_host_edits()
        euler = c.step_index < 3
        rc, res = self._dev.step(self._fill_params(t, dt_used, euler))
        for name, idx in zip(_STAGE_NAMES, res.stage_bad):
            if idx >= 0:  # dispersion.py:92-98
                raise FloatingPointError(f"non-finite stage value: {name} at interior cell "
                                         f"(j={idx // nx}, i={idx % nx}) at t={t:.6g}")
        self.last_scheme = "euler" if euler else "ab3"
        if rc == nat.BSQ_ERR_SINGULAR:
            if self.solver == "cr":  # which of _kernels.py:419-446 fired
                raise ZeroDivisionError(nat.lib().bsq_last_error().decode(errors="replace"))
            raise ZeroDivisionError("singular tridiagonal system: zero pivot")
        g = self.bathy.grid
        if res.clamped > 0.0:
            self.clamped_volume += res.clamped * g.dx * g.dy
        dev = res.max_dev
        if not math.isfinite(dev) or dev > self.blowup_bound:
            raise InstabilityError(
                f"surface deviation {dev:.3g} exceeded the blow-up bound "
                f"{self.blowup_bound:.3g} at step {c.step_index}, t={t + dt_used:.6g}",
                step_index=c.step_index, sim_time=t + dt_used, state=self._pending_state())
        extrema_start = self._extrema
        self._extrema = (res.max_rate, res.max_speed, res.max_depth)
        if c.mode == "adaptive":
            for name, idx in zip(("w", "P", "Q"), res.state_bad):
                if idx >= 0:  # stepper.py:88-94
                    raise FloatingPointError(
                        f"non-finite {name} at interior cell (j={idx // nx}, i={idx % nx})")
            cand = cfl_candidate(res.max_rate, c.cfl_target, c.dt_min, c.dt_max)
            self._chain = lazy_ema(cand, self._chain, c.alpha)
            c.dt = self._chain if c.step_index + 1 >= 3 else c.dt_init
        self._dev.commit()
        if self.history.n < 3:
            self.history.n += 1
        c.dt_prev2 = c.dt_prev
        c.dt_prev = dt_used
        c.sim_time = t + dt_used
        rec = StepRecord(step_index=c.step_index, sim_time=c.sim_time, dt=dt_used,
                         max_cfl=dt_used * extrema_start[0], max_speed=extrema_start[1],
                         max_depth=extrema_start[2])
        self.records.append(rec)
        c.step_index += 1
        return rec

    # -- run loop ----------------------------------------------------------------
    def run(self, until: float, on_step=None) -> list[StepRecord]:
        """Advance to ``until``, truncating the last step (stepper.py:329-340)."""
        c = self.controller
        eps = 1e-12 * max(1.0, abs(until))
        while c.sim_time < until - eps:
            remaining = until - c.sim_time
            dt = c.dt if c.dt <= remaining else remaining
            rec = self.advance(dt)
            if on_step is not None:
                on_step(self, rec)
        return self.records

    def close(self):
        self._dev.close()


# ---------------------------------------------------------------------------
# module-level helpers the reference exposes (stepper.py:82-142).  They act on
# host arrays outside the step loop; the Simulator never calls them.


def compute_cfl_dt(state, bathy, phys, cfl_target: float, dt_min: float = DT_MIN_DEFAULT,
                   dt_max: float = math.inf) -> float:
    ii = bathy.grid.interior
    for name, arr in (("w", state.w), ("P", state.p), ("Q", state.q)):
        vals = arr[ii]
        if not np.isfinite(vals).all():
            j, i = np.argwhere(~np.isfinite(vals))[0]
            raise FloatingPointError(f"non-finite {name} at interior cell (j={int(j)}, i={int(i)})")
    h = np.maximum(state.w[ii] - bathy.bed_eff[ii], 0.0)
    hstar = np.maximum(h, bathy.h_eps)
    c = np.sqrt(phys.g * h)
    su = np.abs(state.p[ii]) / hstar + c
    sv = np.abs(state.q[ii]) / hstar + c
    g = bathy.grid
    rate = float(np.max(np.maximum(su * (1.0 / g.dx), sv * (1.0 / g.dy))))
    return cfl_candidate(rate, cfl_target, dt_min, dt_max)


def predict_w(state, history, steps):
    wts = multistep.ab3_weights(steps, ratio_policy="clamp")
    w_int = state.w[GHOST:-GHOST, GHOST:-GHOST]
    return multistep.ab3_step(w_int, history.newest.e, history.middle.e, history.oldest.e, wts)


def predict_uvstar(ustar, vstar, history, steps):
    wts = multistep.ab3_weights(steps, ratio_policy="clamp")
    sc, sp, sp2 = multistep.increment_weights(steps, ratio_policy="clamp")
    s0, s1, s2 = history.newest, history.middle, history.oldest
    base_u = ustar + (wts.w_cur * s0.f + wts.w_prev * s1.f + wts.w_prev2 * s2.f)
    base_v = vstar + (wts.w_cur * s0.g + wts.w_prev * s1.g + wts.w_prev2 * s2.g)
    return (base_u + (sc * s0.fstar + sp * s1.fstar + sp2 * s2.fstar),
            base_v + (sc * s0.gstar + sp * s1.gstar + sp2 * s2.gstar))
