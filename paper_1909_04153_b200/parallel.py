"""y-strip sharding of the Boussinesq step across GPUs.

Rank r owns interior rows [row0_r, row0_r + ny_r) of the global grid with
the full x extent.  A step is the single-GPU step cut at its exchange
points (include/bsq.h BSQ_PH_*):

  GHOST     physical ghost strips            -> halo: 2 rows of w, P, Q
  STAGE     fused stage + t+dt ghost strips
  SOLVE1F   x lines (rank local) + y lines forward sweep, pipelined across
            ranks: rank r continues each column's recurrence from rank r-1's
            last dw (exactly the single-GPU Thomas operation sequence)
  SOLVE1B   y lines back substitution, pipelined from the top rank down
                                             -> halo: 1 row of P1, Q1
  CORRECT   cross-correction right-hand sides
  SOLVE2F/B second solve, as above
  FINAL     finalize; reductions combined across ranks (max, NaN flag,
            first bad cell as a global row-major index, clamped volume
            summed in rank order)

Every per-cell operation therefore sees the same operands as on one GPU, so
a sharded run is bitwise identical to the single-GPU run (and so to the
reference) -- checked by tests/test_gpu_sharded.py with the ranks emulated
in one process on one GPU.

Two transports: ``LocalComm`` keeps all strips in this process (device
copies on one stream, sequential pipeline -- used for emulation/tests) and
``DistComm`` holds one strip per process and moves halos and boundary
vectors with torch.distributed (NCCL over NVLink on a multi-GPU box; its
host-side logic is exercised with gloo on CPU by tests/test_parallel_host.py).
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _native as nat
from .device import DeviceStep
from .grid import GHOST
from . import boundary as bc
from .stepper import Simulator

_N, _S = 0, 1  # side indices (bsq.h order N, S, E, W)
_STATE = (nat.ARR_W, nat.ARR_P, nat.ARR_Q)
_PENDING_PQ = (nat.ARR_P_NEW, nat.ARR_Q_NEW)


def split_rows(ny: int, world: int) -> list[tuple[int, int]]:
    """(row0, ny_r) per rank: as equal as possible, earlier ranks one larger."""
    if world < 1 or ny < 5 * world:
        raise ValueError(f"cannot split {ny} rows over {world} strips of >= 5 rows")
    base, extra = divmod(ny, world)
    out, r0 = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append((r0, n))
        r0 += n
    return out


def strip_band(lo_g: int, len_g: int, row0: int, ny: int):
    """Local part of a global N/S sponge band: (local lo, length, offset
    into the global factor array)."""
    lo = max(lo_g - row0, 0)
    hi = min(lo_g + len_g - row0, ny)
    if hi <= lo:
        return 0, 0, 0
    return lo, hi - lo, row0 + lo - lo_g


class _StripStatic:
    """The static fields of one strip: rows of the global padded arrays."""

    def __init__(self, bathy, row0: int, ny: int):
        rows = slice(row0, row0 + ny + 2 * GHOST)
        self.bed_eff = bathy.bed_eff[rows]
        self.depth = bathy.depth[rows]
        self.depth_dx = bathy.depth_dx[rows]
        self.depth_dy = bathy.depth_dy[rows]
        self.bed_face_x = bathy.bed_face_x[rows]
        self.bed_face_y = bathy.bed_face_y[row0:row0 + ny + 2 * GHOST - 1]


# ---------------------------------------------------------------------------
# transports


class LocalComm:
    """All strips in this process (one GPU): exchanges are device copies on
    one stream, the y-line pipeline runs the strips in rank order."""

    def __init__(self, world: int):
        self.world = world
        self.local = list(range(world))

    def is_local(self, r):
        return True

    # setup: cw tails travel rank -> rank + 1
    def pass_tail(self, tails: dict, r: int, tail):
        tails[r] = tail

    def get_tail(self, tails: dict, r: int, nx: int):
        return tails[r - 1]

    def any_flag(self, flags: list) -> bool:
        return any(flags)

    def max_scalar(self, x: float) -> float:
        return x

    def halo(self, strips, ids, nrows: int, stream, inner=None):
        """Copy ``nrows`` boundary rows of arrays ``ids`` between neighbouring
        strips; ``inner()`` queues the work that reads no halo row (it runs
        while the transfers are in flight under DistComm)."""
        if inner is not None:
            inner()
        with torch.cuda.stream(stream):
            for r in range(self.world - 1):
                lo, up = strips[r], strips[r + 1]
                n = lo.ny
                for a in ids:
                    L, U = lo.rows(a), up.rows(a)
                    U[GHOST - nrows:GHOST].copy_(L[n + GHOST - nrows:n + GHOST])
                    L[n + GHOST:n + GHOST + nrows].copy_(U[GHOST:GHOST + nrows])

    def pipeline(self, strips, ph_f: int, ph_b: int, stream):
        with torch.cuda.stream(stream):
            for r in range(self.world):
                if r > 0:
                    strips[r].vector(nat.ARR_DW_IN).copy_(strips[r - 1].vector(nat.ARR_DW_OUT))
                strips[r].phase(ph_f)
            for r in reversed(range(self.world)):
                if r < self.world - 1:
                    strips[r].vector(nat.ARR_X_IN).copy_(strips[r + 1].vector(nat.ARR_X_OUT))
                strips[r].phase(ph_b)

    def reduce(self, parts: list, nx: int, rows0: list):
        return _combine(parts, nx, rows0)

    def gather_state(self, locals_: dict, shape, ranges):
        return _assemble(locals_, shape, ranges)

    def gather_values(self, per: dict, n: int):
        """per[r] = (values (n, k), owned (n,) bool): the owners' rows."""
        return _pick_owned(per.values(), n)

    # BSQ_Y_SPIKE: static spike coefficients once, solve boundary rows per solve
    def gather_spike_table(self, per: dict, nx: int) -> np.ndarray:
        return np.stack([per[r] for r in range(self.world)])

    def max_rate(self, strips, stream) -> None:
        """Every strip's device max CFL rate <- the max over the strips
        (stream-ordered; max is exact, so this equals the host fold)."""
        with torch.cuda.stream(stream):
            vs = [strips[r].result_rate() for r in sorted(strips)]
            m = torch.stack(vs).amax(0)
            for v in vs:
                v.copy_(m)

    def spike_bounds(self, strips, arr: int, stream) -> dict:
        with torch.cuda.stream(stream):
            parts = []
            for r in range(self.world):
                R, n = strips[r].rows(arr), strips[r].ny
                parts.append(torch.stack([R[GHOST, GHOST:-GHOST], R[GHOST + n - 1, GHOST:-GHOST]]))
            yb = torch.stack(parts).contiguous()
        return {r: yb for r in range(self.world)}

    def gather_rows(self, per: dict, nx: int, ranges):
        """per[r] = strip r's interior rows (n_r, nx) -> (ny, nx)."""
        return np.concatenate([per[r] for r in range(self.world)], axis=0)


class DistComm:
    """One strip per process; halos, boundary vectors and reductions over
    torch.distributed (NCCL on GPUs; gloo for the CPU tests of this logic)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.local = [self.rank]
        # a non-NCCL backend (gloo: the CPU tests, and ranks sharing one GPU in
        # the functional multi-process GPU test) moves device rows through
        # host memory; NCCL sends device memory directly
        self.staged = dist.get_backend(group) != "nccl"

    def _wire(self, t):
        """What goes on the wire for tensor ``t`` (a host copy when staged)."""
        return t.cpu() if (self.staged and t.is_cuda) else t

    def _landing(self, t):
        """Where the transport receives into for destination ``t``: ``t``
        itself, or a host buffer copied into it afterwards when staged."""
        return torch.empty(t.shape, dtype=t.dtype, device="cpu") if (self.staged and t.is_cuda) \
            else t

    def _dev(self):
        return torch.device("cuda", torch.cuda.current_device()) \
            if self.dist.get_backend(self.group) == "nccl" else torch.device("cpu")

    def is_local(self, r):
        return r == self.rank

    def pass_tail(self, tails: dict, r: int, tail):
        if r + 1 < self.world:
            self.dist.send(torch.from_numpy(np.ascontiguousarray(tail)).to(self._dev()), r + 1,
                           group=self.group)

    def get_tail(self, tails: dict, r: int, nx: int):
        buf = torch.empty(nx, dtype=torch.float64, device=self._dev())
        self.dist.recv(buf, r - 1, group=self.group)
        return buf.cpu().numpy()

    def any_flag(self, flags: list) -> bool:
        t = torch.tensor([1 if any(flags) else 0], dtype=torch.int64, device=self._dev())
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return bool(t.item())

    def reduce_scalar(self, x: float, op: str) -> float:
        """All-reduce of one float64 ("max" or "min"); exact (no rounding)."""
        t = torch.tensor([x], dtype=torch.float64, device=self._dev())
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX if op == "max" else self.dist.ReduceOp.MIN,
                             group=self.group)
        return float(t.item())

    def max_scalar(self, x: float) -> float:
        return self.reduce_scalar(x, "max")

    def _exchange(self, send_up, send_dn, recv_up, recv_dn, inner=None):
        """Post the four transfers with the neighbours (None = no neighbour),
        queue ``inner()`` on the current stream while they are in flight, then
        make the current stream wait for them."""
        d, r, ops = self.dist, self.rank, []
        wire = []  # (staged landing buffer, device destination)
        if send_up is not None:
            land = self._landing(recv_up)
            wire.append((land, recv_up))
            ops.append(d.P2POp(d.isend, self._wire(send_up), r + 1, group=self.group))
            ops.append(d.P2POp(d.irecv, land, r + 1, group=self.group))
        if send_dn is not None:
            land = self._landing(recv_dn)
            wire.append((land, recv_dn))
            ops.append(d.P2POp(d.isend, self._wire(send_dn), r - 1, group=self.group))
            ops.append(d.P2POp(d.irecv, land, r - 1, group=self.group))
        works = d.batch_isend_irecv(ops) if ops else []
        if inner is not None:
            inner()  # interior rows: overlap the transfers
        for w in works:
            w.wait()
        for land, dst in wire:
            if land is not dst:
                dst.copy_(land)

    def halo(self, strips, ids, nrows: int, stream, inner=None):
        s = strips[self.rank]
        n = s.ny
        up, dn = self.rank + 1 < self.world, self.rank > 0
        with torch.cuda.stream(stream):
            views = [s.rows(a) for a in ids]
            send_up = torch.cat([v[n + GHOST - nrows:n + GHOST] for v in views]) if up else None
            send_dn = torch.cat([v[GHOST:GHOST + nrows] for v in views]) if dn else None
            recv_up = torch.empty_like(send_up) if up else None
            recv_dn = torch.empty_like(send_dn) if dn else None
            self._exchange(send_up, send_dn, recv_up, recv_dn, inner)
            for k, v in enumerate(views):
                if up:
                    v[n + GHOST:n + GHOST + nrows].copy_(recv_up[k * nrows:(k + 1) * nrows])
                if dn:
                    v[GHOST - nrows:GHOST].copy_(recv_dn[k * nrows:(k + 1) * nrows])

    def _recv_into(self, dst, src_rank):
        land = self._landing(dst)
        self.dist.recv(land, src_rank, group=self.group)
        if land is not dst:
            dst.copy_(land)

    def pipeline(self, strips, ph_f: int, ph_b: int, stream):
        d, r, s = self.dist, self.rank, strips[self.rank]
        with torch.cuda.stream(stream):
            if r > 0:
                self._recv_into(s.vector(nat.ARR_DW_IN), r - 1)
            s.phase(ph_f)
            if r + 1 < self.world:
                d.send(self._wire(s.vector(nat.ARR_DW_OUT)), r + 1, group=self.group)
                self._recv_into(s.vector(nat.ARR_X_IN), r + 1)
            s.phase(ph_b)
            if r > 0:
                d.send(self._wire(s.vector(nat.ARR_X_OUT)), r - 1, group=self.group)

    def reduce(self, parts: list, nx: int, rows0: list):
        """One all_gather per step: every rank's reductions (maxima, NaN flag as
        NaN, clamped volume, global first-bad indices) packed into 14
        doubles, folded on every rank in rank order like LocalComm."""
        mine = _combine(parts, nx, rows0)
        vec = torch.tensor([mine["max_rate"], mine["max_speed"], mine["max_depth"],
                            mine["max_dev"], mine["clamped"]]
                           + [float(b) for b in mine["stage_bad"] + mine["state_bad"]],
                           dtype=torch.float64, device=self._dev())
        bufs = [torch.empty_like(vec) for _ in range(self.world)]
        self.dist.all_gather(bufs, vec, group=self.group)
        rows = torch.stack(bufs).cpu().numpy()
        out = {"max_rate": 0.0, "max_speed": 0.0, "max_depth": 0.0, "max_dev": 0.0,
               "clamped": 0.0, "stage_bad": [-1] * 5, "state_bad": [-1] * 3}
        nan = False
        for r in rows:  # rank order: the clamped sum is deterministic
            out["max_rate"] = max(out["max_rate"], float(r[0]))
            out["max_speed"] = max(out["max_speed"], float(r[1]))
            out["max_depth"] = max(out["max_depth"], float(r[2]))
            if math.isnan(r[3]):
                nan = True
            else:
                out["max_dev"] = max(out["max_dev"], float(r[3]))
            out["clamped"] += float(r[4])
            for i, key, k in [(5 + j, "stage_bad", j) for j in range(5)] + \
                    [(10 + j, "state_bad", j) for j in range(3)]:
                g = int(r[i])
                if g >= 0:
                    cur = out[key][k]
                    out[key][k] = g if cur < 0 else min(cur, g)
        if nan:
            out["max_dev"] = math.nan
        return out

    def gather_state(self, locals_: dict, shape, ranges):
        (w, p, q), = locals_.values()
        dev = self._dev()
        outs = []
        for a in (w, p, q):
            t = torch.from_numpy(np.ascontiguousarray(a)).to(dev)
            n_max = max(n for _, n in ranges) + 2 * GHOST
            buf = torch.zeros((n_max, a.shape[1]), dtype=t.dtype, device=dev)
            buf[:t.shape[0]] = t
            bufs = [torch.empty_like(buf) for _ in range(self.world)]
            self.dist.all_gather(bufs, buf, group=self.group)
            outs.append([b.cpu().numpy() for b in bufs])
        per = {r: tuple(outs[k][r][:ranges[r][1] + 2 * GHOST] for k in range(3))
               for r in range(self.world)}
        return _assemble(per, shape, ranges)

    def gather_values(self, per: dict, n: int):
        (vals, owned), = per.values()
        dev = self._dev()
        v = torch.from_numpy(np.ascontiguousarray(vals, dtype=np.float64)).to(dev)
        m = torch.from_numpy(np.ascontiguousarray(owned, dtype=np.int64)).to(dev)
        vs = [torch.empty_like(v) for _ in range(self.world)]
        ms = [torch.empty_like(m) for _ in range(self.world)]
        self.dist.all_gather(vs, v, group=self.group)
        self.dist.all_gather(ms, m, group=self.group)
        return _pick_owned([(a.cpu().numpy(), b.cpu().numpy().astype(bool)) for a, b in zip(vs, ms)],
                           n)

    def gather_rows(self, per: dict, nx: int, ranges):
        (mine,), dev = per.values(), self._dev()
        n_max = max(n for _, n in ranges)
        buf = torch.zeros((n_max, nx), dtype=torch.float64, device=dev)
        buf[:mine.shape[0]] = torch.from_numpy(np.ascontiguousarray(mine)).to(dev)
        bufs = [torch.empty_like(buf) for _ in range(self.world)]
        self.dist.all_gather(bufs, buf, group=self.group)
        return np.concatenate([b.cpu().numpy()[:ranges[r][1]] for r, b in enumerate(bufs)], axis=0)

    def gather_spike_table(self, per: dict, nx: int) -> np.ndarray:
        (mine,) = per.values()
        t = torch.from_numpy(np.ascontiguousarray(mine)).to(self._dev())
        bufs = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(bufs, t, group=self.group)
        return np.stack([b.cpu().numpy() for b in bufs])

    def max_rate(self, strips, stream) -> None:
        """All-reduce (max) of this rank's device max CFL rate, in place on
        the library stream (NCCL reads device memory; gloo stages through the
        host)."""
        v = strips[self.rank].result_rate()
        with torch.cuda.stream(stream):
            wire = self._wire(v)
            self.dist.all_reduce(wire, op=self.dist.ReduceOp.MAX, group=self.group)
            if wire is not v:
                v.copy_(wire)

    def spike_bounds(self, strips, arr: int, stream) -> dict:
        s = strips[self.rank]
        with torch.cuda.stream(stream):
            R, n = s.rows(arr), s.ny
            mine = torch.stack([R[GHOST, GHOST:-GHOST], R[GHOST + n - 1, GHOST:-GHOST]]).contiguous()
            wire = self._wire(mine)
            bufs = [torch.empty_like(wire) for _ in range(self.world)]
            self.dist.all_gather(bufs, wire, group=self.group)
            yb = torch.stack(bufs).to(mine.device).contiguous()
        return {self.rank: yb}


def _pick_owned(parts, n: int):
    out = None
    for vals, owned in parts:
        if out is None:
            out = np.zeros((n,) + vals.shape[1:])
        out[owned] = vals[owned]
    return out


def _combine(parts: list, nx: int, rows0: list) -> dict:
    """Cross-strip reduction of per-strip step results, in rank order."""
    out = {"max_rate": 0.0, "max_speed": 0.0, "max_depth": 0.0, "max_dev": 0.0, "clamped": 0.0,
           "stage_bad": [-1] * 5, "state_bad": [-1] * 3}
    nan = False
    for res, row0 in zip(parts, rows0):
        out["max_rate"] = max(out["max_rate"], res.max_rate)
        out["max_speed"] = max(out["max_speed"], res.max_speed)
        out["max_depth"] = max(out["max_depth"], res.max_depth)
        if math.isnan(res.max_dev):
            nan = True
        else:
            out["max_dev"] = max(out["max_dev"], res.max_dev)
        out["clamped"] += res.clamped
        for key, src in (("stage_bad", res.stage_bad), ("state_bad", res.state_bad)):
            for k, b in enumerate(src):
                if b >= 0:
                    g = b + row0 * nx  # global row-major interior index
                    cur = out[key][k]
                    out[key][k] = g if cur < 0 else min(cur, g)
    if nan:
        out["max_dev"] = math.nan
    return out


def _assemble(per: dict, shape, ranges):
    """Global padded arrays from per-strip padded arrays (interior rows of
    every strip, ghost rows of the edge strips)."""
    full = [np.empty(shape) for _ in range(3)]
    last = len(ranges) - 1
    for r, (row0, n) in enumerate(ranges):
        lo = 0 if r == 0 else GHOST
        hi = n + 2 * GHOST if r == last else n + GHOST
        for k in range(3):
            full[k][row0 + lo:row0 + hi] = per[r][k][lo:hi]
    return tuple(full)


# ---------------------------------------------------------------------------


class ShardedDevice:
    """Drop-in for DeviceStep over y-strips (the Simulator drives it)."""

    def __init__(self, sim: "ShardedSimulator", desc, bathy, device, world: int, comm,
                 coupling: str = "pipeline", local_inputs: bool = False):
        if coupling not in ("pipeline", "spike"):
            raise ValueError(f"coupling must be 'pipeline' or 'spike', got {coupling!r}")
        self.sim, self.comm, self.world = sim, comm, world
        # local_inputs: bathy / state arrays are this process's strip only
        self.local_inputs = local_inputs
        self.spike = coupling == "spike" and world > 1
        self.nx, self.ny = desc.nx, desc.ny
        self.shape = (desc.ny + 2 * GHOST, desc.nx + 2 * GHOST)
        self.ranges = split_rows(desc.ny, world)
        dev = torch.device(device if device is not None else "cuda")
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        self.stream = torch.cuda.Stream(dev)
        self.strips: dict[int, DeviceStep] = {}
        self._bands = []  # per rank: [(lo, len, off)] for N, S
        tails: dict = {}
        sing = []
        for r, (row0, n) in enumerate(self.ranges):
            bands = []
            for s in (_N, _S):
                bands.append(strip_band(desc.sponge_lo[s], desc.sponge_len[s], row0, n)
                             if desc.sponge_len[s] else (0, 0, 0))
            self._bands.append(bands)
            if not comm.is_local(r):
                continue
            d = nat.Desc.from_buffer_copy(desc)
            d.ny, d.row0, d.ny_global = n, row0, desc.ny
            d.south_internal = 1 if r > 0 else 0
            d.north_internal = 1 if r < world - 1 else 0
            d.y_coupling = nat.Y_SPIKE if self.spike else nat.Y_PIPELINE
            for s, (lo, ln, _) in zip((_N, _S), bands):
                d.sponge_lo[s], d.sponge_len[s] = lo, ln
            # the pipelined recurrence continues the south strip's factorization;
            # spike blocks are factored alone
            cws = comm.get_tail(tails, r, desc.nx) if r > 0 and not self.spike else None
            strip = DeviceStep(d, _StripStatic(bathy, 0 if local_inputs else row0, n), device=dev,
                               stream=self.stream,
                               cw_south=cws)
            self.strips[r] = strip
            if not self.spike:
                comm.pass_tail(tails, r, strip.factor_tail())
            sing.append(strip.pivot_flags()[1])
        self.singular = comm.any_flag(sing)
        self.cross = bool(desc.cross_correction)
        if self.spike:
            table = comm.gather_spike_table({r: s.spike_coeffs() for r, s in self.strips.items()},
                                            desc.nx)
            for r, s in self.strips.items():
                s.set_spike_table(table, r)
        first = self.strips[min(self.strips)]
        self.workspace = first.workspace
        self._res = nat.StepResult()

    # -- state -----------------------------------------------------------------------
    def _rows(self, r):
        row0, n = self.ranges[r]
        return slice(0 if self.local_inputs else row0, (0 if self.local_inputs else row0) + n + 2 * GHOST)

    def upload(self, w, p, q):
        for r, s in self.strips.items():
            rows = self._rows(r)
            s.upload(w[rows], p[rows], q[rows])

    def download(self, pending: bool = False, out=None):
        if self.local_inputs:  # this process's strip, in the strip's own shape
            (s,) = self.strips.values()
            full = s.download(pending=pending)
            if out is not None:
                for dst, src in zip(out, full):
                    dst[...] = src
                return out
            return full
        per = {r: s.download(pending=pending) for r, s in self.strips.items()}
        full = self.comm.gather_state(per, self.shape, self.ranges)
        if out is not None:
            for dst, src in zip(out, full):
                dst[...] = src
            return out
        return full

    def download_local(self, out):
        """Copy only this process's strips into the matching rows of the
        global arrays ``out`` (w, p, q): the distributed-I/O path."""
        for r, s in self.strips.items():
            rows = self._rows(r)
            w, p, q = s.download()
            out[0][rows], out[1][rows], out[2][rows] = w, p, q
        return out

    # -- observers: each strip samples the gauges in its rows -------------------
    def set_gauges(self, cells):
        self._gauges = [(int(j), int(i)) for j, i in cells]
        self._gslots = {}
        for r, s in self.strips.items():
            row0, n = self.ranges[r]
            mine = [k for k, (j, _) in enumerate(self._gauges) if row0 <= j - GHOST < row0 + n]
            s.set_gauges([(self._gauges[k][0] - row0, self._gauges[k][1]) for k in mine])
            self._gslots[r] = mine

    def gauge_values(self) -> np.ndarray:
        n = len(getattr(self, "_gauges", []))
        per = {}
        for r, s in self.strips.items():
            vals, owned = np.zeros((n, 3)), np.zeros(n, dtype=bool)
            mine = self._gslots[r]
            if mine:
                vals[mine] = s.gauge_values()
                owned[mine] = True
            per[r] = (vals, owned)
        return self.comm.gather_values(per, n)

    def max_tracker(self, op: int):
        for s in self.strips.values():
            s.max_tracker(op)

    def download_max(self) -> np.ndarray:
        per = {r: s.download_max() for r, s in self.strips.items()}
        return self.comm.gather_rows(per, self.nx, self.ranges)

    def history(self, level: int, field: int) -> np.ndarray:
        out = np.empty((self.ny, self.nx))
        for r, s in self.strips.items():
            row0, n = self.ranges[r]
            out[row0:row0 + n] = s.history(level, field)
        return out

    def speed_extrema(self):
        vals = [s.speed_extrema() for s in self.strips.values()]
        res = [nat.StepResult() for _ in vals]
        for rs, v in zip(res, vals):
            rs.max_rate, rs.max_speed, rs.max_depth = v
            rs.max_dev = 0.0
            for k in range(5):
                rs.stage_bad[k] = -1
            for k in range(3):
                rs.state_bad[k] = -1
        m = self.comm.reduce(res, self.nx, [self.ranges[r][0] for r in self.strips])
        return m["max_rate"], m["max_speed"], m["max_depth"]

    # -- the sharded step ----------------------------------------------------------------
    def _strip_params(self, params, r):
        """params with this strip's part of the N/S sponge factors."""
        p = nat.StepParams.from_buffer_copy(params)
        for s, (lo, ln, off) in zip((_N, _S), self._bands[r]):
            fac = self.sim._fac_keep[s]
            p.sponge_fac[s] = nat.ptr(fac[off:]) if (ln and fac is not None) else None
        return p

    def step(self, params):
        order = sorted(self.strips)
        strips = self.strips
        sp = {r: self._strip_params(params, r) for r in order}
        for r in order:
            strips[r].phase(nat.PH_GHOST, sp[r])

        def each(ph):
            return lambda: [strips[r].phase(ph) for r in order]
        # the stage's and the correction's interior rows run while the halo
        # rows they do not read are in flight
        self.comm.halo(strips, _STATE, 2, self.stream, inner=each(nat.PH_STAGE_INNER))
        each(nat.PH_STAGE_EDGE)()
        self._ysolve(1)
        self.comm.halo(strips, _PENDING_PQ, 1, self.stream, inner=each(nat.PH_CORRECT_INNER))
        each(nat.PH_CORRECT_EDGE)()
        self._ysolve(2)
        if params.spec:
            # speculation: k_final alone, the max CFL rate reduced over the
            # ranks on the device, then PH_FINAL's device controller queues the
            # next step's ghosts and inner stage rows behind the result copy
            for r in order:
                strips[r].phase(nat.PH_FINAL_LAUNCH)
            self.comm.max_rate(strips, self.stream)
        parts = []
        for r in order:
            _, res = strips[r].phase(nat.PH_FINAL)
            parts.append(nat.StepResult.from_buffer_copy(res))
        m = self.comm.reduce(parts, self.nx, [self.ranges[r][0] for r in order])
        out = self._res
        out.max_rate, out.max_speed, out.max_depth = m["max_rate"], m["max_speed"], m["max_depth"]
        out.max_dev, out.clamped = m["max_dev"], m["clamped"]
        for k in range(5):
            out.stage_bad[k] = m["stage_bad"][k]
        for k in range(3):
            out.state_bad[k] = m["state_bad"][k]
        rc = nat.BSQ_ERR_SINGULAR if self.singular else nat.BSQ_OK
        return rc, out

    def _ysolve(self, solve: int):
        """The line solves of one phase: x rows are local; y columns continue
        across strips (rank pipeline) or are coupled afterwards (spike)."""
        ph_f, ph_b = (nat.PH_SOLVE1F, nat.PH_SOLVE1B) if solve == 1 else \
            (nat.PH_SOLVE2F, nat.PH_SOLVE2B)
        if not self.spike:
            self.comm.pipeline(self.strips, ph_f, ph_b, self.stream)
            return
        for r in sorted(self.strips):
            self.strips[r].phase(ph_f)
        if solve == 2 and not self.cross:
            return
        yb = self.comm.spike_bounds(self.strips, nat.ARR_Q_NEW, self.stream)
        for r, s in self.strips.items():
            s.spike_fix(solve, yb[r])

    def commit(self):
        for s in self.strips.values():
            s.commit()

    def close(self):
        for s in self.strips.values():
            s.close()

    # timing / introspection: the first local strip stands for the rank
    def set_timing(self, on: bool):
        for s in self.strips.values():
            s.set_timing(on)

    def kernel_times(self):
        return self.strips[min(self.strips)].kernel_times()

    def kernels_per_step(self) -> int:
        return sum(s.kernels_per_step() + 2 for s in self.strips.values())

    def stage_rates(self):
        raise NotImplementedError("kernel-level seams are single-grid only")

    solve_momentum = fill_ghosts = stage_rates


class ShardedSimulator(Simulator):
    """Simulator whose grid is split into y-strips, one per rank.

    ``world`` strips emulated in this process when ``comm`` is None (one GPU,
    bitwise-checkable against the single-GPU run), or ``comm=DistComm()``
    under torchrun with one strip per process.  Inputs are the global
    objects; every API is the Simulator's.

    ``global_grid`` (DistComm only): the inputs are this rank's strip instead
    -- ``bathy``/``state`` hold padded rows [row0, row0 + ny_r + 4) of the
    global arrays (scenario.make_strip_case; bathy.grid is the strip's grid)
    and ``global_grid`` is the whole grid, so no rank ever holds global
    arrays.  ``state`` and the downloads are then this rank's strip; the
    blow-up bound uses the global initial amplitude (one all-reduce).
    """

    def __init__(self, *args, world: int | None = None, comm=None, coupling: str = "pipeline",
                 global_grid=None, **kw):
        if comm is None:
            comm = LocalComm(world or 1)
        if global_grid is not None and len(comm.local) != 1:
            raise ValueError("strip-local inputs need one strip per process (DistComm)")
        self._comm = comm
        self._world = comm.world
        self._coupling = coupling
        self._global_grid = global_grid
        super().__init__(*args, **kw)

    def _make_device(self, desc, bathy, device):
        if self.solver != "thomas":
            raise NotImplementedError("sharded solves use the Thomas pipeline")
        return ShardedDevice(self, desc, bathy, device, self._world, self._comm, self._coupling,
                             local_inputs=self._global_grid is not None)

    def _validate_inputs(self, state, bathy, boundaries):
        if self._global_grid is None:
            return super()._validate_inputs(state, bathy, boundaries)
        row0, n = split_rows(self._global_grid.ny, self._world)[self._comm.rank]
        g = bathy.grid
        if (g.nx, g.ny) != (self._global_grid.nx, n):
            raise ValueError(f"strip grid {g.nx}x{g.ny} is not rank {self._comm.rank}'s "
                             f"{self._global_grid.nx}x{n} rows of the global grid")
        # a side facing another strip has no boundary policy to validate
        sides = {s: getattr(boundaries, s) for s in bc.SIDES}
        if row0 > 0:
            sides["south"] = bc.Wall()
        if row0 + n < self._global_grid.ny:
            sides["north"] = bc.Wall()
        super()._validate_inputs(state, bathy, bc.Boundaries(**sides))

    def _desc_grid(self, grid):
        return self._global_grid if self._global_grid is not None else grid

    def _global_max(self, x: float) -> float:
        return self._comm.max_scalar(x) if self._global_grid is not None else x

    @property
    def stream(self):
        return self._dev.stream
