"""Host logic of the multi-GPU path on CPU: DistComm (torch.distributed,
gloo, world_size 2) must move halos, pipeline the y-line boundary values and
reduce step results exactly like the in-process LocalComm the GPU tests
validate bitwise.  Strips are CPU stand-ins whose 'kernels' are simple
exact recurrences, so any mis-ordered or mis-routed transfer changes bits."""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1909_04153_b200 import _native as nat
from paper_1909_04153_b200.parallel import (DistComm, LocalComm, _assemble, _combine,
                                             split_rows)

NX, NY, WORLD = 6, 12, 2


class FakeStrip:
    """CPU strip: padded fields, boundary vectors, and phases that consume
    the halo / boundary values like the device kernels do."""

    def __init__(self, rank, row0, ny):
        self.rank, self.row0, self.ny, self.nx = rank, row0, ny, NX
        g = torch.Generator().manual_seed(1234 + rank)
        self.f = {a: torch.rand((ny + 4, NX + 4), generator=g, dtype=torch.float64)
                  for a in (nat.ARR_W, nat.ARR_P, nat.ARR_Q, nat.ARR_P_NEW, nat.ARR_Q_NEW)}
        self.v = {a: torch.zeros(NX, dtype=torch.float64)
                  for a in (nat.ARR_DW_IN, nat.ARR_DW_OUT, nat.ARR_X_IN, nat.ARR_X_OUT)}
        self.col = torch.zeros(NX, dtype=torch.float64)
        self.rate = torch.tensor([0.75 + 0.5 * rank], dtype=torch.float64)

    def result_rate(self):
        return self.rate

    def rows(self, a):
        return self.f[a]

    def vector(self, a):
        return self.v[a]

    def phase(self, ph, params=None):
        w = self.f[nat.ARR_W]
        if ph == nat.PH_SOLVE1F:  # running column recurrence over this strip's rows
            acc = self.v[nat.ARR_DW_IN].clone() if self.rank > 0 else torch.zeros(NX, dtype=torch.float64)
            for j in range(2, self.ny + 2):
                acc = (acc * 0.5 + w[j, 2:-2]) / 1.25
            self.v[nat.ARR_DW_OUT].copy_(acc)
            self.col = acc
        elif ph == nat.PH_SOLVE1B:
            x = self.v[nat.ARR_X_IN].clone() if self.rank < WORLD - 1 else self.col.clone()
            for j in range(self.ny + 1, 1, -1):
                x = w[j, 2:-2] - 0.3 * x
            self.v[nat.ARR_X_OUT].copy_(x)
            self.col = x
        return 0, None


def run_local():
    ranges = split_rows(NY, WORLD)
    strips = {r: FakeStrip(r, *ranges[r]) for r in range(WORLD)}
    comm = LocalComm(WORLD)
    comm.halo(strips, (nat.ARR_W, nat.ARR_P, nat.ARR_Q), 2, None)
    comm.halo(strips, (nat.ARR_P_NEW, nat.ARR_Q_NEW), 1, None)
    comm.pipeline(strips, nat.PH_SOLVE1F, nat.PH_SOLVE1B, None)
    return {r: ({a: t.clone() for a, t in s.f.items()}, s.col.clone()) for r, s in strips.items()}


def _spike_coef(rank):
    return np.arange(4 * NX, dtype=np.float64).reshape(4, NX) * (rank + 1) + 0.125


def _worker(rank, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        ranges = split_rows(NY, WORLD)
        strips = {rank: FakeStrip(rank, *ranges[rank])}
        comm = DistComm()
        # inner(): the interior work queued while the halo is in flight; it
        # must see the halo rows before the exchange (snapshot of one ghost row)
        seen = []
        s0 = strips[rank]

        def inner():
            seen.append(s0.f[nat.ARR_W][1].clone())
        comm.halo(strips, (nat.ARR_W, nat.ARR_P, nat.ARR_Q), 2, None, inner=inner)
        comm.halo(strips, (nat.ARR_P_NEW, nat.ARR_Q_NEW), 1, None)
        comm.pipeline(strips, nat.PH_SOLVE1F, nat.PH_SOLVE1B, None)
        # reductions of per-strip step results
        res = nat.StepResult()
        res.max_rate, res.max_speed, res.max_depth = 1.0 + rank, 2.0 - rank, 0.5 * rank
        res.max_dev = math.nan if rank == 1 else 0.25
        res.clamped = 0.1 * (rank + 1)
        for k in range(5):
            res.stage_bad[k] = -1
        for k in range(3):
            res.state_bad[k] = -1
        res.stage_bad[2] = 3 if rank == 1 else -1
        res.state_bad[0] = 7 if rank == 0 else 1
        red = comm.reduce([res], NX, [ranges[rank][0]])
        # state gather
        s = strips[rank]
        per = {rank: tuple(s.f[a].numpy() for a in (nat.ARR_W, nat.ARR_P, nat.ARR_Q))}
        full = comm.gather_state(per, (NY + 4, NX + 4), ranges)
        tails = {}
        if rank == 0:
            comm.pass_tail(tails, 0, np.arange(NX, dtype=np.float64) * 0.5)
            got_tail = None
        else:
            got_tail = comm.get_tail(tails, 1, NX)
        any_flag = comm.any_flag([rank == 1])
        # spike coupling: static table once, first/last solved rows per solve
        table = comm.gather_spike_table({rank: _spike_coef(rank)}, NX)
        yb = comm.spike_bounds(strips, nat.ARR_Q_NEW, None)[rank].numpy().copy()
        # speculation on strips: the step's max CFL rate reduced in place
        comm.max_rate(strips, None)
        out_q.put((rank, {a: t.numpy().copy() for a, t in s.f.items()}, s.col.numpy().copy(),
                   red, [a.copy() for a in full], got_tail, any_flag, table, yb,
                   [t.numpy() for t in seen], float(s.rate[0])))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def dist_results():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(WORLD):
        item = q.get(timeout=120)
        got[item[0]] = item[1:]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return got


def test_distcomm_halo_and_pipeline_match_localcomm(dist_results):
    ref = run_local()
    for r in range(WORLD):
        fields, col = dist_results[r][0], dist_results[r][1]
        for a, t in ref[r][0].items():
            assert np.array_equal(fields[a], t.numpy()), (r, a)
        assert np.array_equal(col, ref[r][1].numpy()), r


def test_distcomm_reductions(dist_results):
    ranges = split_rows(NY, WORLD)
    for r in range(WORLD):
        red = dist_results[r][2]
        assert red["max_rate"] == 2.0 and red["max_speed"] == 2.0 and red["max_depth"] == 0.5
        assert math.isnan(red["max_dev"])
        assert red["clamped"] == 0.1 + 0.2  # rank order
        # global row-major indices: local index + row0 * nx
        assert red["stage_bad"] == [-1, -1, 3 + ranges[1][0] * NX, -1, -1]
        assert red["state_bad"] == [7, -1, -1]


def test_distcomm_gather_setup_tails_flags(dist_results):
    ranges = split_rows(NY, WORLD)
    per = {}
    for r in range(WORLD):
        f = dist_results[r][0]
        per[r] = tuple(f[a] for a in (nat.ARR_W, nat.ARR_P, nat.ARR_Q))
    want = _assemble(per, (NY + 4, NX + 4), ranges)
    for r in range(WORLD):
        for a, b in zip(dist_results[r][3], want):
            assert np.array_equal(a, b)
    assert np.array_equal(dist_results[1][4], np.arange(NX) * 0.5)
    assert dist_results[0][5] and dist_results[1][5]


def test_distcomm_spike_exchange_matches_localcomm(dist_results):
    ranges = split_rows(NY, WORLD)
    strips = {r: FakeStrip(r, *ranges[r]) for r in range(WORLD)}
    comm = LocalComm(WORLD)
    comm.halo(strips, (nat.ARR_W, nat.ARR_P, nat.ARR_Q), 2, None)
    comm.halo(strips, (nat.ARR_P_NEW, nat.ARR_Q_NEW), 1, None)
    comm.pipeline(strips, nat.PH_SOLVE1F, nat.PH_SOLVE1B, None)
    want_tab = comm.gather_spike_table({r: _spike_coef(r) for r in range(WORLD)}, NX)
    want_yb = comm.spike_bounds(strips, nat.ARR_Q_NEW, None)[0].numpy()
    assert want_yb.shape == (WORLD, 2, NX)
    for r in range(WORLD):
        table, yb = dist_results[r][6], dist_results[r][7]
        assert np.array_equal(table, want_tab)
        assert np.array_equal(yb, want_yb)


def test_distcomm_halo_runs_inner_work_before_the_rows_land(dist_results):
    """halo(..., inner=f) calls f once, after posting the transfers and
    before the received rows are written (rank 1's south ghost row 1 still
    holds its initial value inside f, and the neighbour's row afterwards)."""
    ranges = split_rows(NY, WORLD)
    init = FakeStrip(1, *ranges[1]).f[nat.ARR_W][1].numpy()
    seen = dist_results[1][8]
    assert len(seen) == 1 and np.array_equal(seen[0], init)
    assert not np.array_equal(dist_results[1][0][nat.ARR_W][1], init)
    assert len(dist_results[0][8]) == 1


def test_combine_matches_reference_semantics():
    a, b = nat.StepResult(), nat.StepResult()
    for res, v in ((a, 1.0), (b, 3.0)):
        res.max_rate = res.max_speed = res.max_depth = v
        res.max_dev = v
        res.clamped = v
        for k in range(5):
            res.stage_bad[k] = -1
        for k in range(3):
            res.state_bad[k] = -1
    b.stage_bad[0] = 0
    a.stage_bad[0] = 11
    m = _combine([a, b], 4, [0, 3])
    assert m["max_rate"] == 3.0 and m["clamped"] == 4.0
    assert m["stage_bad"][0] == 11  # min(11, 0 + 3*4 = 12)


def test_max_rate_reduced_in_place_on_every_strip(dist_results):
    """The device controller of each strip sees the global max rate (the value
    the host fold of the step results computes)."""
    want = 0.75 + 0.5 * (WORLD - 1)
    for r in range(WORLD):
        assert dist_results[r][9] == want
    ranges = split_rows(NY, WORLD)
    strips = {r: FakeStrip(r, *ranges[r]) for r in range(WORLD)}
    LocalComm(WORLD).max_rate(strips, None)
    assert all(float(s.rate[0]) == want for s in strips.values())
