"""The multi-process y-strip path on one GPU: two ranks (processes) share
cuda:0 and exchange over gloo, which makes DistComm stage its device rows
through host memory.  This runs everything the NCCL multi-GPU bench runs --
bench.py's own rank launcher, strip-local inputs, ShardedSimulator with the
real kernels, DistComm halos / pipeline vectors / spike rows / reductions --
except NCCL itself (one GPU cannot host two NCCL ranks).  Functional only:
the two ranks time-share the GPU, so no number here is a scaling figure."""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bench_two_ranks_over_gloo_one_json_line():
    env = dict(os.environ, BSQ_DIST_BACKEND="gloo", OMP_NUM_THREADS="2")
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--steps", "2", "--warmup", "3", "--scale", "32", "--no-cpu",
                          "--no-configs"], cwd=ROOT, env=env, capture_output=True, text=True,
                         timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["config"]["parallelism"] == "y-strip x2"


def _worker(rank, world, port, coupling, steps, path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_1909_04153_b200 import stepper
    from paper_1909_04153_b200.parallel import DistComm, ShardedSimulator
    from paper_1909_04153_b200.scenario import make_strip_case
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = DistComm()
    case = make_strip_case("C4", rank, world, reduce=comm.reduce_scalar, scale=16)
    sim = ShardedSimulator(case.bathy, case.state.copy(), case.boundaries,
                           stepper.TimeController(dt_init=case.dt_init), phys=case.phys,
                           comm=comm, coupling=coupling, global_grid=case.grid)
    recs = [sim.advance() for _ in range(steps)]
    st = sim._dev.comm.gather_state({rank: sim._dev.download()}, sim._dev.shape,
                                    sim._dev.ranges)
    if rank == 0:
        np.savez(path, w=st[0], p=st[1], q=st[2],
                 rec=np.array([(r.dt, r.max_cfl, r.max_speed, r.max_depth) for r in recs]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("coupling", ["pipeline", "spike"])
def test_sharded_two_processes_match_one_grid(coupling, tmp_path):
    from paper_1909_04153_b200 import stepper
    from paper_1909_04153_b200.scenario import make_case
    steps = 12
    path = str(tmp_path / "dist.npz")
    mp.spawn(_worker, args=(2, _port(), coupling, steps, path), nprocs=2, join=True)
    z = np.load(path)
    case = make_case("C4", scale=16)
    sim = stepper.Simulator(case.bathy, case.state.copy(), case.boundaries,
                            stepper.TimeController(dt_init=case.dt_init), phys=case.phys)
    recs = np.array([(r.dt, r.max_cfl, r.max_speed, r.max_depth)
                     for r in (sim.advance() for _ in range(steps))])
    st = sim.state
    if coupling == "pipeline":  # the exact rank pipeline: bitwise one grid
        assert np.array_equal(recs, z["rec"])
        for f in ("w", "p", "q"):
            assert np.array_equal(getattr(st, f).view(np.uint64), z[f].view(np.uint64)), f
    else:  # partitioned column solves: equal up to rounding
        for f in ("w", "p", "q"):
            a, b = getattr(st, f), z[f]
            assert np.linalg.norm(a - b) <= 1e-12 * np.linalg.norm(a), f


def _nccl_worker(rank, port, steps, path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_1909_04153_b200 import stepper
    from paper_1909_04153_b200.parallel import DistComm, ShardedSimulator
    from paper_1909_04153_b200.scenario import make_case
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    comm = DistComm()
    assert not comm.staged  # device tensors go to NCCL directly
    case = make_case("C4", scale=16)
    sim = ShardedSimulator(case.bathy, case.state.copy(), case.boundaries,
                           stepper.TimeController(dt_init=case.dt_init), phys=case.phys, comm=comm)
    recs = [sim.advance() for _ in range(steps)]
    st = sim.state
    np.savez(path, w=st.w, p=st.p, q=st.q,
             rec=np.array([(r.dt, r.max_cfl, r.max_speed, r.max_depth) for r in recs]))
    dist.destroy_process_group()


def test_nccl_single_rank_sharded_step_matches_one_grid(tmp_path):
    """The NCCL transport on the one GPU a box has: a single-rank process
    group drives the sharded step (NCCL all-reduce of the device CFL rate on a
    workspace view, all_gather of the step results) and equals the single-grid
    Simulator bitwise."""
    from paper_1909_04153_b200 import stepper
    from paper_1909_04153_b200.scenario import make_case
    steps = 12
    path = str(tmp_path / "nccl.npz")
    mp.spawn(_nccl_worker, args=(_port(), steps, path), nprocs=1, join=True)
    z = np.load(path)
    case = make_case("C4", scale=16)
    sim = stepper.Simulator(case.bathy, case.state.copy(), case.boundaries,
                            stepper.TimeController(dt_init=case.dt_init), phys=case.phys)
    recs = np.array([(r.dt, r.max_cfl, r.max_speed, r.max_depth)
                     for r in (sim.advance() for _ in range(steps))])
    assert np.array_equal(recs, z["rec"])
    for f in ("w", "p", "q"):
        assert np.array_equal(getattr(sim.state, f).view(np.uint64), z[f].view(np.uint64)), f
