"""Rebuild a golden run's inputs (tests/golden/run_*.npz) as product-side
objects, without the reference package."""

from __future__ import annotations

import os

import numpy as np

from paper_1909_04153_b200 import boundary as bc
from paper_1909_04153_b200.grid import Bathymetry, FieldState, Grid, PhysParams

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SIDES = ("north", "south", "east", "west")
RUNS = ["c1", "hump", "hump_cr", "maker_sponge", "rip_irregular", "runup", "dry_clamp",
        "blowup", "fixed_single_pass", "lake", "island"]


def load(name):
    return np.load(os.path.join(GOLDEN, f"run_{name}.npz"), allow_pickle=False)


def inputs(z):
    """(bathy, state, boundaries, phys, controller kwargs, sim kwargs)."""
    grid = Grid(int(z["nx"]), int(z["ny"]), float(z["dx"]), float(z["dy"]),
                float(z["x0"]), float(z["y0"]))
    bathy = Bathymetry(grid=grid, ws=float(z["ws"]), bed=np.pad(z["bed"], 2, mode="symmetric"),
                       bed_eff=z["bed_eff"].copy(), depth=z["depth"].copy(),
                       depth_dx=z["depth_dx"].copy(), depth_dy=z["depth_dy"].copy(),
                       bed_face_x=z["bed_face_x"].copy(), bed_face_y=z["bed_face_y"].copy(),
                       h_eps=float(z["h_eps"]))
    state = FieldState(z["w0"].copy(), z["p0"].copy(), z["q0"].copy())
    comps = {k: [] for k in range(4)}
    for row in z["maker_comps"]:
        comps[int(row[0])].append(bc.WaveComponent(row[1], row[2], row[3], row[4]))
    sponges = {int(r[0]): (float(r[1]), float(r[2])) for r in z["sponges"]}
    pols = {}
    for k, side in enumerate(SIDES):
        kind = str(z["side_kinds"][k])
        if kind == "wall":
            pols[side] = bc.Wall()
        elif kind == "sine":
            pols[side] = bc.SineMaker(tuple(comps[k]))
        elif kind == "irregular":
            pols[side] = bc.IrregularMaker(tuple(comps[k]))
        else:
            pols[side] = bc.Sponge(*sponges[k])
    bounds = bc.Boundaries(**pols)
    phys = PhysParams(g=float(z["g"]), b_disp=float(z["b_disp"]), c_f=float(z["c_f"]))
    ckw = dict(dt_init=float(z["dt_init"]), mode=str(z["mode"]))
    h_dry = float(z["h_dry"])
    skw = dict(solver=str(z["solver"]), cross_correction=bool(z["cross_correction"]),
               h_dry=None if np.isnan(h_dry) else h_dry)
    return bathy, state, bounds, phys, ckw, skw
