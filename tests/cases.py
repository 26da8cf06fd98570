"""Shared test problems: the small plans pinned in tests/golden/golden.npz."""

import numpy as np

from paper_2602_15883_b200 import config as fconfig
from paper_2602_15883_b200.runtime import TrainConfig, build_plan

CASES = {
    "p1": dict(kind="2d", counts=(1, 1), m=1),
    "p2": dict(kind="2d", counts=(2, 1), m=1),
    "t2": dict(kind="2d", counts=(1, 1), m=2),
    "p8": dict(kind="2d", counts=(2, 2), m=2),
    "d3": dict(kind="3d", counts=(2, 2, 2), m=1),
}


def problem(tag):
    c = CASES[tag]
    if c["kind"] == "2d":
        return fconfig.cylinder2d_problem(n_pde=1600, n_ghost=40, per_snapshot=12, grid_nx=9, snapshots=10,
                                          hidden_layers=2, width=16, activation="tanh",
                                          counts=c["counts"], time_splits=c["m"])
    return fconfig.cylinder3d_problem(n_pde=1600, n_ghost=40, per_snapshot=10, grid_nx=5, snapshots=6,
                                      hidden_layers=2, width=16, activation="sin",
                                      counts=c["counts"], time_splits=c["m"])


def train_config(tag, golden):
    epochs, lr, factor, interval, clip, _ = golden[f"{tag}/meta"]
    pb = problem(tag)
    return pb, TrainConfig(epochs=int(epochs), batch_size=500, learning_rate=float(lr), weights=pb.weights,
                           anchor=pb.anchor, lr_factor=float(factor), lr_interval=int(interval), comm_interval=1,
                           clip_norm=None if clip < 0 else float(clip), seed=0)


def training_plan(tag, golden):
    pb, tc = train_config(tag, golden)
    return pb, build_plan(pb.subdomains, pb.datasets, pb.expert_config, tc)


def oracle_ranks(plan):
    """Oracle input for train_serial built from a TrainingPlan."""
    ranks = {}
    for ws in plan.worker_specs:
        d = ws.datasets
        w = ws.effective_weights
        from paper_2602_15883_b200.network import init_params

        ranks[ws.rank] = dict(
            flat=init_params(ws.expert_config, ws.param_seed).flat.copy(),
            data=dict(obs_pts=d.obs_points, obs_vel=d.obs_velocity, colloc=d.colloc_points,
                      ghosts=[(g.kind, g.points, None, None) for g in d.ghosts]),
            weights=dict(obs=w.obs, pde=w.pde, ghost_u=w.ghost_u, ghost_p_space=w.ghost_p_space,
                         ghost_p_time=w.ghost_p_time, velocity=w.velocity),
            outgoing=[(e.dest, e.ghost_index, e.points) for e in ws.outgoing],
            normalize=ws.normalize_outgoing,
        )
    return ranks
