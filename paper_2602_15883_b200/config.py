"""Problem construction for the benchmark configurations.

`decomposition_for_procs` is the reference's canonical strong-scaling table
(pkg/src/flowrec/config.py:331-349).  `cylinder2d_problem` / `cylinder3d_problem`
assemble the synthetic cylinder-wake-shaped problems of BASELINE.md section 3 /
SURVEY section 8(d): the reference's Taylor-Green / Beltrami stand-ins on the
paper's boxes, snapshot observation plans, budgets, anchor and weights.
"""

from dataclasses import dataclass

from . import benchmarks
from .decomposition import (Budget, GlobalDomain, ReferenceTable, build_all_rank_datasets,
                            partition, snapshot_observations)
from .network import ExpertConfig
from .physics import LossWeights


class ConfigError(ValueError):
    pass


def decomposition_for_procs(regime, n_procs):
    """Spatial splits first, then a temporal bisection (2D) / third axis (3D)."""
    table_2d = {1: ((1, 1), 1), 2: ((2, 1), 1), 4: ((2, 2), 1), 8: ((2, 2), 2)}
    table_3d = {1: ((1, 1, 1), 1), 2: ((2, 1, 1), 1), 4: ((2, 2, 1), 1), 8: ((2, 2, 2), 1)}
    table = table_3d if regime.n_space == 3 else table_2d
    if n_procs not in table:
        raise ConfigError(f"no canonical decomposition for P={n_procs} (choose from {sorted(table)})")
    counts, m = table[n_procs]
    if m > 1 and not regime.has_time:
        raise ConfigError(f"P={n_procs} needs a temporal split; {regime.kind} is steady")
    return counts, m


@dataclass
class Problem:
    """Everything `build_plan` needs, plus the reference table for evaluation."""

    solution: object
    domain: GlobalDomain
    subdomains: list
    datasets: dict
    expert_config: ExpertConfig
    weights: LossWeights
    anchor: tuple
    budget: Budget
    table: ReferenceTable


def cylinder2d_problem(n_procs=1, n_pde=500_000, n_ghost=1000, per_snapshot=200, grid_nx=33,
                       snapshots=50, hidden_layers=4, width=64, activation="tanh", seed=0,
                       counts=None, time_splits=None, colloc_on_device=False):
    """2D cylinder-wake-shaped config: Taylor-Green at Re=100
    on [-7.5, 17.5] x [-8, 8], t in [0, 7.35], 50 snapshots, delta 2.0 / 1.0."""
    sol = benchmarks.TaylorGreen2D(re=100.0, spatial_box=((-7.5, 17.5), (-8.0, 8.0)), time_interval=(0.0, 7.35))
    return _assemble(sol, n_procs, n_pde, n_ghost, per_snapshot, grid_nx, snapshots, hidden_layers, width,
                     activation, seed, (2.0, 1.0), LossWeights(10.0, 5.0, 1.0, 1.0, 1.0), counts, time_splits,
                     colloc_on_device)


def cylinder3d_problem(n_procs=8, n_pde=600_000, n_ghost=5000, per_snapshot=1250, grid_nx=17,
                       snapshots=80, hidden_layers=8, width=64, activation="sin", seed=0,
                       counts=None, time_splits=None, colloc_on_device=False):
    """3D wake-shaped config: Beltrami at Re=300 on
    [-5, 20] x [-5, 5] x [0, 10], t in [0, 11.85]; weights (10, 10, 1, 1),
    velocity weights (1, 5, 100)."""
    sol = benchmarks.Beltrami3D(a=1.0, d=1.0, re=300.0, spatial_box=((-5.0, 20.0), (-5.0, 5.0), (0.0, 10.0)),
                                time_interval=(0.0, 11.85))
    w = LossWeights(10.0, 10.0, 1.0, 1.0, 1.0, velocity=(1.0, 5.0, 100.0))
    return _assemble(sol, n_procs, n_pde, n_ghost, per_snapshot, grid_nx, snapshots, hidden_layers, width,
                     activation, seed, (2.0, 2.0), w, counts, time_splits, colloc_on_device)


def _assemble(sol, n_procs, n_pde, n_ghost, per_snapshot, grid_nx, snapshots, hidden_layers, width,
              activation, seed, deltas, weights, counts, time_splits, colloc_on_device=False):
    regime = sol.regime
    domain = GlobalDomain.from_solution(sol)
    if counts is None:
        counts, time_splits = decomposition_for_procs(regime, n_procs)
    pts = benchmarks.grid_points(sol, grid_nx, snapshots)
    vel, p = sol.velocity_pressure(pts)
    table = ReferenceTable(regime=regime, points=pts, velocity=vel, pressure=p)
    obs = snapshot_observations(table, per_snapshot, seed=0)
    budget = Budget(n_obs=obs.n, n_pde=n_pde, n_ghost_per_interface=n_ghost)
    subs = partition(domain, counts, time_splits, delta_space=deltas[0], delta_time=deltas[1])
    datasets = build_all_rank_datasets(subs, budget, obs, seed, colloc_on_device=colloc_on_device)
    cfg = ExpertConfig.for_regime(regime, hidden_layers, width, activation)
    anchor = tuple(lo + 0.25 * (hi - lo) for lo, hi in domain.spatial_box)
    return Problem(sol, domain, subs, datasets, cfg, weights, anchor, budget, table)
