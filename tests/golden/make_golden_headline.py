"""Golden fixtures for the BENCHMARKED network, [3, 64x4, 3] tanh on the
cylinder-wake box, produced by the UNMODIFIED reference (`flowrec`).

    PYTHONPATH=baseline/_ref python tests/golden/make_golden_headline.py

Writes tests/golden/golden_headline.npz:

* ``ep/<rank>/*``: `LocalObjective.epoch` (runtime/objective.py:164-199) on
  two ranks of the P=8 (2,2)x2 decomposition (N_pde 20,000 global, 1,000
  ghost points per interface, 200 observations per snapshot), each with
  spatial AND temporal ghost sets and non-trivial ghost targets: rank 0 is a
  master (`LossWeights.as_master()`, physics.py:190-200), rank 3 a slave.
* ``tr/*``: the reference's serial `train()` (runtime/driver.py:127-144) of
  that (2,2)x2 plan for 3 epochs: per-rank history and final parameters.
* ``full/*``: one UNSAMPLED P=1 epoch of the headline config C (N_pde =
  500,000, N_obs = 10,000; `LocalObjective.epoch`): the loss parts, total and
  the flat gradient only (the datasets are regenerated bit-exactly by the
  engine's input side; a SHA-256 of the reference's collocation array pins that).

Takes about a minute on one core (the full epoch dominates).
"""

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

import flowrec  # noqa: E402
from flowrec import benchmarks  # noqa: E402
from flowrec.config import decomposition_for_procs  # noqa: E402
from flowrec.decomposition import (Budget, GlobalDomain, ReferenceTable, build_all_rank_datasets,  # noqa: E402
                                   partition, snapshot_observations)
from flowrec.network import ExpertConfig, init_params, predict  # noqa: E402
from flowrec.physics import LossWeights  # noqa: E402
from flowrec.runtime import LocalObjective, TrainConfig, build_plan, train  # noqa: E402
from threadpoolctl import threadpool_limits  # noqa: E402

assert flowrec.backend_name() == "cython", flowrec.backend_name()


def headline_problem(counts, m, n_pde):
    """The engine's config.cylinder2d_problem, stated with the reference's API."""
    sol = benchmarks.TaylorGreen2D(re=100.0, spatial_box=((-7.5, 17.5), (-8.0, 8.0)), time_interval=(0.0, 7.35))
    domain = GlobalDomain.from_solution(sol)
    pts = benchmarks.grid_points(sol, 33, 50)
    vel, p = sol.velocity_pressure(pts)
    table = ReferenceTable(regime=sol.regime, points=pts, velocity=vel, pressure=p)
    obs = snapshot_observations(table, 200, seed=0)
    budget = Budget(n_obs=obs.n, n_pde=n_pde, n_ghost_per_interface=1000)
    subs = partition(domain, counts, m, delta_space=2.0, delta_time=1.0)
    ds = build_all_rank_datasets(subs, budget, obs, 0)
    cfg = ExpertConfig.for_regime(sol.regime, 4, 64, "tanh")
    anchor = tuple(lo + 0.25 * (hi - lo) for lo, hi in domain.spatial_box)
    return sol, subs, ds, cfg, LossWeights(10.0, 5.0, 1.0, 1.0, 1.0), anchor


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def main():
    out = {}
    t0 = time.perf_counter()
    with threadpool_limits(limits=1):
        # ---- LocalObjective.epoch on a master and a slave rank of (2,2)x2 ----
        sol, subs, ds, cfg, weights, anchor = headline_problem((2, 2), 2, 20_000)
        tc = TrainConfig(epochs=3, batch_size=25_000, learning_rate=1e-3, weights=weights, anchor=anchor,
                         lr_factor=0.2, lr_interval=2000, comm_interval=1, seed=0)
        plan = build_plan(subs, ds, cfg, tc)
        assert sorted(plan.masters) == [0, 4], plan.masters
        rng = np.random.default_rng(2602)
        for r in (0, 3):
            ws = plan.worker_specs[r]
            d = ws.datasets
            kinds = sorted({g.kind for g in d.ghosts})
            assert kinds == ["spatial", "temporal"], kinds
            # targets of the size and scale of real neighbour predictions
            nb = init_params(cfg, plan.worker_specs[d.ghosts[0].neighbor].param_seed)
            targets = []
            for g in d.ghosts:
                y = predict(nb, g.points)
                targets.append((y[:, :2] + 0.05 * rng.normal(size=(g.points.shape[0], 2)),
                                y[:, 2] + 0.05 * rng.normal(size=g.points.shape[0])))
            params = init_params(cfg, ws.param_seed)
            obj = LocalObjective(cfg, plan.regime, d, ws.effective_weights, batch_size=25_000)
            obj.set_ghost_targets(targets)
            parts, grad, total = obj.epoch(params, np.random.default_rng(0))
            k = f"ep/{r}"
            out[f"{k}/role"] = np.array(ws.role == "master")
            w = ws.effective_weights
            out[f"{k}/weights"] = np.array([w.obs, w.pde, w.ghost_u, w.ghost_p_space, w.ghost_p_time])
            out[f"{k}/params"] = params.flat
            out[f"{k}/colloc_sha"] = np.array(sha(d.colloc_points))
            out[f"{k}/obs_points"], out[f"{k}/obs_velocity"] = d.obs_points, d.obs_velocity
            for gi, (g, (u, p)) in enumerate(zip(d.ghosts, targets)):
                out[f"{k}/ghost{gi}"], out[f"{k}/ghost{gi}_u"], out[f"{k}/ghost{gi}_p"] = g.points, u, p
            out[f"{k}/parts"] = np.array(parts.astuple())
            out[f"{k}/total"] = np.array(total)
            out[f"{k}/grad"] = grad
            print(f"epoch rank {r} ({ws.role}): parts {parts.astuple()} |g| {np.linalg.norm(grad):.4e}")

        # ---- serial train() of the same (2,2)x2 plan, 3 epochs ----
        res = train(plan, backend="serial")
        for r in sorted(res.params):
            out[f"tr/r{r}/final"] = res.params[r].flat
            out[f"tr/r{r}/history"] = res.history[r]
        print(f"train (2,2)x2 done ({time.perf_counter() - t0:.1f} s)")

        # ---- one unsampled P=1 epoch of config C (500,000 collocation points) ----
        counts, m = decomposition_for_procs(sol.regime, 1)
        sol, subs, ds, cfg, weights, anchor = headline_problem(counts, m, 500_000)
        d = ds[0]
        assert d.n_colloc == 500_000 and d.n_obs == 10_000 and not d.ghosts
        tc1 = TrainConfig(epochs=1, batch_size=25_000, learning_rate=1e-3, weights=weights, anchor=anchor, seed=0)
        plan1 = build_plan(subs, ds, cfg, tc1)
        ws = plan1.worker_specs[0]
        params = init_params(cfg, ws.param_seed)
        obj = LocalObjective(cfg, plan1.regime, d, ws.effective_weights, batch_size=25_000)
        t1 = time.perf_counter()
        parts, grad, total = obj.epoch(params, np.random.default_rng(0))
        out["full/seconds"] = np.array(time.perf_counter() - t1)
        out["full/colloc_sha"] = np.array(sha(d.colloc_points))
        out["full/obs_sha"] = np.array(sha(d.obs_points))
        out["full/params"] = params.flat
        out["full/parts"] = np.array(parts.astuple())
        out["full/total"] = np.array(total)
        out["full/grad"] = grad
        w = ws.effective_weights
        out["full/weights"] = np.array([w.obs, w.pde, w.ghost_u, w.ghost_p_space, w.ghost_p_time])
        print(f"full P=1 epoch: parts {parts.astuple()} in {float(out['full/seconds']):.1f} s")

    path = os.path.join(HERE, "golden_headline.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes,", len(out), "arrays")


if __name__ == "__main__":
    sys.exit(main())
