"""Generate golden fixtures by running the UNMODIFIED reference (`flowrec`).

Run in the build container (the reference is not present on GPU boxes):

    PYTHONPATH=baseline/_ref python tests/golden/make_golden.py

`baseline/_ref` is the reference installed with
`pip install --no-index --no-build-isolation --no-deps --target baseline/_ref <copy of /root/reference/pkg>`
(Cython kernels built).  Every array below comes from the reference's own API:
partition / datasets / masters / routes (decomposition.py, driver.build_plan),
init_params (network.py), tapes (autodiff), LocalObjective.epoch, adam_step,
and the serial training driver.  Fixtures are small so they can be committed.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

import flowrec  # noqa: E402
from flowrec import autodiff as ad  # noqa: E402
from flowrec import benchmarks  # noqa: E402
from flowrec.decomposition import (Budget, GhostSet, GlobalDomain, RankDatasets,  # noqa: E402
                                   ReferenceTable, build_all_rank_datasets, partition,
                                   snapshot_observations)
from flowrec.network import ExpertConfig, init_params  # noqa: E402
from flowrec.physics import FlowRegime, LossWeights, residual_structure  # noqa: E402
from flowrec.runtime import AdamState, LocalObjective, TrainConfig, adam_step, build_plan, train  # noqa: E402

assert flowrec.backend_name() == "cython", flowrec.backend_name()


def problem_2d(counts, m, n_pde, n_ghost, per_snapshot, nx=9, snaps=10, width=16, layers=2, act="tanh", seed=0):
    sol = benchmarks.TaylorGreen2D(re=100.0, spatial_box=((-7.5, 17.5), (-8.0, 8.0)), time_interval=(0.0, 7.35))
    return _problem(sol, counts, m, n_pde, n_ghost, per_snapshot, nx, snaps, width, layers, act, seed, (2.0, 1.0),
                    LossWeights(10.0, 5.0, 1.0, 1.0, 1.0))


def problem_3d(counts, m, n_pde, n_ghost, per_snapshot, nx=5, snaps=6, width=16, layers=2, act="sin", seed=0):
    sol = benchmarks.Beltrami3D(a=1.0, d=1.0, re=300.0, spatial_box=((-5.0, 20.0), (-5.0, 5.0), (0.0, 10.0)),
                                time_interval=(0.0, 11.85))
    return _problem(sol, counts, m, n_pde, n_ghost, per_snapshot, nx, snaps, width, layers, act, seed, (2.0, 2.0),
                    LossWeights(10.0, 10.0, 1.0, 1.0, 1.0, velocity=(1.0, 5.0, 100.0)))


def _problem(sol, counts, m, n_pde, n_ghost, per_snapshot, nx, snaps, width, layers, act, seed, deltas, weights):
    domain = GlobalDomain.from_solution(sol)
    pts = benchmarks.grid_points(sol, nx, snaps)
    vel, p = sol.velocity_pressure(pts)
    table = ReferenceTable(regime=sol.regime, points=pts, velocity=vel, pressure=p)
    obs = snapshot_observations(table, per_snapshot, seed=0)
    budget = Budget(n_obs=obs.n, n_pde=n_pde, n_ghost_per_interface=n_ghost)
    subs = partition(domain, counts, m, delta_space=deltas[0], delta_time=deltas[1])
    ds = build_all_rank_datasets(subs, budget, obs, seed)
    cfg = ExpertConfig.for_regime(sol.regime, layers, width, act)
    anchor = tuple(lo + 0.25 * (hi - lo) for lo, hi in domain.spatial_box)
    return sol, subs, ds, cfg, weights, anchor, table, obs


def dump_plan(out, tag, plan, obs, table):
    out[f"{tag}/masters"] = np.array(sorted(plan.masters))
    out[f"{tag}/obs_points"] = obs.points
    out[f"{tag}/obs_velocity"] = obs.velocity
    out[f"{tag}/table_velocity"] = table.velocity
    out[f"{tag}/table_pressure"] = table.pressure
    for ws in plan.worker_specs:
        r = ws.rank
        d = ws.datasets
        out[f"{tag}/r{r}/role"] = np.array(ws.role == "master")
        out[f"{tag}/r{r}/param_seed"] = np.array(ws.param_seed, dtype=np.uint64)
        out[f"{tag}/r{r}/init"] = init_params(ws.expert_config, ws.param_seed).flat
        out[f"{tag}/r{r}/obs_points"] = d.obs_points
        out[f"{tag}/r{r}/obs_velocity"] = d.obs_velocity
        out[f"{tag}/r{r}/colloc"] = d.colloc_points
        out[f"{tag}/r{r}/ghost_neighbors"] = np.array([g.neighbor for g in d.ghosts], dtype=np.int64)
        out[f"{tag}/r{r}/ghost_kinds"] = np.array([g.kind == "temporal" for g in d.ghosts])
        for gi, g in enumerate(d.ghosts):
            out[f"{tag}/r{r}/ghost{gi}"] = g.points
        out[f"{tag}/r{r}/out_dest"] = np.array([e.dest for e in ws.outgoing], dtype=np.int64)
        out[f"{tag}/r{r}/out_gi"] = np.array([e.ghost_index for e in ws.outgoing], dtype=np.int64)
        w = ws.effective_weights
        out[f"{tag}/r{r}/weights"] = np.array([w.obs, w.pde, w.ghost_u, w.ghost_p_space, w.ghost_p_time])


def main():
    out = {}
    # ---------------- decomposition / plans / training (small) ----------------
    cases = {
        "p1": dict(kind="2d", counts=(1, 1), m=1),
        "p2": dict(kind="2d", counts=(2, 1), m=1),
        "t2": dict(kind="2d", counts=(1, 1), m=2),
        "p8": dict(kind="2d", counts=(2, 2), m=2),
        "d3": dict(kind="3d", counts=(2, 2, 2), m=1),
    }
    for tag, c in cases.items():
        if c["kind"] == "2d":
            sol, subs, ds, cfg, weights, anchor, table, obs = problem_2d(c["counts"], c["m"], 1600, 40, 12)
            epochs, lr, clip = 4, 1e-3, None
        else:
            sol, subs, ds, cfg, weights, anchor, table, obs = problem_3d(c["counts"], c["m"], 1600, 40, 10)
            epochs, lr, clip = 3, 1e-3, 1.0
        tc = TrainConfig(epochs=epochs, batch_size=500, learning_rate=lr, weights=weights, anchor=anchor,
                         lr_factor=0.5, lr_interval=2, comm_interval=1, clip_norm=clip, seed=0)
        plan = build_plan(subs, ds, cfg, tc)
        dump_plan(out, tag, plan, obs, table)
        out[f"{tag}/meta"] = np.array([epochs, lr, 0.5, 2, -1.0 if clip is None else clip, len(subs)])
        res = train(plan, backend="serial")
        for r in sorted(res.params):
            out[f"{tag}/r{r}/final"] = res.params[r].flat
            out[f"{tag}/r{r}/history"] = res.history[r]
        print(tag, "ranks", len(subs), "masters", sorted(plan.masters))

    # ---------------- tapes: jets, PDE loss + grad, MSE ----------------
    rng = np.random.default_rng(123)
    tape_cases = [
        ("unsteady2d", [3, 16, 16, 3], "tanh", 80.0),
        ("unsteady2d", [3, 16, 16, 16, 3], "sin", 100.0),
        ("steady2d", [2, 16, 16, 3], "tanh", 40.0),
        ("unsteady3d", [4, 16, 16, 4], "sin", 300.0),
        ("unsteady2d", [3, 64, 64, 64, 64, 3], "tanh", 100.0),
        ("unsteady2d", [3, 150, 150, 150, 3], "sin", 100.0),   # wide (layer-wise kernels)
        ("unsteady3d", [4, 200, 200, 4], "sin", 300.0),
        ("steady2d", [2, 256, 256, 3], "tanh", 40.0),
    ]
    for i, (kind, arch, act, re) in enumerate(tape_cases):
        regime = FlowRegime(kind, re)
        cfg = ExpertConfig(arch[0], len(arch) - 2, arch[1], act, arch[-1])
        params = init_params(cfg, 10 + i)
        n = 37
        pts = rng.uniform(-3.0, 3.0, (n, arch[0]))
        jt = ad.build_jet_tape(arch, n, act)
        jet = ad.forward_jet(jt, params, pts)
        pt = ad.build_pde_tape(arch, n, act, residual_structure(regime), coef=0.5 / n)
        pt.bind_params(params.tape_arrays())
        pt.bind_inputs(points=pts)
        pt.forward()
        g = pt.backward()
        nv = regime.n_vel
        tu = rng.normal(size=(n, nv))
        tp = rng.normal(size=n)
        vw = [1.0, 2.0, 3.0][:nv]
        mt = ad.build_mse_tape(arch, n, act, n_vel=nv, vel_weights=vw, vel_coef=0.25, p_coef=0.75,
                               p_channel=regime.p_channel)
        mt.bind_params(params.tape_arrays())
        mt.bind_inputs(points=pts, target_u=tu, target_p=tp)
        mt.forward()
        gm = mt.backward()
        t = f"tape{i}"
        out[f"{t}/params"] = params.flat
        out[f"{t}/pts"] = pts
        out[f"{t}/jet_value"], out[f"{t}/jet_grad"], out[f"{t}/jet_lap"] = jet.value, jet.grad, jet.lap
        out[f"{t}/sq_pde"] = np.array(pt.scalar("sq_pde"))
        out[f"{t}/grad_pde"] = g
        out[f"{t}/tu"], out[f"{t}/tp"] = tu, tp
        out[f"{t}/sq_u"], out[f"{t}/sq_p"] = np.array(mt.scalar("sq_u")), np.array(mt.scalar("sq_p"))
        out[f"{t}/grad_mse"] = gm
        out[f"{t}/meta"] = np.array([{"steady2d": 0, "unsteady2d": 1, "unsteady3d": 2}[kind], re,
                                     act == "sin", 0.5 / n, 0.25, 0.75] + vw + [0.0] * (3 - len(vw)))
        out[f"{t}/arch"] = np.array(arch)

    # ---------------- LocalObjective.epoch (composite, master weights) ----------------
    regime = FlowRegime("unsteady2d", 40.0)
    cfg = ExpertConfig.for_regime(regime, 3, 16, "tanh")
    params = init_params(cfg, 4)
    ds = RankDatasets(
        obs_points=rng.uniform(0, 1, (23, 3)), obs_velocity=rng.normal(size=(23, 2)),
        colloc_points=rng.uniform(0, 1, (57, 3)),
        ghosts=(GhostSet(1, "spatial", rng.uniform(0, 1, (11, 3))),
                GhostSet(2, "temporal", rng.uniform(0, 1, (13, 3))),
                GhostSet(3, "spatial", rng.uniform(0, 1, (7, 3)))),
    )
    targets = [(rng.normal(size=(g.points.shape[0], 2)), rng.normal(size=g.points.shape[0])) for g in ds.ghosts]
    for tag, w in (("obj", LossWeights(10.0, 4.0, 1.0, 1.5, 2.0, velocity=(1.0, 3.0))),
                   ("objm", LossWeights(10.0, 4.0, 1.0, 1.5, 2.0).as_master())):
        obj = LocalObjective(cfg, regime, ds, w, batch_size=16)
        obj.set_ghost_targets(targets)
        parts, grad, total = obj.epoch(params, np.random.default_rng(0))
        out[f"{tag}/parts"] = np.array(parts.astuple())
        out[f"{tag}/grad"] = grad
        out[f"{tag}/total"] = np.array(total)
        out[f"{tag}/weights"] = np.array([w.obs, w.pde, w.ghost_u, w.ghost_p_space, w.ghost_p_time] +
                                         list(w.velocity or (1.0, 1.0)))
    out["obj/params"] = params.flat
    out["obj/obs_points"], out["obj/obs_velocity"], out["obj/colloc"] = ds.obs_points, ds.obs_velocity, ds.colloc_points
    for gi, (g, (u, p)) in enumerate(zip(ds.ghosts, targets)):
        out[f"obj/ghost{gi}"], out[f"obj/ghost{gi}_u"], out[f"obj/ghost{gi}_p"] = g.points, u, p
        out[f"obj/ghost{gi}_kind"] = np.array(g.kind == "temporal")

    # ---------------- Adam ----------------
    n = 50
    p = rng.normal(size=n)
    st = AdamState.zeros(n)
    seq = []
    for k in range(5):
        gr = rng.normal(size=n) * (10.0 if k == 2 else 1.0)
        seq.append(gr.copy())
        adam_step(p, gr, st, lr=1e-2 * (0.5 ** k), clip_norm=3.0)
    rng2 = np.random.default_rng(999)
    p0 = rng2.normal(size=n)
    p = p0.copy()
    st = AdamState.zeros(n)
    grads, ps, ms, vs = [], [], [], []
    for k in range(5):
        gr = rng2.normal(size=n) * (10.0 if k == 2 else 1.0)
        grads.append(gr.copy())
        adam_step(p, gr, st, lr=1e-2 * (0.5 ** k), clip_norm=3.0)
        ps.append(p.copy()); ms.append(st.m.copy()); vs.append(st.v.copy())
    out["adam/p0"], out["adam/grads"] = p0, np.array(grads)
    out["adam/params"], out["adam/m"], out["adam/v"] = np.array(ps), np.array(ms), np.array(vs)

    path = os.path.join(HERE, "golden.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes,", len(out), "arrays")


if __name__ == "__main__":
    sys.exit(main())
