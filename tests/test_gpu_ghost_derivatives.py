"""Opt-in C^1 interface coupling (TrainConfig.ghost_derivative_weight > 0):
ghost messages also carry the sender's first derivatives of the velocity at
the receiver's ghost points, and the receiver adds
lambda_gd / N_ghost * sum w_c (d u_c/d x_i - target)^2.  The reference couples
values only (worker.py:179-197; SURVEY 8e says this extension defaults off for
parity), so the kernel is pinned to the float64 oracle restatement of the same
term, and the default (weight 0) path is unchanged (every other test)."""

import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype,tol", [("float64", 1e-10), ("float32", 1e-4)])
@pytest.mark.parametrize("kind,act,din", [("unsteady2d", "tanh", 3), ("unsteady3d", "sin", 4), ("steady2d", "tanh", 2)])
def test_ghost_jet_head_matches_oracle(kind, act, din, dtype, tol):
    from oracle import flowrec_oracle as O
    from paper_2602_15883_b200 import engine
    from paper_2602_15883_b200.network import ExpertConfig, init_params

    nv = din - 1 if kind != "steady2d" else 2
    cfg = ExpertConfig(din, 3, 64, act, nv + 1)
    p = init_params(cfg, 4).flat
    rng = np.random.default_rng(9)
    pts = rng.uniform(-2, 2, (777, din))
    tdu = rng.normal(0, 0.3, (777, din, nv))
    vw = [1.0, 5.0, 100.0][:nv]
    sq_ref, g_ref = O.ghost_jet_loss_grad(p, cfg.arch, act, pts, tdu, vw, 0.37)
    plan = engine.get_plan(cfg, kind, 100.0, dtype)
    sq, g = engine.ghost_jet_loss_grad(plan, p, pts, tdu, vw, 0.37)
    assert abs(sq - sq_ref) <= tol * sq_ref
    assert rel_l2(g, g_ref) < tol


def _objective(golden, weight):
    from paper_2602_15883_b200.decomposition import GhostSet, RankDatasets
    from paper_2602_15883_b200.network import ExpertConfig
    from paper_2602_15883_b200.physics import FlowRegime, LossWeights
    from paper_2602_15883_b200.runtime import LocalObjective

    w = golden["obj/weights"]
    weights = LossWeights(*w[:5], velocity=tuple(w[5:7]))
    ghosts, targets = [], []
    rng = np.random.default_rng(3)
    for gi in range(3):
        kind = "temporal" if bool(golden[f"obj/ghost{gi}_kind"]) else "spatial"
        pts = golden[f"obj/ghost{gi}"]
        ghosts.append(GhostSet(gi + 1, kind, pts))
        targets.append((golden[f"obj/ghost{gi}_u"], golden[f"obj/ghost{gi}_p"],
                        rng.normal(0, 0.2, (pts.shape[0], 3, 2))))
    ds = RankDatasets(golden["obj/obs_points"], golden["obj/obs_velocity"], golden["obj/colloc"], tuple(ghosts))
    regime = FlowRegime("unsteady2d", 40.0)
    obj = LocalObjective(ExpertConfig.for_regime(regime, 3, 16, "tanh"), regime, ds, weights, 16, dtype="float64",
                         ghost_derivative_weight=weight)
    obj.set_ghost_targets(targets if weight > 0 else [t[:2] for t in targets])
    return obj, ghosts, targets, weights


def test_objective_adds_the_derivative_term(golden):
    """epoch(weight) = epoch(0) + the GJ head over every ghost set with
    coefficient weight / N_ghost_total (FP64 build, 1e-10)."""
    from oracle import flowrec_oracle as O

    lam = 0.7
    obj0, ghosts, targets, weights = _objective(golden, 0.0)
    obj1, _, _, _ = _objective(golden, lam)
    p = golden["obj/params"]
    parts0, g0, t0 = obj0.epoch(p, None)
    parts1, g1, t1 = obj1.epoch(p, None)
    assert parts0.astuple() == parts1.astuple()
    n_tot = sum(g.points.shape[0] for g in ghosts)
    sq, gx = 0.0, np.zeros_like(g0)
    for g, t in zip(ghosts, targets):
        s, gg = O.ghost_jet_loss_grad(p, obj0.config.arch, "tanh", g.points, t[2], weights.velocity, lam / n_tot)
        sq += s
        gx += gg
    assert abs((t1 - t0) - lam * sq / n_tot) <= 1e-10 * abs(t1)
    assert rel_l2(g1 - g0, gx) < 1e-9


def test_exchange_carries_the_senders_derivatives(golden):
    """In-process trainer with the extension: after one exchange each rank's
    derivative targets are the neighbour's jet at those ghost points, and the
    drop-in message protocol carries the same du."""
    import torch

    from cases import training_plan
    from paper_2602_15883_b200 import engine
    from paper_2602_15883_b200.runtime import RankWorker, build_plan
    from paper_2602_15883_b200.runtime.driver import LocalTrainer
    import dataclasses

    pb, plan0 = training_plan("p8", golden)
    tc = dataclasses.replace(plan0.train_config, ghost_derivative_weight=0.5)
    plan = build_plan(pb.subdomains, pb.datasets, pb.expert_config, tc)
    tr = LocalTrainer(plan, dtype="float64")
    tr.enqueue_exchange()
    torch.cuda.synchronize()
    n_in, nv = plan.regime.n_inputs, plan.regime.n_vel
    for r, w in tr.workers.items():
        for gi, g in enumerate(w.ws.datasets.ghosts):
            src = tr.workers[g.neighbor]
            jet = engine.forward_jet(src.plan, src.flat.cpu().numpy(), g.points)
            got = w.objective.target_du_slice(gi).cpu().numpy()
            assert np.allclose(got, jet[:, 1:1 + n_in, :nv], rtol=1e-12, atol=1e-12), (r, gi)
    # drop-in protocol: messages carry du
    ws = plan.worker_specs[0]
    msgs = RankWorker(ws, dtype="float64").outgoing_messages(0)
    assert all(m.du is not None and m.du.shape == (m.points.shape[0], n_in, nv) for m in msgs)


def test_extension_trains_and_is_deterministic(golden):
    import dataclasses

    from cases import training_plan
    from paper_2602_15883_b200.runtime import build_plan, train

    pb, plan0 = training_plan("p8", golden)
    tc = dataclasses.replace(plan0.train_config, ghost_derivative_weight=0.5)
    plan = build_plan(pb.subdomains, pb.datasets, pb.expert_config, tc)
    a = train(plan, backend="serial")
    b = train(plan, backend="serial", use_graphs=False)
    base = train(plan0, backend="serial")
    for r in a.params:
        assert np.array_equal(a.params[r].flat, b.params[r].flat)
        assert np.all(np.isfinite(a.history[r]))
        assert not np.array_equal(a.params[r].flat, base.params[r].flat)  # the term acts
