"""Pin the CPU oracle (oracle/flowrec_oracle.py) against fixtures produced by
the reference itself (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from cases import CASES, oracle_ranks, training_plan
from conftest import max_rel, rel_l2
from oracle import flowrec_oracle as O

KINDS = {0: "steady2d", 1: "unsteady2d", 2: "unsteady3d"}


def tape_case(golden, i):
    t = f"tape{i}"
    meta = golden[f"{t}/meta"]
    arch = [int(a) for a in golden[f"{t}/arch"]]
    kind, re, act = KINDS[int(meta[0])], float(meta[1]), ("sin" if meta[2] else "tanh")
    return t, arch, kind, re, act, meta


@pytest.mark.parametrize("i", range(8))
def test_oracle_jets_match_reference(golden, i):
    t, arch, kind, re, act, _ = tape_case(golden, i)
    Y, _ = O.jet_forward(golden[f"{t}/params"], arch, act, golden[f"{t}/pts"])
    assert max_rel(Y["v"], golden[f"{t}/jet_value"]) < 1e-13
    grad = np.stack(Y["g"], axis=2)
    lap = np.stack(Y["l"], axis=2)
    assert max_rel(grad, golden[f"{t}/jet_grad"]) < 1e-12
    assert max_rel(lap, golden[f"{t}/jet_lap"]) < 1e-12


@pytest.mark.parametrize("i", range(8))
def test_oracle_pde_loss_and_gradient(golden, i):
    t, arch, kind, re, act, meta = tape_case(golden, i)
    sq, g, _ = O.pde_loss_grad(golden[f"{t}/params"], arch, act, kind, re, golden[f"{t}/pts"], float(meta[3]))
    assert abs(sq - float(golden[f"{t}/sq_pde"])) <= 1e-12 * abs(float(golden[f"{t}/sq_pde"]))
    assert rel_l2(g, golden[f"{t}/grad_pde"]) < 1e-12


@pytest.mark.parametrize("i", range(8))
def test_oracle_mse_loss_and_gradient(golden, i):
    t, arch, kind, re, act, meta = tape_case(golden, i)
    nv = O.REGIMES[kind][1]
    su, sp, g = O.mse_loss_grad(golden[f"{t}/params"], arch, act, golden[f"{t}/pts"], golden[f"{t}/tu"],
                                golden[f"{t}/tp"], meta[6 : 6 + nv], float(meta[4]), float(meta[5]))
    assert abs(su - float(golden[f"{t}/sq_u"])) <= 1e-12 * abs(su)
    assert abs(sp - float(golden[f"{t}/sq_p"])) <= 1e-12 * abs(sp)
    assert rel_l2(g, golden[f"{t}/grad_mse"]) < 1e-12


def objective_data(golden):
    ghosts = []
    for gi in range(3):
        kind = "temporal" if bool(golden[f"obj/ghost{gi}_kind"]) else "spatial"
        ghosts.append((kind, golden[f"obj/ghost{gi}"], golden[f"obj/ghost{gi}_u"], golden[f"obj/ghost{gi}_p"]))
    return dict(obs_pts=golden["obj/obs_points"], obs_vel=golden["obj/obs_velocity"],
                colloc=golden["obj/colloc"], ghosts=ghosts)


@pytest.mark.parametrize("tag", ["obj", "objm"])
def test_oracle_local_epoch(golden, tag):
    w = golden[f"{tag}/weights"]
    weights = dict(obs=w[0], pde=w[1], ghost_u=w[2], ghost_p_space=w[3], ghost_p_time=w[4],
                   velocity=tuple(w[5:7]) if tag == "obj" else None)
    parts, grad, total = O.local_epoch(golden["obj/params"], [3, 16, 16, 16, 3], "tanh", "unsteady2d", 40.0,
                                       objective_data(golden), weights)
    assert max_rel(parts, golden[f"{tag}/parts"]) < 1e-12
    assert abs(total - float(golden[f"{tag}/total"])) < 1e-12 * abs(total)
    assert rel_l2(grad, golden[f"{tag}/grad"]) < 1e-12


def test_oracle_adam(golden):
    p = golden["adam/p0"].copy()
    m, v, step = np.zeros_like(p), np.zeros_like(p), 0
    for k, g in enumerate(golden["adam/grads"]):
        step, _ = O.adam_update(p, g.copy(), m, v, step, 1e-2 * (0.5 ** k), clip_norm=3.0)
        assert np.max(np.abs(p - golden["adam/params"][k])) <= 1e-15
        assert np.max(np.abs(m - golden["adam/m"][k])) <= 1e-15


@pytest.mark.parametrize("tag", ["p1", "t2", "p8", "d3"])
def test_oracle_serial_training_matches_reference(golden, tag):
    """Exchange (incl. anchor normalisation on masters), objective and Adam
    over several epochs against the reference's serial driver."""
    pb, plan = training_plan(tag, golden)
    tc = plan.train_config
    ranks = oracle_ranks(plan)
    hist = O.train_serial(ranks, pb.expert_config.arch, pb.expert_config.activation, plan.regime.kind,
                          plan.regime.reynolds, tc.epochs, tc.lr, tc.comm_interval, tc.clip_norm, tc.anchor)
    for r in ranks:
        assert rel_l2(hist[r], golden[f"{tag}/r{r}/history"]) < 1e-11, r
        assert rel_l2(ranks[r]["flat"], golden[f"{tag}/r{r}/final"]) < 1e-12, r


@pytest.mark.parametrize("rank", [0, 3])
def test_oracle_headline_epoch_matches_reference(rank):
    """The oracle on the benchmarked network: LocalObjective.epoch of a master
    and a slave rank of (2,2)x2 with spatial + temporal ghosts
    (golden_headline.npz, written by the reference)."""
    import os

    from conftest import ROOT
    from paper_2602_15883_b200 import config as fconfig

    hg = np.load(os.path.join(ROOT, "tests", "golden", "golden_headline.npz"))
    pb = fconfig.cylinder2d_problem(n_pde=20_000, counts=(2, 2), time_splits=2)
    d = pb.datasets[rank]
    k = f"ep/{rank}"
    w = hg[f"{k}/weights"]
    ghosts = [(g.kind, g.points, hg[f"{k}/ghost{gi}_u"], hg[f"{k}/ghost{gi}_p"]) for gi, g in enumerate(d.ghosts)]
    parts, grad, total = O.local_epoch(
        hg[f"{k}/params"], pb.expert_config.arch, "tanh", "unsteady2d", 100.0,
        dict(obs_pts=d.obs_points, obs_vel=d.obs_velocity, colloc=d.colloc_points, ghosts=ghosts),
        dict(obs=w[0], pde=w[1], ghost_u=w[2], ghost_p_space=w[3], ghost_p_time=w[4], velocity=None))
    assert max_rel(parts, hg[f"{k}/parts"]) < 1e-12
    assert abs(total - float(hg[f"{k}/total"])) <= 1e-12 * abs(total)
    assert rel_l2(grad, hg[f"{k}/grad"]) < 1e-11
