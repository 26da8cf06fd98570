"""Error and resource contracts of the training path (GPU):

* input finiteness is checked at upload / target installation with the
  reference's message (autodiff/tape.py:251-255, 298-326);
* the in-kernel exchange wait honours train(..., exchange_timeout)
  (runtime/driver.py:150-181, 259) and surfaces as DeadlockError;
* a capped persistent grid is launched the same whether or not the epoch is
  gated (the workspace is sized for the cap);
* graph replays respect the worker's history capacity;
* clip_norm = 0.0 clips (to zero), as the reference's `is not None` test does
  (runtime/optim.py:20-28);
* C^1 derivative targets survive a save / resume.
"""

import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu


def _small_plan(epochs=4, comm_interval=1, width=32, n_pde=2000, gd=0.0, counts=(2, 1), time_splits=2):
    from paper_2602_15883_b200 import config as fconfig
    from paper_2602_15883_b200.runtime import TrainConfig, build_plan

    pb = fconfig.cylinder2d_problem(n_pde=n_pde, n_ghost=40, per_snapshot=12, grid_nx=9, snapshots=10,
                                    hidden_layers=2, width=width, activation="tanh", counts=counts,
                                    time_splits=time_splits)
    tc = TrainConfig(epochs=epochs, batch_size=500, learning_rate=1e-3, weights=pb.weights, anchor=pb.anchor,
                     lr_factor=0.5, lr_interval=2, comm_interval=comm_interval, seed=0,
                     ghost_derivative_weight=gd)
    return pb, build_plan(pb.subdomains, pb.datasets, pb.expert_config, tc)


def _datasets_with(ds, **repl):
    from paper_2602_15883_b200.decomposition import RankDatasets

    f = dict(obs_points=ds.obs_points, obs_velocity=ds.obs_velocity, colloc_points=ds.colloc_points,
             ghosts=ds.ghosts)
    f.update(repl)
    return RankDatasets(f["obs_points"], f["obs_velocity"], f["colloc_points"], tuple(f["ghosts"]))


@pytest.mark.parametrize("field", ["colloc_points", "obs_points", "obs_velocity", "ghost"])
def test_nonfinite_inputs_rejected_with_index(field):
    from paper_2602_15883_b200.decomposition import GhostSet
    from paper_2602_15883_b200.runtime import LocalObjective

    pb, plan = _small_plan()
    ds = plan.worker_specs[0].datasets
    if field == "ghost":
        g = ds.ghosts[0]
        pts = g.points.copy()
        pts[5, 1] = np.inf
        bad = _datasets_with(ds, ghosts=(GhostSet(g.neighbor, g.kind, pts),) + tuple(ds.ghosts[1:]))
        name, idx = "input 'points'", "(5, 1)"
    else:
        arr = getattr(ds, field).copy()
        arr[7, 0] = np.nan
        bad = _datasets_with(ds, **{field: arr})
        name = "input 'target_u'" if field == "obs_velocity" else "input 'points'"
        idx = "(7, 0)"
    with pytest.raises(ValueError, match=f"non-finite value in {name} at index {idx}".replace("(", r"\(")
                       .replace(")", r"\)")):
        LocalObjective(pb.expert_config, pb.domain.regime, bad, plan.worker_specs[0].effective_weights, 500)


def test_nonfinite_ghost_targets_and_params_rejected():
    from paper_2602_15883_b200.network import init_params
    from paper_2602_15883_b200.runtime import LocalObjective

    pb, plan = _small_plan()
    ws = plan.worker_specs[0]
    obj = LocalObjective(pb.expert_config, pb.domain.regime, ws.datasets, ws.effective_weights, 500)
    vals = [(np.zeros((g.points.shape[0], 2)), np.zeros(g.points.shape[0])) for g in ws.datasets.ghosts]
    vals[1][1][3] = np.nan
    with pytest.raises(ValueError, match=r"non-finite value in input 'target_p' at index \(3,\)"):
        obj.set_ghost_targets(vals)
    vals[1][1][3] = 0.0
    obj.set_ghost_targets(vals)
    p = init_params(pb.expert_config, 0)
    flat = p.flat.copy()
    # W1 (32 x 32) follows W0 (3 x 32) and b0 (32): entry (2, 5) of W1
    flat[3 * 32 + 32 + 2 * 32 + 5] = np.inf
    with pytest.raises(ValueError, match=r"non-finite value in parameter at index \(2, 5\)"):
        obj.epoch(flat, None)


def test_exchange_timeout_reaches_the_gate():
    """A transport slower than exchange_timeout trips the in-kernel wait."""
    from paper_2602_15883_b200.runtime import DeadlockError
    from paper_2602_15883_b200.runtime.driver import LocalTrainer

    _, plan = _small_plan(epochs=2)
    # every gate is published 300 ms late; the wait gives up after 20 ms
    tr = LocalTrainer(plan, overlap=True, signal_delay_ns=300_000_000, exchange_timeout=0.02)
    with pytest.raises(DeadlockError):
        tr.run(1)
    ok = LocalTrainer(plan, overlap=True, signal_delay_ns=30_000_000, exchange_timeout=5.0)
    ok.run(1)


def test_capped_grid_same_with_and_without_gate():
    """max_ctas smaller than the tile count: ungated (cap-only) launches write
    exactly the capped grid's partial rows (they used the full grid
    and overran the capped workspace)."""
    import torch

    from paper_2602_15883_b200.engine import get_plan, new_kparams, prepare, to_device
    from paper_2602_15883_b200.network import init_params
    from paper_2602_15883_b200.runtime.objective import DeviceObjective

    pb, plan = _small_plan(n_pde=40000, width=64)
    ws = plan.worker_specs[0]
    ep = get_plan(pb.expert_config, pb.domain.regime.kind, pb.domain.regime.reynolds, "float32")
    flat = to_device(init_params(pb.expert_config, 3).flat, torch.float64, ep.device)
    kp = new_kparams(ep)
    prepare(ep, flat, kp)
    grads = []
    for cap in (0, 4):
        obj = DeviceObjective(ep, pb.domain.regime, ws.datasets, ws.effective_weights, max_ctas=cap)
        assert obj.ws.tiles > obj.grid
        # sentinel rows past the capped workspace must stay untouched
        guard = torch.full((obj.gpart.numel() + 4096,), 7.0, dtype=torch.float64, device=ep.device)
        obj.gpart = guard[: obj.gpart.numel()]
        obj.mark_targets_set()
        obj.enqueue(kp)
        torch.cuda.synchronize()
        assert torch.all(guard[obj.gpart.numel():] == 7.0)
        grads.append(obj.grad.cpu().numpy())
        if cap:
            assert obj.grid < 8
    assert rel_l2(grads[1], grads[0]) < 1e-12


def test_graph_replay_checks_history_capacity():
    from paper_2602_15883_b200.runtime.driver import LocalTrainer

    _, plan = _small_plan(epochs=4)
    tr = LocalTrainer(plan, epochs=3)
    tr.run(3)
    with pytest.raises(RuntimeError, match="capacity"):
        tr.run(1, start=3)


def test_workers_own_their_optimiser_counters():
    from paper_2602_15883_b200.runtime.driver import LocalTrainer

    _, plan = _small_plan(epochs=2)
    tr = LocalTrainer(plan)
    ptrs = {w.sync_counter.data_ptr() for w in tr.workers.values()}
    assert len(ptrs) == len(tr.workers)


@pytest.mark.parametrize("clip", [0.0, 0.5, None])
def test_clip_norm_semantics_match_reference(clip):
    from paper_2602_15883_b200.runtime import AdamState, adam_step

    rng = np.random.default_rng(1)
    p = rng.normal(size=50)
    g = rng.normal(size=50)
    # the reference's float64 sequence (runtime/optim.py:20-49)
    pr, gr, m, v = p.copy(), g.copy(), np.zeros(50), np.zeros(50)
    norm = float(np.sqrt(np.dot(gr, gr)))
    if clip is not None and norm > clip:
        gr *= clip / norm
    m *= 0.9
    m += (1.0 - 0.9) * gr
    v *= 0.999
    v += (1.0 - 0.999) * gr * gr
    pr -= 1e-3 * (m / (1.0 - 0.9)) / (np.sqrt(v / (1.0 - 0.999)) + 1e-8)
    st = AdamState.zeros(50)
    n = adam_step(p, g, st, lr=1e-3, clip_norm=clip)
    assert abs(n - norm) <= 1e-14 * norm
    assert np.max(np.abs(p - pr)) <= 1e-15
    assert np.max(np.abs(g - gr)) <= 1e-15


def test_resume_keeps_derivative_targets(tmp_path):
    """ghost_derivative_weight > 0 and a resume in the middle of a
    comm_interval: the derivative targets come back from the FRTS file."""
    from paper_2602_15883_b200 import checkpoint as ck
    from paper_2602_15883_b200.runtime.driver import LocalTrainer

    _, plan = _small_plan(epochs=4, comm_interval=3, gd=0.5)
    full = LocalTrainer(plan)
    full.run(4)
    a = LocalTrainer(plan)
    a.run(2)
    ck.save_trainer_state(tmp_path / "st", a)
    b = LocalTrainer(plan)
    start = ck.load_trainer_state(tmp_path / "st", b)
    b.run(2, start=start)
    for r in full.workers:
        assert np.array_equal(full.workers[r].flat.cpu().numpy(), b.workers[r].flat.cpu().numpy()), r
