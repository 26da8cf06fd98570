"""Parity of the BENCHMARKED network ([3, 64x4, 3] tanh, cylinder-wake box)
against fixtures written by the unmodified reference
(tests/golden/make_golden_headline.py -> golden_headline.npz):

* `LocalObjective.epoch` on a master and a slave rank of the P=8 (2,2)x2
  decomposition, each with spatial and temporal ghosts and neighbour-shaped
  targets (runtime/objective.py:164-199, physics.py:190-200);
* the reference's serial `train()` of that plan for 3 epochs
  (runtime/driver.py:127-144);
* one unsampled 500,000-point P=1 epoch of config C.

FP32 (the product path) is held to SURVEY 8(c)'s bar: every loss term within
1e-5 relative, the flat gradient within 1e-5 norm-wise; the FP64 build of the
same kernels within 1e-10 (indexing, not rounding).  Measured errors are
reported (pytest -s, or FR_PARITY_LOG=<file>).
"""

import os

import numpy as np
import pytest

from conftest import ROOT, per_term_rel, rel_l2, report

pytestmark = pytest.mark.gpu

F32_TERM = 1e-5
F32_GRAD = 1e-5
F32_PARAMS = 1e-6
F64_TERM = 1e-10
F64_GRAD = 1e-10


@pytest.fixture(scope="module")
def hg():
    return np.load(os.path.join(ROOT, "tests", "golden", "golden_headline.npz"))


def _sha(a):
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def _plan8():
    from paper_2602_15883_b200 import config as fconfig
    from paper_2602_15883_b200.runtime import TrainConfig, build_plan

    pb = fconfig.cylinder2d_problem(n_pde=20_000, counts=(2, 2), time_splits=2)
    tc = TrainConfig(epochs=3, batch_size=25_000, learning_rate=1e-3, weights=pb.weights, anchor=pb.anchor,
                     lr_factor=0.2, lr_interval=2000, comm_interval=1, seed=0)
    return pb, build_plan(pb.subdomains, pb.datasets, pb.expert_config, tc)


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("rank", [0, 3])
def test_headline_local_objective_epoch(hg, rank, dtype):
    from paper_2602_15883_b200.runtime import LocalObjective

    pb, plan = _plan8()
    ws = plan.worker_specs[rank]
    k = f"ep/{rank}"
    d = ws.datasets
    assert _sha(d.colloc_points) == str(hg[f"{k}/colloc_sha"])
    assert bool(hg[f"{k}/role"]) == (ws.role == "master")
    w = ws.effective_weights
    assert np.array_equal([w.obs, w.pde, w.ghost_u, w.ghost_p_space, w.ghost_p_time], hg[f"{k}/weights"])
    targets = []
    for gi, g in enumerate(d.ghosts):
        assert np.array_equal(g.points, hg[f"{k}/ghost{gi}"])
        targets.append((hg[f"{k}/ghost{gi}_u"], hg[f"{k}/ghost{gi}_p"]))
    obj = LocalObjective(pb.expert_config, plan.regime, d, w, 25_000, dtype=dtype)
    obj.set_ghost_targets(targets)
    parts, grad, total = obj.epoch(hg[f"{k}/params"], None)
    e_term = per_term_rel(parts.astuple(), hg[f"{k}/parts"])
    e_total = abs(total - float(hg[f"{k}/total"])) / abs(float(hg[f"{k}/total"]))
    e_grad = rel_l2(grad, hg[f"{k}/grad"])
    report(f"headline_epoch/r{rank}/{dtype}", term=e_term, total=e_total, grad=e_grad)
    tol_t, tol_g = (F64_TERM, F64_GRAD) if dtype == "float64" else (F32_TERM, F32_GRAD)
    assert e_term < tol_t and e_total < tol_t
    assert e_grad < tol_g


@pytest.mark.parametrize("overlap", [False, True])
def test_headline_serial_train_p8(hg, overlap):
    """The (2,2)x2 plan, 3 epochs, all 8 ranks on one GPU (CUDA graphs after
    the first epoch; overlap=True: in-kernel gated exchange)."""
    from paper_2602_15883_b200.runtime.driver import LocalTrainer

    _, plan = _plan8()
    tr = LocalTrainer(plan, overlap=overlap)
    tr.run(3)
    worst_h = worst_p = 0.0
    for r, w in tr.workers.items():
        w.sync_history()
        hist = np.array(w.history)
        ref = hg[f"tr/r{r}/history"]
        assert np.array_equal(hist[:, 0], ref[:, 0])
        eh = per_term_rel(hist[:, 1:6], ref[:, 1:6])
        ep = rel_l2(w.flat.cpu().numpy(), hg[f"tr/r{r}/final"])
        worst_h, worst_p = max(worst_h, eh), max(worst_p, ep)
        assert eh < F32_TERM, (r, eh)
        assert ep < F32_PARAMS, (r, ep)
    report(f"headline_train_p8/overlap={overlap}", history_term=worst_h, params=worst_p)


def test_headline_full_p1_epoch(hg):
    """One unsampled 500,000-point epoch of config C (the benchmarked step)."""
    from paper_2602_15883_b200 import config as fconfig
    from paper_2602_15883_b200.runtime import LocalObjective, TrainConfig, build_plan

    pb = fconfig.cylinder2d_problem(n_procs=1)
    tc = TrainConfig(epochs=1, batch_size=25_000, learning_rate=1e-3, weights=pb.weights, anchor=pb.anchor, seed=0)
    plan = build_plan(pb.subdomains, pb.datasets, pb.expert_config, tc)
    ws = plan.worker_specs[0]
    d = ws.datasets
    assert d.n_colloc == 500_000 and d.n_obs == 10_000
    assert _sha(d.colloc_points) == str(hg["full/colloc_sha"])
    assert _sha(d.obs_points) == str(hg["full/obs_sha"])
    obj = LocalObjective(pb.expert_config, plan.regime, d, ws.effective_weights, 25_000)
    parts, grad, total = obj.epoch(hg["full/params"], None)
    e_term = per_term_rel(parts.astuple(), hg["full/parts"])
    e_total = abs(total - float(hg["full/total"])) / float(hg["full/total"])
    e_grad = rel_l2(grad, hg["full/grad"])
    report("headline_full_p1/float32", term=e_term, total=e_total, grad=e_grad)
    assert e_term < F32_TERM and e_total < F32_TERM
    assert e_grad < F32_GRAD
