"""Split-TF32 tensor-core path of the W <= 64 fused epoch kernel
(FR_MATH_TF32X3: tcgen05.mma kind::tf32, A_hi B_hi + A_hi B_lo + A_lo B_hi,
FP32 accumulation in TMEM) held to the SAME parity bar as the FP32 SIMT path
(per-term losses and the flat gradient within 1e-5 of the
reference's float64 fixtures)."""

import os

import numpy as np
import pytest

from conftest import ROOT, per_term_rel, rel_l2, report

pytestmark = pytest.mark.gpu

TERM, GRAD, PARAMS = 1e-5, 1e-5, 1e-6


def _plan8(math):
    from paper_2602_15883_b200 import config as fconfig
    from paper_2602_15883_b200.runtime import TrainConfig, build_plan

    pb = fconfig.cylinder2d_problem(n_pde=20_000, counts=(2, 2), time_splits=2)
    tc = TrainConfig(epochs=3, batch_size=25_000, learning_rate=1e-3, weights=pb.weights, anchor=pb.anchor,
                     lr_factor=0.2, lr_interval=2000, comm_interval=1, seed=0, math=math)
    return pb, build_plan(pb.subdomains, pb.datasets, pb.expert_config, tc)


@pytest.fixture(scope="module")
def hg():
    return np.load(os.path.join(ROOT, "tests", "golden", "golden_headline.npz"))


@pytest.mark.parametrize("rank", [0, 3])
def test_tf32x3_epoch_matches_reference(hg, rank):
    from paper_2602_15883_b200.runtime import LocalObjective

    pb, plan = _plan8("tf32x3")
    ws = plan.worker_specs[rank]
    k = f"ep/{rank}"
    obj = LocalObjective(pb.expert_config, plan.regime, ws.datasets, ws.effective_weights, 25_000, math="tf32x3")
    assert obj.plan.info.math == 2
    obj.set_ghost_targets([(hg[f"{k}/ghost{gi}_u"], hg[f"{k}/ghost{gi}_p"]) for gi in range(len(ws.datasets.ghosts))])
    parts, grad, total = obj.epoch(hg[f"{k}/params"], None)
    e = dict(term=per_term_rel(parts.astuple(), hg[f"{k}/parts"]),
             total=abs(total - float(hg[f"{k}/total"])) / abs(float(hg[f"{k}/total"])),
             grad=rel_l2(grad, hg[f"{k}/grad"]))
    report(f"tf32x3_epoch/r{rank}", **e)
    assert e["term"] < TERM and e["total"] < TERM
    assert e["grad"] < GRAD


def test_tf32x3_full_p1_epoch(hg):
    from paper_2602_15883_b200 import config as fconfig
    from paper_2602_15883_b200.runtime import LocalObjective

    pb = fconfig.cylinder2d_problem(n_procs=1)
    obj = LocalObjective(pb.expert_config, pb.domain.regime, pb.datasets[0], pb.weights, 25_000, math="tf32x3")
    parts, grad, total = obj.epoch(hg["full/params"], None)
    e = dict(term=per_term_rel(parts.astuple(), hg["full/parts"]),
             total=abs(total - float(hg["full/total"])) / float(hg["full/total"]), grad=rel_l2(grad, hg["full/grad"]))
    report("tf32x3_full_p1", **e)
    assert e["term"] < TERM and e["grad"] < GRAD


def test_tf32x3_train_p8(hg):
    from paper_2602_15883_b200.runtime.driver import LocalTrainer

    _, plan = _plan8("tf32x3")
    tr = LocalTrainer(plan)
    tr.run(3)
    worst_h = worst_p = 0.0
    for r, w in tr.workers.items():
        w.sync_history()
        eh = per_term_rel(np.array(w.history)[:, 1:6], hg[f"tr/r{r}/history"][:, 1:6])
        ep = rel_l2(w.flat.cpu().numpy(), hg[f"tr/r{r}/final"])
        worst_h, worst_p = max(worst_h, eh), max(worst_p, ep)
    report("tf32x3_train_p8", history_term=worst_h, params=worst_p)
    assert worst_h < TERM and worst_p < PARAMS


@pytest.mark.parametrize("kind,act", [("unsteady3d", "sin"), ("steady2d", "tanh"), ("unsteady2d", "sin")])
def test_tf32x3_other_regimes_match_simt(kind, act):
    """3D (256-thread tiles, two M blocks), steady 2D (240-row tiles) and sin:
    the tensor-core epoch agrees with the FP32 SIMT epoch to FP32 accuracy."""
    import torch

    from paper_2602_15883_b200.engine import get_plan, new_kparams, prepare, to_device
    from paper_2602_15883_b200.network import ExpertConfig, init_params
    from paper_2602_15883_b200.physics import FlowRegime, LossWeights
    from paper_2602_15883_b200.decomposition import GhostSet, RankDatasets
    from paper_2602_15883_b200.runtime.objective import DeviceObjective

    regime = FlowRegime(kind, 100.0)
    cfg = ExpertConfig.for_regime(regime, 4, 64, act)
    rng = np.random.default_rng(4)
    d = regime.n_inputs
    ds = RankDatasets(rng.uniform(-2, 2, (700, d)), rng.normal(size=(700, regime.n_vel)),
                      rng.uniform(-2, 2, (9000, d)), (GhostSet(1, "temporal" if regime.has_time else "spatial",
                                                              rng.uniform(-2, 2, (300, d))),))
    w = LossWeights(10.0, 5.0, 1.0, 1.0, 1.0)
    out = {}
    for math in ("simt", "tf32x3"):
        plan = get_plan(cfg, kind, 100.0, "float32", math)
        flat = to_device(init_params(cfg, 9).flat, torch.float64, plan.device)
        kp = new_kparams(plan)
        prepare(plan, flat, kp)
        obj = DeviceObjective(plan, regime, ds, w)
        obj.set_ghost_targets([(rng.normal(size=(300, regime.n_vel)) * 0 + 0.1, np.full(300, 0.2))])
        obj.enqueue(kp)
        torch.cuda.synchronize()
        out[math] = (obj.sums.cpu().numpy().copy(), obj.grad.cpu().numpy().copy())
    e_l = per_term_rel(out["tf32x3"][0], out["simt"][0], floor=1e-300)
    e_g = rel_l2(out["tf32x3"][1], out["simt"][1])
    report(f"tf32x3_vs_simt/{kind}/{act}", loss=e_l, grad=e_g)
    assert e_l < TERM and e_g < GRAD
