"""The drop-in boundary exercised against the REAL reference package
(`flowrec`, installed unmodified under baseline/_ref):

* the reference's own `flowrec.runtime.driver.train`
  patched with the `backend="cuda"` dispatch; `flowrec.config`-style inputs ->
  `flowrec.runtime.build_plan` -> `train(plan, backend="cuda")` returns a
  flowrec `TrainResult` matching flowrec's own serial backend;
* `flowrec._kernels.set_backend("cuda")` routes the
  reference's tape activations (`_ActJet`, tape.py:73-124) through
  fr_jet_act_forward/backward on its host arrays.

The conversion of the reference's plan objects is host-only and runs on CPU.
"""

import os
import sys

import numpy as np
import pytest

from conftest import ROOT, per_term_rel, rel_l2, report

REF = os.path.join(ROOT, "baseline", "_ref")
pytestmark = pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "flowrec")),
                                reason="reference not installed under baseline/_ref")


@pytest.fixture(scope="module")
def flowrec():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import flowrec as F

    return F


def _ref_plan(F, counts=(2, 2), m=2, n_pde=20_000, epochs=3, width=64, layers=4):
    from flowrec import benchmarks as B
    from flowrec.decomposition import (Budget, GlobalDomain, ReferenceTable, build_all_rank_datasets, partition,
                                       snapshot_observations)
    from flowrec.network import ExpertConfig
    from flowrec.physics import LossWeights
    from flowrec.runtime import TrainConfig, build_plan

    sol = B.TaylorGreen2D(re=100.0, spatial_box=((-7.5, 17.5), (-8.0, 8.0)), time_interval=(0.0, 7.35))
    domain = GlobalDomain.from_solution(sol)
    pts = B.grid_points(sol, 33, 50)
    vel, p = sol.velocity_pressure(pts)
    obs = snapshot_observations(ReferenceTable(regime=sol.regime, points=pts, velocity=vel, pressure=p), 200, seed=0)
    subs = partition(domain, counts, m, delta_space=2.0, delta_time=1.0)
    ds = build_all_rank_datasets(subs, Budget(n_obs=obs.n, n_pde=n_pde, n_ghost_per_interface=1000), obs, 0)
    cfg = ExpertConfig.for_regime(sol.regime, layers, width, "tanh")
    anchor = tuple(lo + 0.25 * (hi - lo) for lo, hi in domain.spatial_box)
    tc = TrainConfig(epochs=epochs, batch_size=25_000, learning_rate=1e-3, weights=LossWeights(10.0, 5.0, 1.0, 1.0, 1.0),
                     anchor=anchor, lr_factor=0.2, lr_interval=2000, comm_interval=1, seed=0)
    return build_plan(subs, ds, cfg, tc)


def test_reference_plan_converts_exactly(flowrec):
    """Host side of the whole-path drop-in: the reference's plan objects become
    the engine's with identical roles, weights, routes, seeds and datasets."""
    from paper_2602_15883_b200 import config as fconfig
    from paper_2602_15883_b200.interop import from_reference_plan
    from paper_2602_15883_b200.runtime import TrainConfig, build_plan

    rp = _ref_plan(flowrec)
    ours = from_reference_plan(rp)
    pb = fconfig.cylinder2d_problem(n_pde=20_000, counts=(2, 2), time_splits=2)
    tc = TrainConfig(epochs=3, batch_size=25_000, learning_rate=1e-3, weights=pb.weights, anchor=pb.anchor,
                     lr_factor=0.2, lr_interval=2000, comm_interval=1, seed=0)
    mine = build_plan(pb.subdomains, pb.datasets, pb.expert_config, tc)
    assert ours.masters == mine.masters == rp.masters
    for a, b, r in zip(ours.worker_specs, mine.worker_specs, rp.worker_specs):
        assert (a.rank, a.role, a.param_seed) == (b.rank, b.role, b.param_seed) == (r.rank, r.role, r.param_seed)
        assert a.effective_weights == b.effective_weights
        assert [(e.dest, e.ghost_index) for e in a.outgoing] == [(e.dest, e.ghost_index) for e in r.outgoing]
        assert np.array_equal(a.datasets.colloc_points, r.datasets.colloc_points)
        assert np.array_equal(a.datasets.obs_velocity, b.datasets.obs_velocity)
        for ga, gr in zip(a.datasets.ghosts, r.datasets.ghosts):
            assert (ga.neighbor, ga.kind) == (gr.neighbor, gr.kind) and np.array_equal(ga.points, gr.points)


@pytest.mark.gpu
def test_reference_train_backend_cuda(flowrec, monkeypatch):
    """INTEGRATION.md section 1 applied to the reference's own driver module."""
    import flowrec.runtime.driver as RD

    from paper_2602_15883_b200.interop import train_reference_plan

    stock_train = RD.train

    def train(plan, backend="serial", exchange_timeout=600.0):  # the reference-side patch
        if backend == "cuda":
            return train_reference_plan(plan, exchange_timeout=exchange_timeout)
        return stock_train(plan, backend=backend, exchange_timeout=exchange_timeout)

    monkeypatch.setattr(RD, "train", train)
    plan = _ref_plan(flowrec)
    ref = RD.train(plan, backend="serial")
    got = RD.train(plan, backend="cuda")
    assert isinstance(got, RD.TrainResult)
    assert sorted(got.params) == sorted(ref.params)
    worst_h = worst_p = 0.0
    for r in ref.params:
        assert isinstance(got.params[r], flowrec.network.ExpertParams)
        assert got.params[r].seed == ref.params[r].seed
        assert got.exchange_log[r] == ref.exchange_log[r]
        assert np.array_equal(got.history[r][:, 0], ref.history[r][:, 0])
        eh = per_term_rel(got.history[r][:, 1:6], ref.history[r][:, 1:6])
        ep = rel_l2(got.params[r].flat, ref.params[r].flat)
        worst_h, worst_p = max(worst_h, eh), max(worst_p, ep)
    report("reference_train_backend_cuda", history_term=worst_h, params=worst_p)
    assert worst_h < 1e-5 and worst_p < 1e-6
    assert got.median_epoch_time() > 0.0


@pytest.mark.gpu
def test_reference_kernels_seam_on_gpu(flowrec):
    """the reference's tapes with the "cuda" seam
    match its Cython backend (float64)."""
    from flowrec import _kernels as K
    from flowrec import autodiff as ad
    from flowrec.network import ExpertConfig, init_params
    from flowrec.physics import FlowRegime, residual_structure

    from paper_2602_15883_b200.interop import install_kernels_backend

    install_kernels_backend(K)
    rng = np.random.default_rng(7)
    for act, kind, arch in (("tanh", "unsteady2d", [3, 32, 32, 3]), ("sin", "unsteady3d", [4, 24, 24, 4])):
        regime = FlowRegime(kind, 100.0)
        params = init_params(ExpertConfig(arch[0], len(arch) - 2, arch[1], act, arch[-1]), 3)
        pts = rng.uniform(-2, 2, (41, arch[0]))
        out = {}
        for backend in ("cython", "cuda"):
            prev = K.set_backend(backend)
            try:
                t = ad.build_pde_tape(arch, 41, act, residual_structure(regime), coef=0.1)
                t.bind_params(params.tape_arrays())
                t.bind_inputs(points=pts)
                t.forward()
                out[backend] = (t.scalar("sq_pde"), t.backward().copy())
            finally:
                K.set_backend(prev)
        assert abs(out["cuda"][0] - out["cython"][0]) <= 1e-12 * abs(out["cython"][0])
        assert rel_l2(out["cuda"][1], out["cython"][1]) < 1e-12
    prev = K.set_backend("cuda")
    try:
        z = np.zeros((7, 4))
        with pytest.raises(ValueError, match="unknown activation kind"):
            K.jet_act_forward(5, z, z.copy(), None, z[:1].copy(), z[:1].copy(), 1, 3)
    finally:
        K.set_backend(prev)
