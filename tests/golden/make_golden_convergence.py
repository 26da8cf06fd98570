"""A longer training run of the benchmarked network, by the UNMODIFIED
reference (`flowrec`), to pin multi-epoch behaviour -- loss trajectories,
the coupling across interfaces and the reconstructed fields -- not just one
step.

    PYTHONPATH=baseline/_ref python tests/golden/make_golden_convergence.py

Writes tests/golden/golden_convergence.npz: the (2,2)x2 P=8 plan of
golden_headline's `tr` case (N_pde 20,000, [3,64x4,3] tanh, 1,000 ghosts per
interface, anchor-normalised masters) trained 150 epochs with the reference's
serial `train()` (runtime/driver.py:127-144), then per-rank histories and final
parameters, `evaluation.interface_jump` (evaluation.py:220-279) of the initial
and trained experts, and `evaluation.field_errors` (evaluation.py:107-121) of
the trained stitched field on the reference grid.  About 3 minutes on one core.
"""

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

import flowrec  # noqa: E402
from flowrec import evaluation as ev  # noqa: E402
from flowrec.network import ExpertParams, init_params  # noqa: E402
from flowrec.runtime import TrainConfig, build_plan, train  # noqa: E402
from make_golden_headline import headline_problem  # noqa: E402

assert flowrec.backend_name() == "cython", flowrec.backend_name()
EPOCHS = 150


def main():
    out = {}
    sol, subs, ds, cfg, weights, anchor = headline_problem((2, 2), 2, 20_000)
    tc = TrainConfig(epochs=EPOCHS, batch_size=25_000, learning_rate=1e-3, weights=weights, anchor=anchor,
                     lr_factor=0.2, lr_interval=2000, comm_interval=1, seed=0)
    plan = build_plan(subs, ds, cfg, tc)
    probes = ev.ProbeSpec(n_per_interface=256, eps_frac=1e-4, seed=0)
    init = {ws.rank: init_params(cfg, ws.param_seed) for ws in plan.worker_specs}
    j0 = ev.interface_jump(init, subs, probes)
    t0 = time.perf_counter()
    res = train(plan, backend="serial")
    print(f"trained {EPOCHS} epochs in {time.perf_counter() - t0:.1f} s")
    j1 = ev.interface_jump(res.params, subs, probes)
    for r in sorted(res.params):
        out[f"r{r}/history"] = res.history[r]
        out[f"r{r}/final"] = res.params[r].flat
    out["jump0"] = np.array([[j.rank_a, j.rank_b, j.kind == "temporal", j.max_jump_u, j.max_jump_p] for j in j0])
    out["jump1"] = np.array([[j.rank_a, j.rank_b, j.kind == "temporal", j.max_jump_u, j.max_jump_p] for j in j1])
    from flowrec import benchmarks as B

    pts = B.grid_points(sol, 33, 50)
    vel, p = sol.velocity_pressure(pts)
    st = ev.stitch(res.params, subs, pts)
    from flowrec.decomposition import ReferenceTable

    fe = ev.field_errors(st, ReferenceTable(regime=sol.regime, points=pts, velocity=vel, pressure=p), plan.masters,
                         anchor)
    out["field_errors"] = np.array([fe[k] for k in sorted(fe)])
    out["field_error_keys"] = np.array(sorted(fe))
    out["meta"] = np.array([EPOCHS, 1e-3])
    path = os.path.join(HERE, "golden_convergence.npz")
    np.savez_compressed(path, **out)
    h = np.stack([res.history[r] for r in sorted(res.history)])
    print("mean obs/pde/ghost_u at epoch 0 and end:", h[:, 0, 1:4].mean(0), h[:, -1, 1:4].mean(0))
    print("max jump u/p before:", out["jump0"][:, 3].max(), out["jump0"][:, 4].max(),
          "after:", out["jump1"][:, 3].max(), out["jump1"][:, 4].max())
    print("field errors:", dict(zip(sorted(fe), out["field_errors"])))
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    sys.exit(main())
