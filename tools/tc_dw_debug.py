"""Per-block gradient comparison of the split-TF32 epoch kernel against the
FP32 SIMT one (debugging aid for the tensor-core weight gradient)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(kind, act, n_obs=700, n_pde=9000, n_gh=300):
    import torch

    from paper_2602_15883_b200.decomposition import GhostSet, RankDatasets
    from paper_2602_15883_b200.engine import get_plan, new_kparams, prepare, to_device
    from paper_2602_15883_b200.network import ExpertConfig, init_params
    from paper_2602_15883_b200.physics import FlowRegime, LossWeights
    from paper_2602_15883_b200.runtime.objective import DeviceObjective

    regime = FlowRegime(kind, 100.0)
    cfg = ExpertConfig.for_regime(regime, 4, 64, act)
    rng = np.random.default_rng(4)
    d = regime.n_inputs
    ds = RankDatasets(rng.uniform(-2, 2, (n_obs, d)), rng.normal(size=(n_obs, regime.n_vel)),
                      rng.uniform(-2, 2, (n_pde, d)), (GhostSet(1, "temporal" if regime.has_time else "spatial",
                                                                rng.uniform(-2, 2, (n_gh, d))),))
    w = LossWeights(10.0, 5.0, 1.0, 1.0, 1.0)
    out = {}
    for math in ("simt", "tf32x3"):
        plan = get_plan(cfg, kind, 100.0, "float32", math)
        flat = to_device(init_params(cfg, 9).flat, torch.float64, plan.device)
        kp = new_kparams(plan)
        prepare(plan, flat, kp)
        obj = DeviceObjective(plan, regime, ds, w)
        obj.set_ghost_targets([(np.zeros((n_gh, regime.n_vel)) + 0.1, np.full(n_gh, 0.2))])
        obj.enqueue(kp)
        torch.cuda.synchronize()
        out[math] = (obj.sums.cpu().numpy().copy(), obj.grad.cpu().numpy().copy())
    g0, g1 = out["simt"][1], out["tf32x3"][1]
    pos = 0
    print(f"{kind} {act} obs={n_obs} pde={n_pde} gh={n_gh}: sums simt {out['simt'][0]} tc {out['tf32x3'][0]}")
    for li, ((fi, fo), _) in enumerate(cfg.layer_shapes):
        for name, n in (("W", fi * fo), ("b", fo)):
            a, b = g0[pos:pos + n], g1[pos:pos + n]
            print(f"  layer {li} {name}: rel {np.linalg.norm(a - b) / max(np.linalg.norm(a), 1e-300):.3e}  |g| {np.linalg.norm(a):.3e}")
            pos += n


if __name__ == "__main__":
    for kind, act in (("unsteady3d", "sin"), ("unsteady2d", "sin"), ("steady2d", "tanh")):
        run(kind, act)
        run(kind, act, n_obs=700, n_pde=0, n_gh=300) if False else None
