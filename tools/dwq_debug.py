"""Compare TF32 wide-path gradients across kernel variants (FR_TC_DWQ, FR_TC_FWD,
FR_TC_DX set in the environment by the caller); prints per-case loss terms and
max |g| differences against a saved reference file."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_15883_b200 import engine
from paper_2602_15883_b200.network import ExpertConfig, init_params

tag = sys.argv[1]
out = {}
for kind, d, w, L, act in [("unsteady2d", 3, 150, 4, "sin"), ("unsteady3d", 4, 200, 3, "sin"),
                           ("steady2d", 2, 128, 3, "tanh")]:
    cfg = ExpertConfig(d, L, w, act, d if kind != "steady2d" else 3)
    p = init_params(cfg, 1).flat
    rng = np.random.default_rng(2)
    n = 5003
    pts = rng.uniform(-2.0, 2.0, (n, d))
    plan = engine.get_plan(cfg, kind, 100.0, "float32", math="tf32")
    sq, g = engine.pde_loss_grad(plan, p, pts, 1.0 / n)
    nv = cfg.arch[-1] - 1
    su, sp, gm = engine.mse_loss_grad(plan, p, pts[:777], rng.standard_normal((777, nv)), rng.standard_normal(777),
                                     np.ones(nv), 0.3, 0.7)
    out[kind] = (np.float64([sq, su, sp]), g, gm)
np.save(f"gpurun_out/dwq_dbg_{tag}.npy", np.array([out], dtype=object), allow_pickle=True)
print(tag, "done")
