import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import flowrec_oracle as O
from paper_2602_15883_b200 import engine
from paper_2602_15883_b200.network import ExpertConfig, init_params
def rel(a,b): return float(np.linalg.norm(a-b)/np.linalg.norm(b))
for kind, din, nv in [("steady2d", 2, 2), ("unsteady2d", 3, 2)]:
    for L in (2, 3, 4):
        for dt in ("float64", "float32"):
            cfg = ExpertConfig(din, L, 64, "tanh", nv + 1)
            p = init_params(cfg, 4).flat
            rng = np.random.default_rng(9)
            pts = rng.uniform(-2, 2, (300, din)); tdu = rng.normal(0, 0.3, (300, din, nv))
            sr, gr = O.ghost_jet_loss_grad(p, cfg.arch, "tanh", pts, tdu, [1.0, 5.0], 0.37)
            plan = engine.get_plan(cfg, kind, 100.0, dt)
            s, g = engine.ghost_jet_loss_grad(plan, p, pts, tdu, [1.0, 5.0], 0.37)
            sq2, g2, _ = O.pde_loss_grad(p, cfg.arch, "tanh", kind, 100.0, pts, 0.5)
            s3, g3 = engine.pde_loss_grad(plan, p, pts, 0.5)
            print(kind, L, dt, "GJ loss %.1e grad %.1e" % (abs(s-sr)/sr, rel(g, gr)), "PDE loss %.1e grad %.1e" % (abs(s3-sq2)/sq2, rel(g3, g2)))
