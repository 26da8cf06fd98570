"""Run the TF32 wide PDE launch sequence a few times (ncu target).

    ncu --set full -k regex:tcw_fwd -c 1 python tools/profile_tc.py [width] [layers] [n]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2602_15883_b200 import engine
    from paper_2602_15883_b200.network import ExpertConfig, init_params

    w = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    L = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 100_000
    act = os.environ.get("ACT", "tanh")
    kind = os.environ.get("KIND", "unsteady2d")
    d = 4 if kind == "unsteady3d" else 3
    cfg = ExpertConfig(d, L, w, act, d)
    p = init_params(cfg, 3).flat
    rng = np.random.default_rng(5)
    cols = [rng.uniform(0, 7.35, n), rng.uniform(-7.5, 17.5, n), rng.uniform(-8, 8, n)]
    if d == 4:
        cols.append(rng.uniform(0, 10, n))
    pts = np.column_stack(cols)
    plan = engine.get_plan(cfg, kind, 100.0, "float32", math=os.environ.get("MATH", "tf32"))
    for _ in range(int(os.environ.get("REPS", "2"))):
        sq, g = engine.pde_loss_grad(plan, p, pts, 1.0 / n)
    torch.cuda.synchronize()
    print("loss", sq)


if __name__ == "__main__":
    main()
