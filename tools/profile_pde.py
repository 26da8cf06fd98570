"""Launch the fused PDE kernel at the P=1 bench size (for ncu captures).

    python tools/profile_pde.py [--n 500000] [--reps 3] [--act tanh] [--width 64] [--layers 4]
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    from paper_2602_15883_b200 import _lib as X
    from paper_2602_15883_b200 import engine
    from paper_2602_15883_b200.network import ExpertConfig, init_params

    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=500_000)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--act", default="tanh")
    ap.add_argument("--width", type=int, default=64)
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--dtype", default="float32")
    a = ap.parse_args()
    cfg = ExpertConfig(3, a.layers, a.width, a.act, 3)
    plan = engine.get_plan(cfg, "unsteady2d", 100.0, a.dtype)
    flat = torch.as_tensor(init_params(cfg, 0).flat).cuda()
    kp = engine.new_kparams(plan)
    engine.prepare(plan, flat, kp)
    rng = np.random.default_rng(0)
    pts = np.column_stack([rng.uniform(0, 7.35, a.n), rng.uniform(-7.5, 17.5, a.n), rng.uniform(-8, 8, a.n)])
    pts_d = engine.to_device(pts, plan.tdtype, plan.device)
    ws = plan.workspace(X.MODE_PDE, a.n)
    gp = torch.empty(ws.gpart_elems, dtype=torch.float64, device="cuda")
    lp = torch.empty(ws.lpart_elems, dtype=torch.float64, device="cuda")
    sc = torch.empty(ws.scratch_bytes, dtype=torch.uint8, device="cuda")
    times = []
    for _ in range(a.reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        X.call("fr_pde_fwd_bwd", plan.h, X.ptr(kp), X.ptr(pts_d), a.n, 1e-5, X.ptr(gp), X.ptr(lp), X.ptr(sc),
               X.stream_ptr())
        e.record()
        torch.cuda.synchronize()
        times.append(s.elapsed_time(e))
    fpp = 6 * 6 * (a.layers - 1) * a.width ** 2 + 6 * 3 * a.width + 6 * 6 * a.width * 3 + 45 * a.layers * a.width
    print(f"grid {ws.grid} x {ws.threads} thr, smem {ws.smem_bytes} B, ppt {ws.points_per_tile}; "
          f"ms {['%.3f' % t for t in times]}; TFLOP/s {fpp * a.n / min(times) * 1e-9:.2f}")


if __name__ == "__main__":
    main()
