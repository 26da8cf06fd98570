"""TF32 tensor-core wide path vs the float64 oracle (and vs the FP32 SIMT wide
path) on cylinder-box points: prints loss / gradient relative errors."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def rel_l2(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def main():
    from oracle import flowrec_oracle as O
    from paper_2602_15883_b200 import engine
    from paper_2602_15883_b200.network import ExpertConfig, init_params

    cases = [("unsteady2d", 3, 3, 128, 3, "tanh"), ("unsteady2d", 3, 3, 150, 3, "sin"),
             ("steady2d", 2, 3, 96, 2, "tanh"), ("unsteady3d", 4, 4, 200, 2, "sin"),
             ("unsteady2d", 3, 3, 300, 2, "tanh")]
    n = int(os.environ.get("N", "600"))
    for kind, din, dout, w, L, act in cases:
        cfg = ExpertConfig(din, L, w, act, dout)
        p = init_params(cfg, 3).flat
        rng = np.random.default_rng(5)
        cols = [rng.uniform(0, 7.35, n), rng.uniform(-7.5, 17.5, n), rng.uniform(-8, 8, n)]
        if din == 4:
            cols.append(rng.uniform(-4, 4, n))
        pts = np.column_stack(cols if din >= 3 else cols[1:])
        coef = 5.0 / n
        t0 = time.time()
        sq_ref, g_ref, _ = O.pde_loss_grad(p, cfg.arch, act, kind, 100.0, pts, coef)
        nv = dout - 1
        tu = rng.standard_normal((n, nv)) * 0.1
        tp = rng.standard_normal(n) * 0.1
        velw = [1.0] * nv
        su_ref, sp_ref, gm_ref = O.mse_loss_grad(p, cfg.arch, act, pts, tu, tp, velw, 2.0, 3.0)
        t1 = time.time()
        out = [f"{kind} w={w} L={L} {act} (oracle {t1 - t0:.1f}s)"]
        for math in ("simt", "tf32"):
            plan = engine.get_plan(cfg, kind, 100.0, "float32", math=math)
            sq, g = engine.pde_loss_grad(plan, p, pts, coef)
            su, sp, gm = engine.mse_loss_grad(plan, p, pts, tu, tp, velw, 2.0, 3.0)
            sq2, g2 = engine.pde_loss_grad(plan, p, pts, coef)
            det = (sq2 == sq) and np.array_equal(g, g2)
            out.append(f"  {math}: pde loss {abs(sq - sq_ref) / sq_ref:.2e} grad {rel_l2(g, g_ref):.2e} | "
                       f"mse u {abs(su - su_ref) / su_ref:.2e} p {abs(sp - sp_ref) / sp_ref:.2e} "
                       f"grad {rel_l2(gm, gm_ref):.2e} | det {det}")
        print("\n".join(out), flush=True)


if __name__ == "__main__":
    main()
