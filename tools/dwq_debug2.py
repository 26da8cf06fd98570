"""Isolate tcw_dwq_kernel differences: prints, per case, the max relative
difference of each hidden layer's dW / db between FR_TC_DWQ=1 and =0 (the two
runs happen in subprocesses)."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = [("unsteady2d", 3, 160, 2, "tanh", "mse"), ("unsteady2d", 3, 160, 3, "tanh", "mse"),
         ("unsteady3d", 4, 192, 2, "sin", "pde"), ("unsteady3d", 4, 200, 2, "sin", "pde"),
         ("unsteady2d", 3, 160, 2, "tanh", "pde")]
if len(sys.argv) > 1:
    sys.path.insert(0, ROOT)
    from paper_2602_15883_b200 import engine
    from paper_2602_15883_b200.network import ExpertConfig, init_params
    res = []
    for kind, d, w, L, act, head in CASES:
        cfg = ExpertConfig(d, L, w, act, d if kind != "steady2d" else 3)
        p = init_params(cfg, 1).flat
        rng = np.random.default_rng(2)
        n = 512
        pts = rng.uniform(-2.0, 2.0, (n, d))
        plan = engine.get_plan(cfg, kind, 100.0, "float32", math="tf32")
        nv = cfg.arch[-1] - 1
        if head == "pde":
            _, g = engine.pde_loss_grad(plan, p, pts, 1.0 / n)
        else:
            _, _, g = engine.mse_loss_grad(plan, p, pts, rng.standard_normal((n, nv)), rng.standard_normal(n),
                                          np.ones(nv), 0.3, 0.7)
        res.append(g)
    np.save(sys.argv[1], np.array(res, dtype=object), allow_pickle=True)
else:
    out = {}
    envs = {"1": dict(FR_TC_DWQ="1"), "0": dict(FR_TC_DWQ="0"), "1b": dict(FR_TC_DWQ="1"),
            "ns1": dict(FR_TC_DWQ="1", FR_DWQ_NS="1")}
    for m, e in envs.items():
        f = f"/tmp/dwq2_{m}.npy"
        subprocess.run([sys.executable, __file__, f], env=dict(os.environ, **e), check=True)
        out[m] = np.load(f, allow_pickle=True)
    for ci in range(len(CASES)):
        print("case", ci, "rerun identical:", np.array_equal(out["1"][ci], out["1b"][ci]),
              "ns1 == default:", np.array_equal(out["1"][ci], out["ns1"][ci]),
              "ns1 == old:", np.abs(out["ns1"][ci] - out["0"][ci]).max())
    for ci, (kind, d, w, L, act, head) in enumerate(CASES):
        arch = [d] + [w] * L + [d if kind != "steady2d" else 3]
        a, b = out["1"][ci], out["0"][ci]
        off = 0
        msg = []
        for l in range(L + 1):
            for nm, sz in (("W", arch[l] * arch[l + 1]), ("b", arch[l + 1])):
                r = np.abs(a[off:off + sz] - b[off:off + sz]).max() / max(np.abs(b[off:off + sz]).max(), 1e-30)
                msg.append(f"{nm}{l}={r:.1e}")
                off += sz
        print(kind, w, L, act, head, " ".join(msg), flush=True)
        np.save(f"gpurun_out/dwq2_case{ci}.npy", np.stack([a, b]))
