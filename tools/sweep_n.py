"""Epoch-kernel time against the per-rank collocation count (fixed-cost probe).

    python tools/sweep_n.py [--n 62500,125000,250000,500000] [--procs 1]

For each n builds the P=1 (or --procs P, rank 0) cylinder-wake problem, runs
two eager epochs, then times the fused epoch kernel alone (CUDA events, median
of 10 back-to-back launches) and the whole captured epoch.  Prints one line per
n with ms, ms per PDE tile-wave and the FP32 TFLOP/s of the algorithmic work.
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    import bench
    from paper_2602_15883_b200 import _lib as X
    from paper_2602_15883_b200.config import cylinder2d_problem
    from paper_2602_15883_b200.runtime import TrainConfig, build_plan
    from paper_2602_15883_b200.runtime.driver import LocalTrainer

    ap = argparse.ArgumentParser()
    ap.add_argument("--n", default="62500,125000,250000,500000")
    ap.add_argument("--procs", type=int, default=1)
    a = ap.parse_args()
    for n in [int(x) for x in a.n.split(",")]:
        pb = cylinder2d_problem(n_procs=a.procs, n_pde=n * a.procs, hidden_layers=4, width=64, activation="tanh")
        tc = TrainConfig(epochs=40, batch_size=25000, learning_rate=1e-3, weights=pb.weights, anchor=pb.anchor)
        tr = LocalTrainer(build_plan(pb.subdomains, pb.datasets, pb.expert_config, tc), epochs=40)
        tr.run(3, use_graphs=True, record_times=False)
        torch.cuda.synchronize()
        w = tr.workers[0]
        k = bench._time_epoch_kernel(torch, X, w, reps=10)
        ep = tr.run(10, start=3, use_graphs=True, record_times=True)
        fl = bench.flops_per_point() * w.objective.n_colloc + bench.flops_per_value_point() * k["n_mse"]
        print(f"P={a.procs} n_rank={w.objective.n_colloc:7d} n_mse={k['n_mse']:5d} kernel {k['ms']:.3f} ms "
              f"({fl / k['ms'] * 1e-9:.1f} TFLOP/s)  epoch(all {len(tr.workers)} ranks) "
              f"{np.median(ep) * 1e3:.3f} ms", flush=True)


if __name__ == "__main__":
    main()
