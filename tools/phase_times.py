"""Per-phase cycle breakdown of the fused epoch kernel (instrumented build).

    python -m paper_2602_15883_b200.build --force -D FR_PHASE_TIMERS \\
        --lib paper_2602_15883_b200/_lib_timers/libflowrec_b200.so
    FLOWREC_B200_LIB=paper_2602_15883_b200/_lib_timers/libflowrec_b200.so python tools/phase_times.py

Thread 0 of every CTA reads clock64() after each phase barrier; the sums over
CTAs give each phase's share of the kernel (the slowest warp of each phase).
"""

import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

PHASES = ["load points", "layer-0 fwd", "hidden fwd GEMM", "hidden fwd epilogue + stage",
          "output fwd", "head", "output bwd", "act-bwd + rebuild H", "dW compute", "dW combine write",
          "dW combine sum + dX GEMM", "dX store + stage", "layer-0 bwd", "dW0 / db0"]


def main():
    import torch

    from paper_2602_15883_b200 import _lib as X
    from paper_2602_15883_b200.config import cylinder2d_problem
    from paper_2602_15883_b200.runtime import TrainConfig, build_plan
    from paper_2602_15883_b200.runtime.driver import LocalTrainer

    n = int(os.environ.get("N_PDE", "500000"))
    pb = cylinder2d_problem(n_procs=1, n_pde=n, hidden_layers=4, width=64, activation="tanh")
    tc = TrainConfig(epochs=8, batch_size=25000, learning_rate=1e-3, weights=pb.weights, anchor=pb.anchor,
                     math=os.environ.get("MATH") or None)
    tr = LocalTrainer(build_plan(pb.subdomains, pb.datasets, pb.expert_config, tc))
    tr.run(2, use_graphs=False, record_times=False)
    torch.cuda.synchronize()
    lib = X.lib()
    f = lib.fr_debug_phase_cycles_f32
    f.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
    buf = (C.c_ulonglong * 32)()
    f(buf, 1)
    tr.run(4, start=2, use_graphs=False, record_times=False)
    torch.cuda.synchronize()
    f(buf, 1)
    tot = sum(buf[: len(PHASES)])
    for i, name in enumerate(PHASES):
        print(f"{i:2d} {name:28s} {buf[i] / tot * 100:6.2f}%")
    print("total CTA-cycles", tot)
    for i, name in ((10, "tc3 dX A_lo transform"), (11, "tc3 MMA wait"), (12, "tc3 drain D"), (13, "tc dW chunk wait"),
                    (14, "tc dW staging"), (15, "tc dW stage barrier"), (9, "tc dW drain")):
        if buf[16 + i]:
            print(f"   {name:28s} {buf[16 + i] / tot * 100:6.2f}%")


if __name__ == "__main__":
    main()
