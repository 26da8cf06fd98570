"""Descriptor sweep for MN-major TF32 operands (fr_debug_tc_raw2): which shared
word does the tensor core read for A(m, k) under each (layout type, LBO, SBO)?
Prints the word map for a few (m, k) per combination; 0 = read zero."""
import itertools
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def word_map(X, torch, a_mn, lbo, sbo, lt):
    out = []
    for shift in (0, 10):
        C = torch.zeros((128, 32), dtype=torch.float32, device="cuda")
        X.call("fr_debug_tc_raw2", C.data_ptr(), a_mn, lbo, sbo, lt, shift, None)
        torch.cuda.synchronize()
        out.append(C.cpu().numpy()[:, :8].astype(np.int64))
    lo, hi = out
    w = np.where(lo > 0, (hi - 1) * 1024 + (lo - 1), -1)
    return w


def main():
    import torch

    from paper_2602_15883_b200 import _lib as X

    combos = [(0, 0, 2048, 128)]
    for lt in (1,):
        for lbo, sbo in itertools.product((16, 128, 256, 512, 1024, 2048), repeat=2):
            combos.append((1, lt, lbo, sbo))
    for a_mn, lt, lbo, sbo in combos:
        w = word_map(X, torch, a_mn, lbo, sbo, lt)
        nz = int((w >= 0).sum())
        ms = (0, 1, 2, 3, 4, 5, 8, 31, 32, 127)
        rows = " | ".join(f"m{m}:" + ",".join(str(v) for v in w[m, :8]) for m in ms[:6])
        print(f"mn={a_mn} lt={lt} lbo={lbo:5d} sbo={sbo:5d} nonzero={nz:4d}  {rows}", flush=True)
        if nz:
            print("   m8..:", " | ".join(f"m{m}:" + ",".join(str(v) for v in w[m, :8]) for m in ms[6:]), flush=True)




def gemm_check():
    import torch

    from paper_2602_15883_b200 import _lib as X

    rng = np.random.default_rng(0)
    N, K = 64, 32
    A = rng.standard_normal((128, K)).astype(np.float32)
    B = rng.standard_normal((N, K)).astype(np.float32)
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    dA = torch.from_numpy(A).cuda()
    dB = torch.from_numpy(B).cuda()
    for layout in (0, 1, 2, 3, 5, 6, 7, 13, 14, 15):
        dC = torch.zeros((128, N), dtype=torch.float32, device="cuda")
        X.call("fr_debug_tc_gemm_tf32", dA.data_ptr(), dB.data_ptr(), dC.data_ptr(), N, K, layout, None)
        torch.cuda.synchronize()
        C = dC.cpu().numpy()
        print(f"gemm layout={layout}: max|C-ref| = {np.abs(C - ref).max():.3e}  max|C| = {np.abs(C).max():.3e}", flush=True)


if __name__ == "__main__":
    gemm_check()
    main()
