"""Probe the tcgen05 TF32 accumulation rounding: A, B exactly representable in
TF32 (products exact), C = A B^T on the tensor core vs the exact float64 sum;
a one-signed error (relative to sign(C)) means the accumulator truncates.

    python tools/tc_accum_probe.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_15883_b200 import _lib as X  # noqa: E402


def tf32(a):
    u = a.astype(np.float32).view(np.uint32) & np.uint32(0xFFFFE000)
    return u.view(np.float32)


def main():
    rng = np.random.default_rng(0)
    for K in (8, 64):
        N = 64
        errs, rel = [], []
        for trial in range(20):
            A = tf32(rng.normal(size=(128, K)))
            B = tf32(rng.normal(size=(N, K)))
            exact = A.astype(np.float64) @ B.astype(np.float64).T
            a = torch.tensor(A, device="cuda")
            b = torch.tensor(B, device="cuda")
            c = torch.empty((128, N), dtype=torch.float32, device="cuda")
            rc = X.lib().fr_debug_tc_gemm_tf32(X.ptr(a), X.ptr(b), X.ptr(c), N, K, 0, X.stream_ptr())
            assert rc == 0, rc
            C = c.cpu().numpy().astype(np.float64)
            d = (C - exact) * np.sign(exact)  # > 0: rounded away from zero, < 0: toward zero
            f32 = (exact.astype(np.float32).astype(np.float64) - exact) * np.sign(exact)
            errs.append(d.ravel())
            rel.append((np.abs(C - exact) / np.abs(exact).clip(1e-30)).ravel())
        e = np.concatenate(errs)
        r = np.concatenate(rel)
        print(f"K={K}: toward-zero {np.mean(e < 0):.3f} away {np.mean(e > 0):.3f} exact {np.mean(e == 0):.3f}; "
              f"median rel {np.median(r):.3e} max rel {np.max(r):.3e}")


if __name__ == "__main__":
    main()
