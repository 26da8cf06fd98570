"""GPU: tcgen05 TF32 tensor-core plumbing (UMMA descriptors, TMEM, tcgen05.ld).

The wide-expert tensor-core path stages k-quad activation tiles as canonical
K-major SWIZZLE_NONE UMMA operands; this checks one 128 x N x K MMA chain
against a float64 matmul of the TF32-rounded operands."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _tf32(x):
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    return (b & np.uint32(0xFFFFE000)).view(np.float32)


@pytest.mark.parametrize("N,K", [(16, 8), (64, 32), (128, 64), (256, 64), (96, 40)])
def test_tc_gemm_tf32(N, K):
    """K-major A and B (the only TF32 operand layout the wide kernels use:
    MN-major TF32 descriptors read zeros on sm_100a, tools/tc_layout_probe.py)."""
    layout = 0
    import torch

    from paper_2602_15883_b200 import _lib as X

    rng = np.random.default_rng(N * 1000 + K)
    A = rng.standard_normal((128, K)).astype(np.float32)
    B = rng.standard_normal((N, K)).astype(np.float32)
    dA = torch.from_numpy(A).cuda()
    dB = torch.from_numpy(B).cuda()
    dC = torch.zeros((128, N), dtype=torch.float32, device="cuda")
    X.call("fr_debug_tc_gemm_tf32", dA.data_ptr(), dB.data_ptr(), dC.data_ptr(), N, K, layout, None)
    torch.cuda.synchronize()
    C = dC.cpu().numpy().astype(np.float64)
    ref = _tf32(A).astype(np.float64) @ _tf32(B).astype(np.float64).T
    full = A.astype(np.float64) @ B.astype(np.float64).T
    scale = np.abs(A).astype(np.float64) @ np.abs(B).astype(np.float64).T
    # truncation vs round-to-nearest of the TF32 conversion: bound by 2^-10 per product
    err = np.abs(C - ref) / scale
    assert err.max() < 2.0 ** -10, (err.max(), np.abs(C - full).max())
