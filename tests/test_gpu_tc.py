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


@pytest.mark.parametrize("layout", [0, 5, 6, 7])
@pytest.mark.parametrize("N,K", [(16, 8), (64, 32), (128, 64), (256, 64), (96, 40)])
def test_tc_gemm_tf32(N, K, layout):
    """K-major A and B (layout 0, what the kernels use), and MN-major A / B / both
    (5 / 6 / 7) in the SWIZZLE_128B_BASE32B canonical layout -- the only one in
    which sm_100a reads MN-major TF32 (SWIZZLE_NONE MN-major reads zeros,
    tools/tc_mn_probe.py); LBO = MN-group stride, SBO = K-group stride."""
    if layout and N % 32:
        pytest.skip("BASE32B MN-major atoms span 32 MN elements")
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


_PERSIST_SCRIPT = r"""
import hashlib, os, sys
import numpy as np
sys.path.insert(0, os.environ["FR_ROOT"])
from paper_2602_15883_b200 import engine
from paper_2602_15883_b200.network import ExpertConfig, init_params
out = []
for kind, d, w, L, act in [("unsteady2d", 3, 150, 4, "sin"), ("unsteady3d", 4, 200, 3, "sin"),
                           ("steady2d", 2, 128, 3, "tanh")]:
    cfg = ExpertConfig(d, L, w, act, d if kind != "steady2d" else 3)
    p = init_params(cfg, 1).flat
    rng = np.random.default_rng(2)
    n = 5003  # a ragged last tile
    pts = rng.uniform(-2.0, 2.0, (n, d))
    plan = engine.get_plan(cfg, kind, 100.0, "float32", math="tf32")
    sq, g = engine.pde_loss_grad(plan, p, pts, 1.0 / n)
    nv = cfg.arch[-1] - 1
    su, sp, gm = engine.mse_loss_grad(plan, p, pts[:777], rng.standard_normal((777, nv)), rng.standard_normal(777),
                                     np.ones(nv), 0.3, 0.7)
    out.append(hashlib.sha256(np.float64([sq, su, sp]).tobytes() + g.tobytes() + gm.tobytes()).hexdigest())
print(" ".join(out))
"""


def test_tc_persistent_kernels_bit_identical_to_tile_kernels():
    """The persistent TF32 forward / adjoint kernels (default) compute exactly
    what the one-tile-per-CTA kernels do (FR_TC_FWD=tile / FR_TC_DX=tile):
    same MMA K order, same per-point epilogue arithmetic, so losses and both
    PDE and MSE gradients are bit-identical, incl. a ragged last tile, the 3D
    per-unit activation split and the steady regime."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for mode in ("persistent", "tile"):
        env = dict(os.environ, FR_ROOT=root, FR_TC_FWD=mode, FR_TC_DX=mode)
        r = subprocess.run([sys.executable, "-c", _PERSIST_SCRIPT], env=env, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        res[mode] = r.stdout.split()
    assert len(res["persistent"]) == 3
    assert res["persistent"] == res["tile"]


def test_tc_dw_from_kquad_slabs_bit_identical_to_transposed_copies():
    """The weight gradient with Zbar read straight from the k-quad adjoint
    slabs (default, tcw_dwq_kernel: BASE32B MN-major B operand, tensor-map
    TMA) equals the one from the row-quad-major Zbar^T copies (FR_TC_DWQ=0):
    same rows per K-step, pad rows zero, so losses and gradients are
    bit-identical -- ragged last tile, 3D (N block not a multiple of 32),
    steady, MSE."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for mode in ("1", "0"):
        env = dict(os.environ, FR_ROOT=root, FR_TC_DWQ=mode)
        r = subprocess.run([sys.executable, "-c", _PERSIST_SCRIPT], env=env, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        res[mode] = r.stdout.split()
    assert len(res["1"]) == 3
    assert res["1"] == res["0"]



@pytest.mark.parametrize("WP", [128, 160, 208])
def test_tma_kquad_view(WP):
    """The tensor-map TMA view of a k-quad slab buffer (csrc/tma.cuh, what the
    weight-gradient kernel loads with: one cp.async.bulk.tensor per operand
    and 32-row group) lands a group as the [quad][row][4] stage."""
    import torch

    from paper_2602_15883_b200 import _lib as X

    nt, nq = 3, WP // 4
    rng = np.random.default_rng(WP)
    src = rng.standard_normal((nt, nq, 128, 4)).astype(np.float32)
    dS = torch.from_numpy(src).cuda()
    for tile, g in ((2, 1), (0, 3)):
        d0 = torch.zeros(32 * WP, dtype=torch.float32, device="cuda")
        X.call("fr_debug_tma_kquad", dS.data_ptr(), d0.data_ptr(), WP, nt, tile, g, None)
        torch.cuda.synchronize()
        assert np.array_equal(d0.cpu().numpy().reshape(nq, 32, 4), src[tile, :, 32 * g:32 * g + 32, :])


def test_tc_adjoint_32_unit_steps_bit_identical_to_16():
    """The persistent adjoint's 32-unit epilogue steps (default where the
    buffers fit; the last step of an N block may be 16 units, e.g. the 3D
    208-unit case) compute exactly what 16-unit steps do (FR_TC_DX_CQ=4)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for mode in ("8", "4"):
        env = dict(os.environ, FR_ROOT=root, FR_TC_DX_CQ=mode)
        r = subprocess.run([sys.executable, "-c", _PERSIST_SCRIPT], env=env, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        res[mode] = r.stdout.split()
    assert len(res["8"]) == 3
    assert res["8"] == res["4"]


@pytest.mark.parametrize("width,tcw,wpad", [(72, 80, 128), (150, 160, 192), (200, 208, 256), (256, 256, 256),
                                            (300, 320, 320)])
def test_tc_tensor_width(width, tcw, wpad):
    """TF32 plans run on their own tensor width (hidden width rounded to the
    16-deep K chunk, to 32 above 256 units) while the parameter layout keeps
    its 64-unit padding; FP64 and W <= 64 plans have none."""
    from paper_2602_15883_b200 import engine
    from paper_2602_15883_b200.network import ExpertConfig

    cfg = ExpertConfig(3, 3, width, "sin", 3)
    info = engine.get_plan(cfg, "unsteady2d", 100.0, "float32", math="tf32").info
    assert (info.tc_width, info.width_pad) == (tcw, wpad)
    assert engine.get_plan(cfg, "unsteady2d", 100.0, "float64").info.tc_width == 0
    assert engine.get_plan(ExpertConfig(3, 3, 64, "tanh", 3), "unsteady2d", 100.0, "float32").info.tc_width == 0
