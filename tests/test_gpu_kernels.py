"""GPU parity of the fused jet-MLP kernels against the reference's fixtures.

Two builds of the same kernel templates are checked:
  * float64 (parity build): must agree with the reference's float64 tapes to
    1e-10 -- this isolates indexing / algorithm errors from rounding;
  * float32 (product path): the tolerances below are the stated FP32 bounds.
"""

import numpy as np
import pytest

from conftest import max_rel, rel_l2, report

pytestmark = pytest.mark.gpu

KINDS = {0: "steady2d", 1: "unsteady2d", 2: "unsteady3d"}
RE = {}

# stated FP32 tolerances (relative): jets (value, gradient and
# Laplacian streams, max-abs relative to the largest entry) / losses /
# gradients (norm-wise) -- measured errors are <= 1.1e-6 (profiles/r2_parity_errors.jsonl)
F32_JET = 1e-5
F32_LOSS = 1e-5
F32_GRAD = 1e-5
# stated TF32 tensor-core tolerances (wide FP32 experts, relative): one TF32
# rounding (2^-11) per product, accumulated in FP32 through the layer chain
TF32_LOSS = 5e-3
TF32_GRAD = 5e-3
WIDE_TAPES = (5, 6, 7)


def _case(golden, i):
    from paper_2602_15883_b200.network import ExpertConfig

    t = f"tape{i}"
    meta = golden[f"{t}/meta"]
    arch = [int(a) for a in golden[f"{t}/arch"]]
    act = "sin" if meta[2] else "tanh"
    cfg = ExpertConfig(arch[0], len(arch) - 2, arch[1], act, arch[-1])
    return t, cfg, KINDS[int(meta[0])], float(meta[1]), meta


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("i", range(8))
def test_jet_forward(golden, i, dtype):
    from paper_2602_15883_b200 import engine

    t, cfg, kind, re, _ = _case(golden, i)
    plan = engine.get_plan(cfg, kind, re, dtype, math="simt")
    y = engine.forward_jet(plan, golden[f"{t}/params"], golden[f"{t}/pts"])
    d = cfg.input_dim
    val, grad, lap = y[:, 0], np.transpose(y[:, 1 : 1 + d], (0, 2, 1)), np.transpose(y[:, 1 + d :], (0, 2, 1))
    tol = 1e-12 if dtype == "float64" else F32_JET
    v = engine.forward_values(plan, golden[f"{t}/params"], golden[f"{t}/pts"])
    e = dict(value=max_rel(val, golden[f"{t}/jet_value"]), grad=max_rel(grad, golden[f"{t}/jet_grad"]),
             lap=max_rel(lap, golden[f"{t}/jet_lap"]), predict=max_rel(v, golden[f"{t}/jet_value"]))
    report(f"jet/{t}/{dtype}", **e)
    assert e["value"] < tol and e["predict"] < tol
    assert e["grad"] < tol and e["lap"] < tol


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("i", range(8))
def test_pde_loss_and_gradient(golden, i, dtype):
    from paper_2602_15883_b200 import engine

    t, cfg, kind, re, meta = _case(golden, i)
    plan = engine.get_plan(cfg, kind, re, dtype, math="simt")
    sq, g = engine.pde_loss_grad(plan, golden[f"{t}/params"], golden[f"{t}/pts"], float(meta[3]))
    ref_sq = float(golden[f"{t}/sq_pde"])
    tol_l, tol_g = (1e-11, 1e-10) if dtype == "float64" else (F32_LOSS, F32_GRAD)
    e_l, e_g = abs(sq - ref_sq) / abs(ref_sq), rel_l2(g, golden[f"{t}/grad_pde"])
    report(f"pde/{t}/{dtype}", loss=e_l, grad=e_g)
    assert e_l <= tol_l, (sq, ref_sq)
    assert e_g < tol_g


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("i", range(8))
def test_mse_loss_and_gradient(golden, i, dtype):
    from paper_2602_15883_b200 import engine

    t, cfg, kind, re, meta = _case(golden, i)
    nv = cfg.output_dim - 1
    plan = engine.get_plan(cfg, kind, re, dtype, math="simt")
    su, sp, g = engine.mse_loss_grad(plan, golden[f"{t}/params"], golden[f"{t}/pts"], golden[f"{t}/tu"],
                                     golden[f"{t}/tp"], list(meta[6 : 6 + nv]), float(meta[4]), float(meta[5]))
    tol_l, tol_g = (1e-12, 1e-11) if dtype == "float64" else (F32_LOSS, F32_GRAD)
    e = dict(sq_u=abs(su - float(golden[f"{t}/sq_u"])) / abs(su), sq_p=abs(sp - float(golden[f"{t}/sq_p"])) / abs(sp),
             grad=rel_l2(g, golden[f"{t}/grad_mse"]))
    report(f"mse/{t}/{dtype}", **e)
    assert e["sq_u"] <= tol_l and e["sq_p"] <= tol_l
    assert e["grad"] < tol_g


def test_rerun_bit_identical(golden):
    """Fixed-order reductions: a rerun reproduces loss and gradient bit for bit
    (the reference's contract, tape.py:1-6 / test_tape.py:75-95)."""
    from paper_2602_15883_b200 import engine

    t, cfg, kind, re, meta = _case(golden, 4)
    plan = engine.get_plan(cfg, kind, re, "float32")
    pts = np.random.default_rng(0).uniform(-3, 3, (20000, 3))
    a = engine.pde_loss_grad(plan, golden[f"{t}/params"], pts, 1e-4)
    b = engine.pde_loss_grad(plan, golden[f"{t}/params"], pts, 1e-4)
    assert a[0] == b[0]
    assert np.array_equal(a[1], b[1])


def test_loss_is_additive_over_point_sets(golden):
    """Mini-batch invariance (objective.py:46-64): the PDE loss/gradient of a
    set equals the sum over any split of it."""
    from paper_2602_15883_b200 import engine

    t, cfg, kind, re, meta = _case(golden, 4)
    plan = engine.get_plan(cfg, kind, re, "float64")
    pts = np.random.default_rng(1).uniform(-3, 3, (3001, 3))
    sq, g = engine.pde_loss_grad(plan, golden[f"{t}/params"], pts, 1.0)
    sq1, g1 = engine.pde_loss_grad(plan, golden[f"{t}/params"], pts[:1234], 1.0)
    sq2, g2 = engine.pde_loss_grad(plan, golden[f"{t}/params"], pts[1234:], 1.0)
    assert abs(sq - (sq1 + sq2)) <= 1e-12 * sq
    assert rel_l2(g1 + g2, g) < 1e-12


@pytest.mark.parametrize("act", ["tanh", "sin"])
def test_f32_matches_oracle_at_cylinder_scale(act):
    """[3,64x4,3] on cylinder-box points (|x| up to 17.5): FP32 kernels vs the
    float64 oracle on 8192 collocation points."""
    from oracle import flowrec_oracle as O
    from paper_2602_15883_b200 import engine
    from paper_2602_15883_b200.network import ExpertConfig, init_params

    cfg = ExpertConfig(3, 4, 64, act, 3)
    p = init_params(cfg, 3).flat
    rng = np.random.default_rng(5)
    pts = np.column_stack([rng.uniform(0, 7.35, 8192), rng.uniform(-7.5, 17.5, 8192), rng.uniform(-8, 8, 8192)])
    coef = 5.0 / pts.shape[0]
    sq_ref, g_ref, _ = O.pde_loss_grad(p, cfg.arch, act, "unsteady2d", 100.0, pts, coef)
    plan = engine.get_plan(cfg, "unsteady2d", 100.0, "float32")
    sq, g = engine.pde_loss_grad(plan, p, pts, coef)
    report(f"cylinder_scale/{act}", loss=abs(sq - sq_ref) / sq_ref, grad=rel_l2(g, g_ref))
    assert abs(sq - sq_ref) <= F32_LOSS * sq_ref, (sq, sq_ref)
    assert rel_l2(g, g_ref) < F32_GRAD


@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("accumulate", [0, 1])
def test_reference_seam_jet_act(kind, accumulate):
    """fr_jet_act_forward/backward == the reference's _kernels semantics
    (numpy_backend.py:43-89), restated in the oracle's factor helper."""
    import torch

    from paper_2602_15883_b200 import _lib as X

    rng = np.random.default_rng(7)
    B, d, W = 33, 3, 12
    z = rng.normal(size=((1 + 2 * d) * B, W))
    s = np.zeros_like(z)
    aux = np.cos(z[:B]) if kind == 1 else None
    s[:B] = np.tanh(z[:B]) if kind == 0 else np.sin(z[:B])
    sbar = rng.normal(size=z.shape)
    zbar0 = rng.normal(size=z.shape)
    dev = torch.device("cuda")
    T = lambda a: torch.as_tensor(a, device=dev).contiguous()
    zt, st, sb, zb = T(z), T(s), T(sbar), T(zbar0)
    at = T(aux) if aux is not None else None
    d1 = torch.empty((B, W), dtype=torch.float64, device=dev)
    d2 = torch.empty_like(d1)
    X.call("fr_jet_act_forward", kind, X.ptr(zt), X.ptr(st), X.ptr(at), X.ptr(d1), X.ptr(d2), B, d, W,
           X.stream_ptr())
    X.call("fr_jet_act_backward", kind, X.ptr(zt), X.ptr(st), X.ptr(at), X.ptr(sb), X.ptr(zb), B, d, W,
           accumulate, X.stream_ptr())
    # numpy restatement
    sv = s[:B]
    if kind == 0:
        f1 = 1.0 - sv * sv
        f2 = -2.0 * (sv * f1)
        f3 = -2.0 * (f1 * f1 + sv * f2)
    else:
        f1, f2, f3 = aux, -sv, -aux
    s_ref = s.copy()
    acc = sbar[:B] * f1
    zb_ref = zbar0.copy() if accumulate else np.zeros_like(z)
    for j in range(d):
        g = slice((1 + j) * B, (2 + j) * B)
        l = slice((1 + d + j) * B, (2 + d + j) * B)
        s_ref[g] = f1 * z[g]
        s_ref[l] = f2 * z[g] * z[g] + f1 * z[l]
        acc = acc + (sbar[g] * (f2 * z[g]) + sbar[l] * (f3 * z[g] * z[g] + f2 * z[l]))
        tg = sbar[g] * f1 + (2.0 * f2) * z[g] * sbar[l]
        tl = sbar[l] * f1
        zb_ref[g] = zb_ref[g] + tg if accumulate else tg
        zb_ref[l] = zb_ref[l] + tl if accumulate else tl
    zb_ref[:B] = zb_ref[:B] + acc if accumulate else acc
    assert np.max(np.abs(st.cpu().numpy() - s_ref)) <= 1e-15
    assert np.max(np.abs(d1.cpu().numpy() - f1)) <= 1e-15
    assert max_rel(zb.cpu().numpy(), zb_ref) <= 1e-15


@pytest.mark.parametrize("i", WIDE_TAPES)
def test_tf32_pde_loss_and_gradient(golden, i):
    """Wide FP32 experts on the tcgen05 TF32 path (the default math for widths
    65..512) against the reference's float64 tapes, at the stated TF32 bound."""
    from paper_2602_15883_b200 import engine

    t, cfg, kind, re, meta = _case(golden, i)
    plan = engine.get_plan(cfg, kind, re, "float32", math="tf32")
    assert plan.info.math == 1
    sq, g = engine.pde_loss_grad(plan, golden[f"{t}/params"], golden[f"{t}/pts"], float(meta[3]))
    ref_sq = float(golden[f"{t}/sq_pde"])
    report(f"tf32_pde/{t}", loss=abs(sq - ref_sq) / abs(ref_sq), grad=rel_l2(g, golden[f"{t}/grad_pde"]))
    assert abs(sq - ref_sq) <= TF32_LOSS * abs(ref_sq), (sq, ref_sq)
    assert rel_l2(g, golden[f"{t}/grad_pde"]) < TF32_GRAD


@pytest.mark.parametrize("i", WIDE_TAPES)
def test_tf32_mse_loss_and_gradient(golden, i):
    from paper_2602_15883_b200 import engine

    t, cfg, kind, re, meta = _case(golden, i)
    nv = cfg.output_dim - 1
    plan = engine.get_plan(cfg, kind, re, "float32", math="tf32")
    su, sp, g = engine.mse_loss_grad(plan, golden[f"{t}/params"], golden[f"{t}/pts"], golden[f"{t}/tu"],
                                     golden[f"{t}/tp"], list(meta[6 : 6 + nv]), float(meta[4]), float(meta[5]))
    report(f"tf32_mse/{t}", sq_u=abs(su - float(golden[f"{t}/sq_u"])) / abs(su),
           sq_p=abs(sp - float(golden[f"{t}/sq_p"])) / abs(sp), grad=rel_l2(g, golden[f"{t}/grad_mse"]))
    assert abs(su - float(golden[f"{t}/sq_u"])) <= TF32_LOSS * abs(su)
    assert abs(sp - float(golden[f"{t}/sq_p"])) <= TF32_LOSS * abs(sp)
    assert rel_l2(g, golden[f"{t}/grad_mse"]) < TF32_GRAD


@pytest.mark.parametrize("width,layers,act,kind", [(128, 4, "tanh", "unsteady2d"), (150, 3, "sin", "unsteady2d"),
                                                   (96, 2, "tanh", "steady2d"), (200, 2, "sin", "unsteady3d"),
                                                   (300, 2, "tanh", "unsteady2d")])
def test_tf32_matches_oracle_at_cylinder_scale(width, layers, act, kind):
    """TF32 path on cylinder-box points, including a width > 256 (two N blocks),
    a 3D regime and the steady regime; plus bit-identical reruns."""
    from oracle import flowrec_oracle as O
    from paper_2602_15883_b200 import engine
    from paper_2602_15883_b200.network import ExpertConfig, init_params

    din = {"steady2d": 2, "unsteady2d": 3, "unsteady3d": 4}[kind]
    cfg = ExpertConfig(din, layers, width, act, din if din == 4 else 3)
    p = init_params(cfg, 3).flat
    rng = np.random.default_rng(5)
    n = 1000
    cols = [rng.uniform(0, 7.35, n), rng.uniform(-7.5, 17.5, n), rng.uniform(-8, 8, n), rng.uniform(-4, 4, n)]
    pts = np.column_stack(cols[:din] if din >= 3 else cols[1:3])
    coef = 5.0 / n
    sq_ref, g_ref, _ = O.pde_loss_grad(p, cfg.arch, act, kind, 100.0, pts, coef)
    plan = engine.get_plan(cfg, kind, 100.0, "float32", math="tf32")
    sq, g = engine.pde_loss_grad(plan, p, pts, coef)
    assert abs(sq - sq_ref) <= TF32_LOSS * sq_ref, (sq, sq_ref)
    assert rel_l2(g, g_ref) < TF32_GRAD
    sq2, g2 = engine.pde_loss_grad(plan, p, pts, coef)
    assert sq2 == sq and np.array_equal(g2, g)
    nv = cfg.output_dim - 1
    tu, tp = rng.standard_normal((n, nv)) * 0.1, rng.standard_normal(n) * 0.1
    su_ref, sp_ref, gm_ref = O.mse_loss_grad(p, cfg.arch, act, pts, tu, tp, [1.0] * nv, 2.0, 3.0)
    su, sp, gm = engine.mse_loss_grad(plan, p, pts, tu, tp, [1.0] * nv, 2.0, 3.0)
    assert abs(su - su_ref) <= TF32_LOSS * su_ref and abs(sp - sp_ref) <= TF32_LOSS * sp_ref
    assert rel_l2(gm, gm_ref) < TF32_GRAD


def test_math_mode_selection():
    """TF32 is the default for wide FP32 experts, split TF32 (tf32x3) for the
    FP32 W <= 64 fused epoch kernel; FP64, narrow-width and single-hidden-layer
    plans refuse the tensor-core modes."""
    from paper_2602_15883_b200 import _lib as X
    from paper_2602_15883_b200 import engine
    from paper_2602_15883_b200.network import ExpertConfig

    assert engine.Plan(ExpertConfig(3, 3, 150, "sin", 3), "unsteady2d", 100.0).info.math == 1
    assert engine.Plan(ExpertConfig(3, 4, 64, "tanh", 3), "unsteady2d", 100.0).info.math == 2
    assert engine.Plan(ExpertConfig(3, 4, 64, "tanh", 3), "unsteady2d", 100.0, math="simt").info.math == 0
    assert engine.Plan(ExpertConfig(3, 4, 64, "tanh", 3), "unsteady2d", 100.0, "float64").info.math == 0
    assert engine.Plan(ExpertConfig(3, 2, 16, "tanh", 3), "unsteady2d", 100.0).info.math == 0
    with pytest.raises(X.FlowrecError, match="split-TF32"):
        engine.Plan(ExpertConfig(3, 4, 64, "tanh", 3), "unsteady2d", 100.0, "float64", math="tf32x3")
    with pytest.raises(X.FlowrecError, match="split-TF32"):
        engine.Plan(ExpertConfig(3, 1, 64, "tanh", 3), "unsteady2d", 100.0, math="tf32x3")
    assert engine.Plan(ExpertConfig(3, 3, 150, "sin", 3), "unsteady2d", 100.0, "float64").info.math == 0
    with pytest.raises(X.FlowrecError, match="FP32"):
        engine.Plan(ExpertConfig(3, 3, 150, "sin", 3), "unsteady2d", 100.0, "float64", math="tf32")
    with pytest.raises(X.FlowrecError, match="65..512"):
        engine.Plan(ExpertConfig(3, 4, 64, "tanh", 3), "unsteady2d", 100.0, math="tf32")
    assert engine.Plan(ExpertConfig(3, 3, 150, "sin", 3), "unsteady2d", 100.0, math="simt").info.math == 0
