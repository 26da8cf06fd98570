"""GPU: public prediction API and error contracts.

predict / predict_jet (network.py:142-177) reconstruct u/v/p fields and their
derivatives; checked against the float64 oracle on a cylinder-box grid for a
fused-width and a wide expert."""

import numpy as np
import pytest

from conftest import max_rel

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("width,act", [(64, "tanh"), (150, "sin")])
def test_predict_fields_on_grid(width, act):
    from oracle import flowrec_oracle as O
    from paper_2602_15883_b200 import benchmarks
    from paper_2602_15883_b200.network import ExpertConfig, init_params, predict, predict_jet

    sol = benchmarks.TaylorGreen2D(re=100.0, spatial_box=((-7.5, 17.5), (-8.0, 8.0)), time_interval=(0.0, 7.35))
    pts = benchmarks.grid_points(sol, 21, 5)
    cfg = ExpertConfig(3, 3, width, act, 3)
    params = init_params(cfg, 11)
    ref = O.value_forward(params.flat, cfg.arch, act, pts)
    for dtype, tol in (("float64", 1e-12), ("float32", 1e-5)):
        uvp = predict(params, pts, dtype=dtype)
        assert uvp.shape == (pts.shape[0], 3)
        assert max_rel(uvp, ref) < tol
    jet = predict_jet(params, pts[:500], dtype="float64")
    Y, _ = O.jet_forward(params.flat, cfg.arch, act, pts[:500])
    assert max_rel(jet.value, Y["v"]) < 1e-12
    assert max_rel(jet.grad, np.stack(Y["g"], axis=2)) < 1e-11
    assert max_rel(jet.lap, np.stack(Y["l"], axis=2)) < 1e-11
    one = predict(params, pts[3], dtype="float64")
    assert one.shape == (3,) and max_rel(one, ref[3]) < 1e-12


def test_plan_validation_errors():
    from paper_2602_15883_b200 import _lib as X
    from paper_2602_15883_b200.engine import Plan
    from paper_2602_15883_b200.network import ExpertConfig, init_params, predict

    with pytest.raises(X.FlowrecError, match="inputs"):
        Plan(ExpertConfig(2, 2, 16, "tanh", 3), "unsteady2d", 100.0)  # regime wants 3 inputs
    with pytest.raises(X.FlowrecError, match="outputs"):
        Plan(ExpertConfig(3, 2, 16, "tanh", 4), "unsteady2d", 100.0)
    with pytest.raises(ValueError, match="coordinates"):
        predict(init_params(ExpertConfig(3, 2, 16, "tanh", 3), 0), np.zeros((4, 2)))


def test_empty_point_sets_and_single_points():
    from paper_2602_15883_b200 import engine
    from paper_2602_15883_b200.network import ExpertConfig, init_params

    cfg = ExpertConfig(3, 2, 16, "tanh", 3)
    plan = engine.get_plan(cfg, "unsteady2d", 100.0, "float64")
    flat = init_params(cfg, 1).flat
    sq, g = engine.pde_loss_grad(plan, flat, np.zeros((0, 3)), 1.0)
    assert sq == 0.0 and not g.any()
    from oracle import flowrec_oracle as O

    p = np.array([[0.3, -1.0, 2.0]])
    sq1, g1 = engine.pde_loss_grad(plan, flat, p, 1.0)
    sq_ref, g_ref, _ = O.pde_loss_grad(flat, cfg.arch, "tanh", "unsteady2d", 100.0, p, 1.0)
    assert abs(sq1 - sq_ref) <= 1e-12 * sq_ref
    assert max_rel(g1, g_ref) < 1e-11


def test_no_cpu_fallback_library_is_the_compute_path():
    """The engine's numbers come from libflowrec_b200.so: the library's own
    launch counter moves when the API computes."""
    from paper_2602_15883_b200 import _lib as X
    from paper_2602_15883_b200.network import ExpertConfig, init_params, predict

    before = X.kernel_launches()
    predict(init_params(ExpertConfig(3, 2, 16, "tanh", 3), 0), np.zeros((10, 3)))
    assert X.kernel_launches() > before


@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_nccl_transport_self_exchange(dtype):
    """fr_nccl_init / fr_exchange on a one-rank communicator: a grouped round
    of sends to and receives from this rank moves every buffer (the C-ABI
    transport of SURVEY 8b; multi-rank rounds need more GPUs than this box)."""
    import ctypes as C

    import torch

    from paper_2602_15883_b200 import _lib as X

    uid = C.create_string_buffer(128)
    X.call("fr_nccl_get_unique_id", uid)
    comm = C.c_void_p()
    X.call("fr_nccl_init", uid, 1, 0, C.byref(comm))
    T = torch.float32 if dtype == "float32" else torch.float64
    src = [torch.arange(n, dtype=T, device="cuda") * (k + 1) for k, n in enumerate((1000, 3000, 7))]
    dst = [torch.zeros_like(t) for t in src]
    ptrs = lambda ts: (C.c_void_p * len(ts))(*[t.data_ptr() for t in ts])  # noqa: E731
    cnts = (C.c_longlong * 3)(*[t.numel() for t in src])
    peers = (C.c_int * 3)(0, 0, 0)
    X.call("fr_exchange", comm, 3, peers, ptrs(src), cnts, 3, peers, ptrs(dst), cnts,
           X.F32 if dtype == "float32" else X.F64, X.stream_ptr())
    torch.cuda.synchronize()
    for a, b in zip(src, dst):
        assert torch.equal(a, b)
    bad = (C.c_int * 1)(1)
    with pytest.raises(X.FlowrecError, match="peer 1"):
        X.call("fr_exchange", comm, 1, bad, ptrs(src[:1]), cnts, 0, None, None, None, X.F32, X.stream_ptr())
    X.call("fr_nccl_destroy", comm)
