"""Device-resident engine objects over the C ABI (plans, buffers, launches).

PyTorch is used only for device memory, streams and graphs; every arithmetic
step on the training path is one of the library's sm_100a kernels.
"""

import ctypes as C
import threading

import numpy as np
import torch

from . import _lib as X

_DTYPES = {"float32": X.F32, "f32": X.F32, "float64": X.F64, "f64": X.F64,
           torch.float32: X.F32, torch.float64: X.F64}
TORCH_DTYPE = {X.F32: torch.float32, X.F64: torch.float64}


def dtype_code(dtype):
    try:
        return _DTYPES[dtype]
    except KeyError:
        raise ValueError(f"unsupported compute dtype {dtype!r} (float32 or float64)") from None


def require_cuda():
    if not torch.cuda.is_available():
        raise X.FlowrecError("a CUDA device is required (the engine has no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


MATH_CODES = {"simt": 0, "tf32": 1, "tf32x3": 2}


class Plan:
    """A validated (architecture, activation, regime, dtype) for the kernels."""

    def __init__(self, config, regime_kind, reynolds, dtype="float32", math=None):
        """`math`: None keeps the library default (TF32 tensor cores for FP32
        experts wider than 64 units, FP32 SIMT otherwise); "simt" / "tf32"
        force the contraction math of the PDE / MSE training kernels."""
        self.device = require_cuda()
        self.config = config
        self.regime_kind = regime_kind
        self.code = dtype_code(dtype)
        self.tdtype = TORCH_DTYPE[self.code]
        arch = list(config.arch)
        carr = (C.c_int * len(arch))(*arch)
        h = C.c_void_p()
        X.call("fr_plan_create", carr, len(arch), X.ACT_CODES[config.activation],
               X.REGIME_CODES[regime_kind], 1.0 / float(reynolds), self.code, C.byref(h))
        self.h = h
        if math is not None:
            if math not in MATH_CODES:
                raise ValueError(f"unknown math {math!r}; expected one of {sorted(MATH_CODES)}")
            X.call("fr_plan_set_math", h, MATH_CODES[math])
        info = X.PlanInfo()
        X.call("fr_plan_get_info", h, C.byref(info))
        self.info = info

    def workspace(self, mode, n):
        ws = X.Workspace()
        X.call("fr_plan_workspace", self.h, mode, int(n), C.byref(ws))
        return ws

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            try:
                X.lib().fr_plan_destroy(h)
            except Exception:
                pass
            self.h = None


_plans = {}
_plans_lock = threading.Lock()


def get_plan(config, regime_kind, reynolds, dtype="float32", math=None):
    key = (config, regime_kind, float(reynolds), dtype_code(dtype), math, torch.cuda.current_device())
    with _plans_lock:
        p = _plans.get(key)
        if p is None:
            p = Plan(config, regime_kind, reynolds, dtype, math)
            _plans[key] = p
        return p


def to_device(arr, dtype, device):
    return torch.as_tensor(np.ascontiguousarray(arr)).to(device=device, dtype=dtype).contiguous()


def prepare(plan, flat_d, kparams, stream=None):
    """f64 flat params (device) -> padded kernel params (+ transposes)."""
    X.call("fr_prepare_params", plan.h, X.ptr(flat_d), X.ptr(kparams), X.stream_ptr(stream))


def new_kparams(plan):
    return torch.empty(plan.info.kp_elems, dtype=plan.tdtype, device=plan.device)


def _kparams_for(plan, flat):
    flat_d = flat if torch.is_tensor(flat) else to_device(flat, torch.float64, plan.device)
    kp = new_kparams(plan)
    prepare(plan, flat_d, kp)
    return kp


def launch_value(plan, kparams, pts_d, out_d, stream=None):
    n = pts_d.shape[0]
    X.call("fr_value_fwd", plan.h, X.ptr(kparams), X.ptr(pts_d), n, X.ptr(out_d), X.stream_ptr(stream))


def forward_values(plan, flat, points):
    """(n, n_out) float64 numpy values of the network at `points`."""
    kp = _kparams_for(plan, flat)
    pts = to_device(np.atleast_2d(points), plan.tdtype, plan.device)
    out = torch.empty((pts.shape[0], plan.info.n_out), dtype=plan.tdtype, device=plan.device)
    launch_value(plan, kp, pts, out)
    return out.double().cpu().numpy()


def forward_jet(plan, flat, points):
    """(n, 1 + 2d, n_out) float64 numpy: value, d/dx_j, d2/dx_j^2 blocks."""
    kp = _kparams_for(plan, flat)
    pts = to_device(np.atleast_2d(points), plan.tdtype, plan.device)
    s = 1 + 2 * plan.info.n_in
    out = torch.empty((pts.shape[0], s, plan.info.n_out), dtype=plan.tdtype, device=plan.device)
    X.call("fr_jet_fwd", plan.h, X.ptr(kp), X.ptr(pts), pts.shape[0], X.ptr(out), X.stream_ptr())
    return out.double().cpu().numpy()


def adam_schedule(epochs, lr_fn, beta1=0.9, beta2=0.999, start_step=0):
    """Rows {lr, 1 - beta1^t, 1 - beta2^t} for t = start_step+1 .. start_step+epochs,
    evaluated with the reference's Python float arithmetic (optim.py:40-58)."""
    rows = np.empty((epochs, 3))
    for i in range(epochs):
        t = start_step + i + 1
        rows[i] = (lr_fn(start_step + i), 1.0 - beta1 ** t, 1.0 - beta2 ** t)
    return rows


def _train_call(plan, mode, n, launch):
    ws = plan.workspace(mode, n)
    dev = plan.device
    gpart = torch.empty(max(ws.gpart_elems, 1), dtype=torch.float64, device=dev)
    lpart = torch.empty(max(ws.lpart_elems, 2), dtype=torch.float64, device=dev)
    scratch = torch.empty(max(ws.scratch_bytes, 16), dtype=torch.uint8, device=dev)
    launch(gpart, lpart, scratch)
    grad = torch.zeros(plan.info.n_params, dtype=torch.float64, device=dev)
    X.call("fr_reduce_grad", plan.h, X.ptr(gpart), ws.grid, X.ptr(grad), 0, None, X.stream_ptr())
    sums = torch.zeros(2, dtype=torch.float64, device=dev)
    rows = (C.c_int * 1)(ws.loss_rows)
    X.call("fr_reduce_loss", X.ptr(lpart), rows, 1, X.ptr(sums), X.stream_ptr())
    s = sums.cpu().numpy()
    return float(s[0]), float(s[1]), grad.cpu().numpy()


def pde_loss_grad(plan, flat, points, coef):
    """(sum_n |r_n|^2, gradient of coef * sum_n |r_n|^2) for one point set."""
    kp = _kparams_for(plan, flat)
    pts = to_device(np.atleast_2d(points), plan.tdtype, plan.device)
    n = pts.shape[0]

    def launch(gp, lp, sc):
        X.call("fr_pde_fwd_bwd", plan.h, X.ptr(kp), X.ptr(pts), n, float(coef), X.ptr(gp), X.ptr(lp),
               X.ptr(sc), X.stream_ptr())

    sq, _, g = _train_call(plan, X.MODE_PDE, n, launch)
    return sq, g


def ghost_jet_loss_grad(plan, flat, points, target_du, vel_w, coef):
    """(sq, gradient of coef * sq) of the opt-in ghost-derivative head:
    sq = sum_n sum_i sum_c w_c (d u_c / d x_i - target_du[n, i, c])^2."""
    kp = _kparams_for(plan, flat)
    pts = to_device(np.atleast_2d(points), plan.tdtype, plan.device)
    td = to_device(target_du, plan.tdtype, plan.device)
    n = pts.shape[0]
    vw = (C.c_double * 4)(*(list(vel_w) + [1.0] * (4 - len(vel_w))))

    def launch(gp, lp, sc):
        X.call("fr_ghost_jet_fwd_bwd", plan.h, X.ptr(kp), X.ptr(pts), X.ptr(td), n, vw, float(coef), X.ptr(gp),
               X.ptr(lp), X.ptr(sc), X.stream_ptr())

    sq, _, g = _train_call(plan, X.MODE_GJ, n, launch)
    return sq, g


def mse_loss_grad(plan, flat, points, target_u, target_p, vel_w, vel_coef, p_coef):
    """(sq_u, sq_p, gradient) of the MSE head; target_p None omits the p term."""
    kp = _kparams_for(plan, flat)
    pts = to_device(np.atleast_2d(points), plan.tdtype, plan.device)
    tu = to_device(target_u, plan.tdtype, plan.device)
    tp = None if target_p is None else to_device(target_p, plan.tdtype, plan.device)
    n = pts.shape[0]
    vw = (C.c_double * 4)(*(list(vel_w) + [1.0] * (4 - len(vel_w))))

    def launch(gp, lp, sc):
        X.call("fr_mse_fwd_bwd", plan.h, X.ptr(kp), X.ptr(pts), X.ptr(tu), X.ptr(tp), n, vw, float(vel_coef),
               float(p_coef), X.ptr(gp), X.ptr(lp), X.ptr(sc), X.stream_ptr())

    return _train_call(plan, X.MODE_MSE, n, launch)
