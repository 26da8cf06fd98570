"""Adam with global-norm clipping and the step-decay schedule (device).

Mirrors pkg/src/flowrec/runtime/optim.py:8-58.  The update runs in one fused
kernel (fr_adam_step): fixed-order norm reduction, finiteness check, optional
clip, bias-corrected moments in f64, and (on the training path) refresh of the
kernel copy of the parameters.  Learning rates and bias-correction factors are
evaluated on the host with Python float arithmetic, exactly as the reference.
"""

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from .. import _lib as X
from ..engine import adam_schedule, require_cuda


def lr_at(epoch, lr0, factor=1.0, interval=1):
    """lr0 * factor ** floor(epoch / interval) (optim.py:52-58)."""
    if epoch < 0:
        raise ValueError("epoch must be nonnegative")
    if interval < 1:
        raise ValueError("decay interval must be >= 1")
    return lr0 * factor ** (epoch // interval)


@dataclass
class AdamState:
    """First/second moments and step counter (numpy or device tensors)."""

    m: object
    v: object
    step: int = 0

    @classmethod
    def zeros(cls, n, device=None):
        if device is None:
            return cls(m=np.zeros(n), v=np.zeros(n))
        z = lambda: torch.zeros(n, dtype=torch.float64, device=device)
        return cls(m=z(), v=z())


def new_sync_counter(device):
    """Zero-initialised device int for the optimiser's last-block step update.
    It self-resets after every launch, but launches that may run concurrently
    (workers on different streams of one GPU) each need their own."""
    return torch.zeros(1, dtype=torch.int32, device=device)


def launch_adam(params, grad, m, v, step, sched, row_base, *, beta1=0.9, beta2=0.999, eps=1e-8,
                clip_norm=None, flags, grad_norm=None, plan=None, kparams=None, history=None,
                loss=None, norm_parts=None, stream=None, sync_counter=None):
    """Enqueue fr_adam_step on device tensors (graph-capturable).

    loss: None or dict(lpart=<tensor>, seg_rows=[4 ints], n_obs=..., w_obs=..., ...).
    sync_counter: this caller's counter (new_sync_counter); None allocates a
    fresh one, which a graph-captured or repeated caller must not rely on."""
    a = X.AdamArgs()
    a.n = params.numel()
    a.params, a.grad, a.m, a.v = (t.data_ptr() for t in (params, grad, m, v))
    a.step, a.sched, a.row_base = step.data_ptr(), sched.data_ptr(), int(row_base)
    a.beta1, a.beta2, a.eps = float(beta1), float(beta2), float(eps)
    # None -> NaN: the kernel's `norm > clip_norm` is then false, as the
    # reference's `clip_norm is not None and norm > clip_norm` (optim.py:26)
    a.clip_norm = float("nan") if clip_norm is None else float(clip_norm)
    if norm_parts is not None:
        a.norm_parts, a.n_norm_parts = norm_parts.data_ptr(), norm_parts.numel()
    a.flags = flags.data_ptr()
    a.grad_norm = None if grad_norm is None else grad_norm.data_ptr()
    a.kparams = None if kparams is None else kparams.data_ptr()
    a.history = None if history is None else history.data_ptr()
    if sync_counter is None:
        sync_counter = new_sync_counter(params.device)
    a.sync_counter = sync_counter.data_ptr()
    for k, val in (loss or {}).items():
        if k == "lpart":
            a.lpart = val.data_ptr()
        elif k == "seg_rows":
            a.seg_rows[:] = list(val)
        else:
            setattr(a, k, val)
    X.call("fr_adam_step", None if plan is None else plan.h, C.byref(a), X.stream_ptr(stream))


def clip_by_global_norm(grad, clip_norm):
    """Rescale grad in place to 2-norm <= clip_norm; returns the pre-clip norm
    (optim.py:20-28).  Runs the optimiser kernel's reduction on the device."""
    dev = require_cuda()
    host = not torch.is_tensor(grad)
    g = torch.as_tensor(grad).to(dev, torch.float64) if host else grad
    n = g.numel()
    red = torch.zeros(n, dtype=torch.float64, device=dev)
    # zero moments + lr 0: the kernel then only clips (params unchanged)
    sched = torch.tensor([0.0, 1.0, 1.0], dtype=torch.float64, device=dev)
    step = torch.zeros(1, dtype=torch.int64, device=dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    norm = torch.zeros(1, dtype=torch.float64, device=dev)
    launch_adam(red.clone(), g, red.clone(), red.clone(), step, sched, 0, clip_norm=clip_norm, flags=flags,
                grad_norm=norm)
    if int(flags.item()) & X.FLAG_NONFINITE_GRAD:
        raise ValueError("non-finite gradient norm")
    if host:
        grad[...] = g.cpu().numpy()
    return float(norm.item())


def adam_step(params, grad, state: AdamState, lr, beta1=0.9, beta2=0.999, eps=1e-8, clip_norm=None):
    """One in-place Adam update (optim.py:31-49) on the GPU.

    numpy inputs are copied to the device and back (drop-in use); float64 CUDA
    tensors are updated in place.  Raises ValueError on a non-finite gradient
    norm, like the reference.  Returns the pre-clip gradient norm.
    """
    dev = require_cuda()
    dev_t = lambda a: a if torch.is_tensor(a) else torch.as_tensor(a).to(dev, torch.float64)
    p_d, g_d, m_d, v_d = (dev_t(a) for a in (params, grad, state.m, state.v))
    if p_d.shape != g_d.shape or p_d.shape != m_d.shape:
        raise ValueError("parameter/gradient/state shape mismatch")
    t = state.step
    sched = torch.tensor(adam_schedule(1, lambda e: lr, beta1, beta2, start_step=t)[0],
                         dtype=torch.float64, device=dev)
    step_d = torch.tensor([t], dtype=torch.int64, device=dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    norm = torch.zeros(1, dtype=torch.float64, device=dev)
    launch_adam(p_d, g_d, m_d, v_d, step_d, sched, t, beta1=beta1, beta2=beta2, eps=eps, clip_norm=clip_norm,
                flags=flags, grad_norm=norm)
    if int(flags.item()) & X.FLAG_NONFINITE_GRAD:
        raise ValueError("non-finite gradient norm")
    state.step = t + 1
    for host, dev_v in ((params, p_d), (grad, g_d), (state.m, m_d), (state.v, v_d)):
        if not torch.is_tensor(host):
            host[...] = dev_v.cpu().numpy()
    return float(norm.item())
