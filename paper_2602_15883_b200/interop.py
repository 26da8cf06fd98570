"""Drop-in glue for the reference package itself (`flowrec`).

Two integration levels:

1. Whole path: `train_reference_plan(plan)` takes a `flowrec` TrainingPlan
   (built by `flowrec.runtime.build_plan`, driver.py:71-121) and returns a
   `flowrec` TrainResult (driver.py:57-68), training on the GPU.  It is what
   the reference's `train(plan, backend="cuda")` dispatches to.  The
   reference's frozen dataclasses are converted field by field into this
   package's field-compatible ones (same class names, same fields).
2. The reference's native seam, `flowrec._kernels` (_kernels/__init__.py:
   22-68): `CudaKernels` implements `jet_act_forward` / `jet_act_backward` on
   the caller's HOST float64 arrays (the reference keeps its tape buffers in
   NumPy) through `fr_jet_act_forward/backward`, and `install_kernels_backend`
   teaches `flowrec._kernels._select` the name "cuda", so
   `flowrec._kernels.set_backend("cuda")` routes every `_ActJet` through the GPU.

Nothing here imports `flowrec` at module load; the caller passes its objects.
"""

import dataclasses

import numpy as np

from . import decomposition, network, physics
from .runtime import driver as _driver
from .runtime import worker as _worker

_ENGINE_CLASSES = {}
for _m in (decomposition, physics, network, _worker, _driver):
    for _name in dir(_m):
        _c = getattr(_m, _name)
        if isinstance(_c, type) and dataclasses.is_dataclass(_c):
            _ENGINE_CLASSES.setdefault(_name, _c)


def to_engine(obj):
    """Convert (recursively) reference dataclass instances into this
    package's classes of the same name; arrays and scalars pass through."""
    if dataclasses.is_dataclass(obj) and not isinstance(obj, type):
        name = type(obj).__name__
        cls = _ENGINE_CLASSES.get(name)
        if cls is None:
            raise TypeError(f"no engine counterpart for reference type {name}")
        if isinstance(obj, cls):
            return obj
        kw = {f.name: to_engine(getattr(obj, f.name)) for f in dataclasses.fields(obj) if f.init}
        return cls(**kw)
    if isinstance(obj, tuple):
        return tuple(to_engine(x) for x in obj)
    if isinstance(obj, list):
        return [to_engine(x) for x in obj]
    if isinstance(obj, dict):
        return {k: to_engine(v) for k, v in obj.items()}
    if isinstance(obj, frozenset):
        return frozenset(to_engine(x) for x in obj)
    return obj


def from_reference_plan(plan):
    """A flowrec TrainingPlan -> this package's TrainingPlan (same roles,
    effective weights, routes and parameter seeds: build_plan is re-run on the
    converted subdomains / datasets / configs, driver.py:71-121)."""
    subs = to_engine(tuple(plan.subdomains))
    datasets = {ws.rank: to_engine(ws.datasets) for ws in plan.worker_specs}
    ours = _driver.build_plan(subs, datasets, to_engine(plan.expert_config), to_engine(plan.train_config))
    for a, b in zip(ours.worker_specs, plan.worker_specs):
        if (a.rank, a.role, a.param_seed, a.normalize_outgoing) != (b.rank, b.role, b.param_seed, b.normalize_outgoing):
            raise ValueError(f"rank {b.rank}: converted plan disagrees with the reference's")
    return ours


def train_reference_plan(plan, exchange_timeout=600.0, dtype="float32", result_type=None, params_type=None):
    """Train a flowrec TrainingPlan on the GPU (every rank resident on the
    current device, CUDA-graph epochs) and return a flowrec TrainResult.

    result_type / params_type default to flowrec.runtime.driver.TrainResult /
    flowrec.network.ExpertParams (imported lazily from the caller's flowrec)."""
    if result_type is None or params_type is None:
        from flowrec.network import ExpertParams as params_type  # noqa: N813
        from flowrec.runtime.driver import TrainResult as result_type  # noqa: N813
    res = _driver.train(from_reference_plan(plan), backend="cuda", exchange_timeout=exchange_timeout, dtype=dtype)
    params = {r: params_type(plan.expert_config, np.array(p.flat), seed=p.seed) for r, p in res.params.items()}
    return result_type(params=params, history=res.history, epoch_times=res.epoch_times,
                       exchange_log=res.exchange_log, wall_time_s=res.wall_time_s)


class CudaKernels:
    """`flowrec._kernels` backend on the GPU for host float64 arrays.

    Same signatures and in-place semantics as _kernels/numpy_backend.py:43-89
    (value rows of `s` are set by the caller; derivative blocks written; the
    adjoint written or accumulated into `zbar`; d1/d2 filled with the
    activation factors, d3 is scratch).  An unknown kind raises ValueError as
    the numpy backend does (the Cython one silently uses sin)."""

    ACT_TANH, ACT_SIN = 0, 1

    def __init__(self):
        import torch

        from . import _lib as X
        from .engine import require_cuda

        self._torch, self._X = torch, X
        self.device = require_cuda()

    def _dev(self, a):
        return None if a is None else self._torch.from_numpy(np.ascontiguousarray(a)).to(self.device)

    def jet_act_forward(self, kind, z, s, aux, d1, d2, batch, n_inputs):
        if kind not in (self.ACT_TANH, self.ACT_SIN):
            raise ValueError(f"unknown activation kind {kind}")
        X = self._X
        zd, sd, ad = self._dev(z), self._dev(s), self._dev(aux if kind == self.ACT_SIN else None)
        d1d = self._torch.empty(d1.shape, dtype=self._torch.float64, device=self.device)
        d2d = self._torch.empty_like(d1d)
        X.call("fr_jet_act_forward", int(kind), X.ptr(zd), X.ptr(sd), X.ptr(ad), X.ptr(d1d), X.ptr(d2d),
               int(batch), int(n_inputs), int(z.shape[1]), X.stream_ptr())
        s[...] = sd.cpu().numpy()
        d1[...] = d1d.cpu().numpy()
        d2[...] = d2d.cpu().numpy()

    def jet_act_backward(self, kind, z, s, aux, sbar, zbar, d1, d2, d3, batch, n_inputs, accumulate):
        if kind not in (self.ACT_TANH, self.ACT_SIN):
            raise ValueError(f"unknown activation kind {kind}")
        X = self._X
        zd, sd, ad = self._dev(z), self._dev(s), self._dev(aux if kind == self.ACT_SIN else None)
        sbd, zbd = self._dev(sbar), self._dev(zbar)
        X.call("fr_jet_act_backward", int(kind), X.ptr(zd), X.ptr(sd), X.ptr(ad), X.ptr(sbd), X.ptr(zbd),
               int(batch), int(n_inputs), int(z.shape[1]), int(bool(accumulate)), X.stream_ptr())
        zbar[...] = zbd.cpu().numpy()


def install_kernels_backend(kernels_module):
    """Teach a `flowrec._kernels` module the backend name "cuda" (the one-line
    `_select` branch of INTEGRATION.md section 2); returns the backend object."""
    impl = CudaKernels()
    prev_select = kernels_module._select

    def _select(name):
        if name == "cuda":
            return impl, "cuda"
        return prev_select(name)

    kernels_module._select = _select
    return impl
