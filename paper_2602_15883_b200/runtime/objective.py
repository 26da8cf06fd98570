"""Per-rank composite objective on the GPU.

`DeviceObjective` is the resident form used by the training loop: datasets
live in HBM, one epoch is a fixed sequence of kernel launches (obs MSE -> PDE
-> ghost-spatial MSE -> ghost-temporal MSE -> fixed-order reductions), with no
host synchronisation, so it can be captured in a CUDA graph.

`LocalObjective` keeps the reference's API (pkg/src/flowrec/runtime/objective.py:67-199):
the same coefficients (lambda/N folded into each loss head, ghost-u normalised
over the union of ghost kinds, ghost-p per kind, :96-140), the same unweighted
`LossParts` and the same non-finite guard.  Mini-batching in the reference is
pure gradient accumulation (:46-64); the GPU processes every point of a
dataset in one persistent launch, so `batch_size` only validates.
"""

import ctypes

import numpy as np
import torch

from .. import _lib as X
from ..decomposition import DeviceUniform
from ..engine import get_plan, new_kparams, prepare, to_device
from ..physics import LossParts, compose_loss

SEG_OBS, SEG_PDE, SEG_GS, SEG_GT = 0, 1, 2, 3
KINDS = ("spatial", "temporal")


def check_finite(name, arr):
    """ValueError naming the first non-finite entry, as the reference's tape
    binding does (autodiff/tape.py:251-255).  The reference checks each
    shuffled mini-batch as it binds it, so its index is batch-relative; here
    every dataset is checked once, whole, at upload, and the index is the
    dataset row."""
    a = arr.detach().cpu().numpy() if torch.is_tensor(arr) else np.asarray(arr, dtype=np.float64)
    if not np.all(np.isfinite(a)):
        idx = tuple(int(i) for i in np.argwhere(~np.isfinite(a))[0])
        raise ValueError(f"non-finite value in {name} at index {idx}")


class DeviceObjective:
    """Resident datasets, workspaces and the per-epoch launch sequence."""

    def __init__(self, plan, regime, datasets, weights, max_ctas=0, ghost_derivative_weight=0.0,
                 target_alloc=None):
        """target_alloc(kind, name, shape) -> zeroed device tensor: where the
        ghost-target rows live (default: torch allocations; the peer-memory
        transport passes views of its IPC block so neighbours can store into
        them directly)."""
        self.plan = plan
        if target_alloc is None:
            target_alloc = lambda kind, name, shape: torch.zeros(shape, dtype=plan.tdtype, device=plan.device)  # noqa: E731
        self.target_alloc = target_alloc
        self.max_ctas = int(max_ctas)  # persistent-grid cap (SMs left free for the exchange transport)
        # opt-in C^1 interface extension (0: the reference's value-only coupling)
        self.gd_weight = float(ghost_derivative_weight)
        if self.gd_weight < 0:
            raise ValueError("ghost derivative weight must be non-negative")
        self.gd_launches = []
        self.regime = regime
        self.weights = weights
        dev, T = plan.device, plan.tdtype
        nv = regime.n_vel
        self.n_obs = datasets.n_obs
        self.n_colloc = datasets.n_colloc
        if self.n_obs == 0 and weights.obs > 0:
            raise ValueError("observation dataset is empty but the observation weight is positive")
        if self.n_colloc == 0:
            raise ValueError("collocation dataset is empty")
        vw = weights.velocity if weights.velocity is not None else (1.0,) * nv
        if len(vw) != nv:
            raise ValueError(f"need one velocity weight per component ({nv}), got {len(vw)}")
        self.vel_w = (ctypes.c_double * 4)(*(list(vw) + [1.0] * (4 - nv)))

        # the reference validates every input it binds (tape.py:298-313); the
        # datasets are resident here, so they are checked once
        device_colloc = isinstance(datasets.colloc_points, DeviceUniform)  # sampled on the GPU
        if not device_colloc:
            check_finite("input 'points'", datasets.colloc_points)  # (a device sample is finite by construction)
        if self.n_obs:
            check_finite("input 'points'", datasets.obs_points)
            check_finite("input 'target_u'", datasets.obs_velocity)
        for g in datasets.ghosts:
            check_finite("input 'points'", g.points)
        self.obs_pts = to_device(datasets.obs_points.reshape(-1, regime.n_inputs), T, dev)
        self.obs_vel = to_device(datasets.obs_velocity.reshape(-1, nv), T, dev)
        self.col_pts = (datasets.colloc_points.to_device("float32" if T == torch.float32 else "float64", dev)
                        if device_colloc else to_device(datasets.colloc_points, T, dev))

        # ghost sets grouped per kind in ghost-index order (objective.py:115-141)
        self.ghost_slices = {}  # ghost index -> (kind, offset, n)
        self.ghost = {}
        counts = {k: 0 for k in KINDS}
        per_kind = {k: [] for k in KINDS}
        for gi, g in enumerate(datasets.ghosts):
            n = g.points.shape[0]
            self.ghost_slices[gi] = (g.kind, counts[g.kind], n)
            counts[g.kind] += n
            per_kind[g.kind].append(g.points)
        self.n_ghost = counts
        self.n_ghost_total = counts["spatial"] + counts["temporal"]
        for kind in KINDS:
            if counts[kind] == 0:
                continue
            p_w = weights.ghost_p_space if kind == "spatial" else weights.ghost_p_time
            self.ghost[kind] = {
                "pts": to_device(np.vstack(per_kind[kind]), T, dev),
                "tu": target_alloc(kind, "tu", (counts[kind], nv)),
                "tp": target_alloc(kind, "tp", (counts[kind],)),
                "vel_coef": weights.ghost_u / self.n_ghost_total,
                "p_coef": p_w / counts[kind],
            }
        self.targets_set = {k: False for k in self.ghost}

        # one persistent launch per epoch covers every loss head (obs, PDE,
        # ghost-spatial, ghost-temporal); loss-partial blocks are packed in the
        # reference's dataset order so the optimiser kernel can reduce them
        self.set_order = []  # (segment id, kind or None) of the MSE sets, in launch order
        if self.n_obs:
            self.set_order.append((SEG_OBS, None))
        for kind, seg in (("spatial", SEG_GS), ("temporal", SEG_GT)):
            if counts[kind]:
                self.set_order.append((seg, kind))
        self.wide = plan.info.width_pad > 64
        if self.wide and self.gd_weight > 0:
            raise ValueError("the ghost-derivative extension needs hidden width <= 64")
        if self.wide:
            self._init_wide(plan, counts, weights, dev)
            return
        n_sets = (ctypes.c_longlong * 3)(*([self._set_n(sg, k) for sg, k in self.set_order] + [0] * 3)[:3])
        ws = X.Workspace()
        X.call("fr_epoch_workspace_capped", plan.h, self.n_colloc, n_sets, len(self.set_order), self.max_ctas,
               ctypes.byref(ws))
        self.ws = ws
        self.grid = ws.grid
        present = [SEG_OBS] if self.n_obs else []
        present += [SEG_PDE] + [sg for sg, k in self.set_order if k is not None]
        self.seg_rows = (ctypes.c_int * 4)(*[ws.grid if sg in present else 0 for sg in range(4)])
        self.total_rows = ws.grid
        npad = plan.info.np_pad
        self.lpart = torch.zeros(len(present) * ws.grid * 2, dtype=torch.float64, device=dev)
        block = {sg: self.lpart.data_ptr() + 8 * 2 * ws.grid * i for i, sg in enumerate(present)}
        self.lpart_blocks = (ctypes.c_void_p * 4)(block[SEG_PDE], *[block[sg] for sg, _ in self.set_order])
        self._init_ghost_derivatives(plan, ws.grid, npad, dev)
        self.scratch = torch.empty(max(ws.scratch_bytes, 16), dtype=torch.uint8, device=dev)
        self.sets = (X.MseSet * 3)()
        for i, (sg, kind) in enumerate(self.set_order):
            st = self.sets[i]
            if kind is None:
                st.pts, st.target_u, st.target_p = self.obs_pts.data_ptr(), self.obs_vel.data_ptr(), None
                st.n, st.vel_coef, st.p_coef = self.n_obs, weights.obs / self.n_obs, 0.0
            else:
                g = self.ghost[kind]
                st.pts, st.target_u, st.target_p = g["pts"].data_ptr(), g["tu"].data_ptr(), g["tp"].data_ptr()
                st.n, st.vel_coef, st.p_coef = counts[kind], g["vel_coef"], g["p_coef"]
        self.grad = torch.zeros(plan.info.n_params, dtype=torch.float64, device=dev)
        self.norm_parts = torch.zeros(X.lib().fr_reduce_grad_parts(plan.h), dtype=torch.float64, device=dev)
        self.sums = torch.zeros(8, dtype=torch.float64, device=dev)
        # ghost sets follow obs in set_order: the overlapped exchange gates them
        self.first_ghost_set = 1 if self.n_obs else 0
        # ungated launches of a capped workspace still launch the capped grid
        self.cap_gate = X.EpochGate(None, 0, self.max_ctas, None, 0) if self.max_ctas else None

    def _init_ghost_derivatives(self, plan, epoch_rows, npad, dev):
        """Extension buffers: per ghost kind the derivative targets (N, n_in,
        n_vel) and one FR_MODE_GJ launch whose gradient-partial rows follow the
        epoch kernel's in `gpart` (so fr_reduce_grad folds them in)."""
        self.gd_launches = []
        self.gpart = None
        rows = epoch_rows
        if self.gd_weight > 0 and self.ghost:
            n_in, nv = self.regime.n_inputs, self.regime.n_vel
            lrow = 0
            for kind, g in self.ghost.items():
                n = g["pts"].shape[0]
                g["tdu"] = self.target_alloc(kind, "tdu", (n, n_in, nv))
                ws = plan.workspace(X.MODE_GJ, n)
                self.gd_launches.append((kind, n, rows, lrow, ws))
                rows += ws.grid
                lrow += ws.loss_rows
            self.gd_lpart = torch.zeros(max(lrow, 1) * 2, dtype=torch.float64, device=dev)
            self.gd_rows = (ctypes.c_int * 1)(lrow)
            self.gd_sums = torch.zeros(2, dtype=torch.float64, device=dev)
            self.gd_scratch = torch.empty(max(max(w.scratch_bytes for *_, w in self.gd_launches), 16),
                                          dtype=torch.uint8, device=dev)
        self.total_rows = rows
        self.gpart = torch.empty(rows * npad, dtype=torch.float64, device=dev)

    def make_gate(self, gate_word, flags, timeout_s=600.0):
        """fr_epoch_gate for the overlapped exchange (ghost sets wait on
        gate_word for at most timeout_s: the reference's exchange_timeout,
        driver.py:150-181, 259)."""
        if self.wide:
            raise ValueError("the overlapped exchange needs the fused epoch kernel (hidden width <= 64)")
        if not timeout_s > 0:
            raise ValueError("exchange timeout must be positive")
        timeout_ms = min(int(round(float(timeout_s) * 1000.0)), 2**32 - 1)
        return X.EpochGate(gate_word.data_ptr(), self.first_ghost_set, self.max_ctas, flags.data_ptr(),
                           max(timeout_ms, 1))

    def _init_wide(self, plan, counts, weights, dev):
        """Wide experts (hidden width > 64): one layer-wise launch sequence per
        dataset, each writing its own block of gradient / loss partial rows."""
        npad = plan.info.np_pad
        launches = [(SEG_PDE, X.MODE_PDE, None)] + [(sg, X.MODE_MSE, k) for sg, k in self.set_order]
        launches.sort(key=lambda t: t[0])  # reference order: obs, pde, ghost-spatial, ghost-temporal
        self.wide_launches = []
        grow = lrow = 0
        scratch = 0
        seg_rows = [0, 0, 0, 0]
        for sg, mode, kind in launches:
            n = self.n_colloc if mode == X.MODE_PDE else self._set_n(sg, kind)
            ws = plan.workspace(mode, n)
            self.wide_launches.append((sg, mode, kind, n, grow, lrow))
            seg_rows[sg] = ws.loss_rows
            grow += ws.grid
            lrow += ws.loss_rows
            scratch = max(scratch, ws.scratch_bytes)
        self.total_rows = grow
        self.seg_rows = (ctypes.c_int * 4)(*seg_rows)
        self.gpart = torch.zeros(grow * npad, dtype=torch.float64, device=dev)
        self.lpart = torch.zeros(max(lrow, 1) * 2, dtype=torch.float64, device=dev)
        self.scratch = torch.empty(max(scratch, 16), dtype=torch.uint8, device=dev)
        self.grad = torch.zeros(plan.info.n_params, dtype=torch.float64, device=dev)
        self.norm_parts = torch.zeros(X.lib().fr_reduce_grad_parts(plan.h), dtype=torch.float64, device=dev)
        self.sums = torch.zeros(8, dtype=torch.float64, device=dev)

    def _enqueue_wide(self, kparams, st):
        plan, npad = self.plan, self.plan.info.np_pad
        kp, sc = X.ptr(kparams), X.ptr(self.scratch)
        for sg, mode, kind, n, grow, lrow in self.wide_launches:
            gp = self.gpart.data_ptr() + 8 * grow * npad
            lp = self.lpart.data_ptr() + 16 * lrow
            if mode == X.MODE_PDE:
                X.call("fr_pde_fwd_bwd", plan.h, kp, X.ptr(self.col_pts), n, self.weights.pde / self.n_colloc,
                       gp, lp, sc, st)
            elif kind is None:
                X.call("fr_mse_fwd_bwd", plan.h, kp, X.ptr(self.obs_pts), X.ptr(self.obs_vel), None, n,
                       self.vel_w, self.weights.obs / self.n_obs, 0.0, gp, lp, sc, st)
            else:
                g = self.ghost[kind]
                X.call("fr_mse_fwd_bwd", plan.h, kp, X.ptr(g["pts"]), X.ptr(g["tu"]), X.ptr(g["tp"]), n,
                       self.vel_w, g["vel_coef"], g["p_coef"], gp, lp, sc, st)

    def _set_n(self, seg, kind):
        return self.n_obs if kind is None else self.n_ghost[kind]

    # -- ghost targets --------------------------------------------------------
    def target_slice(self, gi):
        """Device views (u, p) of ghost set gi's target rows."""
        kind, off, n = self.ghost_slices[gi]
        g = self.ghost[kind]
        return g["tu"][off : off + n], g["tp"][off : off + n]

    def target_du_slice(self, gi):
        """Device view (n, n_in, n_vel) of ghost set gi's derivative targets
        (extension; None when ghost_derivative_weight == 0)."""
        kind, off, n = self.ghost_slices[gi]
        tdu = self.ghost[kind].get("tdu")
        return None if tdu is None else tdu[off : off + n]

    def ghost_derivative_loss(self):
        """Unweighted extension term of the last epoch run with sums:
        sum w_c (d u_c/d x_i - target)^2 / N_ghost_total (0 when disabled)."""
        if not self.gd_launches:
            return 0.0
        return float(self.gd_sums[0].item()) / self.n_ghost_total

    def set_ghost_targets(self, values):
        """values aligned with datasets.ghosts: (u (g, n_vel), p (g,)) arrays/tensors."""
        nv = self.regime.n_vel
        for gi, (kind, off, n) in self.ghost_slices.items():
            u, p = values[gi][0], values[gi][1]
            du = values[gi][2] if len(values[gi]) > 2 else None
            tdu = self.target_du_slice(gi)
            if tdu is not None:
                if du is None:
                    raise ValueError("ghost derivative coupling is on: messages must carry derivatives")
                du_t = du if torch.is_tensor(du) else torch.as_tensor(np.asarray(du, dtype=np.float64))
                if tuple(du_t.shape) != tuple(tdu.shape):
                    raise ValueError("ghost derivative target shape mismatch")
                tdu.copy_(du_t)
            u_t = u if torch.is_tensor(u) else torch.as_tensor(np.asarray(u, dtype=np.float64))
            p_t = p if torch.is_tensor(p) else torch.as_tensor(np.asarray(p, dtype=np.float64))
            if tuple(u_t.shape) != (n, nv) or tuple(p_t.shape) != (n,):
                raise ValueError("ghost target shape mismatch")
            # the reference binds the targets as tape inputs (tape.py:298-313)
            check_finite("input 'target_u'", u_t)
            check_finite("input 'target_p'", p_t)
            if du is not None:
                check_finite("input 'target_du'", du_t)
            tu, tp = self.target_slice(gi)
            tu.copy_(u_t)
            tp.copy_(p_t)
        for kind in self.ghost:
            self.targets_set[kind] = True

    def mark_targets_set(self):
        for kind in self.ghost:
            self.targets_set[kind] = True

    # -- launches -------------------------------------------------------------
    def loss_coeffs(self):
        w = self.weights
        return dict(lpart=self.lpart, seg_rows=list(self.seg_rows), n_obs=float(self.n_obs), n_colloc=float(self.n_colloc),
                    n_ghost_total=float(self.n_ghost_total), n_ghost_space=float(self.n_ghost["spatial"]),
                    n_ghost_time=float(self.n_ghost["temporal"]), w_obs=w.obs, w_pde=w.pde,
                    w_ghost_u=w.ghost_u, w_ghost_p_space=w.ghost_p_space, w_ghost_p_time=w.ghost_p_time)

    def enqueue(self, kparams, stream=None, with_sums=True, gate=None):
        """Launch the epoch's loss/gradient kernel and the fixed-order gradient
        reduction (no sync).  with_sums also reduces the loss partials into
        `sums` (the training loop leaves that to the optimiser kernel).  With a
        `gate` (make_gate) the ghost heads wait inside the kernel for the
        exchange instead of the launch waiting for it."""
        for kind in self.ghost:
            if not self.targets_set[kind]:
                raise RuntimeError(f"{kind} ghost targets were never set; run an exchange first")
        plan = self.plan
        st = X.stream_ptr(stream)
        if self.wide:
            self._enqueue_wide(kparams, st)
        else:
            X.call("fr_epoch_fwd_bwd_gated", plan.h, X.ptr(kparams), X.ptr(self.col_pts), self.n_colloc,
                   self.weights.pde / self.n_colloc, self.sets, len(self.set_order), self.vel_w,
                   X.ptr(self.gpart), self.lpart_blocks, X.ptr(self.scratch),
                   ctypes.byref(gate if gate is not None else self.cap_gate)
                   if (gate is not None or self.cap_gate is not None) else None, st)
        npad = plan.info.np_pad
        for kind, n, grow, lrow, _ in self.gd_launches:
            g = self.ghost[kind]
            X.call("fr_ghost_jet_fwd_bwd", plan.h, X.ptr(kparams), X.ptr(g["pts"]), X.ptr(g["tdu"]), n, self.vel_w,
                   self.gd_weight / self.n_ghost_total, self.gpart.data_ptr() + 8 * grow * npad,
                   self.gd_lpart.data_ptr() + 16 * lrow, X.ptr(self.gd_scratch), st)
        X.call("fr_reduce_grad", plan.h, X.ptr(self.gpart), self.total_rows, X.ptr(self.grad), 0,
               X.ptr(self.norm_parts), st)
        if with_sums and self.gd_launches:
            X.call("fr_reduce_loss", X.ptr(self.gd_lpart), self.gd_rows, 1, X.ptr(self.gd_sums), st)
        if with_sums:
            X.call("fr_reduce_loss", X.ptr(self.lpart), self.seg_rows, 4, X.ptr(self.sums), st)

    def parts_from_sums(self, sums):
        """Unweighted LossParts from the reduced sums (objective.py:183-191)."""
        s = [float(v) for v in sums]
        ng = self.n_ghost
        return LossParts(
            obs=s[0] / self.n_obs if self.n_obs else 0.0,
            pde=s[2] / self.n_colloc,
            ghost_u=(s[4] + s[6]) / self.n_ghost_total if self.n_ghost_total else 0.0,
            ghost_p_space=s[5] / ng["spatial"] if ng["spatial"] else 0.0,
            ghost_p_time=s[7] / ng["temporal"] if ng["temporal"] else 0.0,
        )


class LocalObjective:
    """Drop-in `LocalObjective(config, regime, datasets, weights, batch_size)`.

    `epoch(params, rng, grad_out=None) -> (LossParts, grad, total)` runs on the
    GPU; `params` is an ExpertParams (or flat f64 vector) and the returned grad
    is a float64 numpy vector in the reference's flat layout.
    """

    def __init__(self, config, regime, datasets, weights, batch_size, dtype="float32", math=None,
                 ghost_derivative_weight=0.0):
        if batch_size < 1:
            raise ValueError("batch size must be >= 1")
        self.config = config
        self.regime = regime
        self.weights = weights
        self.batch = int(batch_size)
        self.plan = get_plan(config, regime.kind, regime.reynolds, dtype, math)
        self.dev = DeviceObjective(self.plan, regime, datasets, weights,
                                   ghost_derivative_weight=ghost_derivative_weight)
        self.n_obs, self.n_colloc = self.dev.n_obs, self.dev.n_colloc
        self.n_ghost, self.n_ghost_total = self.dev.n_ghost, self.dev.n_ghost_total
        self.n_params = config.n_params
        self._kp = new_kparams(self.plan)

    def set_ghost_targets(self, values):
        self.dev.set_ghost_targets(values)

    def epoch(self, params, rng=None, grad_out=None):
        flat = params.flat if hasattr(params, "flat") else np.asarray(params, dtype=np.float64)
        flat_d = to_device(flat, torch.float64, self.plan.device)
        if not torch.isfinite(flat_d).all():
            # the reference reports the index inside the offending tape array
            # (W0, b0, W1, ... ; tape.py:314-326)
            bad = int(torch.nonzero(~torch.isfinite(flat_d))[0])
            off = 0
            for wshape, bshape in self.config.layer_shapes:
                for shp in (wshape, bshape):
                    size = int(np.prod(shp))
                    if bad < off + size:
                        idx = tuple(int(i) for i in np.unravel_index(bad - off, shp))
                        raise ValueError(f"non-finite value in parameter at index {idx}")
                    off += size
            raise ValueError("non-finite value in parameter")
        prepare(self.plan, flat_d, self._kp)
        self.dev.enqueue(self._kp)
        grad = self.dev.grad.cpu().numpy()
        parts = self.dev.parts_from_sums(self.dev.sums.cpu().numpy())
        if grad_out is None:
            grad_out = np.zeros(self.n_params)
        grad_out += grad
        total = compose_loss(parts, self.weights)
        if self.dev.gd_launches:  # opt-in C^1 extension term
            total += self.dev.gd_weight * self.dev.ghost_derivative_loss()
        if not np.isfinite(total):
            raise FloatingPointError(
                f"non-finite training loss: obs={parts.obs} pde={parts.pde} ghost_u={parts.ghost_u} "
                f"ghost_p_space={parts.ghost_p_space} ghost_p_time={parts.ghost_p_time}"
            )
        return parts, grad_out, total
