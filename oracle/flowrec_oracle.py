"""CPU oracle for the training hot path -- TEST INFRASTRUCTURE ONLY.

A float64 NumPy restatement of the reference's per-rank training step
(arXiv 2602.15883, package `flowrec`, /root/reference/pkg/src/flowrec).  Only
`tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline leg may use
it, and only as the checker / CPU baseline; the product path never imports it.

Pinned against the reference itself: tests/golden/*.npz are produced by
tests/golden/make_golden.py, which runs the reference's own tapes, objective,
optimiser and serial driver in this container; tests/test_oracle.py checks
this module against every fixture to 1e-12.

What is restated (reference file:line):
  jet forward through the stacked-jet affine + activation chain
      autodiff/tape.py:22-124, _kernels/numpy_backend.py:23-89, builders.py:24-38
  NS residual term table                   physics.py:70-93, builders.py:51-64
  PDE / MSE losses and their reverse sweep builders.py:85-141, tape.py:335-371
  composite per-rank epoch                 runtime/objective.py:67-199
  Adam + clip + step-decay LR              runtime/optim.py:20-58
  ghost exchange + anchor normalisation    runtime/worker.py:24-46,170-228
  serial training loop                     runtime/driver.py:127-144
"""

import numpy as np

# ----------------------------------------------------------------------------
# network pieces
# ----------------------------------------------------------------------------


def unflatten(flat, arch):
    """flat W0 (fi x fo row-major), b0, W1, b1, ... -> [(W, b)] (network.py:72-115)."""
    layers, pos = [], 0
    for fi, fo in zip(arch[:-1], arch[1:]):
        w = flat[pos : pos + fi * fo].reshape(fi, fo)
        pos += fi * fo
        layers.append((w, flat[pos : pos + fo]))
        pos += fo
    assert pos == flat.size
    return layers


def _factors(act, z):
    """sigma, sigma', sigma'', sigma''' at z (numpy_backend.py:23-40)."""
    if act == "tanh":
        s = np.tanh(z)
        d1 = 1.0 - s * s
        d2 = -2.0 * s * d1
        d3 = -2.0 * (d1 * d1 + s * d2)
    elif act == "sin":
        s, c = np.sin(z), np.cos(z)
        d1, d2, d3 = c, -s, -c
    else:
        raise ValueError(act)
    return s, d1, d2, d3


def value_forward(flat, arch, act, x):
    """Plain forward (network.py:142-156)."""
    h = np.asarray(x, dtype=np.float64)
    layers = unflatten(np.asarray(flat, dtype=np.float64), arch)
    for w, b in layers[:-1]:
        h = _factors(act, h @ w + b)[0]
    w, b = layers[-1]
    return h @ w + b


def jet_forward(flat, arch, act, x, lap_inputs=None, value_only=False):
    """Forward jets.  Streams: value, d/dx_j (all inputs), d2/dx_j^2 for j in
    lap_inputs (default all); value_only keeps the value stream alone.
    Returns (Y, cache) with Y["v"], Y["g"][j], Y["l"][k] of shape (n, n_out)."""
    x = np.asarray(x, dtype=np.float64)
    n, d = x.shape
    if value_only:
        lap_inputs = []
    lap_inputs = list(range(d)) if lap_inputs is None else list(lap_inputs)
    layers = unflatten(np.asarray(flat, dtype=np.float64), arch)
    # input jets: value rows = points, grad block j = e_j, lap blocks = 0 (tape.py:426-436)
    H = {"v": x, "g": [] if value_only else [np.tile(np.eye(d)[j], (n, 1)) for j in range(d)],
         "l": [np.zeros((n, d)) for _ in lap_inputs]}
    cache = []
    for li, (w, b) in enumerate(layers):
        Z = {"v": H["v"] @ w + b, "g": [g @ w for g in H["g"]], "l": [l @ w for l in H["l"]]}
        if li == len(layers) - 1:
            cache.append((H, Z, None))
            return Z, cache
        s, d1, d2, _ = _factors(act, Z["v"])
        S = {"v": s, "g": [d1 * zg for zg in Z["g"]],
             "l": [d2 * Z["g"][j] * Z["g"][j] + d1 * zl for j, zl in zip(lap_inputs, Z["l"])]}
        cache.append((H, Z, S))
        H = S


def jet_backward(flat, arch, act, cache, Ybar, lap_inputs):
    """Reverse sweep of jet_forward given output adjoints Ybar (same structure
    as Y).  Returns the flat gradient (tape.py:22-124,335-371)."""
    layers = unflatten(np.asarray(flat, dtype=np.float64), arch)
    grads = [None] * len(layers)
    Zb = Ybar
    for li in range(len(layers) - 1, -1, -1):
        w, _ = layers[li]
        H, Z, S = cache[li]
        if li < len(layers) - 1:
            # activation backward (numpy_backend.py:58-89), Sb -> Zb
            Sb = Zb
            _, d1, d2, d3 = _factors(act, Z["v"])
            zv = Sb["v"] * d1
            zg = [sg * d1 for sg in Sb["g"]]
            for g_i, sg in enumerate(Sb["g"]):
                zv = zv + sg * (d2 * Z["g"][g_i])
            for k, j in enumerate(lap_inputs):
                sl = Sb["l"][k]
                zv = zv + sl * (d3 * Z["g"][j] * Z["g"][j] + d2 * Z["l"][k])
                zg[j] = zg[j] + 2.0 * d2 * Z["g"][j] * sl
            Zb = {"v": zv, "g": zg, "l": [sl * d1 for sl in Sb["l"]]}
        gw = H["v"].T @ Zb["v"]
        for h, zb in zip(H["g"], Zb["g"]):
            gw = gw + h.T @ zb
        for h, zb in zip(H["l"], Zb["l"]):
            gw = gw + h.T @ zb
        grads[li] = (gw, Zb["v"].sum(axis=0))
        if li > 0:
            Zb = {"v": Zb["v"] @ w.T, "g": [z @ w.T for z in Zb["g"]], "l": [z @ w.T for z in Zb["l"]]}
    return np.concatenate([np.concatenate([gw.ravel(), gb]) for gw, gb in grads])


# ----------------------------------------------------------------------------
# regime / residual
# ----------------------------------------------------------------------------

REGIMES = {  # kind -> (n_inputs, n_vel, has_time)
    "steady2d": (2, 2, False),
    "unsteady2d": (3, 2, True),
    "unsteady3d": (4, 3, True),
}


def residual_terms(kind, reynolds):
    """Term table of physics.py:70-93."""
    n_in, nv, has_t = REGIMES[kind]
    inv_re = 1.0 / reynolds
    sp = list(range(int(has_t), int(has_t) + nv))
    comps = []
    for i in range(nv):
        lin = ([(1.0, "grad", i, 0)] if has_t else []) + [(1.0, "grad", nv, sp[i])]
        lin += [(-inv_re, "lap", i, j) for j in sp]
        comps.append((lin, [(1.0, k, i, sp[k]) for k in range(nv)]))
    comps.append(([(1.0, "grad", k, sp[k]) for k in range(nv)], []))
    return comps


def pde_loss_grad(flat, arch, act, kind, reynolds, pts, coef):
    """(sum_n |r_n|^2, d(coef * sum |r|^2)/dtheta, residuals (n, nv+1))."""
    n_in, nv, has_t = REGIMES[kind]
    lap_inputs = list(range(int(has_t), n_in))
    Y, cache = jet_forward(flat, arch, act, pts, lap_inputs)
    lap_pos = {j: k for k, j in enumerate(lap_inputs)}

    def entry(kind_, c, j):
        if kind_ == "val":
            return Y["v"][:, c]
        if kind_ == "grad":
            return Y["g"][j][:, c]
        return Y["l"][lap_pos[j]][:, c]

    terms = residual_terms(kind, reynolds)
    R = np.zeros((pts.shape[0], len(terms)))
    for i, (lin, conv) in enumerate(terms):
        r = np.zeros(pts.shape[0])
        for cf, kd, c, j in lin:
            r = r + cf * entry(kd, c, j)
        for cf, a, b, j in conv:
            r = r + cf * (entry("val", a, None) * entry("grad", b, j))
        R[:, i] = r
    sq = float(np.sum(R * R))
    Rb = 2.0 * coef * R
    Yb = {"v": np.zeros_like(Y["v"]), "g": [np.zeros_like(g) for g in Y["g"]],
          "l": [np.zeros_like(l) for l in Y["l"]]}
    for i, (lin, conv) in enumerate(terms):
        rb = Rb[:, i]
        for cf, kd, c, j in lin:
            if kd == "grad":
                Yb["g"][j][:, c] += cf * rb
            else:
                Yb["l"][lap_pos[j]][:, c] += cf * rb
        for cf, a, b, j in conv:
            Yb["v"][:, a] += cf * rb * entry("grad", b, j)
            Yb["g"][j][:, b] += cf * rb * entry("val", a, None)
    return sq, jet_backward(flat, arch, act, cache, Yb, lap_inputs), R


def mse_loss_grad(flat, arch, act, pts, target_u, target_p, vel_w, vel_coef, p_coef):
    """(sq_u, sq_p, grad) of vel_coef*sum_c w_c|u_c - t_c|^2 + p_coef*|p - t_p|^2
    (builders.py:103-141); target_p None omits the pressure term."""
    pts = np.asarray(pts, dtype=np.float64)
    nv = target_u.shape[1]
    Y, cache = jet_forward(flat, arch, act, pts, value_only=True)
    y = Y["v"]
    w = np.ones(nv) if vel_w is None else np.asarray(vel_w, dtype=np.float64)
    du = y[:, :nv] - target_u
    sq_u = float(sum(w[c] * np.dot(du[:, c], du[:, c]) for c in range(nv)))
    yb = np.zeros_like(y)
    yb[:, :nv] = 2.0 * vel_coef * w * du
    sq_p = 0.0
    if target_p is not None:
        dp = y[:, nv] - target_p
        sq_p = float(np.dot(dp, dp))
        yb[:, nv] = 2.0 * p_coef * dp
    return sq_u, sq_p, jet_backward(flat, arch, act, cache, {"v": yb, "g": [], "l": []}, [])


def ghost_jet_loss_grad(flat, arch, act, pts, target_du, vel_w, coef):
    """Opt-in C^1 interface extension (NOT in the reference, whose ghost
    coupling matches values only, worker.py:179-197): (sq, grad) of
    coef * sum_n sum_i sum_c w_c (d u_c/d x_i - target_du[n, i, c])^2, first
    derivatives of the velocity w.r.t. every input, through the same jet
    forward / reverse sweep as the PDE head (tape.py:22-124)."""
    pts = np.asarray(pts, dtype=np.float64)
    n_in, nv = target_du.shape[1], target_du.shape[2]
    Y, cache = jet_forward(flat, arch, act, pts, [])
    w = np.ones(nv) if vel_w is None else np.asarray(vel_w, dtype=np.float64)
    sq = 0.0
    gb = []
    for i in range(n_in):
        d = Y["g"][i][:, :nv] - target_du[:, i, :]
        sq += float(sum(w[c] * np.dot(d[:, c], d[:, c]) for c in range(nv)))
        b = np.zeros_like(Y["g"][i])
        b[:, :nv] = 2.0 * coef * w * d
        gb.append(b)
    return sq, jet_backward(flat, arch, act, cache, {"v": np.zeros_like(Y["v"]), "g": gb, "l": []}, [])


# ----------------------------------------------------------------------------
# per-rank objective, optimiser, exchange, serial loop
# ----------------------------------------------------------------------------


def local_epoch(flat, arch, act, kind, reynolds, data, weights):
    """One composite epoch (objective.py:164-199).

    data: obs_pts, obs_vel, colloc, ghosts = [(kind, pts, tu, tp)] in ghost order.
    weights: dict obs, pde, ghost_u, ghost_p_space, ghost_p_time, velocity.
    Returns (parts tuple of 5, grad, total)."""
    vw = weights.get("velocity")
    grad = np.zeros(flat.size)
    n_obs = data["obs_pts"].shape[0]
    sq_obs = 0.0
    if n_obs:
        sq_obs, _, g = mse_loss_grad(flat, arch, act, data["obs_pts"], data["obs_vel"], None, vw,
                                     weights["obs"] / n_obs, None)
        grad += g
    n_col = data["colloc"].shape[0]
    sq_pde, g, _ = pde_loss_grad(flat, arch, act, kind, reynolds, data["colloc"], weights["pde"] / n_col)
    grad += g
    by_kind = {"spatial": [], "temporal": []}
    for gk, pts, tu, tp in data["ghosts"]:
        by_kind[gk].append((pts, tu, tp))
    counts = {k: sum(p.shape[0] for p, _, _ in v) for k, v in by_kind.items()}
    n_tot = counts["spatial"] + counts["temporal"]
    gh_u, gh_p = 0.0, {"spatial": 0.0, "temporal": 0.0}
    for k in ("spatial", "temporal"):
        if not counts[k]:
            continue
        pts = np.vstack([p for p, _, _ in by_kind[k]])
        tu = np.vstack([t for _, t, _ in by_kind[k]])
        tp = np.concatenate([t for _, _, t in by_kind[k]])
        pw = weights["ghost_p_space"] if k == "spatial" else weights["ghost_p_time"]
        su, sp, g = mse_loss_grad(flat, arch, act, pts, tu, tp, vw, weights["ghost_u"] / n_tot, pw / counts[k])
        grad += g
        gh_u += su
        gh_p[k] = sp
    parts = (sq_obs / n_obs if n_obs else 0.0, sq_pde / n_col, gh_u / n_tot if n_tot else 0.0,
             gh_p["spatial"] / counts["spatial"] if counts["spatial"] else 0.0,
             gh_p["temporal"] / counts["temporal"] if counts["temporal"] else 0.0)
    names = ("obs", "pde", "ghost_u", "ghost_p_space", "ghost_p_time")
    total = 0.0
    for nm, v in zip(names, parts):
        total = total + weights[nm] * v
    return parts, grad, total


def adam_update(params, grad, m, v, step, lr, beta1=0.9, beta2=0.999, eps=1e-8, clip_norm=None):
    """In place; returns (new step, pre-clip norm) (optim.py:20-49)."""
    norm = float(np.sqrt(np.dot(grad, grad)))
    if not np.isfinite(norm):
        raise ValueError("non-finite gradient norm")
    if clip_norm is not None and norm > clip_norm:
        grad *= clip_norm / norm
    t = step + 1
    m *= beta1
    m += (1.0 - beta1) * grad
    v *= beta2
    v += (1.0 - beta2) * grad * grad
    params -= lr * (m / (1.0 - beta1 ** t)) / (np.sqrt(v / (1.0 - beta2 ** t)) + eps)
    return t, norm


def train_serial(ranks, arch, act, kind, reynolds, epochs, lr_fn, comm_interval=1, clip_norm=None,
                 anchor=None):
    """Serial multi-rank loop (driver.py:127-144, worker.py:170-244).

    ranks: dict rank -> {flat, data (ghost targets filled by the exchange),
    weights, outgoing [(dest, ghost_index, pts)], normalize}.  Mutates flat.
    Returns {rank: history (epochs, 7)}."""
    n_in, nv, has_t = REGIMES[kind]
    order = sorted(ranks)
    state = {r: dict(m=np.zeros(ranks[r]["flat"].size), v=np.zeros(ranks[r]["flat"].size), step=0) for r in order}
    hist = {r: [] for r in order}
    for e in range(epochs):
        if e % comm_interval == 0:
            inbox = {r: [] for r in order}
            for r in order:
                R = ranks[r]
                for dest, gi, pts in R["outgoing"]:
                    y = value_forward(R["flat"], arch, act, pts)
                    p = y[:, nv]
                    if R["normalize"]:
                        anc = np.tile(np.asarray(anchor, dtype=np.float64), (pts.shape[0], 1))
                        if has_t:
                            anc = np.column_stack([pts[:, 0], anc])
                        p = p - value_forward(R["flat"], arch, act, anc)[:, nv]
                    inbox[dest].append((gi, y[:, :nv], p))
            for r in order:
                gh = ranks[r]["data"]["ghosts"]
                for gi, u, p in inbox[r]:
                    gk, pts, _, _ = gh[gi]
                    gh[gi] = (gk, pts, u, p)
        for r in order:
            R = ranks[r]
            lr = lr_fn(e)
            parts, grad, total = local_epoch(R["flat"], arch, act, kind, reynolds, R["data"], R["weights"])
            if not np.isfinite(total):
                raise FloatingPointError("non-finite training loss")
            st = state[r]
            st["step"], _ = adam_update(R["flat"], grad, st["m"], st["v"], st["step"], lr, clip_norm=clip_norm)
            hist[r].append((float(e),) + tuple(parts) + (lr,))
    return {r: np.array(h) for r, h in hist.items()}
