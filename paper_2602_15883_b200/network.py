"""Per-subdomain local experts: configuration, flat parameters, init, prediction.

Host-side contracts mirror `flowrec.network` (pkg/src/flowrec/network.py:19-177):
the flat float64 layout W0 (fan_in x fan_out, row-major), b0, W1, b1, ... and the
seeded Glorot initialisation are reproduced bit-exactly (one-time host work).
`predict` / `predict_jet` run on the GPU through fr_value_fwd / fr_jet_fwd.
"""

from dataclasses import dataclass

import numpy as np

from .jet import Jet
from .physics import FlowRegime

ACTIVATIONS = ("tanh", "sin")


@dataclass(frozen=True)
class ExpertConfig:
    input_dim: int
    hidden_layers: int
    width: int
    activation: str
    output_dim: int
    omega0: float = 1.0

    def __post_init__(self):
        if self.input_dim < 1 or self.output_dim < 1:
            raise ValueError("input/output dims must be positive")
        if self.hidden_layers < 1:
            raise ValueError("need at least one hidden layer")
        if self.width < 1:
            raise ValueError("zero-width layer")
        if self.activation not in ACTIVATIONS:
            raise ValueError(
                f"unsupported activation {self.activation!r} (supported: {sorted(ACTIVATIONS)})"
            )
        if self.omega0 <= 0:
            raise ValueError("omega0 must be positive")

    @classmethod
    def for_regime(cls, regime: FlowRegime, hidden_layers, width, activation, omega0=1.0):
        return cls(regime.n_inputs, hidden_layers, width, activation, regime.n_outputs, omega0)

    @property
    def arch(self):
        return [self.input_dim] + [self.width] * self.hidden_layers + [self.output_dim]

    @property
    def layer_shapes(self):
        a = self.arch
        return [((fi, fo), (fo,)) for fi, fo in zip(a[:-1], a[1:])]

    @property
    def n_params(self):
        return sum(fi * fo + fo for (fi, fo), _ in self.layer_shapes)


class ExpertParams:
    """Flat float64 vector with (W, b) views sharing its memory (network.py:72-115)."""

    def __init__(self, config: ExpertConfig, flat, seed=None):
        flat = np.ascontiguousarray(flat, dtype=np.float64)
        if flat.shape != (config.n_params,):
            raise ValueError(f"flat vector has shape {flat.shape}, config needs ({config.n_params},)")
        self.config = config
        self.flat = flat
        self.seed = seed
        self.layers = []
        pos = 0
        for (fi, fo), _ in config.layer_shapes:
            w = flat[pos : pos + fi * fo].reshape(fi, fo)
            pos += fi * fo
            b = flat[pos : pos + fo]
            pos += fo
            self.layers.append((w, b))

    @property
    def n_params(self):
        return self.flat.size

    def __reduce__(self):
        return (ExpertParams, (self.config, self.flat, self.seed))

    def tape_arrays(self):
        return [a for wb in self.layers for a in wb]

    def copy(self):
        return ExpertParams(self.config, self.flat.copy(), seed=self.seed)


def init_params(config: ExpertConfig, seed: int) -> ExpertParams:
    """Glorot-uniform weights, zero biases; same PCG64 draws as network.py:118-139."""
    if seed < 0:
        raise ValueError("seed must be nonnegative")
    gen = np.random.Generator(np.random.PCG64(np.random.SeedSequence(int(seed))))
    chunks = []
    for li, ((fi, fo), _) in enumerate(config.layer_shapes):
        bound = np.sqrt(6.0 / (fi + fo))
        w = gen.uniform(-bound, bound, size=fi * fo)
        if li == 0 and config.activation == "sin" and config.omega0 != 1.0:
            w *= config.omega0
        chunks += [w, np.zeros(fo)]
    return ExpertParams(config, np.concatenate(chunks), seed=seed)


def _regime_for(config: ExpertConfig):
    kinds = {(2, 3): "steady2d", (3, 3): "unsteady2d", (4, 4): "unsteady3d"}
    kind = kinds.get((config.input_dim, config.output_dim))
    if kind is None:
        raise ValueError(
            f"no flow regime with {config.input_dim} inputs and {config.output_dim} outputs"
        )
    return kind


def predict(params: ExpertParams, points, dtype="float32") -> np.ndarray:
    """Value forward on the GPU (any batch size); (n, n_out) float64 result."""
    from .engine import get_plan, forward_values

    x = np.asarray(points, dtype=np.float64)
    squeeze = x.ndim == 1
    x = np.atleast_2d(x)
    cfg = params.config
    if x.shape[1] != cfg.input_dim:
        raise ValueError(f"points have {x.shape[1]} coordinates, expected {cfg.input_dim}")
    plan = get_plan(cfg, _regime_for(cfg), reynolds=1.0, dtype=dtype)
    out = forward_values(plan, params.flat, x)
    return out[0] if squeeze else out


def predict_jet(params: ExpertParams, points, dtype="float32") -> Jet:
    """Outputs with first and diagonal second input derivatives (GPU jet forward)."""
    from .engine import get_plan, forward_jet

    pts = np.atleast_2d(np.asarray(points, dtype=np.float64))
    cfg = params.config
    if pts.shape[1] != cfg.input_dim:
        raise ValueError(f"points have {pts.shape[1]} coordinates, expected {cfg.input_dim}")
    plan = get_plan(cfg, _regime_for(cfg), reynolds=1.0, dtype=dtype)
    y = forward_jet(plan, params.flat, pts)  # (n, 1 + 2d, n_out)
    d = cfg.input_dim
    value = y[:, 0, :].copy()
    grad = np.ascontiguousarray(np.transpose(y[:, 1 : 1 + d, :], (0, 2, 1)))
    lap = np.ascontiguousarray(np.transpose(y[:, 1 + d :, :], (0, 2, 1)))
    return Jet(value=value, grad=grad, lap=lap)
