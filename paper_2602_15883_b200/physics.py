"""Flow regimes, the Navier-Stokes term table, loss weights and composition.

Mirrors the reference's `flowrec.physics` data contracts
(pkg/src/flowrec/physics.py:17-93, :164-224).  The term table is what the
fused PDE kernel hard-codes per regime (csrc/jetmlp_kernel.cuh, residual head);
`residual_structure` is kept so callers and tests can inspect the formula.
"""

from dataclasses import dataclass

REGIME_KINDS = ("steady2d", "unsteady2d", "unsteady3d")


@dataclass(frozen=True)
class FlowRegime:
    """Dimensionality, steadiness and Reynolds number (physics.py:17-67)."""

    kind: str
    reynolds: float

    def __post_init__(self):
        if self.kind not in REGIME_KINDS:
            raise ValueError(f"unknown regime kind {self.kind!r} (use one of {REGIME_KINDS})")
        if not self.reynolds > 0:
            raise ValueError(f"Reynolds number must be positive, got {self.reynolds}")

    has_time = property(lambda self: self.kind != "steady2d")
    n_space = property(lambda self: 3 if self.kind == "unsteady3d" else 2)
    n_vel = property(lambda self: self.n_space)
    n_inputs = property(lambda self: self.n_space + int(self.has_time))
    n_outputs = property(lambda self: self.n_vel + 1)
    time_index = property(lambda self: 0 if self.has_time else None)
    p_channel = property(lambda self: self.n_vel)
    velocity_names = property(lambda self: ("u", "v", "w")[: self.n_vel])

    @property
    def space_indices(self):
        first = int(self.has_time)
        return tuple(range(first, first + self.n_space))


def residual_structure(regime: FlowRegime):
    """Momentum components then continuity (physics.py:70-93).

    linear entries (coef, "grad"|"lap", out_channel, in_index);
    conv entries (coef, vel_channel, out_channel, in_index) = coef * u_vel * d(out)/d(in).
    """
    inv_re = 1.0 / regime.reynolds
    sp = regime.space_indices
    p = regime.p_channel
    table = []
    for i in range(regime.n_vel):
        linear = [(1.0, "grad", i, regime.time_index)] if regime.has_time else []
        linear.append((1.0, "grad", p, sp[i]))
        linear += [(-inv_re, "lap", i, j) for j in sp]
        conv = [(1.0, k, i, sp[k]) for k in range(regime.n_vel)]
        table.append({"linear": linear, "conv": conv})
    table.append({"linear": [(1.0, "grad", k, sp[k]) for k in range(regime.n_vel)], "conv": []})
    return table


@dataclass(frozen=True)
class LossWeights:
    """Composite-objective weights (physics.py:164-197)."""

    obs: float
    pde: float
    ghost_u: float
    ghost_p_space: float
    ghost_p_time: float
    velocity: tuple = None

    def __post_init__(self):
        for name in ("obs", "pde", "ghost_u", "ghost_p_space", "ghost_p_time"):
            if getattr(self, name) < 0:
                raise ValueError(f"loss weight {name} must be nonnegative, got {getattr(self, name)}")
        if self.velocity is not None:
            vel = tuple(float(w) for w in self.velocity)
            if any(w < 0 for w in vel):
                raise ValueError("velocity component weights must be nonnegative")
            object.__setattr__(self, "velocity", vel)

    def as_master(self):
        """Anchor owner: spatial ghost-pressure weight switched off (one-way gauge)."""
        return LossWeights(self.obs, self.pde, self.ghost_u, 0.0, self.ghost_p_time, self.velocity)


@dataclass(frozen=True)
class LossParts:
    """Five unweighted loss components of one rank (physics.py:200-211)."""

    obs: float = 0.0
    pde: float = 0.0
    ghost_u: float = 0.0
    ghost_p_space: float = 0.0
    ghost_p_time: float = 0.0

    def astuple(self):
        return (self.obs, self.pde, self.ghost_u, self.ghost_p_space, self.ghost_p_time)


def compose_loss(parts, weights: LossWeights):
    """Weighted sum, left to right (physics.py:214-224)."""
    if not isinstance(parts, LossParts):
        parts = LossParts(*parts)
    return (
        weights.obs * parts.obs
        + weights.pde * parts.pde
        + weights.ghost_u * parts.ghost_u
        + weights.ghost_p_space * parts.ghost_p_space
        + weights.ghost_p_time * parts.ghost_p_time
    )
