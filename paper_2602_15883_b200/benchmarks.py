"""Closed-form Navier-Stokes fields used to synthesise training inputs.

The reference ships these as its stand-ins for CFD data
(pkg/src/flowrec/benchmarks.py:62-259); the cylinder presets use Taylor-Green
(2D) and Beltrami (3D) on the paper's boxes (config.py:84-108).  Only the
(u, p) values are needed to build observation sets, so this module evaluates
values, with the same floating-point expression order as the reference so that
observation targets are bit-identical.
"""

import numpy as np

from .physics import FlowRegime


class _Field:
    name = "base"

    def __init__(self, regime, spatial_box, time_interval):
        self.regime = regime
        self.spatial_box = tuple((float(lo), float(hi)) for lo, hi in spatial_box)
        self.time_interval = None if time_interval is None else tuple(float(t) for t in time_interval)

    def _pts(self, points):
        pts = np.atleast_2d(np.asarray(points, dtype=np.float64))
        if pts.shape[1] != self.regime.n_inputs:
            raise ValueError(f"{self.name} expects {self.regime.n_inputs} coordinates, got {pts.shape[1]}")
        return pts

    def velocity_pressure(self, points):
        vals = self.values(self._pts(points))
        nv = self.regime.n_vel
        return vals[:, :nv], vals[:, nv]


class Kovasznay(_Field):
    """Steady 2D wake-like flow (x, y) -> (u, v, p)."""

    name = "kovasznay"

    def __init__(self, re=40.0, spatial_box=((0.0, 1.0), (0.0, 1.0))):
        super().__init__(FlowRegime("steady2d", re), spatial_box, None)
        self.lam = re / 2.0 - np.sqrt(re * re / 4.0 + 4.0 * np.pi * np.pi)

    def values(self, pts):
        x, y = pts[:, 0], pts[:, 1]
        b = 2.0 * np.pi
        ex = np.exp(self.lam * x)
        out = np.empty((pts.shape[0], 3))
        out[:, 0] = 1.0 - ex * np.cos(b * y)
        out[:, 1] = (self.lam / b) * ex * np.sin(b * y)
        out[:, 2] = 0.5 * (1.0 - np.exp(2.0 * self.lam * x))
        return out


class TaylorGreen2D(_Field):
    """Decaying 2D vortex array (t, x, y) -> (u, v, p)."""

    name = "taylor_green"

    def __init__(self, re=100.0, spatial_box=((0.0, 2.0 * np.pi), (0.0, 2.0 * np.pi)),
                 time_interval=(0.0, 1.0)):
        super().__init__(FlowRegime("unsteady2d", re), spatial_box, time_interval)

    def values(self, pts):
        t, x, y = pts[:, 0], pts[:, 1], pts[:, 2]
        decay = np.exp(-(2.0 / self.regime.reynolds) * t)
        out = np.empty((pts.shape[0], 3))
        out[:, 0] = -np.cos(x) * np.sin(y) * decay
        out[:, 1] = np.sin(x) * np.cos(y) * decay
        out[:, 2] = -0.25 * (np.cos(2.0 * x) + np.cos(2.0 * y)) * (decay * decay)
        return out


class Beltrami3D(_Field):
    """Ethier-Steinman flow (t, x, y, z) -> (u, v, w, p), decay exp(-d^2 t / Re)."""

    name = "beltrami"

    def __init__(self, a=1.0, d=1.0, re=1.0, spatial_box=((-1.0, 1.0), (-1.0, 1.0), (-1.0, 1.0)),
                 time_interval=(0.0, 1.0)):
        super().__init__(FlowRegime("unsteady3d", re), spatial_box, time_interval)
        self.a = float(a)
        self.d = float(d)

    def values(self, pts):
        a, d = self.a, self.d
        decay = np.exp(-((1.0 / self.regime.reynolds) * d * d) * pts[:, 0])
        xyz = (pts[:, 1], pts[:, 2], pts[:, 3])
        out = np.empty((pts.shape[0], 4))
        for i in range(3):
            xi, xj, xk = xyz[i], xyz[(i + 1) % 3], xyz[(i + 2) % 3]
            t1 = np.exp(a * xi) * np.sin(a * xj + d * xk)
            t2 = np.exp(a * xk) * np.cos(a * xi + d * xj)
            out[:, i] = -a * (t1 + t2) * decay
        out[:, 3] = -0.5 * (out[:, 0] ** 2 + out[:, 1] ** 2 + out[:, 2] ** 2)
        return out


_FIELDS = {"kovasznay": Kovasznay, "taylor_green": TaylorGreen2D, "beltrami": Beltrami3D}


def get_solution(name, **kwargs):
    if name not in _FIELDS:
        raise ValueError(f"unknown benchmark {name!r} (available: {sorted(_FIELDS)})")
    return _FIELDS[name](**kwargs)


def grid_points(solution, nx, n_snapshots=1):
    """Uniform grid in layout order: t outermost, then row-major space."""
    axes = [np.linspace(lo, hi, nx) for lo, hi in solution.spatial_box]
    if solution.time_interval is not None:
        if n_snapshots < 1:
            raise ValueError("need at least one snapshot")
        t0, t1 = solution.time_interval
        axes = [np.linspace(t0, t1, n_snapshots) if n_snapshots > 1 else np.array([t0])] + axes
    mesh = np.meshgrid(*axes, indexing="ij")
    return np.stack([m.ravel() for m in mesh], axis=1)
