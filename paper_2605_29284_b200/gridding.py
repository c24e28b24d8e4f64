"""Padded prediction grid and stencil lookup.

``PaddedGrid`` is host bookkeeping with the reference's fields and helpers
(gridding.py:38-111).  ``build_padded_grid`` runs the per-observation cell /
padding reduction on the GPU (rk_build_padded_grid; gridding.py:130-178) with
the exact IEEE arithmetic of the reference, so pads are bit-identical.
``neighborhood`` is the single-location lookup (gridding.py:181-205); the
per-observation stencils of a setup are produced inside the weights kernel.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import DomainError, InternalError

__all__ = ["PaddedGrid", "Neighborhood", "build_padded_grid", "neighborhood",
           "fill_distance", "NODE_SNAP_TOL"]

NODE_SNAP_TOL = 1.0e-9


@dataclass(frozen=True)
class PaddedGrid:
    origin: tuple
    spacing: tuple
    interior_dims: tuple
    pad: tuple      # (left, right, bottom, top)

    @property
    def total_dims(self):
        m1, m2 = self.interior_dims
        l, r, b, t = self.pad
        return m1 + l + r, m2 + b + t

    @property
    def padded_origin(self):
        return (self.origin[0] - self.pad[0] * self.spacing[0],
                self.origin[1] - self.pad[2] * self.spacing[1])

    @property
    def n_total(self):
        a, b = self.total_dims
        return a * b

    @property
    def n_interior(self):
        return self.interior_dims[0] * self.interior_dims[1]

    def to_index(self, ix, iy):
        return np.asarray(iy) * self.total_dims[0] + np.asarray(ix)

    def to_coords(self, index):
        index = np.asarray(index)
        m1t = self.total_dims[0]
        px0, py0 = self.padded_origin
        return px0 + (index % m1t) * self.spacing[0], py0 + (index // m1t) * self.spacing[1]

    def node_xs(self):
        return self.padded_origin[0] + self.spacing[0] * np.arange(self.total_dims[0])

    def node_ys(self):
        return self.padded_origin[1] + self.spacing[1] * np.arange(self.total_dims[1])

    def interior_view(self, field):
        l, _, b, _ = self.pad
        m1, m2 = self.interior_dims
        return field[b:b + m2, l:l + m1]

    def interior_xs(self):
        return self.origin[0] + self.spacing[0] * np.arange(self.interior_dims[0])

    def interior_ys(self):
        return self.origin[1] + self.spacing[1] * np.arange(self.interior_dims[1])

    def interior_nodes(self):
        gx, gy = np.meshgrid(self.interior_xs(), self.interior_ys())
        return np.column_stack([gx.ravel(), gy.ravel()])

    def native(self) -> N.RkGrid:
        g = N.RkGrid()
        g.x0, g.y0 = float(self.origin[0]), float(self.origin[1])
        g.hx, g.hy = float(self.spacing[0]), float(self.spacing[1])
        g.m1, g.m2 = int(self.interior_dims[0]), int(self.interior_dims[1])
        for k in range(4):
            g.pad[k] = int(self.pad[k])
        return g


@dataclass(frozen=True)
class Neighborhood:
    center_obs: int
    indices: np.ndarray
    local_offset: tuple


def build_padded_grid(domain, dims, L: int, obs_locs) -> PaddedGrid:
    """Interior grid over ``domain`` (inclusive ends), padded just enough for every
    observation's 2L x 2L block (reference gridding.py:130-178)."""
    dom = (N.C.c_double * 4)(*[float(v) for v in domain])
    obs = np.ascontiguousarray(np.asarray(obs_locs, dtype=float).reshape(-1, 2))
    g = N.RkGrid()
    N.call("rk_build_padded_grid", N.C.byref(dom), int(dims[0]), int(dims[1]), int(L),
           N.ptr(obs) if obs.shape[0] else None, obs.shape[0], N.C.byref(g))
    return PaddedGrid((g.x0, g.y0), (g.hx, g.hy), (int(g.m1), int(g.m2)), tuple(int(v) for v in g.pad))


def _cell(t: float) -> int:
    r = float(np.rint(t))
    return int(r) if abs(t - r) <= NODE_SNAP_TOL else int(math.floor(t))


def neighborhood(grid: PaddedGrid, obs_loc, L: int, center_obs: int = -1) -> Neighborhood:
    """Block whose central box holds ``obs_loc``; row-major over the block."""
    x, y = float(obs_loc[0]), float(obs_loc[1])
    px0, py0 = grid.padded_origin
    hx, hy = grid.spacing
    M1, M2 = grid.total_dims
    tx, ty = (x - px0) / hx, (y - py0) / hy
    if not (-NODE_SNAP_TOL <= tx <= M1 - 1 + NODE_SNAP_TOL
            and -NODE_SNAP_TOL <= ty <= M2 - 1 + NODE_SNAP_TOL):
        raise DomainError(f"location ({x}, {y}) outside padded grid coverage")
    cx, cy = _cell(tx), _cell(ty)
    xl, yl = cx - (L - 1), cy - (L - 1)
    if xl < 0 or yl < 0 or cx + L > M1 - 1 or cy + L > M2 - 1:
        raise InternalError(f"neighborhood of ({x}, {y}) exits the padded grid; padding contract violated")
    rows = np.arange(yl, yl + 2 * L)
    cols = np.arange(xl, xl + 2 * L)
    return Neighborhood(center_obs, (rows[:, None] * M1 + cols[None, :]).ravel(), (tx - cx, ty - cy))


def fill_distance(h: float) -> float:
    if not h > 0:
        raise DomainError(f"spacing must be positive, got {h}")
    return h * math.sqrt(2.0) / 2.0
