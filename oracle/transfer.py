"""Oracle: pointwise Schwarz projection Pi between non-matching structured hex8 meshes.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Pi "performs pointwise projection of the spatial DoFs in Omega_2 onto the boundary
partial_S Omega_1". For a destination point X and a source box:
    t_d = (X_d - lo_d)/h_d,  i_d = clamp(floor(t_d), 0, n_d - 1),  xi_d = t_d - i_d,
    require xi_d in [-1e-8, 1 + 1e-8]           (SURVEY c.1 step 9, reading R11)
    value = sum over the 8 cell corners b of  prod_d (xi_d if b_d = 1 else 1 - xi_d) * U(node_b)
i.e. the trilinear hex8 interpolant of the source field at X.
"""
from __future__ import annotations

import numpy as np

from .fem import Box


class OverlapError(ValueError):
    """A destination point lies outside the source box (overlap violation)."""


CORNERS = np.array([(di, dj, dk) for dk in (0, 1) for dj in (0, 1) for di in (0, 1)])


def locate(box: Box, X, tol=1e-8):
    """Cell index (n_p,3) and local coordinates xi in [0,1]^3 (n_p,3) of points X (n_p,3)."""
    X = np.atleast_2d(np.asarray(X, dtype=np.float64))
    t = (X - box.lo[None, :]) / box.h[None, :]
    cell = np.clip(np.floor(t), 0, np.asarray(box.nel) - 1).astype(np.int64)
    xi = t - cell
    if np.any(xi < -tol) or np.any(xi > 1 + tol):
        raise OverlapError("Schwarz node outside the source box")
    return cell, xi


def projector(box: Box, X):
    """Donor node ids (n_p, 8) and trilinear weights (n_p, 8) of Pi at points X."""
    cell, xi = locate(box, X)
    nodes = np.empty((len(cell), 8), dtype=np.int64)
    w = np.empty((len(cell), 8))
    for b, (di, dj, dk) in enumerate(CORNERS):
        nodes[:, b] = box.node_id(cell[:, 0] + di, cell[:, 1] + dj, cell[:, 2] + dk)
        w[:, b] = ((xi[:, 0] if di else 1 - xi[:, 0]) * (xi[:, 1] if dj else 1 - xi[:, 1])
                   * (xi[:, 2] if dk else 1 - xi[:, 2]))
    return nodes, w


def apply(nodes, w, values_at_nodes):
    """s[p] = sum_b w[p,b] U(nodes[p,b]); values_at_nodes maps (n_p,8) ids -> (..., n_p, 8, 3)."""
    U = values_at_nodes(nodes)
    return np.einsum("pb,...pbc->...pc", w, U)
