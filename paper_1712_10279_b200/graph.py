"""Channel graph setup for vector transport (host side, one-time).

The per-cell graph gradient/divergence run inside the CUDA sweep; this module
only builds the k x ell coefficient matrix D/c the kernels consume and the
spectral bound behind the step size nu.  Semantics follow the reference's
TransportGraph (S/graph.py:22-77), build_incidence (:96-102) and
lambda_max_graph (:126-134).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import DimensionMismatchError, ValidationError


def _is_connected(k, edges):
    nbrs = {v: set() for v in range(k)}
    for a, b in edges:
        nbrs[a].add(b)
        nbrs[b].add(a)
    seen, todo = {0}, [0]
    while todo:
        for v in nbrs[todo.pop()] - seen:
            seen.add(v)
            todo.append(v)
    return len(seen) == k


@dataclass(frozen=True)
class TransportGraph:
    """Connected weighted graph on k channels; edge e = (i, j), i < j,
    traversal cost c_e, orientation +-1."""

    k: int
    edges: tuple
    costs: np.ndarray
    orientations: np.ndarray | None = field(default=None)

    def __post_init__(self):
        if self.k < 1:
            raise ValidationError("graph needs at least one node")
        edges = tuple((int(a), int(b)) for a, b in self.edges)
        costs = np.asarray(self.costs, dtype=np.float64)
        if costs.shape != (len(edges),):
            raise DimensionMismatchError(f"{len(edges)} edges but {costs.shape} cost entries")
        if np.any(costs <= 0) or not np.all(np.isfinite(costs)):
            raise ValidationError("edge costs must be positive and finite")
        if len(set(edges)) != len(edges):
            raise ValidationError("duplicate edge")
        for a, b in edges:
            if a == b:
                raise ValidationError(f"self-loop at node {a}")
            if not 0 <= a < b < self.k:
                raise ValidationError(f"edge ({a}, {b}) must satisfy 0 <= i < j < k")
        orient = np.ones(len(edges)) if self.orientations is None else self.orientations
        orient = np.asarray(orient, dtype=np.float64)
        if orient.shape != (len(edges),) or not np.all(np.abs(orient) == 1):
            raise ValidationError("orientations must be +-1 per edge")
        if not _is_connected(self.k, edges):
            raise ValidationError("graph must be connected")
        object.__setattr__(self, "edges", edges)
        object.__setattr__(self, "costs", costs)
        object.__setattr__(self, "orientations", orient)

    @property
    def num_edges(self) -> int:
        return len(self.edges)

    @property
    def incidence(self) -> np.ndarray:
        D = np.zeros((self.k, self.num_edges))
        for e, (a, b) in enumerate(self.edges):
            D[a, e] = self.orientations[e]
            D[b, e] = -self.orientations[e]
        return D

    def coefficients(self) -> np.ndarray:
        """D / c, the k x ell matrix of the graph gradient x -> x @ (D/c)."""
        return self.incidence / self.costs


def lambda_max_graph(g: TransportGraph) -> float:
    """Largest eigenvalue of D diag(1/c^2) D^T."""
    D = g.incidence
    return float(np.linalg.eigvalsh((D / g.costs ** 2) @ D.T).max())


def triangle_graph(costs=(1.0, 1.0, 1.0)) -> TransportGraph:
    """RGB default: edges (0,1), (0,2), (1,2)."""
    return TransportGraph(3, [(0, 1), (0, 2), (1, 2)], costs)
