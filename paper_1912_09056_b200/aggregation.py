"""Interface-respecting displacement aggregation and mortar-driven multiplier
aggregation (aggregation.py:1-322).

Integer work stays on the host but runs in C++
(`csrc/aggregate.cu`); the node graph itself is built on the device from the
level's K.  Results are bit-exact to the reference.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import DimensionError, SetupError
from .sparse import SparseMatrix

UNASSIGNED = -1
BODY_SLAVE = 0
BODY_MASTER = 1


class NodeGraph:
    """Undirected node graph with body / interface tags (aggregation.py:26-63)."""

    def __init__(self, num_nodes, indptr, indices, body_tag, interface_tag=None):
        self.num_nodes = int(num_nodes)
        self.indptr = np.asarray(indptr, dtype=np.int64)
        self.indices = np.asarray(indices, dtype=np.int64)
        self.body_tag = np.asarray(body_tag, dtype=np.int8)
        self.interface_tag = (np.zeros(num_nodes, dtype=np.int8) if interface_tag is None
                              else np.asarray(interface_tag, dtype=np.int8))

    def neighbors(self, i) -> np.ndarray:
        return self.indices[self.indptr[i]:self.indptr[i + 1]]

    @property
    def adjacency(self):
        return [self.neighbors(i) for i in range(self.num_nodes)]

    @staticmethod
    def from_edges(num_nodes, edges, body_tag=None, interface_tag=None) -> "NodeGraph":
        import scipy.sparse
        body = np.zeros(num_nodes, dtype=np.int8) if body_tag is None else body_tag
        e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
        e = e[e[:, 0] != e[:, 1]]
        G = scipy.sparse.csr_matrix((np.ones(2 * len(e)), (np.concatenate([e[:, 0], e[:, 1]]),
                                                           np.concatenate([e[:, 1], e[:, 0]]))),
                                    shape=(num_nodes, num_nodes))
        G.sum_duplicates()
        G.sort_indices()
        return NodeGraph(num_nodes, G.indptr, G.indices, body, interface_tag)


@dataclass
class Aggregation:
    node_to_agg: np.ndarray
    num_aggs: int
    agg_root: np.ndarray
    singleton_count: int = 0
    overlap_touch_count: int = 0

    def sizes(self) -> np.ndarray:
        return np.bincount(self.node_to_agg, minlength=self.num_aggs)

    def is_partition(self) -> bool:
        if np.any(self.node_to_agg == UNASSIGNED):
            return False
        return bool(np.all(self.sizes() > 0))


@dataclass
class LagrangeMap:
    """Row r of the mortar block <-> slave DOF slave_dofs[r] (aggregation.py:85-106)."""

    slave_dofs: np.ndarray
    row_node: np.ndarray
    lm_node_of_lm_dof: np.ndarray

    @property
    def num_lm_nodes(self) -> int:
        return int(self.lm_node_of_lm_dof.max()) + 1 if len(self.lm_node_of_lm_dof) else 0

    def slave_dof_to_lm_dof(self, dof) -> int:
        idx = np.searchsorted(self.slave_dofs, dof)
        if idx >= len(self.slave_dofs) or self.slave_dofs[idx] != dof:
            raise KeyError(f"DOF {dof} is not a slave interface DOF")
        return int(idx)


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def filtered_node_graph(K: SparseMatrix, dof_node, num_nodes, node_body, interface_tag=None,
                        eps_drop: float = 0.0) -> NodeGraph:
    """Node graph of K, cross-body and dropped entries removed
    (aggregation.py:127-145), built on the device."""
    dof_node = np.ascontiguousarray(dof_node, dtype=np.int64)
    if len(dof_node) != K.num_rows:
        raise DimensionError("dof->node map length does not match K")
    body = np.ascontiguousarray(node_body, dtype=np.int8)
    h, nnz = C.c_void_p(), C.c_int64()
    N.call("camg_node_graph", K.device, _p(dof_node), int(num_nodes), _p(body), float(eps_drop),
           C.byref(h), C.byref(nnz))
    try:
        indptr = np.empty(int(num_nodes) + 1, dtype=np.int64)
        indices = np.empty(max(int(nnz.value), 1), dtype=np.int64)
        N.call("camg_pattern_to_host", h, _p(indptr), _p(indices))
    finally:
        N.lib().camg_csr_destroy(h)
    return NodeGraph(num_nodes, indptr, indices[:int(nnz.value)], body, interface_tag)


def build_filtered_graph(K: SparseMatrix, dofs_per_node: int, dof_class=None, node_body=None,
                         eps_drop: float = 0.0) -> NodeGraph:
    if K.num_rows % dofs_per_node != 0:
        raise DimensionError("K rows are not divisible by dofs_per_node")
    num_nodes = K.num_rows // dofs_per_node
    dof_node = np.arange(K.num_rows, dtype=np.int64) // dofs_per_node
    if node_body is None:
        node_body = np.zeros(num_nodes, dtype=np.int8)
    return filtered_node_graph(K, dof_node, num_nodes, node_body, None, eps_drop)


def aggregate_greedy(graph: NodeGraph, min_agg_size: int = 1) -> Aggregation:
    """Three-phase greedy aggregation, lowest id wins ties (aggregation.py:186-258)."""
    if min_agg_size < 1:
        raise ValueError("min_agg_size must be >= 1")
    n = graph.num_nodes
    agg = np.empty(n, dtype=np.int64)
    roots = np.empty(max(n, 1), dtype=np.int64)
    na, singles = C.c_int64(), C.c_int64()
    ip = np.ascontiguousarray(graph.indptr, dtype=np.int64)
    ix = np.ascontiguousarray(graph.indices, dtype=np.int64)
    N.call("camg_aggregate_greedy", n, _p(ip), _p(ix), int(min_agg_size), _p(agg), C.byref(na), _p(roots),
           C.byref(singles))
    return Aggregation(agg, int(na.value), roots[:na.value].copy(), singleton_count=int(singles.value))


def aggregate_lagrange(disp_aggs: Aggregation, D: SparseMatrix, lmap: LagrangeMap) -> Aggregation:
    """Paper Alg. 1, first touch wins (aggregation.py:261-303)."""
    n_lm = lmap.num_lm_nodes
    lam = np.empty(max(n_lm, 1), dtype=np.int64)
    roots = np.empty(max(n_lm, 1), dtype=np.int64)
    na, ov = C.c_int64(), C.c_int64()
    rp = np.ascontiguousarray(D.row_offsets, dtype=np.int64)
    ci = np.ascontiguousarray(D.col_indices, dtype=np.int64)
    va = np.ascontiguousarray(D.values, dtype=np.float64)
    sd = np.ascontiguousarray(lmap.slave_dofs, dtype=np.int64)
    rn = np.ascontiguousarray(lmap.row_node, dtype=np.int64)
    lm = np.ascontiguousarray(lmap.lm_node_of_lm_dof, dtype=np.int64)
    dn = np.ascontiguousarray(disp_aggs.node_to_agg, dtype=np.int64)
    N.call("camg_aggregate_lagrange", _p(dn), D.num_rows, _p(rp), _p(ci), _p(va), _p(sd), _p(rn), _p(lm),
           len(lm), _p(lam), C.byref(na), _p(roots), C.byref(ov))
    return Aggregation(lam[:n_lm].copy(), int(na.value), roots[:na.value].copy(),
                       overlap_touch_count=int(ov.value))


def check_body_separation(aggs: Aggregation, body_tag) -> bool:
    body_tag = np.asarray(body_tag)
    lo = np.full(aggs.num_aggs, 127, dtype=np.int16)
    hi = np.full(aggs.num_aggs, -128, dtype=np.int16)
    np.minimum.at(lo, aggs.node_to_agg, body_tag)
    np.maximum.at(hi, aggs.node_to_agg, body_tag)
    return bool(np.all(lo == hi))


def dump_aggregation(aggs: Aggregation, body_tag) -> str:
    body_tag = np.asarray(body_tag)
    return "".join(f"{i} {a} {b}\n" for i, (a, b) in enumerate(zip(aggs.node_to_agg, body_tag)))
