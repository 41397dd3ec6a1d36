"""Host-side view of the device-built index tree.

Mirrors reference tree.py (/root/reference/pkg/src/seriesearch/tree.py):
``Node`` (:92-179) and ``SplitPolicy`` (:50-89) with the same attribute names,
so code that walks a reference tree (persistence, tests, tooling) walks this
one.  The tree itself is built on the B200 (csrc/build.cu); these objects are
read back from the C ABI (ssb_index_node) after the build.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import DTYPE

MEAN = "mean"
SD = "sd"


@dataclass
class SplitPolicy:
    """How an internal node routes a series: value < threshold goes left."""

    segment_index: int
    attribute: str  # MEAN or SD
    split_point: int | None
    route_start: int
    route_end: int
    threshold: float
    gain: float = 0.0

    @property
    def is_vsplit(self) -> bool:
        return self.split_point is not None


class Node:
    def __init__(self, node_id: int, endpoints, parent: "Node | None" = None):
        self.node_id = node_id
        self.endpoints = np.asarray(endpoints, dtype=np.int64)
        m = len(self.endpoints)
        self.mu_min = np.full(m, np.inf, dtype=DTYPE)
        self.mu_max = np.full(m, -np.inf, dtype=DTYPE)
        self.sd_min = np.full(m, np.inf, dtype=DTYPE)
        self.sd_max = np.full(m, -np.inf, dtype=DTYPE)
        self.rho = 0
        self.is_leaf = True
        self.parent = parent
        self.left: Node | None = None
        self.right: Node | None = None
        self.policy: SplitPolicy | None = None
        self.file_position: tuple[int, int] | None = None
        self.oversize = False
        self.depth = 0
        self.inherited = 0
        self.split_set = 0

    @property
    def starts(self) -> np.ndarray:
        return np.concatenate([[0], self.endpoints[:-1]])

    @property
    def widths(self) -> np.ndarray:
        return self.endpoints - self.starts

    @property
    def num_segments(self) -> int:
        return len(self.endpoints)

    def segment_bounds(self, i: int) -> tuple[int, int]:
        start = 0 if i == 0 else int(self.endpoints[i - 1])
        return start, int(self.endpoints[i])

    def iter_leaves(self):
        stack = [self]
        while stack:
            node = stack.pop()
            if node.is_leaf:
                yield node
            else:
                stack.append(node.right)
                stack.append(node.left)

    def iter_nodes(self):
        stack = [self]
        while stack:
            node = stack.pop()
            yield node
            if not node.is_leaf:
                stack.append(node.right)
                stack.append(node.left)

    def __repr__(self):
        kind = "leaf" if self.is_leaf else "internal"
        return f"<Node {self.node_id} {kind} m={self.num_segments} rho={self.rho}>"


def tree_from_records(records) -> Node:
    """Rebuild the Node graph from ssb_node_t records (index order = node id)."""
    nodes = []
    for i, r in enumerate(records):
        m = r.m
        nd = Node(i, [r.endpoints[j] for j in range(m)])
        env = np.array([[r.envelope[j][q] for q in range(4)] for j in range(m)], dtype=DTYPE)
        nd.mu_min, nd.mu_max, nd.sd_min, nd.sd_max = (env[:, q].copy() for q in range(4))
        nd.rho = int(r.count)
        nd.is_leaf = bool(r.is_leaf)
        nd.oversize = bool(r.oversize)
        nd.inherited = int(getattr(r, "inherited", 0))  # members it was created with (parent's split set)
        nd.split_set = int(getattr(r, "split_set", 0))  # members its policy was chosen on
        nd.depth = int(r.depth)
        nd.file_position = (int(r.first), int(r.count))
        if not nd.is_leaf:
            nd.policy = SplitPolicy(
                segment_index=int(r.segment),
                attribute=MEAN if r.attribute == 0 else SD,
                split_point=None if r.split_point < 0 else int(r.split_point),
                route_start=int(r.route_start),
                route_end=int(r.route_end),
                threshold=float(r.threshold),
                gain=float(r.gain),
            )
        nodes.append(nd)
    for i, r in enumerate(records):
        if r.parent >= 0:
            nodes[i].parent = nodes[r.parent]
        if r.left >= 0:
            nodes[i].left = nodes[r.left]
            nodes[i].right = nodes[r.right]
    return nodes[0]
