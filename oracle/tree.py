"""Adaptive quadtree (oracle; test infrastructure).

P:87-89 (index sets I_{l;i}), P:202 (subdivide until each leaf holds a constant
number of points; levels 0..L), P:192 (adaptive decomposition in practice),
P:545 (Def. sibs).  Readings: R-S (root = [0,1]^2, half-open boxes), children
ordered SW, SE, NW, NE by quadrant index q = [x >= cx] + 2 [y >= cy]; empty
children pruned; a box splits while it holds more than `leaf` points, up to
depth 30.
"""
from __future__ import annotations

import numpy as np

MAX_DEPTH = 30


class Node:
    __slots__ = ("level", "cx", "cy", "h", "idx", "children", "parent", "quad", "id")

    def __init__(self, level, cx, cy, h, idx, parent=None, quad=0):
        self.level, self.cx, self.cy, self.h = level, cx, cy, h
        self.idx = idx            # original point indices (ascending)
        self.children = []        # existing children, in quadrant order
        self.parent = parent
        self.quad = quad          # quadrant index within the parent (R-R)
        self.id = -1

    @property
    def is_leaf(self):
        return not self.children


class QuadTree:
    def __init__(self, xy: np.ndarray, leaf: int):
        xy = np.asarray(xy, dtype=np.float64)
        if xy.ndim != 2 or xy.shape[1] != 2 or len(xy) < 1:
            raise ValueError("xy must be n x 2 with n >= 1")
        if not np.all(np.isfinite(xy)):
            raise ValueError("non-finite coordinates")
        if leaf < 1:
            raise ValueError("leaf >= 1")
        self.xy = xy
        self.leaf = leaf
        self.root = Node(0, 0.5, 0.5, 0.5, np.arange(len(xy)))
        self.levels = [[self.root]]
        stack = [self.root]
        while stack:
            b = stack.pop()
            if len(b.idx) > leaf and b.level < MAX_DEPTH:
                p = xy[b.idx]
                q = (p[:, 0] >= b.cx).astype(np.int64) + 2 * (p[:, 1] >= b.cy).astype(np.int64)
                hh = 0.5 * b.h
                for k in range(4):
                    sel = b.idx[q == k]
                    if sel.size == 0:
                        continue
                    cx = b.cx + (hh if k & 1 else -hh)
                    cy = b.cy + (hh if k & 2 else -hh)
                    c = Node(b.level + 1, cx, cy, hh, sel, parent=b, quad=k)
                    b.children.append(c)
                    stack.append(c)
        # level lists in a deterministic (depth-first quadrant) order
        self.levels = []
        order = []

        def walk(b):
            order.append(b)
            for c in b.children:
                walk(c)
        import sys
        sys.setrecursionlimit(max(10000, sys.getrecursionlimit()))
        walk(self.root)
        L = max(b.level for b in order)
        self.levels = [[] for _ in range(L + 1)]
        for b in order:
            self.levels[b.level].append(b)
        for i, b in enumerate(order):
            b.id = i
        self.nodes = order
        self.L = L

    def leaves(self):
        return [b for b in self.nodes if b.is_leaf]
