"""O2s - strong-admissibility matrix peeling for Tr(G) (oracle; test infrastructure only).

Next row f4 of SURVEY.md §8(f).  PAPER.md names the variant and its better scaling for
Matern kernels (Table 3 P:760 / P:777) but defers the algorithm to Lin, Lu and
Ying (2011); this module restates that published construction in the paper's notation
(reading R-f4 in DESIGN.md §7f):

* Boxes of level l on a PERFECT quadtree (every leaf at depth L; other trees raise), box
  coordinates (ix, iy) in [0, 2^l)^2.  N(b) = the 3 x 3 boxes around b (b included);
  IL(b) = children of N(parent(b)) that are not in N(b) (the interaction list, l >= 2).
  Every pair of points is covered exactly once: by the level where their boxes enter each
  other's interaction list, or by the leaf-level near field N(b).  Admissible blocks
  G(I_b, I_c), c in IL(b), are numerically low rank (strong admissibility).
* Level l = 2..L: the residual R_l = G - sum_{m<l} G^(m) restricted to rows I_b only
  involves the 6 x 6 window of children of N(parent(b)) -- so with the 36 color classes
  kappa(b) = (ix mod 6, iy mod 6) every window holds at most one box of each class.  Probes
  W_kappa are Gaussian on the boxes of class kappa; Y_kappa = R_l W_kappa; for
  c in IL(b), Y_kappa(c)(I_b, :) = G_bc W_c exactly (up to the error of the peeled levels).
  Every pair {b, c} then gets the two-sided low-rank approximation of Eq. lowrankapprox
  (P:443-445): U1 = orth(Y_bc), U2 = orth(Y_cb), M = (W_b^T U1)^+ (W_b^T Y_bc) (U2^T W_c)^+,
  G_bc ~ U1 M U2^T, G_cb = G_bc^T.  Widths adapt as in the weak variant (R-M).
* Extraction: R_{L+1} = G - sum_l G^(l) holds only leaf near-field blocks; with the 9 classes
  (ix mod 3, iy mod 3) every 3 x 3 neighbourhood holds one box per class, so
  H_kappa = R_{L+1} E_kappa with E_kappa the identity columns on the leaves of class kappa
  gives H_kappa(I_b, :) = G_bb E_b for kappa(b) = kappa, and Tr G = sum_b Tr G_bb.

Library primitives: scipy pivoted QR (orth), numpy pinv.  Probes are an INPUT, as in
oracle/peel.py: probe(rows, cols, level) -> N(0, 1) entries (original point indices).
"""
from __future__ import annotations

import numpy as np

from .peel import eps_rank, orth
from .tree import QuadTree

NCLASS, NCLASS_EXTRACT = 6, 3


def box_coords(b):
    """(ix, iy) of a box of level l (center ((ix + 1/2) / 2^l, (iy + 1/2) / 2^l))."""
    s = 1 << b.level
    return int(round(b.cx * s - 0.5)), int(round(b.cy * s - 0.5))


def check_perfect(tree: QuadTree):
    for lev in range(tree.L + 1):
        if len(tree.levels[lev]) != 4 ** lev:
            raise ValueError("strong-admissibility peeling needs a perfect quadtree "
                             f"(level {lev} has {len(tree.levels[lev])} of {4 ** lev} boxes)")


def interaction_lists(tree: QuadTree, lev: int):
    """{box id: [boxes c in IL(b)]} at level lev (perfect tree)."""
    at = {box_coords(b): b for b in tree.levels[lev]}
    out = {}
    for b in tree.levels[lev]:
        x, y = box_coords(b)
        px, py = x // 2, y // 2
        il = []
        for cx in range(2 * px - 2, 2 * px + 4):
            for cy in range(2 * py - 2, 2 * py + 4):
                if max(abs(cx - x), abs(cy - y)) <= 1:
                    continue
                c = at.get((cx, cy))
                if c is not None:
                    il.append(c)
        out[b.id] = il
    return out


class StrongLevel:
    """G^(l): for every ordered admissible pair (b, c): rows I_b += U_bc M U_cb^T X(I_c)."""

    def __init__(self):
        self.blocks = []

    def apply(self, X):
        Y = np.zeros_like(X)
        for Ib, Ic, U1, M, U2 in self.blocks:
            Y[Ib] += U1 @ (M @ (U2.T @ X[Ic]))
        return Y


def peel_trace_strong(apply_G, tree: QuadTree, eps_peel: float, probe, *, oversample: int = 8,
                      block: int = 8, start: int | None = None, diag: dict | None = None) -> float:
    check_perfect(tree)
    n = len(tree.xy)
    c = oversample
    peeled = []
    cols_per_level, ranks_per_level = [], []

    def residual_apply(X):
        Y = apply_G(X)
        for lvl in peeled:
            Y -= lvl.apply(X)
        return Y

    for lev in range(2, tree.L + 1):
        boxes = tree.levels[lev]
        IL = interaction_lists(tree, lev)
        cls = {b.id: (box_coords(b)[0] % NCLASS, box_coords(b)[1] % NCLASS) for b in boxes}
        classes = sorted(set(cls.values()))
        pairs = [(b, cc) for b in boxes for cc in IL[b.id] if b.id < cc.id]
        if not pairs:
            continue
        maxn = max(len(b.idx) for b in boxes)
        cap = maxn + c
        ncols = min(start if start is not None else c + block, cap)
        Ys = {k: np.zeros((n, 0)) for k in classes}
        Om = {b.id: np.zeros((len(b.idx), 0)) for b in boxes}
        have = 0
        while True:
            new = np.arange(have, ncols)
            for b in boxes:
                Om[b.id] = np.hstack([Om[b.id], probe(b.idx, new, lev)])
            for k in classes:
                W = np.zeros((n, new.size))
                for b in boxes:
                    if cls[b.id] == k:
                        W[b.idx] = Om[b.id][:, have:ncols]
                Ys[k] = np.hstack([Ys[k], residual_apply(W)])
            have = ncols
            worst = 0
            for b, cc in pairs:
                worst = max(worst, eps_rank(Ys[cls[cc.id]][b.idx], eps_peel),
                            eps_rank(Ys[cls[b.id]][cc.idx], eps_peel))
            if worst <= ncols - c or ncols >= cap:
                break
            ncols = min(cap, ncols + block)
        cols_per_level.append(ncols)
        lvl = StrongLevel()
        rks = []
        for b, cc in pairs:
            Ybc = Ys[cls[cc.id]][b.idx]        # ~ G_bc W_c
            Ycb = Ys[cls[b.id]][cc.idx]        # ~ G_cb W_b
            U1, U2 = orth(Ybc, eps_peel), orth(Ycb, eps_peel)
            Wb, Wc = Om[b.id], Om[cc.id]
            M = np.linalg.pinv(Wb.T @ U1, rcond=1e-14) @ (Wb.T @ Ybc) @ np.linalg.pinv(U2.T @ Wc, rcond=1e-14)
            lvl.blocks.append((b.idx, cc.idx, U1, M, U2))
            lvl.blocks.append((cc.idx, b.idx, U2, M.T, U1))
            rks.append(U1.shape[1])
        ranks_per_level.append(rks)
        peeled.append(lvl)
    # extraction with 9 classes of leaves (the leaf near field)
    leaves = tree.levels[tree.L]
    nL = max(len(b.idx) for b in leaves)
    tr, sabs = 0.0, 0.0
    for kx in range(NCLASS_EXTRACT):
        for ky in range(NCLASS_EXTRACT):
            sel = [b for b in leaves if box_coords(b)[0] % 3 == kx and box_coords(b)[1] % 3 == ky]
            if not sel:
                continue
            E = np.zeros((n, nL))
            for b in sel:
                E[b.idx, np.arange(len(b.idx))] = 1.0
            H = residual_apply(E)
            for b in sel:
                dv = H[b.idx, np.arange(len(b.idx))]
                tr += float(np.sum(dv))
                sabs += float(np.sum(np.abs(dv)))
    if diag is not None:
        diag["ranks"] = ranks_per_level
        diag["cols"] = cols_per_level
        diag["cancellation"] = sabs / abs(tr) if tr != 0 else float("inf")
        diag["nL"] = nL
    return tr
