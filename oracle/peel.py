"""O2 - weak-admissibility matrix peeling for Tr(G) (oracle; test infrastructure).

Follows PAPER.md §3 in order and notation:
  randomized two-sided LRA, Eq. lowrankapprox
      A ~ U1 [(W2^T U1)^+ (W2^T A W1) (U2^T W1)^+] U2^T
  level 1 (block-sparse probes W^(1)_k)
  level 2 and Def. sibs
  subsequent levels (j = k mod 4 groups)
  trace extraction H = (G - sum G^(m)) E
  cancellation remark                            P:597-599 (diagnostic sum|diag|/|Tr|)
Readings: R-K (c = 8 oversampling), R-L (width r + c), R-M (block-adaptive:
grow every W_k by `block` columns until every sibling sketch's eps_peel-rank is
<= columns - c), R-N (orth by CPQR truncated at eps_peel relative; + via
lstsq with rcond 1e-14), R-R (group = quadrant index within the parent;
probes only on existing boxes).

G is a black box: `apply_G(X)` maps n x k -> n x k (original point order) and
must be symmetric.  Probes are an INPUT: `probe(rows, cols, level)` returns the
N(0,1) entries for original point indices `rows` and column indices `cols`.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

from .tree import QuadTree


def orth(Y: np.ndarray, eps: float) -> np.ndarray:
    """Well-conditioned basis of range(Y) by CPQR truncated at eps relative (R-N)."""
    if Y.shape[1] == 0 or Y.shape[0] == 0:
        return np.zeros((Y.shape[0], 0))
    Q, R, _ = sla.qr(Y, mode="economic", pivoting=True, check_finite=False)
    d = np.abs(np.diag(R))
    if d[0] == 0.0:
        return np.zeros((Y.shape[0], 0))
    keep = d > eps * d[0]
    k = int(keep.size if keep.all() else np.argmin(keep))
    return Q[:, :k]


def eps_rank(Y: np.ndarray, eps: float) -> int:
    return orth(Y, eps).shape[1]


class LowRankLevel:
    """G^(l): for each ordered sibling pair (i, j): rows I_i += U_ij M_ij U_ji^T X(I_j)."""

    def __init__(self):
        self.blocks = []   # (rows_i, rows_j, U_ij, M_ij, U_ji)

    def apply(self, X: np.ndarray) -> np.ndarray:
        Y = np.zeros_like(X)
        for Ii, Ij, Ui, M, Uj in self.blocks:
            Y[Ii] += Ui @ (M @ (Uj.T @ X[Ij]))
        return Y


def peel_trace(apply_G, tree: QuadTree, eps_peel: float, probe, *, oversample: int = 8,
               block: int = 8, start: int | None = None, max_cols: int | None = None,
               diag: dict | None = None) -> float:
    n = len(tree.xy)
    c = oversample
    peeled: list[LowRankLevel] = []
    ranks_per_level = []
    cols_per_level = []

    def residual_apply(X):
        Y = apply_G(X)
        for lvl in peeled:
            Y -= lvl.apply(X)
        return Y

    for lev in range(1, tree.L + 1):
        boxes = tree.levels[lev]
        if not boxes:
            break
        # sibling groups: parents with >= 2 children at this level
        parents = {}
        for b in boxes:
            parents.setdefault(b.parent.id, []).append(b)
        fam = [ch for ch in parents.values() if len(ch) >= 2]
        if not fam:
            peeled.append(LowRankLevel())
            continue
        maxn = max(len(b.idx) for b in boxes)
        cap = max_cols if max_cols is not None else maxn + c
        ncols = start if start is not None else c + block
        ncols = min(ncols, cap)
        Ys = [np.zeros((n, 0)) for _ in range(4)]
        Om = {b.id: np.zeros((len(b.idx), 0)) for b in boxes}
        have = 0
        while True:
            new = np.arange(have, ncols)
            # probes for the new columns, W_k supported on quadrant-k boxes
            for b in boxes:
                Om[b.id] = np.hstack([Om[b.id], probe(b.idx, new, lev)])
            for k in range(4):
                W = np.zeros((n, new.size))
                for b in boxes:
                    if b.quad == k:
                        W[b.idx] = Om[b.id][:, have:ncols]
                Ys[k] = np.hstack([Ys[k], residual_apply(W)])
            have = ncols
            # adaptivity (R-M): every sibling sketch rank <= columns - c
            worst = 0
            for ch in fam:
                for bi in ch:
                    for bj in ch:
                        if bi is bj:
                            continue
                        worst = max(worst, eps_rank(Ys[bj.quad][bi.idx], eps_peel))
            if worst <= ncols - c or ncols >= cap:
                break
            ncols = min(cap, ncols + block)
        cols_per_level.append(ncols)
        # Eq. lowrankapprox for every ordered sibling pair
        lvl = LowRankLevel()
        rks = []
        for ch in fam:
            for bi in ch:
                for bj in ch:
                    if bi is bj:
                        continue
                    Yij = Ys[bj.quad][bi.idx]      # ~ G_ij W_j
                    Yji = Ys[bi.quad][bj.idx]      # ~ G_ji W_i
                    U1 = orth(Yij, eps_peel)
                    U2 = orth(Yji, eps_peel)
                    Wi, Wj = Om[bi.id], Om[bj.id]
                    A1 = np.linalg.pinv(Wi.T @ U1, rcond=1e-14)
                    A2 = np.linalg.pinv(U2.T @ Wj, rcond=1e-14)
                    M = A1 @ (Wi.T @ Yij) @ A2
                    lvl.blocks.append((bi.idx, bj.idx, U1, M, U2))
                    rks.append(U1.shape[1])
        ranks_per_level.append(rks)
        peeled.append(lvl)
    # extraction
    leaves = tree.leaves()
    nL = max(len(b.idx) for b in leaves)
    E = np.zeros((n, nL))
    for b in leaves:
        E[b.idx, np.arange(len(b.idx))] = 1.0
    H = residual_apply(E)
    tr = 0.0
    sabs = 0.0
    for b in leaves:
        dvals = H[b.idx, np.arange(len(b.idx))]
        tr += float(np.sum(dvals))
        sabs += float(np.sum(np.abs(dvals)))
    if diag is not None:
        diag["ranks"] = ranks_per_level
        diag["cols"] = cols_per_level
        diag["cancellation"] = sabs / abs(tr) if tr != 0 else float("inf")
        diag["nL"] = nL
    return tr
