"""O2 - recursive skeletonization factorization, step by step (oracle; test infrastructure).

Follows PAPER.md §2 in its order and notation:
  Def. id            P:205-210  ID: A(:,R) ~ A(:,S) T
  rank-revealing QR  P:293      ID via (column-pivoted) QR
  proxy trick        P:299-308  A = [Sigma(N, I); K(Gamma, I)] (Eq. proxyid), n_prox = 256
  sparsify/decouple  P:212-239  X_SR, X_RR, L_I, U_I
  level recursion    P:242-250, P:274-283 (Eq. rskelf); modified B_SS, original
                     off-diagonal skeleton blocks
  apply/solve/sqrt/logdet
Readings (SURVEY.md §8(c).3 / DESIGN.md §3): R-A (eps = ID tolerance on
|R_jj| <= eps |R_11|), R-C (near radius 1.8h, 4 rings x 64 angles on
[1.75h, 2.45h], ring radii at the 4 midpoints), R-E (near = active DOFs at
the START of the level), R-F (Sigma_i: apply-only compression),
R-Y (levels L..1 skeletonized, level-0 remainder dense), R-BB, R-CC.

Library primitives used as single steps: scipy QR (with/without column
pivoting), Cholesky, triangular solve, cKDTree ball queries.
"""
from __future__ import annotations

import math

import numpy as np
import scipy.linalg as sla
from scipy.spatial import cKDTree

from .kernels import Kernel
from .tree import QuadTree

R_NEAR = 1.8
R_IN, R_OUT = 1.75, 2.45
N_RINGS, N_ANGLES = 4, 64


class NumericError(RuntimeError):
    pass


def proxy_points(cx: float, cy: float, h: float) -> np.ndarray:
    """Gamma_b: 256 points discretizing the annulus [1.75h, 2.45h] (R-C)."""
    rad = h * (R_IN + (R_OUT - R_IN) * (np.arange(N_RINGS) + 0.5) / N_RINGS)
    ang = 2.0 * math.pi * np.arange(N_ANGLES) / N_ANGLES
    rr = np.repeat(rad, N_ANGLES)
    aa = np.tile(ang, N_RINGS)
    return np.stack([cx + rr * np.cos(aa), cy + rr * np.sin(aa)], axis=1)


def interp_decomp(A: np.ndarray, eps: float):
    """Def. id via QR then column-pivoted QR of R.

    Returns (piv, k, T): skeleton columns piv[:k], redundant piv[k:],
    A(:, piv[k:]) ~ A(:, piv[:k]) @ T.
    """
    m, c = A.shape
    if c == 0:
        return np.zeros(0, dtype=np.int64), 0, np.zeros((0, 0))
    if m == 0:
        return np.arange(c), 0, np.zeros((0, c))
    R = sla.qr(A, mode="r", check_finite=False)[0]
    R = R[:min(m, c)]
    R2, piv = sla.qr(R, mode="r", pivoting=True, check_finite=False)
    d = np.abs(np.diag(R2))
    if d.size == 0 or d[0] == 0.0:
        k = 0                                   # R-BB
    else:
        keep = d > eps * d[0]           # |R_jj| is non-increasing under pivoting
        k = int(keep.size if keep.all() else np.argmin(keep))
    T = sla.solve_triangular(R2[:k, :k], R2[:k, k:], lower=False, check_finite=False) \
        if k > 0 else np.zeros((0, c))
    return piv.astype(np.int64), k, T


class Box:
    __slots__ = ("node", "I", "S", "R", "T", "L", "E", "XRR", "XSR", "BSS")


class RSF:
    """F ~ Sigma (or, with which=name, the apply-only compression of Sigma_i)."""

    def __init__(self, kern: Kernel, xy: np.ndarray, eps: float, leaf: int = 64,
                 which: str | None = None, tree: QuadTree | None = None):
        if eps <= 0:
            raise ValueError("eps > 0")
        self.kern, self.xy, self.eps, self.which = kern, np.asarray(xy, np.float64), eps, which
        self.n = len(self.xy)
        self.tree = tree if tree is not None else QuadTree(self.xy, leaf)
        self.levels = {}          # level -> list[Box]
        self.logdet = 0.0
        self._factor()

    # entries of the matrix being compressed
    def _blk(self, rows, cols):
        if self.which is None:
            return self.kern.sigma_block(self.xy, rows, cols)
        return self.kern.dsigma_block(self.which, self.xy, rows, cols)

    def _prox(self, P, cols):
        if self.which is None:
            return self.kern.sigma_points(P, self.xy[cols])
        return self.kern.dsigma_points(self.which, P, self.xy[cols])

    def _factor(self):
        tree, xy = self.tree, self.xy
        active = np.ones(self.n, dtype=bool)
        skel = {}      # node id -> (S indices, modified B_SS)
        for lev in range(tree.L, 0, -1):
            act_idx = np.flatnonzero(active)          # snapshot at the level start (R-E)
            kd = cKDTree(xy[act_idx]) if act_idx.size else None
            boxes = []
            for nd in tree.levels[lev]:
                bx = Box()
                bx.node = nd
                if nd.is_leaf:
                    I = nd.idx
                    B = self._blk(I, I)
                else:
                    I, B = self._parent_block(nd, skel)
                bx.I = I
                # near field N_b (R-C, R-E)
                if kd is not None:
                    cand = act_idx[kd.query_ball_point([nd.cx, nd.cy], R_NEAR * nd.h)]
                    cand = cand[np.linalg.norm(xy[cand] - [nd.cx, nd.cy], axis=1) < R_NEAR * nd.h]
                    N = np.setdiff1d(cand, I)
                else:
                    N = np.zeros(0, dtype=np.int64)
                G = proxy_points(nd.cx, nd.cy, nd.h)
                A = np.vstack([self._blk(N, I), self._prox(G, I)])
                piv, k, T = interp_decomp(A, self.eps)
                pS, pR = piv[:k], piv[k:]
                bx.S, bx.R, bx.T = I[pS], I[pR], T
                BSS = B[np.ix_(pS, pS)]
                BSR = B[np.ix_(pS, pR)]
                BRR = B[np.ix_(pR, pR)]
                XSR = BSR - BSS @ T                        # P:212-224 (sparsify)
                XRR = BRR - BSR.T @ T - T.T @ XSR
                if self.which is None:                     # P:225-239 (eliminate)
                    XRR = 0.5 * (XRR + XRR.T)
                    try:
                        Lc = sla.cholesky(XRR, lower=True, check_finite=False) if pR.size else np.zeros((0, 0))
                    except np.linalg.LinAlgError:
                        raise NumericError(f"Cholesky of X_RR failed at level {lev}, box {nd.id}")
                    E = sla.solve_triangular(Lc, XSR.T, lower=True, check_finite=False).T \
                        if pR.size else np.zeros((k, 0))
                    bx.L, bx.E = Lc, E
                    self.logdet += 2.0 * float(np.sum(np.log(np.diag(Lc))))
                    bx.BSS = BSS - E @ E.T
                else:                                      # R-F: apply-only
                    bx.XRR, bx.XSR = XRR, XSR
                    bx.BSS = BSS
                skel[nd.id] = (bx.S, bx.BSS)
                boxes.append(bx)
            for bx in boxes:
                active[bx.R] = False
            self.levels[lev] = boxes
        # top (level 0): dense remainder (R-Y)
        root = tree.root
        if root.is_leaf:
            I0 = root.idx
            B0 = self._blk(I0, I0)
        else:
            I0, B0 = self._parent_block(root, skel)
        self.I0, self.B0 = I0, B0
        if self.which is None:
            B0 = 0.5 * (B0 + B0.T)
            try:
                self.C = sla.cholesky(B0, lower=True, check_finite=False) if I0.size else np.zeros((0, 0))
            except np.linalg.LinAlgError:
                raise NumericError("Cholesky of the top block failed (level 0)")
            self.logdet += 2.0 * float(np.sum(np.log(np.diag(self.C))))

    def _parent_block(self, nd, skel):
        """Parent self block: children's (modified) B_SS on the diagonal, original
        Sigma(S_c, S_c') off the diagonal."""
        parts = [skel[c.id] for c in nd.children]
        I = np.concatenate([p[0] for p in parts]) if parts else np.zeros(0, dtype=np.int64)
        B = self._blk(I, I)
        o = 0
        for S, BSS in parts:
            B[o:o + len(S), o:o + len(S)] = BSS
            o += len(S)
        return I, B

    # ---------------------------------------------------------------- operators
    def _sweep_levels_up(self):
        return range(self.tree.L, 0, -1)

    def solve(self, b):
        """x = F^{-1} b."""
        assert self.which is None
        x = np.array(b, dtype=np.float64, copy=True)
        for lev in self._sweep_levels_up():
            for bx in self.levels[lev]:
                if bx.R.size == 0:
                    continue
                xR = x[bx.R] - bx.T.T @ x[bx.S]
                xR = sla.solve_triangular(bx.L, xR, lower=True, check_finite=False)
                x[bx.S] -= bx.E @ xR
                x[bx.R] = xR
        if self.I0.size:
            y = sla.solve_triangular(self.C, x[self.I0], lower=True, check_finite=False)
            x[self.I0] = sla.solve_triangular(self.C, y, lower=True, trans="T", check_finite=False)
        for lev in range(1, self.tree.L + 1):
            for bx in self.levels[lev]:
                if bx.R.size == 0:
                    continue
                xR = sla.solve_triangular(bx.L, x[bx.R] - bx.E.T @ x[bx.S], lower=True,
                                          trans="T", check_finite=False)
                x[bx.R] = xR
                x[bx.S] -= bx.T @ xR
        return x

    def apply(self, v):
        """y = F v: up sweep M^T P^-T, top C C^T, down sweep P^-1 M."""
        if self.which is not None:
            return self._apply_only(v)
        x = np.array(v, dtype=np.float64, copy=True)
        for lev in self._sweep_levels_up():
            for bx in self.levels[lev]:
                if bx.R.size == 0:
                    continue
                x[bx.S] += bx.T @ x[bx.R]
                x[bx.R] = bx.L.T @ x[bx.R] + bx.E.T @ x[bx.S]
        if self.I0.size:
            x[self.I0] = self.C @ (self.C.T @ x[self.I0])
        self._down(x)
        return x

    def _down(self, x):
        for lev in range(1, self.tree.L + 1):
            for bx in self.levels[lev]:
                if bx.R.size == 0:
                    continue
                x[bx.S] += bx.E @ x[bx.R]
                x[bx.R] = bx.L @ x[bx.R]
                x[bx.R] += bx.T.T @ x[bx.S]

    def sqrt(self, w):
        """z = F^{1/2} w, F^{1/2} = [prod (L U) P] C."""
        assert self.which is None
        x = np.array(w, dtype=np.float64, copy=True)
        if self.I0.size:
            x[self.I0] = self.C @ x[self.I0]
        self._down(x)
        return x

    def _apply_only(self, v):
        """y = F_i v for the apply-only compression (R-F).  Per level
        Sigma_i ~ P^-1 Z P^-T with Z = [[Sigma'_rest, X_SR],[X_RS, X_RR]], so
          up (L->1):  x_S += T x_R;  y_R = X_RS x_S + X_RR x_R   (R rows are final)
          top:        y_0 = B_0 x_0
          down (1->L): y_S += X_SR x_R;  y_R += T^T y_S
        (the X_SR x_R coupling must be added after the coarser levels' P^-1)."""
        x = np.array(v, dtype=np.float64, copy=True)
        y = np.zeros_like(x)
        for lev in self._sweep_levels_up():
            for bx in self.levels[lev]:
                if bx.R.size == 0:
                    continue
                x[bx.S] += bx.T @ x[bx.R]
                y[bx.R] = bx.XSR.T @ x[bx.S] + bx.XRR @ x[bx.R]
        if self.I0.size:
            y[self.I0] = self.B0 @ x[self.I0]
        for lev in range(1, self.tree.L + 1):
            for bx in self.levels[lev]:
                if bx.R.size == 0:
                    continue
                y[bx.S] += bx.XSR @ x[bx.R]
                y[bx.R] += bx.T.T @ y[bx.S]
        return y

    def stats(self):
        out = []
        for lev in range(self.tree.L, 0, -1):
            bs = self.levels[lev]
            out.append(dict(level=lev, boxes=len(bs), I=sum(len(b.I) for b in bs),
                            S=sum(len(b.S) for b in bs),
                            maxI=max((len(b.I) for b in bs), default=0)))
        out.append(dict(level=0, top=len(self.I0)))
        return out
