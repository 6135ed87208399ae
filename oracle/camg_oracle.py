"""ORACLE — TEST INFRASTRUCTURE ONLY.

CPU restatement (numpy/scipy) of the reference solve path and the Galerkin
setup that feeds it, used by `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` as the checker and the
CPU baseline.  It is never imported by the product package
`paper_1912_09056_b200`, whose path runs on the GPU through `libcamg.so`.

Pinned against the reference itself: `tests/golden/make_golden.py` imports
the unmodified reference (`/root/reference/pkg/src/contactamg`) in the build
container and stores its outputs as `tests/golden/*.npz`;
`tests/test_oracle_golden.py` checks this module against every one of them.

Every function cites the reference file:line it restates; paths are relative
to `/root/reference/pkg/src/contactamg/`.
"""

from __future__ import annotations

import time
import warnings
from dataclasses import dataclass, field, replace

import numpy as np
import scipy.linalg
import scipy.sparse
import scipy.sparse.linalg

DROP_TOL = 1e-300          # sparse.py:21
RANK_TOL = 1e-10           # transfer.py:24
BREAKDOWN = 1e-14          # krylov.py:18
UNASSIGNED = -1            # aggregation.py:19
SLAVE = 0                  # aggregation.py:21 / problem.py:28


class OracleError(Exception):
    pass


# ---------------------------------------------------------------------------
# sparse core (sparse.py)


def canon(mat) -> scipy.sparse.csr_matrix:
    """Canonical CSR: duplicates summed, columns sorted, |v| < 1e-300 dropped
    (sparse.py:50-66)."""
    m = scipy.sparse.csr_matrix(mat, dtype=np.float64)
    m.sum_duplicates()
    m.sort_indices()
    tiny = np.abs(m.data) < DROP_TOL
    if tiny.any():
        c = m.tocoo()
        k = ~tiny
        m = scipy.sparse.csr_matrix((c.data[k], (c.row[k], c.col[k])), shape=m.shape)
        m.sum_duplicates()
        m.sort_indices()
    m.indptr = m.indptr.astype(np.int64)
    m.indices = m.indices.astype(np.int64)
    return m


def spmv(A, x):                      # sparse.py:149-154
    return A @ np.asarray(x, dtype=np.float64)


def transpose(A):                    # sparse.py:157-158
    return canon(A.T)


def matmul(A, B):                    # sparse.py:161-166
    return canon(A @ B)


def rap(R, A, P):                    # sparse.py:169-173 ; scipy evaluates (R@A)@P
    return canon(R @ A @ P)


def diagonal(A, mode="plain"):       # sparse.py:176-188
    if mode == "plain":
        return A.diagonal()
    if mode == "abs_rowsum":
        d = np.asarray(abs(A).sum(axis=1)).ravel()
        if np.any(d == 0.0):
            raise OracleError(f"abs_rowsum: zero row {int(np.argmax(d == 0.0))}")
        return d
    raise ValueError(mode)


def lu_factor(dense):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", scipy.linalg.LinAlgWarning)
        return scipy.linalg.lu_factor(dense)


# ---------------------------------------------------------------------------
# saddle operator (saddle.py:11-72)


@dataclass
class Saddle:
    K: scipy.sparse.csr_matrix
    B1: scipy.sparse.csr_matrix
    B2: scipy.sparse.csr_matrix
    Cz: scipy.sparse.csr_matrix

    @property
    def n_u(self):
        return self.K.shape[0]

    @property
    def n_lam(self):
        return self.Cz.shape[0]

    @property
    def n(self):
        return self.n_u + self.n_lam

    @property
    def nnz(self):
        return self.K.nnz + self.B1.nnz + self.B2.nnz + self.Cz.nnz

    def apply(self, u, lam):                       # saddle.py:49-52
        return (self.K @ u + self.B1 @ lam, self.B2 @ u - self.Cz @ lam)

    def residual(self, u, lam, bu, bl):            # saddle.py:54-56
        au, al = self.apply(u, lam)
        return bu - au, bl - al

    def merged(self):                              # saddle.py:58-67
        return canon(scipy.sparse.bmat([[self.K, self.B1], [self.B2, -self.Cz]], format="csr"))

    def merged_dense(self):                        # saddle.py:69-72
        return np.block([[self.K.toarray(), self.B1.toarray()],
                         [self.B2.toarray(), -self.Cz.toarray()]])


# ---------------------------------------------------------------------------
# point smoothers (smoothers.py:29-199)


@dataclass(frozen=True)
class PointCfg:
    kind: str = "sgs"
    sweeps: int = 1
    damping: float = 1.0
    block: int = 1          # mcgs only: DOFs per node of the colouring


@dataclass(frozen=True)
class BlockCfg:
    kind: str = "simplec"
    alpha: float = 0.7
    outer_sweeps: int = 1
    predictor: PointCfg = PointCfg()
    corrector: PointCfg = PointCfg(kind="ilu0")
    a_hat_mode: str = "plain_diag"

    def effective_a_hat_mode(self):                # smoothers.py:64-70
        if self.kind == "simplec":
            return "abs_rowsum"
        if self.kind == "braess_sarazin":
            return "plain_diag"
        return self.a_hat_mode


def ilu0_values(A):
    """ILU(0) on A's pattern, IKJ order, unit lower (smoothers.py:82-123)."""
    n = A.shape[0]
    ip, ix = A.indptr, A.indices
    v = A.data.astype(np.float64).copy()
    where = [dict(zip(ix[ip[i]:ip[i + 1]].tolist(), range(ip[i], ip[i + 1]))) for i in range(n)]
    dpos = np.empty(n, dtype=np.int64)
    for i in range(n):
        if i not in where[i]:
            raise OracleError(f"ILU(0): no diagonal in row {i}")
        dpos[i] = where[i][i]
    for i in range(n):
        for p in range(ip[i], ip[i + 1]):
            k = ix[p]
            if k >= i:
                break
            piv = v[dpos[k]]
            if piv == 0.0:
                raise OracleError(f"ILU(0): zero pivot {k}")
            v[p] /= piv
            lik = v[p]
            for q in range(dpos[k] + 1, ip[k + 1]):
                t = where[i].get(int(ix[q]))
                if t is not None:
                    v[t] -= lik * v[q]
        if v[dpos[i]] == 0.0:
            raise OracleError(f"ILU(0): zero pivot {i}")
    return v


def greedy_colors(A, block=1):
    """Greedy colouring of the symmetrised pattern in natural order -- the
    colouring libcamg uses for its multicolour SGS (GPU-only variant, not in
    the reference; emulated here to check the GPU elementwise).  With
    block > 1 the nodes of `block` consecutive rows are coloured (node graph:
    p != q coupled by a non-zero entry) and every row takes its node's
    colour."""
    A = scipy.sparse.csr_matrix(A)
    if block > 1:
        nn = A.shape[0] // block
        rows = np.repeat(np.arange(A.shape[0]), np.diff(A.indptr)) // block
        cols = A.indices // block
        keep = (rows != cols) & (A.data != 0.0)
        A = scipy.sparse.csr_matrix((np.ones(int(keep.sum())), (rows[keep], cols[keep])), shape=(nn, nn))
        return np.repeat(greedy_colors(A), block)
    G = (abs(A) + abs(A.T)).tocsr()
    G.sort_indices()
    n = A.shape[0]
    col = -np.ones(n, dtype=np.int64)
    for i in range(n):
        nb = G.indices[G.indptr[i]:G.indptr[i + 1]]
        used = set(col[nb][col[nb] >= 0].tolist())
        c = 0
        while c in used:
            c += 1
        col[i] = c
    return col


class Point:
    """Point smoother bound to one matrix (smoothers.py:141-199)."""

    def __init__(self, cfg: PointCfg, A):
        self.cfg, self.A = cfg, A
        n = A.shape[0]
        if cfg.kind in ("mcgs", "mcilu0"):
            # reference SSOR ("sgs") / ILU(0) on the colour-permuted matrix
            perm = np.argsort(greedy_colors(A, cfg.block), kind="stable")
            self.perm = perm
            inner = "sgs" if cfg.kind == "mcgs" else "ilu0"
            self.inner = Point(PointCfg(inner, cfg.sweeps, cfg.damping), canon(A[perm][:, perm]))
            return
        if cfg.kind == "gpu_chebyshev":
            # GPU-only predictor (not in the reference): Chebyshev polynomial
            # of D^-1 A, degree = sweeps, on [lmax/30, 1.1 lmax]
            d = A.diagonal()
            if np.any(d == 0.0):
                raise OracleError("chebyshev: zero diagonal")
            self.dinv = 1.0 / d
            beta = 1.1 * lambda_max(A, d)
            alpha = beta / 30.0
            self.theta, self.delta = 0.5 * (beta + alpha), 0.5 * (beta - alpha)
            return
        if cfg.kind in ("jacobi", "sgs"):
            d = A.diagonal()
            if np.any(d == 0.0):
                raise OracleError(f"{cfg.kind}: zero diagonal row {int(np.argmax(d == 0.0))}")
            if cfg.kind == "jacobi":
                self.dinv = cfg.damping / d
            else:                                   # residual-form SSOR
                Dw = scipy.sparse.diags(d / cfg.damping)
                self.lo = scipy.sparse.linalg.splu((scipy.sparse.tril(A, k=-1) + Dw).tocsc(), permc_spec="NATURAL")
                self.up = scipy.sparse.linalg.splu((scipy.sparse.triu(A, k=1) + Dw).tocsc(), permc_spec="NATURAL")
        elif cfg.kind == "ilu0":
            fv = ilu0_values(A)
            rows = np.repeat(np.arange(n), np.diff(A.indptr))
            low = rows > A.indices
            L = scipy.sparse.csr_matrix((fv[low], (rows[low], A.indices[low])), shape=(n, n)) + scipy.sparse.identity(n, format="csr")
            U = scipy.sparse.csr_matrix((fv[~low], (rows[~low], A.indices[~low])), shape=(n, n))
            self.L = scipy.sparse.linalg.splu(L.tocsc(), permc_spec="NATURAL")
            self.U = scipy.sparse.linalg.splu(U.tocsc(), permc_spec="NATURAL")
        elif cfg.kind == "direct":
            self.lu = lu_factor(A.toarray())
            if np.any(np.diag(self.lu[0]) == 0.0):
                raise OracleError("direct: singular")
        else:
            raise ValueError(cfg.kind)

    def smooth(self, x, b):
        x = np.array(x, dtype=np.float64)
        k = self.cfg.kind
        if k in ("mcgs", "mcilu0"):
            xp = self.inner.smooth(x[self.perm], np.asarray(b)[self.perm])
            out = np.empty_like(xp)
            out[self.perm] = xp
            return out
        if k == "direct":
            return scipy.linalg.lu_solve(self.lu, b)
        if k == "gpu_chebyshev":
            sigma = self.theta / self.delta
            rho = 1.0 / sigma
            d = self.dinv * (b - self.A @ x) / self.theta
            x += d
            for _ in range(1, self.cfg.sweeps):
                rn = 1.0 / (2.0 * sigma - rho)
                d = rn * rho * d + (2.0 * rn / self.delta) * (self.dinv * (b - self.A @ x))
                rho = rn
                x += d
            return x
        for _ in range(self.cfg.sweeps):
            if k == "jacobi":
                x += self.dinv * (b - self.A @ x)
            elif k == "sgs":
                x += self.lo.solve(b - self.A @ x)
                x += self.up.solve(b - self.A @ x)
            else:
                x += self.U.solve(self.L.solve(b - self.A @ x))
        return x

    def apply(self, b):
        return self.smooth(np.zeros(self.A.shape[0]), b)


# ---------------------------------------------------------------------------
# Schur approximation and block smoothers (smoothers.py:209-329)


def a_hat(K, mode):                                 # smoothers.py:209-217
    if mode == "plain_diag":
        d = K.diagonal()
        if np.any(d == 0.0):
            raise OracleError("a_hat: zero diagonal")
        return d
    return diagonal(K, "abs_rowsum")


def schur(op: Saddle, mode, scale=1.0, a_scale=1.0):
    """S~ = scale*Cz + scale*B2 diag(1/(a_scale*A^)) B1 (smoothers.py:220-239)."""
    if mode == "exact":
        Kinv = np.linalg.inv(op.K.toarray())
        S = scale * (op.Cz.toarray() + op.B2.toarray() @ Kinv @ op.B1.toarray())
        return canon(scipy.sparse.csr_matrix(S)), None
    ainv = 1.0 / (a_scale * a_hat(op.K, mode))
    S = scale * op.Cz + scale * (op.B2 @ scipy.sparse.diags(ainv) @ op.B1)
    return canon(S), ainv


class Block:
    """Bound block smoother (smoothers.py:245-329)."""

    def __init__(self, cfg: BlockCfg, op: Saddle, node_block: int = 1, predictor_solver=None):
        self.cfg, self.op = cfg, op
        mode = cfg.effective_a_hat_mode()
        if cfg.kind == "uzawa":
            self.S, _ = schur(op, mode)
        elif cfg.kind == "braess_sarazin":
            self.S, _ = schur(op, mode, a_scale=cfg.alpha)
        else:
            self.S, _ = schur(op, mode, scale=cfg.alpha)
        if mode == "exact":
            direct = Point(PointCfg("direct"), op.K)
            self.ahat_solve = direct.apply
        else:
            inv = 1.0 / a_hat(op.K, mode)
            self.ahat_solve = lambda r, inv=inv: inv * r
        pcfg = cfg.predictor
        if pcfg.kind == "mcgs" and op.K.shape[0] % max(1, node_block) == 0:
            pcfg = replace(pcfg, block=max(1, node_block))
        if cfg.kind == "braess_sarazin":
            self.pred = None
        elif predictor_solver is not None:            # smoothers.py:277-278
            self.pred = predictor_solver
        else:
            self.pred = Point(pcfg, op.K)
        self.corr = Point(cfg.corrector, self.S)

    def _uzawa(self, u, lam, bu, bl):                # smoothers.py:285-291
        op, a = self.op, self.cfg.alpha
        ru, rl = op.residual(u, lam, bu, bl)
        du = self.pred.apply(ru)
        dl = self.corr.apply(-(rl - op.B2 @ du))
        return u + a * du, lam + a * dl

    def _bs(self, u, lam, bu, bl):                   # smoothers.py:293-301
        op, a = self.op, self.cfg.alpha
        ru = bu - op.K @ u - op.B1 @ lam
        uh = u + self.ahat_solve(ru) / a
        dl = self.corr.apply(-(bl + op.Cz @ lam - op.B2 @ uh))
        return uh - self.ahat_solve(op.B1 @ dl) / a, lam + dl

    def _simple(self, u, lam, bu, bl):               # smoothers.py:303-314
        op, a = self.op, self.cfg.alpha
        ru = bu - op.K @ u - op.B1 @ lam
        uh = u + self.pred.apply(ru)
        dl = self.corr.apply(-(bl + op.Cz @ lam - op.B2 @ uh))
        return uh - a * self.ahat_solve(op.B1 @ dl), lam + a * dl

    def sweep(self, u, lam, bu, bl):                 # smoothers.py:316-326
        step = {"uzawa": self._uzawa, "braess_sarazin": self._bs,
                "simple": self._simple, "simplec": self._simple}[self.cfg.kind]
        u, lam = np.array(u, dtype=np.float64), np.array(lam, dtype=np.float64)
        for _ in range(self.cfg.outer_sweeps):
            u, lam = step(u, lam, bu, bl)
        return u, lam

    def apply(self, bu, bl):                         # smoothers.py:328-329
        return self.sweep(np.zeros(self.op.n_u), np.zeros(self.op.n_lam), bu, bl)


# ---------------------------------------------------------------------------
# aggregation (aggregation.py)


def node_graph(K, dof_node, num_nodes, node_body, eps_drop=0.0):
    """Symmetric node adjacency of K without self loops and cross-body edges
    (aggregation.py:127-145 + NodeGraph.from_edges :47-63).  Returns the
    sorted CSR arrays (indptr, indices)."""
    dof_node = np.asarray(dof_node, dtype=np.int64)
    node_body = np.asarray(node_body)
    rows = np.repeat(np.arange(K.shape[0], dtype=np.int64), np.diff(K.indptr))
    ni, nj = dof_node[rows], dof_node[K.indices]
    keep = (ni != nj) & (node_body[ni] == node_body[nj])
    vals = np.abs(K.data)
    if eps_drop > 0.0:
        dg = np.abs(K.diagonal())
        keep &= vals > eps_drop * np.sqrt(dg[rows] * dg[K.indices])
    else:
        keep &= vals > 0.0
    a, b = ni[keep], nj[keep]
    G = scipy.sparse.csr_matrix((np.ones(2 * len(a)), (np.concatenate([a, b]), np.concatenate([b, a]))),
                                shape=(num_nodes, num_nodes))
    G.sum_duplicates()
    G.sort_indices()
    return G.indptr.astype(np.int64), G.indices.astype(np.int64)


@dataclass
class Aggregates:
    node_to_agg: np.ndarray
    num_aggs: int
    roots: np.ndarray
    singletons: int = 0
    overlaps: int = 0


def greedy(indptr, indices, n, min_size=1):
    """Three-phase greedy aggregation, lowest id wins ties (aggregation.py:186-258)."""
    agg = np.full(n, UNASSIGNED, dtype=np.int64)
    roots = []
    # phase 1: root every node whose closed neighbourhood is untouched
    for i in range(n):
        if agg[i] != UNASSIGNED:
            continue
        nb = indices[indptr[i]:indptr[i + 1]]
        if (agg[nb] == UNASSIGNED).all():
            agg[i] = len(roots)
            agg[nb] = len(roots)
            roots.append(i)
    # phase 2: attach leftovers to the most-connected neighbour aggregate
    for i in range(n):
        if agg[i] != UNASSIGNED:
            continue
        c = agg[indices[indptr[i]:indptr[i + 1]]]
        c = c[c != UNASSIGNED]
        if len(c) == 0:
            agg[i] = len(roots)
            roots.append(i)
        else:
            agg[i] = int(np.argmax(np.bincount(c)))
    na = len(roots)
    size = np.bincount(agg, minlength=na)
    # phase 3: merge undersized aggregates into their best-connected neighbour
    if min_size > 1:
        order = np.argsort(agg, kind="stable")
        starts = np.concatenate([[0], np.cumsum(size)])
        members = [list(order[starts[a]:starts[a + 1]]) for a in range(na)]
        for a in range(na):
            if size[a] == 0 or size[a] >= min_size:
                continue
            conn = {}
            for v in members[a]:
                for w in indices[indptr[v]:indptr[v + 1]]:
                    t = int(agg[w])
                    if t != a:
                        conn[t] = conn.get(t, 0) + 1
            if not conn:
                continue
            best = min(conn, key=lambda t: (-conn[t], t))
            agg[members[a]] = best
            members[best] += members[a]
            size[best] += size[a]
            size[a] = 0
            members[a] = []
    alive = np.flatnonzero(np.bincount(agg, minlength=na) > 0)
    remap = np.full(na, UNASSIGNED, dtype=np.int64)
    remap[alive] = np.arange(len(alive))
    agg = remap[agg]
    sizes = np.bincount(agg, minlength=len(alive))
    return Aggregates(agg, len(alive), np.asarray(roots, dtype=np.int64)[alive],
                      singletons=int(np.sum(sizes == 1)))


def lagrange(disp: Aggregates, D, slave_dofs, row_node, lm_node_of_lm_dof):
    """Paper Alg. 1 with first-touch (aggregation.py:261-303)."""
    n_lm = int(lm_node_of_lm_dof.max()) + 1 if len(lm_node_of_lm_dof) else 0
    lam = np.full(n_lm, UNASSIGNED, dtype=np.int64)
    owner = {}
    roots = []
    overlap = 0
    for r in np.argsort(slave_dofs, kind="stable"):
        k = int(disp.node_to_agg[int(row_node[r])])
        if k == UNASSIGNED:
            raise OracleError("unaggregated slave node")
        for p in range(D.indptr[r], D.indptr[r + 1]):
            if D.data[p] == 0.0:
                continue
            pn = int(lm_node_of_lm_dof[D.indices[p]])
            tgt = owner.get(k)
            if lam[pn] == UNASSIGNED:
                if tgt is None:
                    tgt = len(roots)
                    owner[k] = tgt
                    roots.append(pn)
                lam[pn] = tgt
            elif tgt is None or lam[pn] != tgt:
                overlap += 1
    return Aggregates(lam, len(roots), np.asarray(roots, dtype=np.int64), overlaps=overlap)


# ---------------------------------------------------------------------------
# transfers (transfer.py)


def constant_nullspace(n_nodes, dpn):               # transfer.py:76-82
    v = np.zeros((dpn * n_nodes, dpn))
    for c in range(dpn):
        v[c::dpn, c] = 1.0
    return v


def tentative(aggs: Aggregates, ns, dof_node):
    """Per-aggregate pivoted QR (transfer.py:86-145).  Returns
    (P, coarse_ns, coarse_dof_agg, dropped)."""
    ns = np.asarray(ns, dtype=np.float64)
    n, k = ns.shape
    agg_of_dof = aggs.node_to_agg[np.asarray(dof_node, dtype=np.int64)]
    if np.any(agg_of_dof == UNASSIGNED):
        raise OracleError("incomplete aggregation")
    order = np.argsort(agg_of_dof, kind="stable")
    cnt = np.bincount(agg_of_dof, minlength=aggs.num_aggs)
    if np.any(cnt == 0):
        raise OracleError("empty aggregate")
    starts = np.concatenate([[0], np.cumsum(cnt)])
    R_rows, C_rows, V_rows, cns, cagg = [], [], [], [], []
    col = 0
    dropped = 0
    for a in range(aggs.num_aggs):
        dofs = order[starts[a]:starts[a + 1]]
        Q, R, piv = scipy.linalg.qr(ns[dofs], mode="economic", pivoting=True)
        dg = np.abs(np.diag(R))
        if len(dg) == 0 or dg[0] <= 0.0:
            raise OracleError(f"aggregate {a}: zero near-kernel block")
        r = int(np.sum(dg > RANK_TOL * dg[0]))
        dropped += k - r
        unperm = np.empty((r, k))
        unperm[:, piv] = R[:r, :]                 # R P^T
        cns.append(unperm)
        for c in range(r):
            R_rows.append(dofs)
            C_rows.append(np.full(len(dofs), col + c, dtype=np.int64))
            V_rows.append(Q[:, c])
            cagg.append(a)
        col += r
    P = canon(scipy.sparse.coo_matrix((np.concatenate(V_rows), (np.concatenate(R_rows), np.concatenate(C_rows))),
                                      shape=(n, col)))
    return P, np.vstack(cns), np.asarray(cagg, dtype=np.int64), dropped


def lambda_max(A, d, iters=10):                      # transfer.py:148-161
    n = A.shape[0]
    v = np.ones(n) / np.sqrt(n)
    lam = 1.0
    for _ in range(iters):
        w = (A @ v) / d
        nw = np.linalg.norm(w)
        if nw == 0.0:
            return 1.0
        lam = nw
        v = w / nw
    return float(lam)


def smooth_prolongator(P, A, omega):                 # transfer.py:164-183
    if omega == 0.0:
        return P, 1.0
    d = A.diagonal()
    if np.any(d == 0.0):
        raise OracleError("zero diagonal")
    lm = lambda_max(A, d)
    DA = canon(A.multiply(1.0 / d[:, None]))
    return canon(P - (omega / lm) * (DA @ P)), lm


# ---------------------------------------------------------------------------
# hierarchy (hierarchy.py)


@dataclass
class Meta:
    """LevelMeta restated (hierarchy.py:70-82)."""
    u_dof_node: np.ndarray
    num_u_nodes: int
    node_body: np.ndarray
    lam_dof_node: np.ndarray
    num_lam_nodes: int
    ns_u: np.ndarray
    ns_lam: np.ndarray
    mortar: scipy.sparse.csr_matrix
    slave_dofs: np.ndarray
    row_node: np.ndarray
    lm_node_of_lm_dof: np.ndarray


@dataclass(frozen=True)
class HierCfg:                                       # hierarchy.py:49-67
    max_levels: int = 3
    max_coarse_size: int = 500
    coarse_solver: str = "merged_lu"
    min_agg_size: int = 6
    smooth_displacement_transfers: bool = True
    omega: float = 4.0 / 3.0
    eps_drop: float = 0.0


@dataclass
class Level:
    op: Saddle
    smoother: Block
    P_u: scipy.sparse.csr_matrix | None = None
    P_lam: scipy.sparse.csr_matrix | None = None
    R_u: scipy.sparse.csr_matrix | None = None
    R_lam: scipy.sparse.csr_matrix | None = None
    info: dict = field(default_factory=dict)


class Hier:
    def __init__(self, levels, cfg, lu, pre, post):
        self.levels, self.cfg, self.lu, self.pre, self.post = levels, cfg, lu, pre, post

    def coarse(self, u, lam, bu, bl):                # hierarchy.py:108-113
        lvl = self.levels[-1]
        if self.cfg.coarse_solver == "merged_lu":
            s = scipy.linalg.lu_solve(self.lu, np.concatenate([bu, bl]))
            return s[:lvl.op.n_u], s[lvl.op.n_u:]
        return lvl.smoother.sweep(u, lam, bu, bl)

    def vcycle(self, l, u, lam, bu, bl):             # hierarchy.py:272-287
        lvl = self.levels[l]
        if l == len(self.levels) - 1:
            return self.coarse(u, lam, bu, bl)
        for _ in range(self.pre):
            u, lam = lvl.smoother.sweep(u, lam, bu, bl)
        ru, rl = lvl.op.residual(u, lam, bu, bl)
        cu, cl = lvl.R_u @ ru, lvl.R_lam @ rl
        nxt = self.levels[l + 1].op
        xu, xl = self.vcycle(l + 1, np.zeros(nxt.n_u), np.zeros(nxt.n_lam), cu, cl)
        u, lam = u + lvl.P_u @ xu, lam + lvl.P_lam @ xl
        for _ in range(self.post):
            u, lam = lvl.smoother.sweep(u, lam, bu, bl)
        return u, lam

    def apply(self, r):                              # hierarchy.py:115-120
        op = self.levels[0].op
        r = np.asarray(r, dtype=np.float64)
        u, lam = self.vcycle(0, np.zeros(op.n_u), np.zeros(op.n_lam), r[:op.n_u], r[op.n_u:])
        return np.concatenate([u, lam])

    @property
    def complexity(self):
        return sum(l.op.nnz for l in self.levels) / self.levels[0].op.nnz


def coarse_meta(opc: Saddle, cns_u, cagg_u, cns_l, cagg_l, disp: Aggregates, lam: Aggregates, meta: Meta):
    """Next level's maps and the B1 mortar surrogate (hierarchy.py:147-177)."""
    body = np.full(disp.num_aggs, -1, dtype=np.int8)
    body[disp.node_to_agg] = meta.node_body
    rows_nnz = np.diff(opc.B1.indptr)
    rows = np.flatnonzero((body[cagg_u] == SLAVE) & (rows_nnz > 0))
    if len(rows) == 0:
        raise OracleError("lost the slave interface")
    return Meta(
        u_dof_node=cagg_u, num_u_nodes=disp.num_aggs, node_body=body,
        lam_dof_node=cagg_l, num_lam_nodes=lam.num_aggs, ns_u=cns_u, ns_lam=cns_l,
        mortar=canon(opc.B1[rows, :]), slave_dofs=rows.astype(np.int64),
        row_node=cagg_u[rows], lm_node_of_lm_dof=cagg_l,
    )


def node_block(meta: Meta) -> int:
    """DOFs per node when every node owns the same consecutive DOF count
    (2, 3 or 6), else 1 -- the node size of the mcgs predictor colouring."""
    n = len(meta.u_dof_node)
    if meta.num_u_nodes == 0 or n % meta.num_u_nodes:
        return 1
    bs = n // meta.num_u_nodes
    if bs not in (2, 3, 6) or not np.array_equal(meta.u_dof_node, np.arange(n) // bs):
        return 1
    return bs


def setup(op: Saddle, meta: Meta, cfg: HierCfg, scfg: BlockCfg, pre=1, post=1) -> Hier:
    """Level loop (hierarchy.py:180-269)."""
    levels = []
    while True:
        if len(levels) + 1 >= cfg.max_levels or op.n < cfg.max_coarse_size:
            levels.append(Level(op, Block(scfg, op, node_block(meta))))
            break
        ip, ix = node_graph(op.K, meta.u_dof_node, meta.num_u_nodes, meta.node_body, cfg.eps_drop)
        disp = greedy(ip, ix, meta.num_u_nodes, cfg.min_agg_size)
        if disp.num_aggs == 0:
            raise OracleError("no aggregates")
        if disp.num_aggs >= meta.num_u_nodes:
            levels.append(Level(op, Block(scfg, op, node_block(meta))))
            break
        lam = lagrange(disp, meta.mortar, meta.slave_dofs, meta.row_node, meta.lm_node_of_lm_dof)
        if np.any(lam.node_to_agg == UNASSIGNED):
            raise OracleError("unreferenced multiplier node")
        Pu, cns_u, cagg_u, dropped = tentative(disp, meta.ns_u, meta.u_dof_node)
        lmax = None
        if cfg.smooth_displacement_transfers:
            Pu, lmax = smooth_prolongator(Pu, op.K, cfg.omega)
        Pl, cns_l, cagg_l, _ = tentative(lam, meta.ns_lam, meta.lam_dof_node)
        Ru, Rl = transpose(Pu), transpose(Pl)
        opc = Saddle(rap(Ru, op.K, Pu), rap(Ru, op.B1, Pl), rap(Rl, op.B2, Pu), rap(Rl, op.Cz, Pl))
        info = dict(u_aggregates=disp.num_aggs, lam_aggregates=lam.num_aggs,
                    u_singletons=disp.singletons, lam_overlap_touches=lam.overlaps,
                    lambda_max=lmax, dropped_ns_columns=dropped,
                    u_agg=disp.node_to_agg, lam_agg=lam.node_to_agg)
        levels.append(Level(op, Block(scfg, op, node_block(meta)), Pu, Pl, Ru, Rl, info))
        meta = coarse_meta(opc, cns_u, cagg_u, cns_l, cagg_l, disp, lam, meta)
        op = opc
    lu = lu_factor(levels[-1].op.merged_dense()) if cfg.coarse_solver == "merged_lu" else None
    return Hier(levels, cfg, lu, pre, post)


# ---------------------------------------------------------------------------
# nested preconditioner (hierarchy.py:289-385)


def node_block_of(dof_node, num_nodes) -> int:
    n = len(dof_node)
    if num_nodes == 0 or n % num_nodes:
        return 1
    bs = n // num_nodes
    if bs not in (2, 3, 6) or not np.array_equal(dof_node, np.arange(n) // bs):
        return 1
    return bs


class ScalarHier:
    """Scalar smoothed-aggregation AMG on K (hierarchy.py:300-363)."""

    def __init__(self, K, meta: Meta, cfg: HierCfg, pcfg: PointCfg):
        self.levels = []                             # (A, P, R, smoother)
        A, dof_node, nn, body, ns = K, meta.u_dof_node, meta.num_u_nodes, meta.node_body, meta.ns_u
        while len(self.levels) + 1 < cfg.max_levels and A.shape[0] >= cfg.max_coarse_size:
            ip, ix = node_graph(A, dof_node, nn, body, cfg.eps_drop)
            aggs = greedy(ip, ix, nn, cfg.min_agg_size)
            if aggs.num_aggs >= nn:
                break
            P, cns, cagg, _ = tentative(aggs, ns, dof_node)
            if cfg.smooth_displacement_transfers:
                P, _ = smooth_prolongator(P, A, cfg.omega)
            R = transpose(P)
            c = pcfg
            if c.kind == "mcgs":
                c = replace(c, block=node_block_of(dof_node, nn))
            self.levels.append((A, P, R, Point(c, A)))
            nbody = np.full(aggs.num_aggs, -1, dtype=np.int8)
            nbody[aggs.node_to_agg] = body
            A, dof_node, nn, body, ns = rap(R, A, P), cagg, aggs.num_aggs, nbody, cns
        self.levels.append((A, None, None, None))
        self.lu = lu_factor(A.toarray())

    def vcycle(self, l, x, b):                       # hierarchy.py:305-315
        A, P, R, sm = self.levels[l]
        if l == len(self.levels) - 1:
            return scipy.linalg.lu_solve(self.lu, b)
        x = sm.smooth(x, b)
        r = b - A @ x
        c = self.vcycle(l + 1, np.zeros(P.shape[1]), R @ r)
        x = x + P @ c
        return sm.smooth(x, b)

    def apply(self, b):
        return self.vcycle(0, np.zeros(len(b)), np.asarray(b, dtype=np.float64))


class Nested:
    """NestedPreconditioner (hierarchy.py:366-376)."""

    def __init__(self, op: Saddle, meta: Meta, scfg: BlockCfg, icfg: HierCfg, ipcfg: PointCfg):
        self.op = op
        self.inner = ScalarHier(op.K, meta, icfg, ipcfg)
        self.outer = Block(scfg, op, node_block(meta), predictor_solver=self.inner)

    def apply(self, r):
        r = np.asarray(r, dtype=np.float64)
        u, lam = self.outer.apply(r[:self.op.n_u], r[self.op.n_u:])
        return np.concatenate([u, lam])


# ---------------------------------------------------------------------------
# GMRES (krylov.py:45-129)


@dataclass
class Report:
    iterations: int = 0
    residual_history: list = field(default_factory=list)
    converged: bool = False
    solve_seconds: float = 0.0


def gmres(apply_A, apply_M, b, rel_tol=1e-8, max_iters=500, restart=100):
    """Right-preconditioned GMRES(m), x0 = 0, MGS + one re-orthogonalisation
    pass, Givens rotations, true residual per restart (krylov.py:45-129)."""
    t0 = time.perf_counter()
    b = np.asarray(b, dtype=np.float64)
    n = len(b)
    rep = Report()
    nb = np.linalg.norm(b)
    rep.residual_history.append(nb)
    if nb == 0.0:
        rep.converged = True
        return np.zeros(n), rep
    tgt = rel_tol * nb
    x = np.zeros(n)
    done = False
    total = 0
    while total < max_iters and not done:
        r = b - apply_A(x)
        beta = np.linalg.norm(r)
        if beta <= tgt:
            done = True
            break
        m = min(restart, max_iters - total)
        V = np.zeros((n, m + 1))
        H = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        g[0] = beta
        V[:, 0] = r / beta
        used = 0
        for j in range(m):
            w = apply_A(apply_M(V[:, j]))
            for _pass in range(2):
                for i in range(j + 1):
                    h = np.dot(V[:, i], w)
                    w -= h * V[:, i]
                    H[i, j] += h
            H[j + 1, j] = np.linalg.norm(w)
            happy = H[j + 1, j] <= BREAKDOWN * max(1.0, abs(H[j, j]))
            if not happy:
                V[:, j + 1] = w / H[j + 1, j]
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            den = np.hypot(H[j, j], H[j + 1, j])
            cs[j], sn[j] = H[j, j] / den, H[j + 1, j] / den
            H[j, j], H[j + 1, j] = den, 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            total += 1
            used = j + 1
            est = abs(g[j + 1])
            rep.residual_history.append(est)
            if happy or est <= tgt or total >= max_iters:
                break
        y = np.zeros(used)
        for i in range(used - 1, -1, -1):
            y[i] = (g[i] - H[i, i + 1:used] @ y[i + 1:used]) / H[i, i]
        x = x + apply_M(V[:, :used] @ y)
        if np.linalg.norm(b - apply_A(x)) <= tgt:
            done = True
    rep.iterations = total
    rep.converged = done
    rep.solve_seconds = time.perf_counter() - t0
    return x, rep


# ---------------------------------------------------------------------------
# convenience: oracle objects from a generated system


def system_from_generated(g):
    """(Saddle, Meta, rhs) for a `paper_1912_09056_b200.problem.GeneratedSystem`."""
    op = Saddle(canon(g.K), canon(g.B1), canon(g.B2), canon(g.Cz))
    d = g.dim
    n_s = len(g.slave_nodes)
    meta = Meta(
        u_dof_node=np.arange(g.n_u, dtype=np.int64) // d,
        num_u_nodes=g.n_u // d,
        node_body=g.node_body.astype(np.int8),
        lam_dof_node=np.arange(g.n_lam, dtype=np.int64) // d,
        num_lam_nodes=n_s,
        ns_u=g.rigid_body_modes(),
        ns_lam=constant_nullspace(n_s, d),
        mortar=canon(g.mortar_block),
        slave_dofs=g.slave_dofs.astype(np.int64),
        row_node=np.repeat(g.slave_nodes, d).astype(np.int64),
        lm_node_of_lm_dof=np.arange(g.n_lam, dtype=np.int64) // d,
    )
    return op, meta, g.rhs.copy()
