"""Two-body mortar contact / mesh-tying problem generator (host side).

The reference generator (`pkg/src/contactamg/problem.py`) is 2-D only, accepts
only matching interfaces (`problem.py:58-69`) and emits only contact rows
(`problem.py:306-353`), so it cannot produce any BASELINE config (SURVEY.md
§0 item 3).  This module is a new generator that keeps the reference's
conventions and extends them:

* slave body = upper block, numbered first; master = lower block
  (`problem.py:83-153`); node id = lexicographic with x fastest;
  DOF = dim * node + component;
* B1 = full mortar coupling, D on slave rows and -M on master rows
  (`problem.py:322-335`); normal rows n.(D u_s - M u_m) in B2 and
  tangential rows t.lam in Cz (`problem.py:337-348`), so the operator is
  [[K, B1], [B2, -Cz]];
* non-matching interfaces use segment-based integration: both interface
  grids are axis-aligned tensor grids, so the mortar matrices factor into
  Kronecker products of exact 1-D overlay integrals;
* Dirichlet nodes are *eliminated* instead of kept as
  unit-diagonal rows;
* contact configs clamp both far faces (the reference
  and the paper clamp both, `problem.py:127-133`, `PAPER.md:2087`).

The stiffness block is assembled from a per-(block, boundary-type) stencil
table.  The same table drives the GPU assembly kernel used for the large
configs (`camg_assemble_stencil` in `csrc/generator.cu`); both sum element
contributions in ascending local-corner order, so host and device K are
bit-identical.
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass, field, replace

import numpy as np
import scipy.sparse

from .errors import AssemblyError, ConfigError

BODY_SLAVE = 0
BODY_MASTER = 1


# ---------------------------------------------------------------------------
# specification


@dataclass(frozen=True)
class BlockSpec:
    elems: tuple          # elements per axis
    origin: tuple         # lower corner
    size: tuple           # edge lengths
    youngs: float = 1.0


@dataclass(frozen=True)
class TwoBodySpec:
    """Two stacked blocks; the vertical axis is the last one."""

    dim: int
    lower: BlockSpec                 # master body
    upper: BlockSpec                 # slave body
    nu: float = 0.3
    coupling: str = "tying"          # "tying" | "contact"
    active_fraction: float | None = None   # contact: Bernoulli(p) active set, None = all
    clamp_upper_top: bool = False
    seed: int = 0
    name: str = ""

    def validate(self):
        if self.dim not in (2, 3):
            raise ConfigError("dim must be 2 or 3")
        for b in (self.lower, self.upper):
            if len(b.elems) != self.dim or min(b.elems) < 1:
                raise ConfigError("element counts must be >= 1 per axis")
            if b.youngs <= 0.0:
                raise ConfigError("youngs modulus must be positive")
        if not (0.0 < self.nu < 0.5):
            raise ConfigError("poisson ratio must lie in (0, 0.5)")
        if self.coupling not in ("tying", "contact"):
            raise ConfigError(f"unknown coupling {self.coupling!r}")
        v = self.dim - 1
        top = self.lower.origin[v] + self.lower.size[v]
        if abs(top - self.upper.origin[v]) > 1e-12:
            raise ConfigError("blocks must touch along the vertical axis")
        for a in range(v):
            if abs(self.lower.origin[a] - self.upper.origin[a]) > 1e-12 or abs(self.lower.size[a] - self.upper.size[a]) > 1e-12:
                raise ConfigError("interface faces must coincide")


def _two_d(lower, upper, e_lower, e_upper, **kw):
    return TwoBodySpec(
        dim=2,
        lower=BlockSpec(lower, (0.0, 0.0), (2.0, 1.0), e_lower),
        upper=BlockSpec(upper, (0.0, 1.0), (2.0, 1.0), e_upper),
        **kw,
    )


def _three_d(lower, upper, e_lower, e_upper, **kw):
    return TwoBodySpec(
        dim=3,
        lower=BlockSpec(lower, (0.0, 0.0, 0.0), (1.0, 1.0, 0.5), e_lower),
        upper=BlockSpec(upper, (0.0, 0.0, 0.5), (1.0, 1.0, 0.5), e_upper),
        **kw,
    )


# BASELINE.json configs[0..4]
CONFIGS = {
    "C1": _two_d((32, 16), (30, 15), 1.0, 1.0, coupling="tying", seed=0, name="C1"),
    "C2": _two_d((256, 128), (240, 120), 1.0, 10.0, coupling="contact",
                 clamp_upper_top=True, seed=1, name="C2"),
    "C3": _three_d((64, 64, 32), (60, 60, 30), 1.0, 1.0, coupling="tying", seed=2, name="C3"),
    "C4": _three_d((128, 128, 64), (120, 120, 60), 1.0, 100.0, coupling="contact",
                   active_fraction=0.5, clamp_upper_top=True, seed=3, name="C4"),
    "C5": _three_d((200, 200, 100), (196, 196, 98), 1.0, 10.0, coupling="contact",
                   clamp_upper_top=True, seed=4, name="C5"),
}


def config_spec(name: str, scale: int = 1) -> TwoBodySpec:
    """BASELINE config `name`, optionally coarsened by an integer factor
    (element counts divided by `scale`, at least 2 per axis) for tests."""
    spec = CONFIGS[name]
    if scale == 1:
        return spec

    def shrink(b):
        return replace(b, elems=tuple(max(2, e // scale) for e in b.elems))

    return replace(spec, lower=shrink(spec.lower), upper=shrink(spec.upper),
                   name=f"{name}/{scale}")


# ---------------------------------------------------------------------------
# element stiffness on an axis-aligned box, lexicographic local corners


def _elasticity_matrix(dim, E, nu):
    lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
    mu = E / (2.0 * (1.0 + nu))
    if dim == 2:  # plane strain, Voigt (xx, yy, xy)
        return np.array([[lam + 2 * mu, lam, 0.0], [lam, lam + 2 * mu, 0.0], [0.0, 0.0, mu]])
    C = np.zeros((6, 6))
    C[:3, :3] = lam
    C[np.arange(3), np.arange(3)] += 2 * mu
    C[3:, 3:] = np.eye(3) * mu
    return C


def element_stiffness(dim: int, h, E: float, nu: float) -> np.ndarray:
    """Q1/hex8 stiffness with 2^dim-point Gauss; corner a = sum_k bit_k(a) 2^k."""
    h = np.asarray(h, dtype=np.float64)
    C = _elasticity_matrix(dim, E, nu)
    nc = 2 ** dim
    corners = np.array([[(a >> k) & 1 for k in range(dim)] for a in range(nc)], dtype=np.float64)
    g = 0.5 / np.sqrt(3.0)
    Ke = np.zeros((dim * nc, dim * nc))
    detJ = float(np.prod(h))
    for gp in itertools.product((0.5 - g, 0.5 + g), repeat=dim):
        gp = np.asarray(gp)
        # reference coords in [0,1]^dim; N_a = prod_k (c_k xi_k + (1-c_k)(1-xi_k))
        dN = np.zeros((nc, dim))
        for a in range(nc):
            f = np.where(corners[a] > 0, gp, 1.0 - gp)
            for k in range(dim):
                df = 1.0 if corners[a, k] > 0 else -1.0
                dN[a, k] = df * np.prod(np.delete(f, k)) / h[k]
        if dim == 2:
            B = np.zeros((3, 2 * nc))
            for a in range(nc):
                B[0, 2 * a] = dN[a, 0]
                B[1, 2 * a + 1] = dN[a, 1]
                B[2, 2 * a] = dN[a, 1]
                B[2, 2 * a + 1] = dN[a, 0]
        else:
            B = np.zeros((6, 3 * nc))
            for a in range(nc):
                x, y, z = dN[a]
                B[0, 3 * a] = x
                B[1, 3 * a + 1] = y
                B[2, 3 * a + 2] = z
                B[3, 3 * a + 1], B[3, 3 * a + 2] = z, y
                B[4, 3 * a], B[4, 3 * a + 2] = z, x
                B[5, 3 * a], B[5, 3 * a + 1] = y, x
        Ke += B.T @ C @ B * (detJ / nc)
    return Ke


# ---------------------------------------------------------------------------
# stencil table: node boundary type x neighbour offset -> dim x dim block


def _offsets(dim):
    """Neighbour offsets in ascending node-id order (last axis slowest)."""
    return [tuple(reversed(o)) for o in itertools.product((-1, 0, 1), repeat=dim)]


def stencil_table(dim: int, Ke: np.ndarray) -> np.ndarray:
    """table[type, offset, r, c] with type = sum_k t_k 3^k, t_k in
    {0: low face, 1: interior, 2: high face} (a grid with one element per
    axis has no interior type, which is never requested).  Each block is the
    sum over the element corners a_p (ascending) of Ke[a_p, a_p + offset]."""
    nc = 2 ** dim
    offs = _offsets(dim)
    ntype = 3 ** dim
    table = np.zeros((ntype, len(offs), dim, dim))
    for t in range(ntype):
        tk = [(t // 3 ** k) % 3 for k in range(dim)]
        for oi, off in enumerate(offs):
            acc = np.zeros((dim, dim))
            for a in range(nc):
                bits = [(a >> k) & 1 for k in range(dim)]
                ok = True
                for k in range(dim):
                    # node is corner bits[k] of the element; the element must
                    # exist (low face: only bits=0; high face: only bits=1)
                    if tk[k] == 0 and bits[k] == 1:
                        ok = False
                    if tk[k] == 2 and bits[k] == 0:
                        ok = False
                    q = bits[k] + off[k]
                    if q < 0 or q > 1:
                        ok = False
                if not ok:
                    continue
                b = sum(((bits[k] + off[k]) << k) for k in range(dim))
                acc = acc + Ke[dim * a: dim * a + dim, dim * b: dim * b + dim]
            table[t, oi] = acc
    return table


# ---------------------------------------------------------------------------
# mortar


def _hat(x, nodes, i):
    """Piecewise linear hat of node i on a sorted 1-D grid."""
    v = np.zeros_like(x)
    if i > 0:
        a, b = nodes[i - 1], nodes[i]
        m = (x >= a) & (x <= b)
        v[m] = (x[m] - a) / (b - a)
    if i < len(nodes) - 1:
        a, b = nodes[i], nodes[i + 1]
        m = (x >= a) & (x <= b)
        v[m] = np.maximum(v[m], (b - x[m]) / (b - a))
    return v


def mortar_1d(xs: np.ndarray, xm: np.ndarray):
    """Exact 1-D mortar integrals on the overlay of two grids.

    D[j, k] = int phi_j^s phi_k^s and M[j, m] = int phi_j^s phi_m^m, both by
    2-point Gauss on every overlay segment (exact for products of linears).
    """
    pts = np.unique(np.concatenate([xs, xm]))
    keep = np.concatenate([[True], np.diff(pts) > 1e-12 * (pts[-1] - pts[0])])
    pts = pts[keep]
    g = 0.5 / np.sqrt(3.0)
    D = np.zeros((len(xs), len(xs)))
    M = np.zeros((len(xs), len(xm)))
    for a, b in zip(pts[:-1], pts[1:]):
        mid = 0.5 * (a + b)
        q = np.array([a + (0.5 - g) * (b - a), a + (0.5 + g) * (b - a)])
        w = 0.5 * (b - a)
        js = np.searchsorted(xs, mid) - 1
        jm = np.searchsorted(xm, mid) - 1
        s_ids = [js, js + 1]
        m_ids = [jm, jm + 1]
        phis = {j: _hat(q, xs, j) for j in s_ids}
        phim = {m: _hat(q, xm, m) for m in m_ids}
        for j in s_ids:
            for k in s_ids:
                D[j, k] += w * float(np.dot(phis[j], phis[k]))
            for m in m_ids:
                M[j, m] += w * float(np.dot(phis[j], phim[m]))
    return D, M


# ---------------------------------------------------------------------------
# generated system


@dataclass
class GeneratedSystem:
    """Everything the solver and the oracle need for one config.

    `K` is None when the caller asked for device-side assembly; the stencil
    description (`stencil`, `blocks`) then drives `camg_assemble_stencil`.
    """

    spec: TwoBodySpec
    dim: int
    n_u: int
    n_lam: int
    K: scipy.sparse.csr_matrix | None
    B1: scipy.sparse.csr_matrix
    B2: scipy.sparse.csr_matrix
    Cz: scipy.sparse.csr_matrix
    rhs: np.ndarray
    node_coords: np.ndarray
    node_body: np.ndarray
    slave_nodes: np.ndarray      # new ids of slave interface nodes (ascending)
    master_nodes: np.ndarray
    active: np.ndarray           # per slave node
    stencil: list = field(default_factory=list)   # per block: (table, grid_nodes, clamp_lo, clamp_hi, node_offset)
    D_face: scipy.sparse.csr_matrix | None = None
    M_face: scipy.sparse.csr_matrix | None = None

    @property
    def num_nodes(self):
        return self.n_u // self.dim

    @property
    def slave_dofs(self):
        d = self.dim
        return (d * self.slave_nodes[:, None] + np.arange(d)[None, :]).ravel()

    @property
    def mortar_block(self) -> scipy.sparse.csr_matrix:
        """Slave-DOF rows of B1: row r <-> slave_dofs[r] (ascending)."""
        return self.B1[self.slave_dofs, :].tocsr()

    def rigid_body_modes(self) -> np.ndarray:
        x = self.node_coords
        n, d = x.shape
        if d == 2:
            v = np.zeros((2 * n, 3))
            v[0::2, 0] = 1.0
            v[1::2, 1] = 1.0
            v[0::2, 2] = -x[:, 1]
            v[1::2, 2] = x[:, 0]
            return v
        v = np.zeros((3 * n, 6))
        for c in range(3):
            v[c::3, c] = 1.0
        v[0::3, 3], v[1::3, 3] = -x[:, 1], x[:, 0]          # about z
        v[1::3, 4], v[2::3, 4] = -x[:, 2], x[:, 1]          # about x
        v[0::3, 5], v[2::3, 5] = x[:, 2], -x[:, 0]          # about y
        return v


def _block_nodes(b: BlockSpec, clamp_lo: bool, clamp_hi: bool, dim: int):
    """Lexicographic grid of a block, with the vertical low/high layers
    optionally removed.  Returns (coords of kept nodes, kept mask, grid dims)."""
    Nn = [e + 1 for e in b.elems]
    axes = [np.linspace(b.origin[k], b.origin[k] + b.size[k], Nn[k]) for k in range(dim)]
    mesh = np.meshgrid(*reversed(axes), indexing="ij")   # last axis slowest
    coords = np.stack([m.ravel() for m in reversed(mesh)], axis=1)
    kept = np.ones(int(np.prod(Nn)), dtype=bool)
    layer = int(np.prod(Nn[:-1]))
    if clamp_lo:
        kept[:layer] = False
    if clamp_hi:
        kept[-layer:] = False
    return coords, kept, Nn


def _assemble_block_host(table, Nn, kept, new_id, dim):
    """CSR pieces of one block (rows = kept nodes in order)."""
    offs = _offsets(dim)
    nnode = int(np.prod(Nn))
    lex = np.arange(nnode)
    idx = []
    rem = lex.copy()
    for k in range(dim):
        idx.append(rem % Nn[k])
        rem //= Nn[k]
    ntype = np.zeros(nnode, dtype=np.int64)
    for k in range(dim):
        t = np.where(idx[k] == 0, 0, np.where(idx[k] == Nn[k] - 1, 2, 1))
        ntype += t * 3 ** k
    rows_nodes = lex[kept]
    R = len(rows_nodes)
    # neighbour validity and columns
    nb_cols = np.full((R, len(offs)), -1, dtype=np.int64)
    for oi, off in enumerate(offs):
        ok = np.ones(R, dtype=bool)
        q = np.zeros(R, dtype=np.int64)
        stride = 1
        for k in range(dim):
            c = idx[k][rows_nodes] + off[k]
            ok &= (c >= 0) & (c < Nn[k])
            q += np.clip(c, 0, Nn[k] - 1) * stride
            stride *= Nn[k]
        ok &= kept[q]
        nb_cols[ok, oi] = new_id[q[ok]]
    vals = table[ntype[rows_nodes]]          # R x noff x dim x dim
    # entries ordered (node, r, offset, c)
    vals = vals.transpose(0, 2, 1, 3)        # R x dim x noff x dim
    cols = dim * nb_cols[:, None, :, None] + np.arange(dim)[None, None, None, :]
    valid = (nb_cols >= 0)[:, None, :, None] & (vals != 0.0)
    valid = np.broadcast_to(valid, vals.shape)
    cols = np.broadcast_to(cols, vals.shape)
    counts = valid.reshape(R * dim, -1).sum(axis=1)
    return counts, cols[valid], vals[valid]


def generate(spec: TwoBodySpec, assemble_K: bool = True) -> GeneratedSystem:
    """Build the saddle system of `spec` on the host.

    With `assemble_K=False` only the stencil description is produced; the
    caller assembles K on the device (large configs).
    """
    spec.validate()
    dim = spec.dim
    contact = spec.coupling == "contact"
    blocks = [
        (spec.upper, False, spec.clamp_upper_top, BODY_SLAVE),
        (spec.lower, True, False, BODY_MASTER),
    ]
    coords_all, body_all, stencil = [], [], []
    offset = 0
    per_block = []
    for b, clo, chi, body in blocks:
        coords, kept, Nn = _block_nodes(b, clo, chi, dim)
        new_id = np.full(len(kept), -1, dtype=np.int64)
        new_id[kept] = offset + np.arange(int(kept.sum()))
        h = [b.size[k] / b.elems[k] for k in range(dim)]
        Ke = element_stiffness(dim, h, b.youngs, spec.nu)
        table = stencil_table(dim, Ke)
        per_block.append((table, Nn, kept, new_id))
        stencil.append(dict(table=table, grid=tuple(Nn), clamp_lo=clo, clamp_hi=chi,
                            node_offset=offset))
        coords_all.append(coords[kept])
        body_all.append(np.full(int(kept.sum()), body, dtype=np.int8))
        offset += int(kept.sum())
    num_nodes = offset
    n_u = dim * num_nodes
    node_coords = np.vstack(coords_all)
    node_body = np.concatenate(body_all)

    K = None
    if assemble_K:
        counts, cols, vals = [], [], []
        for table, Nn, kept, new_id in per_block:
            c, j, v = _assemble_block_host(table, Nn, kept, new_id, dim)
            counts.append(c)
            cols.append(j)
            vals.append(v)
        counts = np.concatenate(counts)
        indptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        K = scipy.sparse.csr_matrix((np.concatenate(vals), np.concatenate(cols), indptr),
                                    shape=(n_u, n_u))
        K.has_sorted_indices = True

    # interface faces: slave = upper bottom layer, master = lower top layer
    (tab_s, Nn_s, kept_s, id_s), (tab_m, Nn_m, kept_m, id_m) = per_block
    layer_s = int(np.prod(Nn_s[:-1]))
    layer_m = int(np.prod(Nn_m[:-1]))
    slave_nodes = id_s[np.arange(layer_s)]
    master_nodes = id_m[len(kept_m) - layer_m + np.arange(layer_m)]
    if np.any(slave_nodes < 0) or np.any(master_nodes < 0):
        raise AssemblyError("interface node was clamped")

    # face mortar matrices (Kronecker of 1-D overlay integrals)
    D_face = M_face = None
    for k in reversed(range(dim - 1)):   # last in-plane axis slowest
        xs = np.linspace(spec.upper.origin[k], spec.upper.origin[k] + spec.upper.size[k], Nn_s[k])
        xm = np.linspace(spec.lower.origin[k], spec.lower.origin[k] + spec.lower.size[k], Nn_m[k])
        D1, M1 = mortar_1d(xs, xm)
        D1 = scipy.sparse.csr_matrix(D1)
        M1 = scipy.sparse.csr_matrix(M1)
        D_face = D1 if D_face is None else scipy.sparse.kron(D_face, D1, format="csr")
        M_face = M1 if M_face is None else scipy.sparse.kron(M_face, M1, format="csr")
    D_face = scipy.sparse.csr_matrix(D_face)
    M_face = scipy.sparse.csr_matrix(M_face)
    D_face.eliminate_zeros()
    M_face.eliminate_zeros()

    n_s = len(slave_nodes)
    n_lam = dim * n_s
    rng = np.random.default_rng(spec.seed)
    if contact and spec.active_fraction is not None:
        active = rng.random(n_s) < spec.active_fraction
    else:
        active = np.ones(n_s, dtype=bool)

    # full constraint matrix B (n_lam x n_u): rows dim*j+c
    Dc = D_face.tocoo()
    Mc = M_face.tocoo()
    r_parts, c_parts, v_parts = [], [], []
    for c in range(dim):
        r_parts += [dim * Dc.row + c, dim * Mc.row + c]
        c_parts += [dim * slave_nodes[Dc.col] + c, dim * master_nodes[Mc.col] + c]
        v_parts += [Dc.data, -Mc.data]
    Bfull = scipy.sparse.csr_matrix(
        (np.concatenate(v_parts), (np.concatenate(r_parts), np.concatenate(c_parts))),
        shape=(n_lam, n_u))
    Bfull.sum_duplicates()
    Bfull.sort_indices()
    B1 = Bfull.T.tocsr()
    B1.sort_indices()

    if not contact:
        B2 = Bfull.copy()
        Cz = scipy.sparse.csr_matrix((n_lam, n_lam))
    else:
        v = dim - 1
        normal_sign = -1.0        # slave outward normal points down
        rows = np.arange(n_lam)
        comp = rows % dim
        node = rows // dim
        normal_row = (comp == v) & active[node]
        scale = np.where(normal_row, normal_sign, 0.0)
        B2 = scipy.sparse.diags(scale) @ Bfull
        B2 = scipy.sparse.csr_matrix(B2)
        B2.eliminate_zeros()
        B2.sort_indices()
        cz_rows = rows[~normal_row]      # tangential rows and every row of inactive nodes
        Cz = scipy.sparse.csr_matrix((np.ones(len(cz_rows)), (cz_rows, cz_rows)),
                                     shape=(n_lam, n_lam))
    rhs = rng.uniform(-1.0, 1.0, n_u + n_lam)

    return GeneratedSystem(
        spec=spec, dim=dim, n_u=n_u, n_lam=n_lam, K=K, B1=B1, B2=B2, Cz=Cz, rhs=rhs,
        node_coords=node_coords, node_body=node_body, slave_nodes=slave_nodes,
        master_nodes=master_nodes, active=active, stencil=stencil,
        D_face=D_face, M_face=M_face,
    )


# ---------------------------------------------------------------------------
# device-side assembly and operator construction


def assemble_K_device(g: GeneratedSystem):
    """K assembled on the device from the stencil tables (bit-identical to
    the host assembly); returns a device-resident SparseMatrix."""
    import ctypes as C

    from . import _native as N
    from .sparse import SparseMatrix

    dim = g.dim
    total = 0
    for blk in g.stencil:
        grid = np.ascontiguousarray(blk["grid"], dtype=np.int64)
        table = np.ascontiguousarray(blk["table"], dtype=np.float64)
        nnz = C.c_int64()
        N.call("camg_stencil_block_counts", dim, grid.ctypes.data_as(C.c_void_p), int(blk["clamp_lo"]),
               int(blk["clamp_hi"]), table.ctypes.data_as(C.c_void_p), C.byref(nnz))
        total += nnz.value
    h = C.c_void_p()
    N.call("camg_csr_alloc", g.n_u, g.n_u, total, C.byref(h))
    row = 0
    for blk in g.stencil:
        grid = np.ascontiguousarray(blk["grid"], dtype=np.int64)
        table = np.ascontiguousarray(blk["table"], dtype=np.float64)
        N.call("camg_assemble_stencil", dim, grid.ctypes.data_as(C.c_void_p), int(blk["clamp_lo"]),
               int(blk["clamp_hi"]), int(blk["node_offset"]), g.n_u, table.ctypes.data_as(C.c_void_p), h, row)
        nk = int(np.prod(blk["grid"])) - (int(np.prod(blk["grid"][:-1])) if blk["clamp_lo"] else 0) \
            - (int(np.prod(blk["grid"][:-1])) if blk["clamp_hi"] else 0)
        row += dim * nk
    return SparseMatrix._wrap(h)


def saddle_operator(g: GeneratedSystem, device_K: bool | None = None):
    """SaddleOperator of a generated system (K on the device)."""
    from .saddle import SaddleOperator
    from .sparse import SparseMatrix

    if g.K is None or device_K:
        K = assemble_K_device(g)
    else:
        K = SparseMatrix.from_scipy(g.K)
    return SaddleOperator(K, SparseMatrix.from_scipy(g.B1), SparseMatrix.from_scipy(g.B2),
                          SparseMatrix.from_scipy(g.Cz))
